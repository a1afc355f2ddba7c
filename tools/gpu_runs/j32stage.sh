#!/bin/bash
cd "$GRAFT_REPO_ROOT"
out=gpurun_out/j32stage.txt
: > $out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "filters_on_paper or every_flag or near_boundary or degenerate or lattice or dimension_limit or switch_off or pairs_equal or songs or work_counters or estimator" > gpurun_out/j32stage_parity.log 2>&1
echo "parity rc=$?" >> $out; tail -1 gpurun_out/j32stage_parity.log >> $out
for v in head . head .; do for wl in songs90; do
  echo "== $v $wl" >> $out
  AB_WORKLOAD=$wl timeout 100 python tools/ab_join.py $( [ $v = . ] && echo . || echo ab/$v ) 4 >> $out 2>&1
done; done
for k in 4 8; do timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --workload songs90 --eps 0.005 --k $k 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('k', d['config']['k'], round(d['ms_per_step'],1), {k: round(v,2) for k,v in d['phases_ms'].items()}, d['roofline']['frac'])" >> $out; done
