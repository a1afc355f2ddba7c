#!/bin/bash
cd "$GRAFT_REPO_ROOT"
out=gpurun_out/est.txt
: > $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "estimator or batches or regrows or entity or expo32" > gpurun_out/est_parity.log 2>&1
echo "parity rc=$?" >> $out; tail -1 gpurun_out/est_parity.log >> $out
for u in 1 0; do for w in "expo32" "songs90 --eps 0.005 --k 6" "songs90 --eps 0.005 --k 8" "uniform16"; do
  echo "== uniform=$u $w" >> $out
  GJ_EST_UNIFORM=$u timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-stats --workload $w 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['phases_ms'], d['pairs'], d['config']['n_batches'])" >> $out 2>&1
done; done
