#!/bin/bash
# per-tile kernel with persistent CTAs (atomic item counter) vs HEAD: parity, launch probe, A/B, projection
cd "$GRAFT_REPO_ROOT"
out=gpurun_out/pp.txt
: > $out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "filters_on_paper_shapes or accumulator_tiles or pairs_equal or every_flag or near_boundary or enable_limit or lattice or degenerate or entity or batches or regrows or dimension_limit or join_counts or work_counters" > gpurun_out/pp_parity.log 2>&1
echo "parity rc=$?" >> $out; tail -1 gpurun_out/pp_parity.log >> $out
echo "== probe new" >> $out; timeout 200 python tools/launch_probe.py 3 24 >> $out 2>&1
for v in head .; do for wl in expo32 uniform16 expo16; do echo "== $v $wl" >> $out; AB_WORKLOAD=$wl timeout 100 python tools/ab_join.py $( [ $v = . ] && echo . || echo ab/$v ) 4 >> $out 2>&1; done; done
sed -i 's#ab/\.#.#' $out
echo "== projection new" >> $out; timeout 300 python tools/scaling_projection.py --workload expo32 2>&1 | grep world >> $out
