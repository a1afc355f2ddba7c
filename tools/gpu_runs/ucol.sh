#!/bin/bash
cd "$GRAFT_REPO_ROOT"
out=gpurun_out/ucol.txt
: > $out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "index_structure or every_flag or work_counters or join_counts or pairs_equal or filters_on_paper or degenerate or lattice or songs and k6 or expo32-default" > gpurun_out/ucol_parity.log 2>&1
echo "parity rc=$?" >> $out; tail -1 gpurun_out/ucol_parity.log >> $out
for v in head . head .; do for wl in songs90 expo32 uniform16; do
  echo "== $v $wl" >> $out
  AB_WORKLOAD=$wl timeout 100 python tools/ab_join.py $( [ $v = . ] && echo . || echo ab/$v ) 4 >> $out 2>&1
done; done
