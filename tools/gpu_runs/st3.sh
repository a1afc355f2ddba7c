#!/bin/bash
cd "$GRAFT_REPO_ROOT"
out=gpurun_out/st3.txt
: > $out
for r in 1 2; do for v in . st3; do for wl in expo32 uniform16 expo16; do
  echo "== $v $wl" >> $out
  AB_WORKLOAD=$wl timeout 100 python tools/ab_join.py $( [ $v = . ] && echo . || echo ab/$v ) 4 >> $out 2>&1
done; done; done
