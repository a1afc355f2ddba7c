#!/bin/bash
# A/B over workloads: legacy per-tile kernel vs persistent kernel builds
cd "$GRAFT_REPO_ROOT"
out=gpurun_out/ws_wl.txt
: > $out
for wl in ${WLS:-expo32 uniform16 expo16 expo64_10m:2000000}; do
  w=${wl%%:*}; n=${wl#*:}; [ "$n" = "$wl" ] && n=""
  for v in ${VARS:-legacy split0 split1}; do
    echo "== $w $n $v" >> $out
    if [ $v = legacy ]; then
      AB_WORKLOAD=$w AB_COUNT=$n GJ_UMMA_WS=0 timeout 200 python tools/ab_join.py ab/split0 3 >> $out 2>&1
    else
      AB_WORKLOAD=$w AB_COUNT=$n GJ_UMMA_WS=1 GJ_WS_EG=${EG:-2} timeout 200 python tools/ab_join.py ab/$v 3 >> $out 2>&1
    fi
  done
done
