cd $GRAFT_REPO_ROOT
export AB_WORKLOAD=expo64_10m
for i in 1 2; do timeout 900 python tools/ab_join.py abtest/B 2 2>&1 | tail -1; GJ_UMMA_CFG=1 timeout 900 python tools/ab_join.py abtest/B 2 2>&1 | sed 's/^B/B-cfg1/' | tail -1; done
