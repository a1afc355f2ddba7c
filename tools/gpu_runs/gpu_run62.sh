cd $GRAFT_REPO_ROOT
export AB_WORKLOAD=expo64_10m AB_COUNT=3000000
for i in 1 2; do timeout 600 python tools/ab_join.py abtest/B 2 2>&1 | tail -1; GJ_UMMA_CFG=6 timeout 600 python tools/ab_join.py abtest/B 2 2>&1 | sed 's/^B/B-cfg6/' | tail -1; done
