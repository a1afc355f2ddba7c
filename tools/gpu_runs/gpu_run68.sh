cd $GRAFT_REPO_ROOT
for i in 1 2; do timeout 300 python tools/ab_join.py abtest/B 3 2>&1 | tail -1; GJ_UMMA_CFG=7 timeout 300 python tools/ab_join.py abtest/B 3 2>&1 | sed 's/^B/B-cfg7/' | tail -1; done
