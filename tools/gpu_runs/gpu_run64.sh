cd $GRAFT_REPO_ROOT
for i in 1 2 3; do for v in A B; do timeout 300 python tools/ab_join.py abtest/$v 3 2>&1 | tail -1; done; done
