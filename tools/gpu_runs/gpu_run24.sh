cd $GRAFT_REPO_ROOT
for cfg in 0 2; do for dbg in 4 8; do echo "CFG=$cfg DEBUG=$dbg"; GJ_UMMA_CFG=$cfg GJ_DEBUG_UMMA=$dbg timeout 300 python tools/prof_join.py --reps 2 --filter 2 --mma-tiles 1 2>&1 | tail -1; done; done
