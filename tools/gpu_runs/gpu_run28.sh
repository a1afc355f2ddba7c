cd $GRAFT_REPO_ROOT
for cfg in 0 3; do echo "CFG=$cfg dbg16"; GJ_UMMA_CFG=$cfg GJ_DEBUG_UMMA=16 timeout 300 python tools/prof_join.py --reps 1 --filter 2 --mma-tiles 1 2>&1 | sort | head -9; done
