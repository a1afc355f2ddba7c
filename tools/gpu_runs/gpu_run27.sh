cd $GRAFT_REPO_ROOT
for cfg in 0 2 3; do echo "CFG=$cfg"; GJ_UMMA_CFG=$cfg timeout 300 python tools/prof_join.py --reps 2 --filter 2 --mma-tiles 1 2>&1 | tail -1; done
echo "CFG=3 dbg16"; GJ_UMMA_CFG=3 GJ_DEBUG_UMMA=16 timeout 300 python tools/prof_join.py --reps 1 --filter 2 --mma-tiles 1 2>&1 | grep -v "^rep" | head -8
echo "CFG=3 dbg20"; GJ_UMMA_CFG=3 GJ_DEBUG_UMMA=20 timeout 300 python tools/prof_join.py --reps 1 --filter 2 --mma-tiles 1 2>&1 | head -8
