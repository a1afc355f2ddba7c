cd $GRAFT_REPO_ROOT
for cfg in 0 3; do for dbg in 0 32 48; do echo "CFG=$cfg dbg$dbg"; GJ_UMMA_CFG=$cfg GJ_DEBUG_UMMA=$dbg timeout 300 python tools/prof_join.py --reps 1 --filter 2 --mma-tiles 1 2>&1 | sort | grep "rep 0\|cta 1002" | head -4; done; done
