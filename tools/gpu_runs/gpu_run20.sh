cd $GRAFT_REPO_ROOT
for dbg in 0 1 2 3; do for mt in 1 2; do echo "DEBUG=$dbg MT=$mt"; GJ_DEBUG_UMMA=$dbg timeout 300 python tools/prof_join.py --reps 2 --filter 2 --mma-tiles $mt 2>&1 | tail -1; done; done
