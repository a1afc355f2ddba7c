cd $GRAFT_REPO_ROOT
for bn in 64 128; do GJ_UMMA_BN=$bn timeout 120 python tools/prof_join.py --count 300000 --reps 2 --filter 2; GJ_UMMA_BN=$bn timeout 300 python tools/prof_join.py --reps 2 --filter 2; done
timeout 1800 python -m pytest tests/test_gpu_parity.py -q -x -k "filt or selftest or paper_shapes" 2>&1 | tail -4
