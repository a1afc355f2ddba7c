cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "accumulator_tiles or paper_shapes or flag_combination or near_the_boundary" 2>&1 | tail -3
for mt in 1 2; do for bn in 64 128; do echo "MT=$mt BN=$bn"; GJ_UMMA_BN=$bn timeout 300 python tools/prof_join.py --reps 2 --filter 2 --mma-tiles $mt 2>&1 | tail -1; done; done
