cd $GRAFT_REPO_ROOT
for cfg in 0 1; do for dbg in 0 1 3; do echo "CFG=$cfg DEBUG=$dbg"; GJ_UMMA_CFG=$cfg GJ_DEBUG_UMMA=$dbg timeout 300 python tools/prof_join.py --reps 2 --filter 2 --mma-tiles 1 2>&1 | tail -1; done; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "accumulator_tiles or paper_shapes" 2>&1 | tail -2
GJ_UMMA_CFG=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "accumulator_tiles or paper_shapes" 2>&1 | tail -2
