cd $GRAFT_REPO_ROOT
for cfg in 0 2 3; do echo "CFG=$cfg"; GJ_UMMA_CFG=$cfg timeout 300 python tools/prof_join.py --reps 2 --filter 2 --mma-tiles 1 2>&1 | tail -1; done
echo "MT=2"; timeout 300 python tools/prof_join.py --reps 2 --filter 2 --mma-tiles 2 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "accumulator_tiles or paper_shapes or near_the_boundary" 2>&1 | tail -2
