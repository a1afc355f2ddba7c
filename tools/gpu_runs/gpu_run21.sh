cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "accumulator_tiles or paper_shapes or near_the_boundary" 2>&1 | tail -2
for cfg in "1 2" "1 1" "2 1"; do set -- $cfg; echo "MT=$1 EPW=$2"; GJ_UMMA_EPW=$2 timeout 300 python tools/prof_join.py --reps 2 --filter 2 --mma-tiles $1 2>&1 | tail -1; done
echo "DEBUG=1 MT=1 EPW=2"; GJ_DEBUG_UMMA=1 timeout 300 python tools/prof_join.py --reps 2 --filter 2 --mma-tiles 1 2>&1 | tail -1
