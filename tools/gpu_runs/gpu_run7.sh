cd $GRAFT_REPO_ROOT
timeout 120 python -m pytest tests/test_gpu_parity.py -q -x -k selftest 2>&1 | tail -15
timeout 300 python tools/prof_join.py --count 300000 --reps 2
timeout 1800 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -15
