cd $GRAFT_REPO_ROOT
timeout 120 python tools/prof_join.py --count 300000 --reps 2 --filter 2
timeout 120 python tools/prof_join.py --count 300000 --reps 1 --filter 3
timeout 300 python tools/prof_join.py --reps 2 --filter 2
timeout 1800 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -6
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_join -s 1 -c 1 -o gpurun_out/prof_join_umma3 python tools/prof_join.py --count 300000 --reps 1 > gpurun_out/prof_join_umma3.out 2>&1
