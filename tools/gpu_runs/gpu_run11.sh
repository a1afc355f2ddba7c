cd $GRAFT_REPO_ROOT
timeout 120 python tools/prof_join.py --count 300000 --reps 2 --filter 2
timeout 300 python tools/prof_join.py --reps 2 --filter 2
timeout 1800 python -m pytest tests/test_gpu_parity.py -q -x -k "filt or selftest or paper_shapes" 2>&1 | tail -4
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_join -s 1 -c 1 -o gpurun_out/prof_join_umma4 python tools/prof_join.py --count 300000 --reps 1 > gpurun_out/prof_join_umma4.out 2>&1
