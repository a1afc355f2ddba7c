cd $GRAFT_REPO_ROOT
timeout 300 python tools/prof_join.py --count 300000 --reps 2
timeout 1800 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -8
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench6.json 2> gpurun_out/bench6.err; tail -3 gpurun_out/bench6.err; cat gpurun_out/bench6.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_join -c 1 -o gpurun_out/prof_join_tc1 python tools/prof_join.py --count 300000 --reps 1 > gpurun_out/prof_join_tc1.out 2>&1
