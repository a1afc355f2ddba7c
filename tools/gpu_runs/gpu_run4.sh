cd $GRAFT_REPO_ROOT
timeout 300 python tools/prof_join.py --count 300000 --reps 2
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench4.json 2> gpurun_out/bench4.err; tail -3 gpurun_out/bench4.err; cat gpurun_out/bench4.json
timeout 1800 python -m pytest tests -m gpu -q -x --durations=10 2>&1 | tail -25 > gpurun_out/pytest_gpu5.txt
cat gpurun_out/pytest_gpu5.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_join -c 1 -o gpurun_out/prof_join_v4 python tools/prof_join.py --count 300000 --reps 1 > gpurun_out/prof_join_v4.out 2>&1
