cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu3.txt
cat gpurun_out/pytest_gpu3.txt
timeout 300 python tools/prof_join.py --count 300000 --reps 2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_join -c 1 -o gpurun_out/prof_join_v2 python tools/prof_join.py --count 300000 --reps 1 > gpurun_out/prof_join_v2.out 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench2.json 2> gpurun_out/bench2.err; tail -3 gpurun_out/bench2.err; cat gpurun_out/bench2.json
