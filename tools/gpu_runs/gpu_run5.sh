cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -8 > gpurun_out/pytest_gpu6.txt
cat gpurun_out/pytest_gpu6.txt
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench5.json 2> gpurun_out/bench5.err; tail -3 gpurun_out/bench5.err; cat gpurun_out/bench5.json
