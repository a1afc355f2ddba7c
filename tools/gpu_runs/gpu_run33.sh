cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_r33.json 2> gpurun_out/bench_r33.err; grep "e2e step\|Error" gpurun_out/bench_r33.err | tail -6
