cd $GRAFT_REPO_ROOT
GJ_TRACE=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_r70.json 2> gpurun_out/bench_r70.err; grep "e2e step\|\[gj\]" gpurun_out/bench_r70.err | tail -40
