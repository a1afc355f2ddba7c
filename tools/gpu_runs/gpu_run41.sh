cd $GRAFT_REPO_ROOT
timeout 600 python tools/e2e_probe.py 2>&1 | tail -4
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_r41.json 2> gpurun_out/bench_r41.err; grep "e2e step" gpurun_out/bench_r41.err
