cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "regrow or host_pipeline" 2>&1 | tail -2
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --workload songs90 --k 6 > gpurun_out/songs6.json 2> gpurun_out/songs6.err; tail -2 gpurun_out/songs6.err; cat gpurun_out/songs6.json | cut -c1-400
