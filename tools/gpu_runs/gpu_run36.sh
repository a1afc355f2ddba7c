cd $GRAFT_REPO_ROOT
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --no-cpu-baseline > gpurun_out/bench_r36_gloo2.json 2> gpurun_out/bench_r36_gloo2.err; tail -3 gpurun_out/bench_r36_gloo2.err | cut -c1-300; cut -c1-700 gpurun_out/bench_r36_gloo2.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_r36_ref.json 2> gpurun_out/bench_r36_ref.err; tail -2 gpurun_out/bench_r36_ref.err | cut -c1-300; cat gpurun_out/bench_r36_ref.json
