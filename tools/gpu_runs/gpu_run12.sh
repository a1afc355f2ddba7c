cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/pytest_gpu_r12.txt; cat gpurun_out/pytest_gpu_r12.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_r12.txt 2>&1; cat gpurun_out/smoke_r12.txt
timeout 900 python bench.py > gpurun_out/bench_r12.json 2> gpurun_out/bench_r12.err; tail -2 gpurun_out/bench_r12.err; cat gpurun_out/bench_r12.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --dist-backend gloo --no-cpu-baseline > gpurun_out/bench_r12_gloo2.json 2> gpurun_out/bench_r12_gloo2.err; tail -3 gpurun_out/bench_r12_gloo2.err; cat gpurun_out/bench_r12_gloo2.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r12.csv python bench.py --steps 3 --warmup 3 > gpurun_out/launches_bench_r12.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_join_umma -s 2 -c 1 -o gpurun_out/prof_bench_join_r12 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --profile > gpurun_out/prof_bench_join_r12.out 2>&1
tail -2 gpurun_out/prof_bench_join_r12.out
