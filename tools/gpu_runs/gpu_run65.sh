cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu_r65.txt; cat gpurun_out/pytest_gpu_r65.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_r65.txt 2>&1; tail -1 gpurun_out/smoke_r65.txt
timeout 900 python bench.py > gpurun_out/bench_r65.json 2> gpurun_out/bench_r65.err; cut -c1-200 gpurun_out/bench_r65.json
timeout 900 python bench.py --impl reference > gpurun_out/bench_r65_ref.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r65.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/launches_bench_r65.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_join_umma -s 2 -c 1 -o gpurun_out/prof_bench_join_r65 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --profile > gpurun_out/prof_bench_join_r65.out 2>&1
B="timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
o=gpurun_out/sweep_r65.jsonl; : > $o
for e in 0.50 0.55 0.60; do $B --workload uniform16 --eps $e >> $o 2>/dev/null; done
$B --workload expo32 --no-reorder >> $o 2>/dev/null
$B --workload expo32 --no-sortidu >> $o 2>/dev/null
for k in 4 5 6 7 8; do $B --workload songs90 --k $k >> $o 2>/dev/null; done
$B --workload songs90 --eps 0.01 >> $o 2>/dev/null
$B --workload expo16 >> $o 2>/dev/null
$B --workload expo64_10m >> $o 2>/dev/null
$B --workload uniform16_small >> $o 2>/dev/null
timeout 900 python tools/scaling_projection.py > gpurun_out/scaling_r65.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --no-cpu-baseline > gpurun_out/bench_r65_gloo2.json 2> gpurun_out/bench_r65_gloo2.err
wc -l $o; grep "^world" gpurun_out/scaling_r65.txt; cut -c1-150 gpurun_out/bench_r65_gloo2.json
