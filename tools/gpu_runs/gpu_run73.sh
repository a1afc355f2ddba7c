cd $GRAFT_REPO_ROOT
B="timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
o=gpurun_out/sweep_r73.jsonl; : > $o
for e in 0.50 0.55 0.60; do $B --workload uniform16 --eps $e >> $o 2>/dev/null; done
$B --workload expo32 --no-reorder >> $o 2>/dev/null
$B --workload expo32 --no-sortidu >> $o 2>/dev/null
for k in 4 5 6 7 8; do $B --workload songs90 --k $k >> $o 2>/dev/null; done
$B --workload songs90 --eps 0.01 >> $o 2>/dev/null
$B --workload expo16 >> $o 2>/dev/null
$B --workload expo64_10m >> $o 2>/dev/null
$B --workload uniform16_small >> $o 2>/dev/null
timeout 900 python tools/scaling_projection.py > gpurun_out/scaling_r73.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_join_umma -s 2 -c 1 -o gpurun_out/prof_bench_join_r73 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --profile > gpurun_out/prof_bench_join_r73.out 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r73.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/launches_bench_r73.out 2>&1
wc -l $o; grep "^world" gpurun_out/scaling_r73.txt
