#!/bin/bash
# Every config point DESIGN reports (BASELINE configs[0..4]), one bench line
# each, then the ncu launch list of the default step and a full ncu capture of
# its join launches (per-join DRAM traffic + pipe utilisation).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
out=gpurun_out/sweep.jsonl
: > $out
run() { timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" >> $out 2>> gpurun_out/sweep.err; }
python bench.py --steps 5 --warmup 3 > gpurun_out/sweep_default.json 2> gpurun_out/sweep_default.err
for e in 0.5 0.55 0.6; do run --workload uniform16 --eps $e; done
run --workload expo32 --no-reorder
run --workload expo32 --no-sortidu
for k in 4 5 6 7 8; do run --workload songs90 --eps 0.005 --k $k; done
run --workload songs90 --eps 0.01 --k 6
run --workload expo16
run --workload uniform16_small
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --workload expo64_10m >> $out 2>> gpurun_out/sweep.err
python bench.py --profile --steps 1 --warmup 1 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_join_umma -s 6 -c 3 -o gpurun_out/join \
    python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_join.log 2>&1
