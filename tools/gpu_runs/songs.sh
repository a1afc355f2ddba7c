#!/bin/bash
cd "$GRAFT_REPO_ROOT"
out=gpurun_out/songs.txt
: > $out
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -x -q -k "songs or filters_on_paper or every_flag or near_boundary or dimension_limit or switch_off or degenerate" > gpurun_out/songs_parity.log 2>&1
echo "parity rc=$?" >> $out; tail -1 gpurun_out/songs_parity.log >> $out
for k in 4 5 6 7 8; do timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --workload songs90 --eps 0.005 --k $k >> gpurun_out/songs.jsonl 2>/dev/null; done
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --workload songs90 --eps 0.01 --k 6 >> gpurun_out/songs.jsonl 2>/dev/null
