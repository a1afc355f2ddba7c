#!/bin/bash
# query-set (deal block) change: parity of the partitioned / batched paths, A/B timing, 8-rank projection
cd "$GRAFT_REPO_ROOT"
out=gpurun_out/deal.txt
: > $out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_distributed.py -m gpu -x -q -k "entity or batches or regrows or work_counters or join_counts or pairs_equal or estimator or neighbor or distributed or nccl or gloo or torchrun" > gpurun_out/deal_parity.log 2>&1
echo "parity rc=$?" >> $out; tail -2 gpurun_out/deal_parity.log >> $out
for B in 1 8 32; do for nb in 3 24; do
  echo "== block $B nb $nb" >> $out
  GJ_DEAL_BLOCK=$B AB_BATCHES=$nb timeout 100 python tools/ab_join.py . 4 >> $out 2>&1
done; done
for B in 1 8; do echo "== projection block $B" >> $out; GJ_DEAL_BLOCK=$B timeout 300 python tools/scaling_projection.py --workload expo32 2>&1 | grep world >> $out; done
