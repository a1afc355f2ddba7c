#!/bin/bash
# quick check of the persistent kernel: parity subset, A/B vs legacy, phase profile (short timeouts)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "${PARITY_K:-filters_on_paper_shapes or accumulator_tiles or pairs_equal or every_flag or near_boundary or enable_limit or lattice or degenerate}" > gpurun_out/wsq_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/wsq_parity.log
: > gpurun_out/wsq_ab.txt
for v in ${AB:-legacy 2 4}; do
  if [ $v = legacy ]; then env="GJ_UMMA_WS=0"; else env="GJ_UMMA_WS=1 GJ_WS_EG=$v"; fi
  echo "== $v" >> gpurun_out/wsq_ab.txt
  env $env timeout 120 python tools/ab_join.py . 5 >> gpurun_out/wsq_ab.txt 2>&1
done
: > gpurun_out/wsq_prof.txt
for eg in ${PROF:-2}; do
  echo "== eg$eg" >> gpurun_out/wsq_prof.txt
  GJ_UMMA_WS=1 GJ_WS_EG=$eg timeout 120 python tools/experiments/ws_prof.py ab/wsprof >> gpurun_out/wsq_prof.txt 2>&1
done
