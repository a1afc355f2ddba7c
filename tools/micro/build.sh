# Build the tcgen05 micro-benchmarks (sm_100a); run them under gpurun, e.g.
#   gpurun -- 'bash tools/micro/build.sh && ./tools/micro/tmem_contention'
set -e
cd "$(dirname "$0")"
for f in umma_rate umma_lat umma_multi umma_slots tmem_ld_bw umma_issue tmem_contention join_pipe tmem_pack; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1809_09930_b200/csrc -o $f $f.cu
done
