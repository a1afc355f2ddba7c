// Micro-benchmark: does tcgen05.ld throughput drop while the tensor core runs
// MMAs into other TMEM columns of the same SM?  One CTA per SM: warp 0 lane 0
// issues M=128 N=256 K=16 f16 MMAs into columns 256..511 (when MMA = 1);
// warps 1..W read columns 0..255 with tcgen05.ld.32x32b.x32 (two loads per
// wait, AND-reduced).  Prints load bytes/clk/SM and MMA issue rate.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1809_09930_b200/csrc -o tmem_contention tmem_contention.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "gj_umma.cuh"
using namespace gj;

__global__ void __launch_bounds__(576, 1) k_cont(int ld_reps, int mma_on, int ld_on, unsigned* out, long long* cyc) {
    __shared__ __align__(1024) __half a[128 * 16];
    __shared__ __align__(1024) __half b[256 * 16];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    __shared__ volatile int stop;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 128 * 16; i += blockDim.x) a[i] = __float2half(0.f);
    for (int i = threadIdx.x; i < 256 * 16; i += blockDim.x) b[i] = __float2half(0.f);
    if (warp == 0) umma::tmem_alloc(&tbase, 512);
    if (threadIdx.x == 0) { umma::mbar_init(&bar, 1); umma::mbar_fence_init(); stop = 0; }
    umma::fence_proxy_async();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tmem = tbase;
    long long t0 = clock64();
    long long nmma = 0;
    if (warp == 0) {
        if (lane == 0 && mma_on) {
            constexpr uint32_t idesc = umma::idesc_f16_f32(128, 256);
            uint32_t ph = 0;
            while (!stop) {
                for (int k = 0; k < 32; ++k)
                    umma::mma_f16(tmem + 256, umma::smem_desc(umma::smem_u32(a), 128, 256),
                                  umma::smem_desc(umma::smem_u32(b), 128, 256), idesc, 1u);
                umma::commit(&bar);
                umma::mbar_wait(&bar, ph);
                ph ^= 1u;
                nmma += 32;
            }
        }
        __syncwarp();
    } else {
        unsigned acc = 0xffffffffu;
        const uint32_t t = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((((warp - 1) >> 2) * 64) & 255);
        if (ld_on) {
            for (int r = 0; r < ld_reps; ++r) {
                uint32_t v[2][32];
                umma::tmem_ld32_nowait(t, v[0]);
                umma::tmem_ld32_nowait(t + 32, v[1]);
                umma::tmem_wait_ld();
#pragma unroll
                for (int x = 0; x < 2; ++x)
#pragma unroll
                    for (int y = 0; y < 32; ++y) acc &= v[x][y];
                acc ^= (unsigned)r;
            }
        } else {
            long long w = clock64();
            while (clock64() - w < 2000000) { }
        }
        if (acc == 0x12345u) out[threadIdx.x] = acc;
    }
    long long t1 = clock64();
    if (warp == 1 && lane == 0) { cyc[blockIdx.x * 2] = t1 - t0; stop = 1; }
    __syncthreads();
    long long t2 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x * 2 + 1] = nmma;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[300] = t2 - t0;
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc(tmem, 512);
}

void run(int warps, int mma_on, int ld_on) {
    unsigned* out; long long* cyc;
    cudaMalloc(&out, 4096 * 4); cudaMalloc(&cyc, 400 * 8);
    const int reps = 4000;
    k_cont<<<148, 32 * (1 + warps)>>>(10, mma_on, ld_on, out, cyc);
    cudaDeviceSynchronize();
    k_cont<<<148, 32 * (1 + warps)>>>(reps, mma_on, ld_on, out, cyc);
    cudaDeviceSynchronize();
    long long h[400];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const double ldb = (double)reps * warps * 2 * 32 * 32 * 4;
    const double c = (double)h[0];
    const double mma_rate = (double)h[1] / (double)h[300];   // MMAs per clk
    printf("ld warps=%2d mma=%d ld=%d : load %.1f B/clk/SM, MMA %.4f /clk (ideal 1/128 = 0.0078) %s\n", warps, mma_on, ld_on,
           ld_on ? ldb / c : 0.0, mma_rate, cudaGetErrorString(cudaGetLastError()));
    cudaFree(out); cudaFree(cyc);
}

int main() {
    for (int w : {8, 16}) { run(w, 0, 1); run(w, 1, 1); }
    run(8, 1, 0);
    return 0;
}
