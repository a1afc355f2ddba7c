// Microbenchmark: cost of the tcgen05 issue loop on B200 (one CTA per SM).
// Variant bits: 1 = commit to an mbarrier per iteration, 2 = wait on that
// barrier (phase of iteration i - depth) before issuing, 4 = epilogue warps
// wait acc-full and arrive acc-empty (the join kernel's handshake).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1809_09930_b200/csrc -o umma_issue umma_issue.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "gj_umma.cuh"
using namespace gj;

template <int NMMA, int N, int SLOTS, int VAR>
__global__ void __launch_bounds__(192, 1) k_issue(int iters, long long* out) {
    __shared__ __align__(1024) __half a[128 * 48];
    __shared__ __align__(1024) __half b[256 * 48];
    __shared__ uint64_t accf[SLOTS], acce[SLOTS];
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 128 * 48; i += blockDim.x) a[i] = __float2half(0.f);
    for (int i = threadIdx.x; i < 256 * 48; i += blockDim.x) b[i] = __float2half(0.f);
    if (warp == 1) umma::tmem_alloc(&tbase, 512);
    if (threadIdx.x == 0) {
        for (int i = 0; i < SLOTS; ++i) { umma::mbar_init(&accf[i], 1); umma::mbar_init(&acce[i], 4); }
        umma::mbar_fence_init();
    }
    umma::fence_proxy_async();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tmem = tbase;
    constexpr uint32_t idesc = umma::idesc_f16_f32(128, N);
    long long t0 = clock64();
    if (warp == 1 && lane == 0) {
        for (int c = 0; c < iters; ++c) {
            const uint32_t ab = c % SLOTS, aph = (c / SLOTS) & 1u;
            if (VAR & 2) umma::mbar_wait(&acce[ab], aph ^ 1u);
            umma::fence_after();
#pragma unroll
            for (int k = 0; k < NMMA; ++k)
                umma::mma_f16(tmem + ab * N, umma::smem_desc(umma::smem_u32(a) + k * 256, 128, 48 * 16),
                              umma::smem_desc(umma::smem_u32(b) + k * 256, 128, 48 * 16), idesc, k > 0);
            if (VAR & 1) umma::commit(&accf[ab]);
        }
    } else if (warp >= 2 && (VAR & 4)) {
        for (int c = 0; c < iters; ++c) {
            const uint32_t ab = c % SLOTS, aph = (c / SLOTS) & 1u;
            umma::mbar_wait(&accf[ab], aph);
            umma::fence_after();
            umma::fence_before();
            __syncwarp();
            if (lane == 0) umma::mbar_arrive(&acce[ab]);
        }
    }
    if (warp == 1 && lane == 0 && !(VAR & 4)) {   // drain: commit + wait once
        umma::commit(&accf[0]);
    }
    umma::fence_before();
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (warp == 1) umma::tmem_dealloc(tmem, 512);
}

template <int NMMA, int N, int SLOTS, int VAR>
void run(const char* name) {
    long long* d; cudaMalloc(&d, 148 * 8);
    const int iters = 20000;
    k_issue<NMMA, N, SLOTS, VAR><<<148, 192>>>(100, d);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_issue<NMMA, N, SLOTS, VAR><<<148, 192>>>(iters, d);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    const double ideal = NMMA * 128.0 * N / 256.0;
    printf("%-44s: %7.1f cyc/iter (ideal %5.0f) %.3f ms %s\n", name, (double)c / iters, ideal, ms,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    run<3, 128, 2, 0>("3 MMA N128, no commit");
    run<3, 128, 2, 1>("3 MMA N128 + commit");
    run<3, 128, 2, 7>("3 MMA N128 + commit + handshake, 2 slots");
    run<3, 128, 4, 7>("3 MMA N128 + commit + handshake, 4 slots");
    run<3, 256, 2, 7>("3 MMA N256 + commit + handshake, 2 slots");
    run<6, 128, 2, 7>("6 MMA N128 + commit + handshake, 2 slots");
    run<6, 128, 4, 7>("6 MMA N128 + commit + handshake, 4 slots");
    run<12, 128, 2, 7>("12 MMA N128 + commit + handshake, 2 slots");
    return 0;
}
