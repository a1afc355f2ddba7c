// Microbenchmark: tcgen05.mma rate with the per-block accumulator handshake
// when MULTI warps issue (warp w issues the blocks c = w mod MULTI, slot c % 4),
// B200, one CTA per SM, 16 epilogue warps (4 per slot) that wait for each
// block's commit, read 32 columns each and release the slot.
// HS: 0 = mbarrier handshake (try_wait + arrive), 1 = named barriers (bar.sync /
// bar.arrive: no shared-memory access on the issuing thread).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1809_09930_b200/csrc -o umma_multi umma_multi.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "gj_umma.cuh"
using namespace gj;

constexpr int KP = 48;
struct Smem {
    alignas(1024) __half a[128 * KP];
    alignas(1024) __half b[128 * KP];
    uint64_t accf[4], acce[4], done[4];
    uint32_t tbase;
};

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int MULTI, int HS, bool READ>
__global__ void __launch_bounds__(640, 1) k_multi(int iters, long long* out) {
    extern __shared__ __align__(1024) unsigned char raw[];
    Smem& S = *reinterpret_cast<Smem*>(raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 128 * KP; i += blockDim.x) {
        S.a[i] = __float2half(((i * 2654435761u >> 20) & 255) / 256.f - 0.5f);
        S.b[i] = __float2half(((i * 2246822519u >> 20) & 255) / 256.f - 0.5f);
    }
    if (warp == 4) umma::tmem_alloc(&S.tbase, 512);
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) {
            umma::mbar_init(&S.accf[i], 1);
            umma::mbar_init(&S.acce[i], 4);
            umma::mbar_init(&S.done[i], 1);
        }
        umma::mbar_fence_init();
    }
    umma::fence_proxy_async();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tmem = S.tbase;
    constexpr uint32_t idesc = umma::idesc_f16_f32(128, 128);
    if (warp < MULTI) {   // issuers
        for (int c = warp; c < iters; c += MULTI) {
            const uint32_t slot = c % 4;
            if (c >= 4) {
                if (HS == 0) {
                    if (lane == 0) umma::mbar_wait(&S.acce[slot], ((c / 4) & 1u) ^ 1u);
                } else {
                    named_sync(1 + slot, 32 * 5);   // 4 epilogue warps arrive, this warp syncs
                }
            }
            if (lane == 0) {
                umma::fence_after();
#pragma unroll
                for (int k = 0; k < KP / 16; ++k)
                    umma::mma_f16(tmem + slot * 128, umma::smem_desc(umma::smem_u32(S.a) + k * 256, 128, KP * 16),
                                  umma::smem_desc(umma::smem_u32(S.b) + k * 256, 128, KP * 16), idesc, k > 0);
                umma::commit(&S.accf[slot]);
            }
            __syncwarp();
        }
        if (lane == 0) {   // drain this warp's MMAs
            umma::commit(&S.done[warp]);
            umma::mbar_wait(&S.done[warp], 0);
        }
    } else if (warp >= 4) {   // 16 epilogue warps, 4 per slot
        const int e = warp - 4, slot = e / 4, q = warp & 3;
        for (int c = slot; c < iters; c += 4) {
            umma::mbar_wait(&S.accf[slot], (c / 4) & 1u);
            umma::fence_after();
            if (READ) {
                uint32_t v[32];
                umma::tmem_ld32_nowait(tmem + ((uint32_t)(32 * q) << 16) + slot * 128 + 32 * (e & 3), v);
                umma::tmem_wait_ld();
                uint32_t x = v[0];
#pragma unroll
                for (int i = 1; i < 32; ++i) x &= v[i];
                if (x == 12345u) out[1000] = x;
            }
            umma::fence_before();
            if (c + 4 < iters) {
                if (HS == 0) {
                    __syncwarp();
                    if (lane == 0) umma::mbar_arrive(&S.acce[slot]);
                } else {
                    named_arrive(1 + slot, 32 * 5);
                }
            }
        }
    }
    umma::fence_before();
    __syncthreads();
    if (warp == 4) umma::tmem_dealloc(tmem, 512);
}

template <int MULTI, int HS, bool READ>
void run(const char* name) {
    long long* d;
    cudaMalloc(&d, 2000 * 8);
    const int iters = 40000;
    auto k = k_multi<MULTI, HS, READ>;
    cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
    printf("%-48s: ", name);
    k<<<148, 640, sizeof(Smem)>>>(400, d);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("warmup failed: %s\n", cudaGetErrorString(cudaGetLastError())); exit(1); }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<148, 640, sizeof(Smem)>>>(iters, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double tflops = 2.0 * 128 * 128 * KP * (double)iters * 148 / (ms * 1e-3) / 1e12;
    printf("%6.1f TFLOP/s  %s\n", tflops, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    setvbuf(stdout, NULL, _IONBF, 0);
    run<1, 0, false>("1 issuer, mbarrier handshake");
    run<2, 0, false>("2 issuers, mbarrier handshake");
    run<4, 0, false>("4 issuers, mbarrier handshake");
    run<1, 1, false>("1 issuer, named-barrier handshake");
    run<2, 1, false>("2 issuers, named-barrier handshake");
    run<4, 1, false>("4 issuers, named-barrier handshake");
    run<1, 0, true>("1 issuer, mbarrier handshake + reads");
    run<4, 0, true>("4 issuers, mbarrier handshake + reads");
    run<1, 1, true>("1 issuer, named-barrier + reads");
    run<4, 1, true>("4 issuers, named-barrier + reads");
    return 0;
}
