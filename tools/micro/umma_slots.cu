// Microbenchmark: tcgen05 join pipeline shape -- SLOTS accumulator slots of N
// columns (SLOTS x N = 512), MULTI issuer warps (issuer w issues the blocks
// c = w mod MULTI; block c goes to slot c % SLOTS; K = 48 per block), 16
// epilogue warps in four groups of four (one warp per TMEM lane quarter);
// group g reads every block whose slot is = g (mod 4): N columns per warp,
// sign-bit AND, release.  B200, one CTA per SM; prints TFLOP/s (useful MMA
// work) and tests per clock per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1809_09930_b200/csrc -o umma_slots umma_slots.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "gj_umma.cuh"
using namespace gj;

constexpr int KP = 48;
struct Smem {
    alignas(1024) __half a[128 * KP];
    alignas(1024) __half b[256 * KP];
    uint64_t accf[8], acce[8], done[8];
    uint32_t tbase;
};

template <int SLOTS, int N, int MULTI, int WPB>
__global__ void __launch_bounds__(640, 1) k_slots(int iters, long long* out) {
    extern __shared__ __align__(1024) unsigned char raw[];
    Smem& S = *reinterpret_cast<Smem*>(raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 128 * KP; i += blockDim.x) {
        S.a[i] = __float2half(((i * 2654435761u >> 20) & 255) / 256.f - 0.5f);
        S.b[i] = __float2half(((i * 2246822519u >> 20) & 255) / 256.f - 0.5f);
    }
    for (int i = threadIdx.x; i < 128 * KP; i += blockDim.x)
        S.b[128 * KP + i] = __float2half(((i * 2654435761u >> 20) & 255) / 256.f - 0.25f);
    if (warp == 4) umma::tmem_alloc(&S.tbase, 512);
    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; ++i) {
            umma::mbar_init(&S.accf[i], 1);
            umma::mbar_init(&S.acce[i], WPB);
            umma::mbar_init(&S.done[i], 1);
        }
        umma::mbar_fence_init();
    }
    umma::fence_proxy_async();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tmem = S.tbase;
    constexpr uint32_t idesc = umma::idesc_f16_f32(128, N);
    if (warp < MULTI) {
        if (lane == 0) {
            for (int c = warp; c < iters; c += MULTI) {
                const uint32_t slot = c % SLOTS;
                if (c >= SLOTS) umma::mbar_wait(&S.acce[slot], ((c / SLOTS) & 1u) ^ 1u);
                umma::fence_after();
#pragma unroll
                for (int k = 0; k < KP / 16; ++k)
                    umma::mma_f16(tmem + slot * N, umma::smem_desc(umma::smem_u32(S.a) + k * 256, 128, KP * 16),
                                  umma::smem_desc(umma::smem_u32(S.b) + k * 256, 128, KP * 16), idesc, k > 0);
                umma::commit(&S.accf[slot]);
            }
            umma::commit(&S.done[warp]);
            umma::mbar_wait(&S.done[warp], 0);
        }
    } else if (warp >= 4) {   // WPB warps read each block: 16 / WPB groups, group g takes c = g mod groups
        constexpr int G = 16 / WPB, CW = N * 4 / WPB;
        const int e = warp - 4, g = e / WPB, q = warp & 3, part = (e % WPB) / 4;
        uint32_t x = 0xffffffffu;
        for (int c = g; c < iters; c += G) {
            const uint32_t slot = c % SLOTS;
            umma::mbar_wait(&S.accf[slot], (c / SLOTS) & 1u);
            umma::fence_after();
            const uint32_t tc = tmem + ((uint32_t)(32 * q) << 16) + slot * N + part * CW;
            if (CW >= 64) {
#pragma unroll
                for (int h = 0; h < CW / 64; ++h) {
                    uint32_t v[2][32];
                    umma::tmem_ld32_nowait(tc + 64 * h, v[0]);
                    umma::tmem_ld32_nowait(tc + 64 * h + 32, v[1]);
                    umma::tmem_wait_ld();
                    if (h == CW / 64 - 1) {
                        umma::fence_before();
                        __syncwarp();
                        if (lane == 0 && c + SLOTS < iters) umma::mbar_arrive(&S.acce[slot]);
                    }
#pragma unroll
                    for (int i = 0; i < 32; ++i) x &= v[0][i] & v[1][i];
                }
            } else {
                uint32_t v[32];
                if (CW == 32) umma::tmem_ld32_nowait(tc, v);
                else umma::tmem_ld16_nowait(tc, *reinterpret_cast<uint32_t(*)[16]>(v));
                umma::tmem_wait_ld();
                umma::fence_before();
                __syncwarp();
                if (lane == 0 && c + SLOTS < iters) umma::mbar_arrive(&S.acce[slot]);
#pragma unroll
                for (int i = 0; i < CW; ++i) x &= v[i];
            }
        }
        if (x == 12345u) out[1000] = x;
    }
    umma::fence_before();
    __syncthreads();
    if (warp == 4) umma::tmem_dealloc(tmem, 512);
}

template <int SLOTS, int N, int MULTI, int WPB>
void run(const char* name) {
    long long* d;
    cudaMalloc(&d, 2000 * 8);
    const int iters = 40000 * 128 / N;
    auto k = k_slots<SLOTS, N, MULTI, WPB>;
    cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
    printf("%-44s: ", name);
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
    const double tests = 128.0 * N * (double)iters * 148;
    const double tflops = 2.0 * KP * tests / (ms * 1e-3) / 1e12;
    printf("%6.1f TFLOP/s (K=48)  %5.1f tests/clk/SM @1.9GHz  %s\n", tflops, tests / 148 / (ms * 1e-3 * 1.9e9),
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    setvbuf(stdout, NULL, _IONBF, 0);
    run<4, 128, 1, 16>("4 x N128, 1 issuer, 16 warps/block");
    run<4, 128, 2, 16>("4 x N128, 2 issuers, 16 warps/block");
    run<2, 256, 1, 16>("2 x N256, 1 issuer, 16 warps/block");
    run<2, 256, 1, 8>("2 x N256, 1 issuer, 8 warps/block");
    run<2, 256, 2, 16>("2 x N256, 2 issuers, 16 warps/block");
    return 0;
}
