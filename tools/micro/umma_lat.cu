// Microbenchmark: where the tcgen05 accumulator round trip goes (B200, one CTA
// per SM).  An issuer thread runs blocks of three K=16 MMAs (M = N = 128) into
// SLOTS accumulator slots; per slot, EPW epilogue warps wait for the block's
// commit and release the slot.  Timestamps (SM clock) per block:
//   issue   issuer starts the block's MMAs          (after its release wait)
//   commit  issuer has issued the MMAs and the commit
//   wake    first epilogue warp returns from the accf wait
//   arrive  last epilogue warp arrives on acce
//   rel     issuer returns from the acce wait for the slot's next block
// Mode 1 measures an isolated block: issue -> commit -> wait on the same thread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1809_09930_b200/csrc -o umma_lat umma_lat.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "gj_umma.cuh"
using namespace gj;

constexpr int KP = 48;
constexpr int NB = 4096;   // blocks
struct Smem {
    alignas(1024) __half a[128 * KP];
    alignas(1024) __half b[128 * KP];
    uint64_t accf[8], acce[8], done;
    uint32_t tbase;
    long long t_issue[NB], t_commit[NB], t_wake[NB], t_arrive[NB], t_rel[NB];
};

template <int SLOTS, int EPW, int ISO>
__global__ void __launch_bounds__(64 + 32 * 16, 1) k_lat(long long* out) {
    extern __shared__ __align__(1024) unsigned char raw[];
    Smem& S = *reinterpret_cast<Smem*>(raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 128 * KP; i += blockDim.x) {
        S.a[i] = __float2half(((i * 2654435761u >> 20) & 255) / 256.f - 0.5f);
        S.b[i] = __float2half(((i * 2246822519u >> 20) & 255) / 256.f - 0.5f);
    }
    for (int i = threadIdx.x; i < NB; i += blockDim.x) S.t_wake[i] = 0x7fffffffffffffffll, S.t_arrive[i] = 0;
    if (warp == 1) umma::tmem_alloc(&S.tbase, 512);
    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; ++i) {
            umma::mbar_init(&S.accf[i], 1);
            umma::mbar_init(&S.acce[i], EPW);
        }
        umma::mbar_init(&S.done, 1);
        umma::mbar_fence_init();
    }
    umma::fence_proxy_async();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tmem = S.tbase;
    constexpr uint32_t idesc = umma::idesc_f16_f32(128, 128);
    constexpr int NS = 512 / 128 < SLOTS ? 4 : SLOTS;
    if (warp == 1 && lane == 0) {
        for (int c = 0; c < NB; ++c) {
            const uint32_t slot = c % NS;
            if (!ISO) {
                umma::mbar_wait(&S.acce[slot], ((c / NS) & 1u) ^ 1u);
                if (c >= NS) S.t_rel[c - NS] = clock64();
            }
            S.t_issue[c] = clock64();
            umma::fence_after();
#pragma unroll
            for (int k = 0; k < KP / 16; ++k)
                umma::mma_f16(tmem + slot * 128, umma::smem_desc(umma::smem_u32(S.a) + k * 256, 128, KP * 16),
                              umma::smem_desc(umma::smem_u32(S.b) + k * 256, 128, KP * 16), idesc, k > 0);
            umma::commit(ISO ? &S.done : &S.accf[slot]);
            S.t_commit[c] = clock64();
            if (ISO) {
                umma::mbar_wait(&S.done, c & 1u);
                S.t_wake[c] = clock64();
            }
        }
    } else if (!ISO && warp >= 2 && (warp - 2) < NS * EPW) {
        const int slot = (warp - 2) / EPW;
        for (int c = slot; c < NB; c += NS) {
            umma::mbar_wait(&S.accf[slot], (c / NS) & 1u);
            const long long w = clock64();
            umma::fence_after();
            umma::fence_before();
            __syncwarp();
            if (lane == 0) {
                atomicMin((unsigned long long*)&S.t_wake[c], (unsigned long long)w);
                atomicMax((unsigned long long*)&S.t_arrive[c], (unsigned long long)clock64());
                umma::mbar_arrive(&S.acce[slot]);
            }
        }
    }
    umma::fence_before();
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        double s[4] = {0, 0, 0, 0};
        int n = 0;
        for (int c = 100; c < NB - 8; ++c, ++n) {
            s[0] += (double)(S.t_commit[c] - S.t_issue[c]);
            s[1] += (double)(S.t_wake[c] - S.t_commit[c]);
            if (!ISO) {
                s[2] += (double)(S.t_arrive[c] - S.t_wake[c]);
                s[3] += (double)(S.t_rel[c] - S.t_arrive[c]);
            }
        }
        out[0] = (long long)(s[0] / n);
        out[1] = (long long)(s[1] / n);
        out[2] = (long long)(s[2] / n);
        out[3] = (long long)(s[3] / n);
        out[4] = (S.t_issue[NB - 9] - S.t_issue[100]) / (NB - 109);
    }
    if (warp == 1) umma::tmem_dealloc(tmem, 512);
}

template <int SLOTS, int EPW, int ISO>
void run(const char* name, int grid) {
    long long* d;
    cudaMalloc(&d, 64 * 8);
    auto k = k_lat<SLOTS, EPW, ISO>;
    cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
    k<<<grid, 64 + 32 * 16, sizeof(Smem)>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[5];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-44s grid %3d: issue->commit %5lld  commit->wake %5lld  wake->arrive %4lld  arrive->rel %4lld  "
           "cycles/block %5lld  %s\n", name, grid, h[0], h[1], h[2], h[3], h[4], cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    setvbuf(stdout, NULL, _IONBF, 0);
    run<4, 1, 1>("isolated block (issue, commit, wait)", 1);
    run<4, 1, 1>("isolated block (issue, commit, wait)", 148);
    run<4, 1, 0>("4 slots x 1 epilogue warp", 1);
    run<4, 1, 0>("4 slots x 1 epilogue warp", 148);
    run<4, 4, 0>("4 slots x 4 epilogue warps", 148);
    run<2, 4, 0>("2 slots x 4 epilogue warps", 148);
    return 0;
}
