// Microbenchmark: the tcgen05 join's block pipeline in isolation (one
// persistent CTA per SM): producer warp (cp.async.bulk of BN x KP fp16 candidate
// blocks from an L2-resident buffer) -> MMA warp (KP/16 tcgen05.mma, M = 128,
// N = BN, into one of SLOTS accumulator slots) -> epilogue warps (tcgen05.ld of
// the slot, AND of the sign bits, __any_sync), the same work per test as
// k_join_umma.  Reports cycles per block and tests per clock per SM, to size
// the accumulator ring / epilogue split before touching the join kernel.
//
// Epilogue split: NEW warps; warp w reads TMEM lane quarter w % 4 and column
// part (w / 4) % CP of every block (CP column parts), and blocks c with
// c % (NEW / (4 CP)) == w / (4 CP) (warp groups take turns on whole blocks).
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1809_09930_b200/csrc -o join_pipe join_pipe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "gj_umma.cuh"
using namespace gj;

// VAR bit 0: no candidate loads (the producer arrives on `full` without a copy);
// bit 1: no accumulator reads (the epilogue releases the slot at once).
// bit 2: mbarrier waits without the suspend-time hint (plain try_wait spin).
// bit 3: stream sequentially through the whole (large) source buffer from a
//        CTA-specific start instead of cycling over the first 512 blocks.
// bit 4: random A operand (the B source is filled by the host: zeros, or random
//        values when main() is given a second argument).
__device__ __forceinline__ void wait_spin(uint64_t* mbar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAITS_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAITS_%=;\n\t}\n" ::"r"(umma::smem_u32(mbar)), "r"(parity));
}
template <int VAR>
__device__ __forceinline__ void wait(uint64_t* mbar, uint32_t parity) {
    if (VAR & 4) wait_spin(mbar, parity); else umma::mbar_wait(mbar, parity);
}

template <int KP, int BN, int SLOTS, int NEW, int CP, int ST>
struct Smem {
    alignas(1024) __half a[128 * KP];
    alignas(1024) __half b[ST][BN * KP];
    uint64_t full[ST], empty[ST], accf[SLOTS], acce[SLOTS];
    uint32_t tbase;
    unsigned hits;
};

template <int KP, int BN, int SLOTS, int NEW, int CP, int ST, int CTAS, int VAR>
__global__ void __launch_bounds__(64 + 32 * NEW, CTAS)
    k_pipe(const __half* __restrict__ bsrc, int nsrc_blocks, int iters, long long* out, unsigned* hits) {
    extern __shared__ __align__(1024) unsigned char raw[];
    auto& S = *reinterpret_cast<Smem<KP, BN, SLOTS, NEW, CP, ST>*>(raw);
    constexpr int GROUPS = NEW / (4 * CP);      // warp groups taking turns on blocks
    constexpr int CW = BN / CP;                 // columns per warp per block
    constexpr int NL = CW / 32;                 // x32 loads per warp per block
    constexpr uint32_t TCOLS = SLOTS * BN <= 128 ? 128 : (SLOTS * BN <= 256 ? 256 : 512);
    static_assert(SLOTS * BN <= 512, "TMEM");
    // a warp group must own whole slots, else a group waiting on block c could
    // see the completion of block c - 2 SLOTS on the same barrier parity
    static_assert(GROUPS >= 1 && SLOTS % GROUPS == 0, "groups must divide slots");
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 128 * KP; i += blockDim.x) {
        const int row = i / KP, k = i % KP;
        const float av = (VAR & 16) ? (float)((row * 131 + k * 71) % 97) / 48.5f - 1.f : (k == 0 ? -1.f : 0.f);
        *reinterpret_cast<__half*>(reinterpret_cast<unsigned char*>(S.a) + umma::tile_off(row, k, KP)) =
            __float2half(av);
    }
    if (warp == 1) umma::tmem_alloc(&S.tbase, TCOLS);
    if (threadIdx.x == 0) {
        for (int i = 0; i < ST; ++i) { umma::mbar_init(&S.full[i], 1); umma::mbar_init(&S.empty[i], 1); }
        for (int i = 0; i < SLOTS; ++i) { umma::mbar_init(&S.accf[i], 1); umma::mbar_init(&S.acce[i], 4 * CP); }
        S.hits = 0;
        umma::mbar_fence_init();
    }
    umma::fence_proxy_async();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tmem = S.tbase;
    constexpr uint32_t kBlockBytes = BN * KP * 2;
    const long long t0 = clock64();
    if (warp == 0) {
        if (lane == 0) {
            for (int c = 0; c < iters; ++c) {
                const uint32_t st = c % ST, ph = (c / ST) & 1u;
                wait<VAR>(&S.empty[st], ph ^ 1u);
                if (VAR & 1) { umma::mbar_arrive(&S.full[st]); continue; }
                umma::mbar_arrive_expect_tx(&S.full[st], kBlockBytes);
                const int sb = (VAR & 8) ? (int)(((long long)blockIdx.x * 977 + c) % nsrc_blocks)
                                         : (c + 7 * blockIdx.x) % 512;
                umma::bulk_g2s(umma::smem_u32(S.b[st]), bsrc + (size_t)sb * BN * KP, kBlockBytes, &S.full[st]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = umma::idesc_f16_f32(128, BN);
            for (int c = 0; c < iters; ++c) {
                const uint32_t st = c % ST, ph = (c / ST) & 1u, ab = c % SLOTS, aph = (c / SLOTS) & 1u;
                wait<VAR>(&S.acce[ab], aph ^ 1u);
                wait<VAR>(&S.full[st], ph);
                umma::fence_after();
#pragma unroll
                for (int ks = 0; ks < KP / 16; ++ks)
                    umma::mma_f16(tmem + ab * BN, umma::smem_desc(umma::smem_u32(S.a) + ks * 256, 128, KP * 16),
                                  umma::smem_desc(umma::smem_u32(S.b[st]) + ks * 256, 128, KP * 16), idesc, ks > 0);
                umma::commit(&S.empty[st]);
                umma::commit(&S.accf[ab]);
            }
        }
    } else {
        const int e = warp - 2, q = warp & 3, cp = (e / 4) % CP, grp = e / (4 * CP);
        unsigned found = 0;
        for (int c = grp; c < iters; c += GROUPS) {
            const uint32_t ab = c % SLOTS, aph = (c / SLOTS) & 1u;
            wait<VAR>(&S.accf[ab], aph);
            umma::fence_after();
            if (VAR & 2) {
                __syncwarp();
                if (lane == 0) umma::mbar_arrive(&S.acce[ab]);
                continue;
            }
            const uint32_t tcol = tmem + ((uint32_t)(32 * q) << 16) + ab * BN + cp * CW;
            uint32_t acc = 0xffffffffu;
            constexpr int NC = NL >= 2 ? 2 : 1;
#pragma unroll
            for (int h = 0; h < NL / NC; ++h) {
                uint32_t v[NC][32];
#pragma unroll
                for (int x = 0; x < NC; ++x) umma::tmem_ld32_nowait(tcol + 32 * (NC * h + x), v[x]);
                umma::tmem_wait_ld();
                if (h == NL / NC - 1) {
                    umma::fence_before();
                    __syncwarp();
                    if (lane == 0) umma::mbar_arrive(&S.acce[ab]);
                }
                uint32_t t[8 * NC];
#pragma unroll
                for (int k = 0; k < 8 * NC; ++k) {
                    const int e0 = 4 * k;
                    t[k] = v[e0 / 32][e0 % 32] & v[(e0 + 1) / 32][(e0 + 1) % 32] & v[(e0 + 2) / 32][(e0 + 2) % 32] &
                           v[(e0 + 3) / 32][(e0 + 3) % 32];
                }
#pragma unroll
                for (int w = 4 * NC; w >= 1; w >>= 1)
#pragma unroll
                    for (int k = 0; k < w; ++k) t[k] &= t[k + w];
                acc &= t[0];
            }
            if (__any_sync(0xffffffffu, !(acc >> 31))) ++found;
        }
        if (lane == 0 && found) atomicAdd(&S.hits, found);
    }
    umma::fence_before();
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) { out[blockIdx.x] = t1 - t0; atomicAdd(hits, S.hits); }
    if (warp == 1) umma::tmem_dealloc(tmem, TCOLS);
}

template <int KP, int BN, int SLOTS, int NEW, int CP, int ST = 4, int CTAS = 1, int VAR = 0>
void run(const char* name, const __half* src, int nsrc_unused) {
    const int nsrc = (int)((size_t)8192 * 256 * 48 / (BN * KP));   // whole buffer in blocks
    using Sm = Smem<KP, BN, SLOTS, NEW, CP, ST>;
    auto kern = k_pipe<KP, BN, SLOTS, NEW, CP, ST, CTAS, VAR>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Sm));
    long long* d; cudaMalloc(&d, 148 * CTAS * 8);
    unsigned* hits; cudaMalloc(&hits, 4); cudaMemset(hits, 0, 4);
    const int iters = 8192 * (128 / BN > 0 ? 128 / BN : 1) * 4;
    kern<<<148 * CTAS, 64 + 32 * NEW, sizeof(Sm)>>>(src, nsrc, 256, d, hits);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<148 * CTAS, 64 + 32 * NEW, sizeof(Sm)>>>(src, nsrc, iters, d, hits);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    unsigned h; cudaMemcpy(&h, hits, 4, cudaMemcpyDeviceToHost);
    const double tests = 128.0 * BN * iters * CTAS;
    printf("%-48s: %7.1f cyc/blk/CTA  %6.1f tests/clk/SM  %.2f Ttests/s  mma-ideal %4.0f cyc  hits %u %s\n", name,
           (double)c / iters, tests / c, tests * 148 / (ms * 1e-3) / 1e12, (KP / 16) * 128.0 * BN / 256.0, h,
           cudaGetErrorString(cudaGetLastError()));
    fflush(stdout);
    cudaFree(d); cudaFree(hits);
}

int main(int argc, char** argv) {
    // 8192 blocks of 256 x 48 fp16 = 201 MB (bit 3 streams through all of it; otherwise
    // the first 512 blocks, 12.6 MB, L2 resident)
    const int nsrc = 8192;
    __half* src; cudaMalloc(&src, (size_t)nsrc * 256 * 48 * 2);
    {
        const size_t tot = (size_t)nsrc * 256 * 48;
        __half* h = (__half*)malloc(tot * 2);
        const bool rnd = argc > 2;
        unsigned x = 12345;
        for (size_t i = 0; i < tot; ++i) {
            x = x * 1664525u + 1013904223u;
            h[i] = __float2half(rnd ? (float)(x >> 8) / 8388608.f - 1.f : 0.f);
        }
        cudaMemcpy(src, h, tot * 2, cudaMemcpyHostToDevice);
        free(h);
    }
    const int pick = argc > 1 ? atoi(argv[1]) : -1;
    int idx = 0;
    if (pick < 0 || pick == idx) run<48,128,2,8,2,7,2,0>("K48 N128 2x(2 slots, 8w) ST7 zeros, L2 src", src, nsrc);
    ++idx;
    if (pick < 0 || pick == idx) run<48,128,2,8,2,7,2,8>("K48 ... streaming 200 MB src", src, nsrc);
    ++idx;
    if (pick < 0 || pick == idx) run<48,128,2,8,2,7,2,16>("K48 ... random A", src, nsrc);
    ++idx;
    if (pick < 0 || pick == idx) run<48,128,2,8,2,7,2,24>("K48 ... random A + streaming", src, nsrc);
    ++idx;
    if (pick < 0 || pick == idx) run<48,128,1,4,1,2,4,0>("K48 current 4x(1 slot) zeros", src, nsrc);
    ++idx;
    if (pick < 0 || pick == idx) run<48,128,1,4,1,2,4,24>("K48 current 4x(1 slot) random A + streaming", src, nsrc);
    ++idx;
    return 0;
}
