// Microbenchmark: sustained tcgen05.mma rate (kind::f16, M = 128, K = 48 per
// block of three MMAs) on B200, one CTA per SM, one issuing thread, four
// accumulator slots, no accumulator handshake -- what the join's MMA issuer
// could reach, as a function of
//   LAYOUT  0 = SWIZZLE_NONE core matrices (the join's layout), 6 = 32B swizzle
//   TS      A operand from TMEM instead of shared memory
//   N       128 or 256 candidates per MMA
//   LOAD    a producer warp streams one 12 KB cp.async.bulk per block into smem
//   READ    16 warps read TMEM (tcgen05.ld.32x32b.x32) continuously
//   RND     random fp16 operands (else zeros)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1809_09930_b200/csrc -o umma_rate umma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "gj_umma.cuh"
using namespace gj;

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    return umma::smem_desc(saddr, lbo, sbo) | ((uint64_t)layout << 61);
}
// WAIT: 0 = try_wait with the suspend-time hint (the join's), 1 = try_wait without a hint, 2 = test_wait poll
template <int WAIT>
__device__ __forceinline__ void wait_ph(uint64_t* mbar, uint32_t parity) {
    if (WAIT == 0) {
        umma::mbar_wait(mbar, parity);
    } else if (WAIT == 1) {
        asm volatile(
            "{\n\t.reg .pred P1;\n"
            "WAITS_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
            "@!P1 bra WAITS_%=;\n\t}\n" ::"r"(umma::smem_u32(mbar)), "r"(parity));
    } else {
        while (!umma::mbar_test(umma::smem_u32(mbar), parity)) {
        }
    }
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}

constexpr int KP = 48;
struct Smem {
    alignas(1024) __half a[128 * KP];
    alignas(1024) __half b[256 * KP];
    alignas(1024) __half ld[4][128 * KP];   // producer target (not read by the MMA)
    uint64_t done, full[4], accf[4], acce[4], stg[4];
    uint32_t tbase;
    volatile uint32_t stop;
    uint32_t credit;
};

template <int LAYOUT, bool TS, int N, bool LOAD, bool READ, bool RND, int SYNC = 0, int WAIT = 0, int ISS = 0>
__global__ void __launch_bounds__(32 * 18, 1) k_rate(int iters, const __half* g, long long* out) {
    extern __shared__ __align__(1024) unsigned char raw[];
    Smem& S = *reinterpret_cast<Smem*>(raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 128 * KP; i += blockDim.x)
        S.a[i] = __float2half(RND ? ((i * 2654435761u >> 20) & 255) / 256.f - 0.5f : 0.f);
    for (int i = threadIdx.x; i < 256 * KP; i += blockDim.x)
        S.b[i] = __float2half(RND ? ((i * 2246822519u >> 20) & 255) / 256.f - 0.5f : 0.f);
    if (warp == 1) umma::tmem_alloc(&S.tbase, 512);
    if (threadIdx.x == 0) {
        umma::mbar_init(&S.done, 1);
        for (int i = 0; i < 4; ++i) {
            umma::mbar_init(&S.full[i], 1);
            umma::mbar_init(&S.accf[i], 1);
            umma::mbar_init(&S.acce[i], 16);
            umma::mbar_init(&S.stg[i], 1);
        }
        S.stop = 0;
        S.credit = 0;
        umma::mbar_fence_init();
    }
    umma::fence_proxy_async();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tmem = S.tbase;
    // slots: N = 128 -> 4 x 128 columns (TS: 3 slots, A at columns 384..407)
    constexpr int SLOTS = TS ? 3 : (N == 128 ? 4 : 2);
    constexpr uint32_t idesc = umma::idesc_f16_f32(128, N);
    constexpr uint32_t sbo = LAYOUT == 0 ? KP * 16 : KP * 16;   // 8-row group stride (bytes)
    constexpr uint32_t lbo = LAYOUT == 0 ? 128 : 16;
    const long long t0 = clock64();
    if (warp == 1 && lane == 0) {
        for (int c = 0; c < iters; ++c) {
            const uint32_t slot = c % SLOTS;
            // SYNC bits: 1 commit accf[slot] per block, 2 + commit stg[slot], 4 fence::after_thread_sync,
            // 8 wait for the epilogue's release of the slot (16 warps wait accf, arrive acce)
            // ISS: 0 = wait per block, 1 = test_wait probe then wait, 2 = wait both slots of a pair
            // every second block, 4 = wait all four slots every fourth block
            if (SYNC & 8) {
                const uint32_t ph = ((c / SLOTS) & 1u) ^ 1u;
                if (ISS == 0) wait_ph<WAIT>(&S.acce[slot], ph);
                else if (ISS == 1) { if (!umma::mbar_test(umma::smem_u32(&S.acce[slot]), ph)) wait_ph<WAIT>(&S.acce[slot], ph); }
                else if (c % ISS == 0) {
                    for (int x = 0; x < ISS; ++x) wait_ph<WAIT>(&S.acce[(c + x) % SLOTS], (((c + x) / SLOTS) & 1u) ^ 1u);
                }
            }
            if (SYNC & 16) umma::mbar_wait(&S.done, 1u);   // a phase that completed long ago
            if (SYNC & 32) { if (*(volatile uint32_t*)&S.credit == 0xdeadbeefu) break; }
            if (SYNC & 64) { if (umma::mbar_test(umma::smem_u32(&S.done), 1u) == false) break; }
            if (SYNC & 4) umma::fence_after();
#pragma unroll
            for (int k = 0; k < KP / 16; ++k) {
                const uint64_t bd = desc(umma::smem_u32(S.b) + k * 256, lbo, sbo, LAYOUT);
                if (TS)
                    mma_ts(tmem + slot * N, tmem + 384 + k * 8, bd, idesc, k > 0);
                else
                    umma::mma_f16(tmem + slot * N, desc(umma::smem_u32(S.a) + k * 256, lbo, sbo, LAYOUT), bd, idesc, k > 0);
            }
            if (SYNC & 1) umma::commit(&S.accf[slot]);
            if ((SYNC & 2) && (ISS < 2 || c % 2 == 1)) umma::commit(&S.stg[slot]);
        }
        umma::commit(&S.done);
        umma::mbar_wait(&S.done, 0);
        S.stop = 1;
    } else if (warp == 0 && LOAD && lane == 0) {
        int c = 0;
        for (; !S.stop; ++c) {
            const int st = c & 3;
            if (c >= 4) umma::mbar_wait(&S.full[st], ((c >> 2) - 1) & 1);
            umma::mbar_arrive_expect_tx(&S.full[st], 128 * KP * 2);
            umma::bulk_g2s(umma::smem_u32(S.ld[st]), g + (size_t)(c % 4096) * 128 * KP, 128 * KP * 2, &S.full[st]);
        }
        for (int x = c - 4 > 0 ? c - 4 : 0; x < c; ++x) umma::mbar_wait(&S.full[x & 3], (x >> 2) & 1);   // drain
    } else if (warp >= 2 && (SYNC & 8)) {   // release each slot as soon as it is complete
        for (int c = 0; c < iters; ++c) {
            const uint32_t slot = c % SLOTS;
            wait_ph<WAIT>(&S.accf[slot], (c / SLOTS) & 1u);
            umma::fence_after();
            if (READ) {
                uint32_t v[32];
                umma::tmem_ld32_nowait(tmem + ((uint32_t)(32 * (warp & 3)) << 16) + slot * N + 32 * ((warp - 2) >> 2), v);
                umma::tmem_wait_ld();
                if (v[0] == 12345u && v[7] == 3u) out[1000] = v[3];
            }
            umma::fence_before();
            __syncwarp();
            if (lane == 0) umma::mbar_arrive(&S.acce[slot]);
        }
    } else if (warp >= 2 && READ) {
        uint32_t acc = 0;
        const uint32_t lane_off = (uint32_t)(32 * (warp & 3)) << 16;
        for (int c = 0; !S.stop; ++c) {
            uint32_t v[32];
            umma::tmem_ld32_nowait(tmem + lane_off + (uint32_t)((c * 32 + 128 * (warp >> 2)) & 511), v);
            umma::tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) acc &= v[i];
        }
        if (acc == 12345) out[1000] = acc;
    }
    umma::fence_before();
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (warp == 1) umma::tmem_dealloc(tmem, 512);
}

template <int LAYOUT, bool TS, int N, bool LOAD, bool READ, bool RND, int SYNC = 0, int WAIT = 0, int ISS = 0>
void run(const char* name, const __half* g) {
    long long* d;
    cudaMalloc(&d, 2000 * 8);
    const int iters = 40000;
    auto k = k_rate<LAYOUT, TS, N, LOAD, READ, RND, SYNC, WAIT, ISS>;
    cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
    printf("%-52s: ", name);
    k<<<148, 32 * 18, sizeof(Smem)>>>(200, g, d);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("warmup failed: %s\n", cudaGetErrorString(cudaGetLastError())); exit(1); }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<148, 32 * 18, sizeof(Smem)>>>(iters, g, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    const double ideal = 3 * 128.0 * N / 256.0;
    const double tflops = 2.0 * 128 * N * KP * (double)iters * 148 / (ms * 1e-3) / 1e12;
    printf("%7.1f cyc/block (ideal %4.0f)  %6.1f TFLOP/s  %s\n", (double)c / iters, ideal, tflops,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    setvbuf(stdout, NULL, _IONBF, 0);
    __half* g;
    cudaMalloc(&g, (size_t)4096 * 128 * KP * 2);
    cudaMemset(g, 0x31, (size_t)4096 * 128 * KP * 2);
    run<0, false, 128, false, false, true, 1>("commit accf", g);
    run<0, false, 128, false, false, true, 17>("commit accf + try_wait on a completed phase", g);
    run<0, false, 128, false, false, true, 65>("commit accf + test_wait on a completed phase", g);
    run<0, false, 128, false, false, true, 33>("commit accf + volatile smem load", g);
    run<0, false, 128, false, false, true, 5>("commit accf + fence::after_thread_sync", g);
    run<0, false, 128, false, false, true, 3>("commit accf + commit stage", g);
    return 0;
}
