// SelfJoinKernel on the 5th-generation tensor cores (tcgen05.mma, TMEM
// accumulators) with the certified distance bound of gj_index.cu (tc_threshold_from) and the
// FP64 decision of every surviving pair (B200-first variant of PAPER.md
// Alg. 1 l.596-607; FP64 semantics unchanged).
//
// CTA = one producer warp, one MMA-issuer warp and 8 epilogue warps per
// 128-query A tile of one cell (M = 128 TMEM lanes), candidates in blocks of
// 128 rows, two accumulator slots, two CTAs per SM (see k_join_umma below).
// The fp16 operands carry augmented columns so that every accumulator is
// (T - ||q^ - c^||^2) / 2 (gj_index.cu tc_threshold_from): a pair survives the
// bound iff its accumulator is > +0, and survivors are decided in FP64.
#include <stdlib.h>

#include <atomic>
#include <string>

#include "gj_internal.cuh"
#include "gj_umma.cuh"

namespace gj {
namespace {

constexpr int kM = 128;         // queries per tile (UMMA M)
constexpr int kN = 128;         // self-test GEMM width
// FP64 decision of one pair: the FP64 kernel's arithmetic (gj_join.cu).
__device__ __forceinline__ double dist2_fp64(const double* __restrict__ a, const double* __restrict__ b,
                                             int n_pad) {
    double acc = 0.0;
    for (int d = 0; d < n_pad; d += 4) {
        const double2 x = *reinterpret_cast<const double2*>(a + d);
        const double2 y = *reinterpret_cast<const double2*>(a + d + 2);
        const double2 u = *reinterpret_cast<const double2*>(b + d);
        const double2 v = *reinterpret_cast<const double2*>(b + d + 2);
        double t;
        t = x.x - u.x; acc = fma(t, t, acc);
        t = x.y - u.y; acc = fma(t, t, acc);
        t = y.x - v.x; acc = fma(t, t, acc);
        t = y.y - v.y; acc = fma(t, t, acc);
    }
    return acc;
}

// FP64 decision of up to 32 staged survivors of the bound, one per lane
// (lanes >= n idle), and emission of the pairs inside eps (both orders when
// symmetric) with one warp-aggregated atomic.  Returns this lane's count
// contribution (kCount).
template <int MODE, bool SYM>
__device__ __forceinline__ unsigned long long decide_batch(const JoinParams& P, const JoinArgs& A, const uint2* sv,
                                                           uint32_t n, int lane) {
    constexpr unsigned long long kMul = SYM ? 2ull : 1ull;
    const bool has = (uint32_t)lane < n;
    const uint2 e = has ? sv[lane] : make_uint2(0u, 0u);
    const bool ok = has && dist2_fp64(P.pts + (size_t)e.x * P.n_pad, P.pts + (size_t)e.y * P.n_pad, P.n_pad) <= P.eps2;
    if (MODE != kEmit) return ok ? kMul : 0ull;
    const unsigned m = __ballot_sync(0xffffffffu, ok);
    if (!m) return 0ull;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd((unsigned long long*)A.count, kMul * (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (ok) {
        const unsigned long long at = base + kMul * (unsigned long long)__popc(m & ((1u << lane) - 1u));
        if (at + kMul <= A.cap) {
            const uint32_t qi = P.orig[e.x], ci = P.orig[e.y];
            uint2* out = reinterpret_cast<uint2*>(A.out);
            out[at] = make_uint2(qi, ci);
            if (SYM) out[at + 1] = make_uint2(ci, qi);
        }
    }
    return 0ull;
}

// Per CTA: one 128-query A tile (M = 128 TMEM lanes) and a ring of
// 128-candidate B blocks; TWO 128-column fp32 accumulator slots (the MMA of
// block c + 1 runs while the epilogue reads block c), 8 epilogue warps
// (TMEM lane quarter = warp % 4, column half = (warp - 2) / 4: 64 columns =
// two tcgen05.ld.32x32b.x32 per warp and block) and TWO CTAs per SM (4 slots,
// 16 epilogue warps, 2 MMA issuers per SM).  Measured on the block pipeline
// alone (tools/micro/join_pipe, K = 48): 71 tests/clk/SM against 36 for four
// CTAs with one slot each (the round-1 kernel) -- a slot must be re-filled
// while another is read, and each block's TMEM read must be split over
// enough warps that one warp's per-block latency chain stays short.
#ifndef GJ_UMMA_N256
#define GJ_UMMA_N256 0
#endif
// (GJ_UMMA_N256 = 1, timing experiment: one CTA per SM with 256-candidate
// blocks, two 256-column slots and 16 epilogue warps)
constexpr int kBN = GJ_UMMA_N256 ? 256 : 128;   // candidates per block (UMMA N)
constexpr int kCtasPerSm = GJ_UMMA_N256 ? 1 : 2;
constexpr int kSlots = 2;                 // accumulator slots per CTA
constexpr int kEpi = kBN / 16;            // epilogue warps: 4 lane quarters x kBN/64 column parts
constexpr int kWarps = 2 + kEpi;          // 0 producer, 1 MMA issuer, 2.. epilogue
constexpr int kThreads = 32 * kWarps;
constexpr int kCW = 64;                   // accumulator columns per epilogue warp and block
constexpr int kTCols = kSlots * kBN;      // TMEM columns per CTA (power of two)
constexpr int kMaxWin = 512;              // adjacent cells handled per setup round
constexpr int kSmemCap = 227 * 1024 / kCtasPerSm - 2048;

template <int KP>
constexpr int umma_stages() {
    // A tile + window arrays + survivor lists + barriers beside the ring
    return (kSmemCap - 128 * KP * 2 - 3 * kMaxWin * 4 - kEpi * 64 * 8 - 512) / (kBN * KP * 2) < 8
               ? (kSmemCap - 128 * KP * 2 - 3 * kMaxWin * 4 - kEpi * 64 * 8 - 512) / (kBN * KP * 2)
               : 8;
}

template <int KP>
struct UmmaSmem {
    alignas(128) __half a[kM * KP];                      // queries (A), canonical K-major layout
    alignas(128) __half b[umma_stages<KP>()][kBN * KP];  // candidate ring (B)
    uint64_t full[umma_stages<KP>()], empty[umma_stages<KP>()], accf[kSlots], acce[kSlots];
    uint32_t tmem_base;
    uint32_t wr[kMaxWin], ws[kMaxWin], nbk[kMaxWin];     // window [r, s), blocks (bit 31: own cell)
    uint2 sv[kEpi][64];                                  // per epilogue warp: staged survivors (qpos, cpos)
    unsigned long long red[kWarps];
};

// Timing experiments (tools/ab_prep.sh builds with -DGJ_UMMA_EXPERIMENT=<bits>;
// the product build has 0): 1 = spin waits without the suspend-time hint,
// 2 = epilogue skips the survivor path, 4 = epilogue releases the slot
// without reading TMEM, 8 = MMA warp commits without issuing MMAs, 16 = the
// survivors are staged but never decided (no FP64 loads), 32 = the sign test
// and its vote run but the survivor path is skipped.
#ifndef GJ_UMMA_EXPERIMENT
#define GJ_UMMA_EXPERIMENT 0
#endif
constexpr int kExp = GJ_UMMA_EXPERIMENT;
// bit 64: clock64 phase counters per role (tools/umma_prof.py reads them through
// gj_debug_umma_prof, which only the experiment build exports)
constexpr bool kProf = (kExp & 64) != 0;
__device__ unsigned long long g_umma_prof[16];

__device__ __forceinline__ void wait_parity(uint32_t mbar, uint32_t parity) {
    if (kExp & 1) {
        asm volatile(
            "{\n\t.reg .pred P1;\n"
            "WAITS_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
            "@!P1 bra WAITS_%=;\n\t}\n" ::"r"(mbar),
            "r"(parity));
        return;
    }
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAITP_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra WAITP_%=;\n\t}\n" ::"r"(mbar),
        "r"(parity), "r"(0x989680u));
}
__device__ __forceinline__ void arrive_addr(uint32_t mbar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(mbar) : "memory");
}

// Warp-specialised tcgen05 join (Alg. 1 l.596-607 with the certified
// bound in front of the FP64 test).  Per CTA (128 queries of one cell): the
// epilogue warps build the A tile (coordinates + augmented columns r_hi,
// r_lo, 1, 1); all threads compute the SORTIDU windows of the adjacent cells
// (thread per cell, union over the CTA's queries, §4.3); then
//   producer : per 128-candidate block, one cp.async.bulk of the contiguous
//              grouped-layout rows [8 floor(r/8) + 128 b, +128) into the ring
//              (full/empty mbarriers, transaction bytes);
//   MMA      : one thread, K/16 tcgen05.mma (M = N = 128) per block into
//              accumulator slot c % 2; commits to empty[stage] and accf[slot];
//   epilogue : 8 warps, each 32 rows x 64 columns of the slot: two
//              tcgen05.ld, release the slot, AND of the 64 sign bits; the rare
//              non-negative entries (survivors of the bound) inside [r, s) (and
//              after the query in its own cell) are staged per warp and decided
//              32 at a time in FP64, one pair per lane.
template <int KP, int MODE, bool SYM>
__global__ void __launch_bounds__(kThreads, kCtasPerSm) k_join_umma(JoinParams P, JoinArgs A) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    UmmaSmem<KP>& S = *reinterpret_cast<UmmaSmem<KP>*>(smem_raw);
    constexpr int ST = umma_stages<KP>();
    constexpr int KS = KP / 16;
    constexpr uint32_t kIdesc = umma::idesc_f16_f32(kM, kBN);
    constexpr uint32_t kSBO = KP * 16;
    constexpr uint32_t kBlockBytes = kBN * KP * 2;
    static_assert(ST >= 2, "candidate ring needs at least two stages");
    static_assert(sizeof(UmmaSmem<KP>) <= kSmemCap, "shared memory");

    const CtaTile ct = cta_tile(P, A, kM);
    if (ct.nq == 0) return;   // sub-block past the end of the tile's cell
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int part = ct.part, split = ct.split;
    const uint32_t g = ct.g, q0 = ct.q0, nq = ct.nq;
    const int n_pad = P.n_pad;
    const double eps = P.eps;

    if (warp == 1) umma::tmem_alloc(&S.tmem_base, kTCols);
    if (tid == 0) {
        for (int i = 0; i < ST; ++i) {
            umma::mbar_init(&S.full[i], 1);
            umma::mbar_init(&S.empty[i], 1);
        }
        for (int i = 0; i < kSlots; ++i) {
            umma::mbar_init(&S.accf[i], 1);
            umma::mbar_init(&S.acce[i], kEpi);
        }
        umma::mbar_fence_init();
    }
    for (int row = tid - 64; row >= 0 && row < kM; row += 32 * kEpi) {   // A tile: thread = query row
        const bool valid = row < (int)nq;
        unsigned char* a_raw = reinterpret_cast<unsigned char*>(S.a);
        for (int kc = 0; kc < KP / 8; ++kc) {
            union { uint4 u; __half h[8]; } cc;
            cc.u = valid ? *reinterpret_cast<const uint4*>(P.pts16 + g16(q0 + row, kc * 8, KP)) : make_uint4(0, 0, 0, 0);
            if (kc == KP / 8 - 1) {   // query-side augmented columns
                query_aug(P.thr16, valid ? P.norm16[q0 + row] : 0.0, valid, cc.h[4], cc.h[5]);
                cc.h[6] = __float2half(1.f);
                cc.h[7] = __float2half(1.f);
            }
            *reinterpret_cast<uint4*>(a_raw + umma::tile_off(row, kc * 8, KP)) = cc.u;
        }
    }
    unsigned long long npairs = 0;
    if (SYM && part == 0 && tid < kM) {   // the self pair (q, q)
        const bool active = tid < (int)nq;
        const uint32_t qid = P.orig[q0 + (active ? tid : 0)];
        if (MODE == kEmit) {
            const unsigned m = __ballot_sync(0xffffffffu, active);
            unsigned long long base = 0;
            if (lane == 0 && m) base = atomicAdd((unsigned long long*)A.count, (unsigned long long)__popc(m));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (active) {
                const unsigned long long at = base + __popc(m & ((1u << lane) - 1u));
                if (at < A.cap) reinterpret_cast<uint2*>(A.out)[at] = make_uint2(qid, qid);
            }
        } else if (active) {
            npairs += 1;
        }
    }
    umma::fence_proxy_async();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tmem = S.tmem_base;
    const uint32_t full0 = umma::smem_u32(&S.full[0]), empty0 = umma::smem_u32(&S.empty[0]);
    const uint32_t accf0 = umma::smem_u32(&S.accf[0]), acce0 = umma::smem_u32(&S.acce[0]);

    const double u_lo = P.pts[(size_t)q0 * n_pad + P.u];
    const double u_hi = P.pts[(size_t)(q0 + nq - 1) * n_pad + P.u];
    const uint32_t nb0 = SYM ? P.nbr_self[g] : P.nbr_off[g], nb1 = P.nbr_off[g + 1];
    uint32_t cnt = 0;   // blocks consumed so far (identical sequence in every role)
    for (uint32_t w0 = nb0; w0 < nb1; w0 += kMaxWin) {
        const int nwin = (int)min((uint32_t)kMaxWin, nb1 - w0);
        for (int i = tid; i < nwin; i += kThreads) {   // windows of this round (thread per adjacent cell)
            const uint32_t B = P.nbr[w0 + i];
            uint32_t r = P.cell_start[B], s = P.cell_start[B + 1];
            if (P.sortidu) {
                uint32_t lo = r, hi = s;
                while (lo < hi) {   // first r with u_lo - r(u) <= eps
                    const uint32_t mid = (lo + hi) >> 1;
                    if (u_lo - P.pts[(size_t)mid * n_pad + P.u] <= eps) hi = mid; else lo = mid + 1;
                }
                const uint32_t rr = lo;
                hi = s;
                while (lo < hi) {   // first s with s(u) - u_hi > eps
                    const uint32_t mid = (lo + hi) >> 1;
                    if (P.pts[(size_t)mid * n_pad + P.u] - u_hi > eps) hi = mid; else lo = mid + 1;
                }
                r = rr;
                s = lo;
            }
            const bool diag = SYM && B == g;
            if (diag) r = max(r, q0 + 1);
            if (split > 1 && s > r) {
                const uint64_t len = s - r;
                s = r + (uint32_t)(len * (part + 1) / split);
                r = r + (uint32_t)(len * part / split);
            }
            S.wr[i] = r;
            S.ws[i] = s;
            S.nbk[i] = (s > r ? (s - (r & ~7u) + kBN - 1) / kBN : 0u) | (diag ? 0x80000000u : 0u);
        }
        __syncthreads();
        if (warp == 0) {   // ---------------- producer
            if (lane == 0) {
                uint32_t c = cnt;
                for (int i = 0; i < nwin; ++i) {
                    const uint32_t nb = S.nbk[i] & 0x7fffffffu;
                    const __half* src = P.pts16 + (size_t)(S.wr[i] & ~7u) * KP;
                    for (uint32_t bi = 0; bi < nb; ++bi, ++c, src += kBN * KP) {
                        const uint32_t st = c % ST, ph = (c / ST) & 1u;
                        wait_parity(empty0 + 8 * st, ph ^ 1u);
                        umma::mbar_arrive_expect_tx(&S.full[st], kBlockBytes);
                        umma::bulk_g2s(umma::smem_u32(S.b[st]), src, kBlockBytes, &S.full[st]);
                    }
                }
            }
        } else if (warp == 1) {   // ---------------- MMA issuer
            if (lane == 0) {
                const uint64_t adesc = umma::smem_desc(umma::smem_u32(S.a), 128, kSBO);
                const uint64_t bdesc = umma::smem_desc(umma::smem_u32(S.b[0]), 128, kSBO);
                uint32_t c = cnt;
                uint32_t total = 0;
                for (int i = 0; i < nwin; ++i) total += S.nbk[i] & 0x7fffffffu;
                unsigned long long mp[5] = {0, 0, 0, 0, 0};   // wait acce, wait full, blocks, mma issue, commits
                const long long mstart = kProf ? clock64() : 0;
                for (uint32_t e = 0; e < total; ++e, ++c) {
                    const uint32_t st = c % ST, ph = (c / ST) & 1u, ab = c & 1u, aph = (c >> 1) & 1u;
                    long long m0 = kProf ? clock64() : 0;
                    wait_parity(acce0 + 8 * ab, aph ^ 1u);
                    long long m1 = kProf ? clock64() : 0;
                    wait_parity(full0 + 8 * st, ph);
                    umma::fence_after();
                    if (kProf) { const long long m2 = clock64(); mp[0] += m1 - m0; mp[1] += m2 - m1; mp[2] += 1; }
                    const uint64_t bd = bdesc + ((st * kBlockBytes) >> 4);
                    long long m3 = kProf ? clock64() : 0;
#pragma unroll
                    for (int ks = 0; ks < ((kExp & 8) ? 0 : KS); ++ks)
                        umma::mma_f16(tmem + ab * kBN, adesc + (uint64_t)(ks * 16), bd + (uint64_t)(ks * 16), kIdesc,
                                      ks > 0 ? 1u : 0u);
                    long long m4 = kProf ? clock64() : 0;
                    // one commit per block: the epilogue frees the ring stage once it has
                    // seen this accumulator complete (the MMA's smem reads are done then)
                    umma::commit(&S.accf[ab]);
                    if (kProf) { const long long m5 = clock64(); mp[3] += m4 - m3; mp[4] += m5 - m4; }
                }
                if (kProf) {
                    atomicAdd(&g_umma_prof[8], mp[0]);
                    atomicAdd(&g_umma_prof[9], mp[1]);
                    atomicAdd(&g_umma_prof[10], mp[2]);
                    atomicAdd(&g_umma_prof[11], (unsigned long long)(clock64() - mstart));
                    atomicAdd(&g_umma_prof[12], mp[3]);
                    atomicAdd(&g_umma_prof[13], mp[4]);
                }
            }
        } else {   // ---------------- epilogue
            const int e = warp - 2;
            const int erow = 32 * (warp & 3) + lane;            // query row = TMEM lane
            const int ecol = e >> 2;                            // column part
            const uint32_t qpos = q0 + erow;
            const bool rvalid = erow < (int)nq;
            const uint32_t tbase = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(ecol * kCW);
            const unsigned lt = (1u << lane) - 1u;
            // Survivors of the bound are staged per warp and decided 32 at a time
            // (one per lane), so a rare FP64 decision never holds the accumulator
            // pipeline for a full memory round trip per pair.
            uint2* sv = S.sv[e];
            uint32_t svn = 0;
            uint32_t c = cnt;
            unsigned long long pr[7] = {0, 0, 0, 0, 0, 0, 0};   // wait, ld, fast, rare, decide, #rare, #decide
            for (int i = 0; i < nwin; ++i) {
                const uint32_t nb = S.nbk[i] & 0x7fffffffu;
                for (uint32_t bi = 0; bi < nb; ++bi, ++c) {
                    const uint32_t ab = c & 1u;
                    long long p0 = kProf ? clock64() : 0;
                    wait_parity(accf0 + 8 * ab, (c >> 1) & 1u);
                    umma::fence_after();
                    if (e == 0 && lane == 0) arrive_addr(empty0 + 8 * (c % ST));   // ring stage of block c is free
                    long long p1 = kProf ? clock64() : 0;
                    if (kProf) pr[0] += p1 - p0;
                    if (kExp & 4) {
                        __syncwarp();
                        if (lane == 0) arrive_addr(acce0 + 8 * ab);
                        continue;
                    }
                    uint32_t v[2][32];
                    umma::tmem_ld32_nowait(tbase + ab * kBN, v[0]);
                    umma::tmem_ld32_nowait(tbase + ab * kBN + 32, v[1]);
                    umma::tmem_wait_ld();
                    umma::fence_before();
                    __syncwarp();
                    if (lane == 0) arrive_addr(acce0 + 8 * ab);
                    if (kProf) { const long long t = clock64(); pr[1] += t - p1; p1 = t; }
                    // sign bits: AND of the 64 accumulators in four independent chains
                    // of 16 (s[h] < 0 iff all 16 accumulators of quarter h are < 0)
                    uint32_t sq[4];
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        uint32_t a = v[h >> 1][(h & 1) * 16];
#pragma unroll
                        for (int j = 1; j < 16; ++j) a &= v[h >> 1][(h & 1) * 16 + j];
                        sq[h] = a;
                    }
                    const bool any = rvalid && !((sq[0] & sq[1] & sq[2] & sq[3]) >> 31);   // rare: some acc > +0
                    const bool rare_blk = (kExp & 2) ? false : __any_sync(0xffffffffu, any);
                    if (kProf) { const long long t = clock64(); pr[2] += t - p1; p1 = t; }
                    if (!rare_blk) continue;
                    if (kExp & 32) continue;
                    if (kProf) pr[5] += 1;
                    // survivor columns of this lane (only the quarters with a hit are
                    // expanded), restricted to the window [r, s) and, in the own cell,
                    // to candidates after the query
                    const uint32_t base = (S.wr[i] & ~7u) + bi * kBN + ecol * kCW;
                    unsigned long long m = 0ull;
                    if (any) {
#pragma unroll
                        for (int h = 0; h < 4; ++h) {
                            if (!(sq[h] >> 31)) {
                                uint32_t bits = 0;
#pragma unroll
                                for (int j = 0; j < 16; ++j) bits |= ((~v[h >> 1][(h & 1) * 16 + j]) >> 31) << j;
                                m |= (unsigned long long)bits << (16 * h);
                            }
                        }
                        const uint32_t wr = S.wr[i], wsd = S.ws[i];
                        uint32_t lo = wr > base ? wr - base : 0u;
                        if ((S.nbk[i] >> 31) && qpos + 1 > base + lo) lo = qpos + 1 - base;
                        const uint32_t hi = wsd > base ? min(wsd - base, 64u) : 0u;
                        const unsigned long long keep_hi = hi >= 64 ? ~0ull : ((1ull << hi) - 1ull);
                        const unsigned long long drop_lo = lo >= 64 ? ~0ull : ((1ull << lo) - 1ull);
                        m &= keep_hi & ~drop_lo;
                    }
                    while (__any_sync(0xffffffffu, m != 0ull)) {   // stage the survivors
                        const bool has = m != 0ull;
                        uint32_t cpos = 0;
                        if (has) {
                            cpos = base + (uint32_t)(__ffsll((long long)m) - 1);
                            m &= m - 1;
                        }
                        const unsigned hb = __ballot_sync(0xffffffffu, has);
                        if (has) sv[svn + __popc(hb & lt)] = make_uint2(qpos, cpos);
                        svn += __popc(hb);
                        if (svn >= 32) {   // a full batch: one FP64 decision per lane
                            __syncwarp();
                            long long pd = kProf ? clock64() : 0;
                            if (!(kExp & 16)) npairs += decide_batch<MODE, SYM>(P, A, sv, 32, lane);
                            if (kProf) { pr[4] += clock64() - pd; pr[6] += 1; }
                            __syncwarp();
                            if ((uint32_t)lane < svn - 32) sv[lane] = sv[32 + lane];
                            svn -= 32;
                            __syncwarp();
                        }
                    }
                    if (kProf) pr[3] += clock64() - p1;
                }
            }
            if (svn) {   // the rest of this round's survivors
                __syncwarp();
                npairs += decide_batch<MODE, SYM>(P, A, sv, svn, lane);
            }
            if (kProf && lane == 0)
                for (int k = 0; k < 7; ++k) atomicAdd(&g_umma_prof[k], pr[k]);
        }
        // every role walked the same block sequence
        for (int i = 0; i < nwin; ++i) cnt += S.nbk[i] & 0x7fffffffu;
        __syncthreads();
    }
    umma::fence_before();
    __syncthreads();
    if (warp == 1) umma::tmem_dealloc(tmem, kTCols);
    if (A.mma_tests && tid == 0 && cnt) atomicAdd(A.mma_tests, (unsigned long long)cnt * kM * kBN);

    if (MODE == kCount) {
        unsigned long long x = npairs;
#pragma unroll
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) S.red[warp] = x;
        __syncthreads();
        if (tid == 0) {
            unsigned long long t = 0;
            for (int w = 0; w < kWarps; ++w) t += S.red[w];
            if (t) atomicAdd((unsigned long long*)A.count, t);
            if (part == 0) atomicAdd((unsigned long long*)A.count + 1, (unsigned long long)nq);
        }
    }
}

// Self-test: D[128][128] = A[128][32] . B[128][32]^T (fp16 in, fp32 out) through
// the same smem layout / descriptors / TMEM path as k_join_umma.
__global__ void __launch_bounds__(128) k_umma_selftest(const __half* __restrict__ Ag, const __half* __restrict__ Bg,
                                                        float* __restrict__ D) {
    constexpr int KP = 32;
    __shared__ __align__(128) __half a[kM * KP];
    __shared__ __align__(128) __half b[kN * KP];
    __shared__ uint64_t mbar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < kM * (KP / 8); i += 128) {
        const int row = i / (KP / 8), kc = i % (KP / 8);
        const uint32_t off = umma::tile_off(row, kc * 8, KP);
        *reinterpret_cast<uint4*>(reinterpret_cast<unsigned char*>(a) + off) =
            *reinterpret_cast<const uint4*>(Ag + row * KP + kc * 8);
        *reinterpret_cast<uint4*>(reinterpret_cast<unsigned char*>(b) + off) =
            *reinterpret_cast<const uint4*>(Bg + row * KP + kc * 8);
    }
    if (warp == 0) umma::tmem_alloc(&tbase, kN);
    if (tid == 0) {
        umma::mbar_init(&mbar, 1);
        umma::mbar_fence_init();
    }
    umma::fence_proxy_async();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tmem = tbase;
    if (tid == 0) {
        for (int ks = 0; ks < KP / 16; ++ks)
            umma::mma_f16(tmem, umma::smem_desc(umma::smem_u32(a) + ks * 256, 128, KP * 16),
                          umma::smem_desc(umma::smem_u32(b) + ks * 256, 128, KP * 16), umma::idesc_f16_f32(kM, kN),
                          ks > 0 ? 1u : 0u);
        umma::commit(&mbar);
    }
    umma::mbar_wait(&mbar, 0);
    umma::fence_after();
    for (int c = 0; c < kN; c += 32) {
        float v[32];
        umma::tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)c, v);
        for (int i = 0; i < 32; ++i) D[(32 * warp + lane) * kN + c + i] = v[i];
    }
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc(tmem, kN);
}

template <int KP, int MODE, bool SYM>
int launch_umma_k(const JoinParams& p, const JoinArgs& a, cudaStream_t s) {
    const size_t smem = sizeof(UmmaSmem<KP>);
    // the attribute is per device: one bit per device, set once
    static std::atomic<unsigned long long> attr_done{0};
    int dev = 0;
    GJ_CUDA(cudaGetDevice(&dev));
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(attr_done.load() & bit)) {
        GJ_CUDA(cudaFuncSetAttribute((const void*)k_join_umma<KP, MODE, SYM>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_done.fetch_or(bit);
    }
    k_join_umma<KP, MODE, SYM><<<grid_ctas(a, (int)p.tile_q, kM), kThreads, smem, s>>>(p, a);
    count_launch();
    GJ_CUDA(cudaGetLastError());
    return GJ_OK;
}

template <int KP>
int launch_umma(const JoinParams& p, JoinMode mode, const JoinArgs& a, bool sym, cudaStream_t s) {
    if (a.n_tiles <= 0) return GJ_OK;
    if (mode == kEmit) return sym ? launch_umma_k<KP, kEmit, true>(p, a, s) : launch_umma_k<KP, kEmit, false>(p, a, s);
    return sym ? launch_umma_k<KP, kCount, true>(p, a, s) : launch_umma_k<KP, kCount, false>(p, a, s);
}

}  // namespace

// One 128-query A tile per CTA (index tiles of 256 queries, gj_options.mma_tiles
// = 2, are covered by two CTAs each), MMA depth K = n + 4 rounded up to 16.
int launch_join_umma(const Index* ix, JoinMode mode, const JoinArgs& a, cudaStream_t s) {
    const JoinParams p = join_params(ix);
    const bool sym = ix->opt.symmetric != 0;
    switch (ix->k16) {
        case 16: return launch_umma<16>(p, mode, a, sym, s);
        case 32: return launch_umma<32>(p, mode, a, sym, s);
        case 48: return launch_umma<48>(p, mode, a, sym, s);
        case 64: return launch_umma<64>(p, mode, a, sym, s);
        case 80: return launch_umma<80>(p, mode, a, sym, s);
        case 96: return launch_umma<96>(p, mode, a, sym, s);
        case 112: return launch_umma<112>(p, mode, a, sym, s);
        case 128: return launch_umma<128>(p, mode, a, sym, s);
        default: break;
    }
    set_error("tcgen05 join: MMA depth " + std::to_string(ix->k16) + " not instantiated");
    return GJ_ERR_INVALID;
}

int selftest_umma(const void* A, const void* B, float* D, cudaStream_t s) {
    k_umma_selftest<<<1, 128, 0, s>>>(reinterpret_cast<const __half*>(A), reinterpret_cast<const __half*>(B), D);
    count_launch();
    GJ_CUDA(cudaGetLastError());
    GJ_CUDA(cudaStreamSynchronize(s));
    return GJ_OK;
}

}  // namespace gj

#if GJ_UMMA_EXPERIMENT & 64
// experiment build only: read and reset the phase counters
extern "C" __attribute__((visibility("default"))) int gj_debug_umma_prof(unsigned long long* out) {
    if (cudaMemcpyFromSymbol(out, gj::g_umma_prof, sizeof(gj::g_umma_prof)) != cudaSuccess) return -2;
    static const unsigned long long zero[16] = {};
    cudaMemcpyToSymbol(gj::g_umma_prof, zero, sizeof(zero));
    return 0;
}
#endif
