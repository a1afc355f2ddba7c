// SelfJoinKernel on the 5th-generation tensor cores (tcgen05.mma, TMEM
// accumulators) with the certified distance bound of gj_join_tc.cu and the
// FP64 decision of every surviving pair (B200-first variant of PAPER.md
// Alg. 1 l.596-607; FP64 semantics unchanged).
//
// CTA = one producer warp, one MMA-issuer warp and 4 x EPW epilogue warps per
// 128-query A tile of one cell (M = 128 TMEM lanes); candidates in blocks of
// BN = 256 (default) or 128 rows (see k_join_umma below for the roles).
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

// Timing experiments (tools/ab_prep.sh <name> <bits> builds an A/B copy with
// -DGJ_UMMA_EXPERIMENT=<bits>; the product build has 0): 1 = the epilogue
// releases each accumulator without reading it, 2 = no candidate loads,
// 4 = accumulator reads without the sign test.
#ifndef GJ_UMMA_EXPERIMENT
#define GJ_UMMA_EXPERIMENT 0
#endif
constexpr int kExp = GJ_UMMA_EXPERIMENT;
// bit 64: clock64 phase counters per role (tools/experiments/umma_prof.py reads
// them through gj_debug_umma_prof, which only the experiment build exports)
constexpr bool kProf = (kExp & 64) != 0;
__device__ unsigned long long g_umma_prof[16];

// Waits on the MMA <-> epilogue handoff: suspend-time-hinted try_wait (default)
// or a plain try_wait spin (-DGJ_UMMA_SPIN, timing experiment).
__device__ __forceinline__ void handoff_wait(uint64_t* mbar, uint32_t parity) {
#ifdef GJ_UMMA_SPIN
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAITS_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAITS_%=;\n\t}\n" ::"r"(umma::smem_u32(mbar)), "r"(parity));
#else
    umma::mbar_wait(mbar, parity);
#endif
}

constexpr int kM = 128;         // queries per tile (UMMA M)
constexpr int kN = 128;         // candidates per block (UMMA N)
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

// Tensor memory: MT accumulator blocks of 128 query rows share every
// candidate block (MT = 2: M = 2 x 128 per B operand, so the candidate stream
// through L2 is halved per test).  An accumulator slot is MT x BN columns,
// 256 / BN slots per CTA: MT = 1 uses 256 columns (two CTAs per SM, four
// slots in flight per SM), MT = 2 all 512 (one CTA per SM).
//
// Epilogue: EPW warps per (A tile, 32-lane TMEM quarter), each reading BN / EPW
// columns.  The accumulator read (4 B per candidate test against 2K MMA
// flops) is as expensive as the MMA itself at K = 48, and TMEM read
// throughput grows with the number of reading warps (tools/micro/tmem_ld_bw:
// ~330 B/clk/SM with 8 warps, ~470 with 16), so MT = 1 runs EPW = 2 (16
// epilogue warps per SM).
constexpr int kMaxWin = 512;             // adjacent cells handled per setup round
template <int MT, int EPW>
constexpr int ws_warps() { return 2 + 4 * MT * EPW; }   // 0 producer, 1 MMA issuer, epilogue
// CTAs per SM: two when a CTA's accumulator slots (MT x SL x BN columns) fit
// in half of the SM's 512 TMEM columns.
// (128-column accumulators: four CTAs per SM up to K = 48, three beyond, where
// A + two ring stages no longer fit a quarter of the shared memory)
template <int KP, int BN, int MT, int SL>
constexpr int ws_ctas_per_sm() { return MT * SL * BN <= 128 ? (KP <= 48 ? 4 : 3) : (MT * SL * BN <= 256 ? 2 : 1); }
template <int KP, int BN, int MT, int SL>
constexpr int ws_budget_kb() {
    return ws_ctas_per_sm<KP, BN, MT, SL>() == 4 ? 40
           : ws_ctas_per_sm<KP, BN, MT, SL>() == 3 ? 64
           : (ws_ctas_per_sm<KP, BN, MT, SL>() == 2 ? 96 : 196);
}
// Candidate ring depth: as many BN-row blocks as fit beside the A tiles in
// ~100 KB (two CTAs per SM) or ~200 KB (one) of shared memory, at most 24.
template <int KP, int BN, int MT, int SL>
constexpr int ws_stages() {
    return (ws_budget_kb<KP, BN, MT, SL>() * 1024 - MT * 128 * KP * 2) / (BN * KP * 2) < 24
               ? (ws_budget_kb<KP, BN, MT, SL>() * 1024 - MT * 128 * KP * 2) / (BN * KP * 2)
               : 24;
}

template <int KP, int BN, int MT, int SL, int EPW>
struct WsSmem {
    alignas(128) __half a[MT][kM * KP];                           // queries (A), canonical K-major layout
    alignas(128) __half b[ws_stages<KP, BN, MT, SL>()][BN * KP];   // candidate ring (B)
    uint64_t full[ws_stages<KP, BN, MT, SL>()], empty[ws_stages<KP, BN, MT, SL>()], accf[2 * SL], acce[2 * SL];
    uint32_t tmem_base, item;
    uint32_t wr[kMaxWin], ws[kMaxWin], nbk[kMaxWin];          // window [r, s), blocks (bit 31: own cell)
    uint2 sv[4 * MT * EPW][64];                               // per epilogue warp: staged survivors (qpos, cpos)
    unsigned long long red[ws_warps<MT, EPW>()];
};

// Warp-specialised tcgen05 join.  Per CTA (MT x 128 queries of one cell): the
// epilogue warps build the A tiles (coordinates + augmented columns r_hi,
// r_lo, 1, 1); all warps compute the SORTIDU windows of the adjacent cells
// (thread per cell, union over the CTA's queries); then
//   producer  : per BN-candidate block, one cp.async.bulk of the contiguous
//               grouped-layout rows [8*floor(r/8) + BN b, +BN) into the ring
//               (full/empty mbarriers, transaction bytes);
//   MMA       : one thread, MT x K/16 tcgen05.mma per block (one per 128-query
//               A tile, same B descriptor) into one accumulator slot, commits
//               to empty[stage] and acc_full[slot];
//   epilogue  : 4 x EPW warps per A tile (TMEM lane quarter = warp % 4, column
//               part BN / EPW); tcgen05.ld, AND of the sign bits (survivor iff
//               acc > +0), release the slot, then stage the rare survivors
//               whose candidate lies in [r, s) (and after the query in its own
//               cell) for a lane-parallel FP64 decision.
template <int KP, int BN, int MT, int SL, int EPW, int MODE, bool SYM>
__global__ void __launch_bounds__(32 * ws_warps<MT, EPW>(), ws_ctas_per_sm<KP, BN, MT, SL>())
    k_join_umma(JoinParams P, JoinArgs A, uint32_t* __restrict__ work_counter, uint32_t n_items) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    WsSmem<KP, BN, MT, SL, EPW>& S = *reinterpret_cast<WsSmem<KP, BN, MT, SL, EPW>*>(smem_raw);
    constexpr int NE = 4 * MT * EPW;       // epilogue warps
    constexpr int NW = ws_warps<MT, EPW>();
    constexpr int NT = 32 * NW;
    constexpr int QT = kM * MT;            // queries per CTA
    constexpr uint32_t TCOLS = MT * SL * BN <= 128 ? 128 : (MT * SL * BN <= 256 ? 256 : 512);   // TMEM columns (power of 2)
    constexpr int KS = KP / 16;
    constexpr int ST = ws_stages<KP, BN, MT, SL>();
    constexpr int NACC = SL;
    constexpr int CW = BN / EPW;           // accumulator columns per epilogue warp
    constexpr int NL = CW / 32;            // 32-column TMEM loads per warp and block
    constexpr uint32_t kIdesc = umma::idesc_f16_f32(kM, BN);
    constexpr uint32_t kSBO = KP * 16;
    constexpr uint32_t kBlockBytes = BN * KP * 2;
    static_assert(NL >= 1 && NL <= 8, "epilogue columns per warp");
    static_assert(ws_stages<KP, BN, MT, SL>() >= 1, "candidate ring needs at least one stage");
    // TMEM loads in flight per wait: 4 (128 columns) when one warp reads a whole
    // 256-column row (EPW = 1, 170 registers at two CTAs per SM), else 2
    constexpr int NC = NL >= 8 ? 4 : (NL < 2 ? NL : 2);
    constexpr int NMW = (NL + 1) / 2;       // 64-bit survivor mask words
    // Half-split accumulator (timing experiment, -DGJ_UMMA_HALVES=1; default
    // shape only): each block's MMA is issued as two N = 64 halves, each with
    // its own full / empty barrier pair, so the next block's first half is
    // computed while the epilogue still reads the second half of this one.
    // Parity-green but not faster (DESIGN "What bounds the tcgen05 join").
#ifndef GJ_UMMA_HALVES
#define GJ_UMMA_HALVES 0   // measured 176-188 vs 172-179 ms on expo32: off
#endif
    constexpr bool HS = GJ_UMMA_HALVES && MT == 1 && SL == 1 && EPW == 1 && BN == 128 && NL / NC == 2;
    constexpr int NBAR = HS ? 2 : NACC;
    constexpr uint32_t kIdescH = umma::idesc_f16_f32(kM, BN / 2);

    // One A tile per CTA (MT = 1): persistent CTAs pull (tile, part) items
    // from an atomic counter (TMEM, barriers and the block pipeline set up
    // once; the last items are the lightest, so no static tail).  MT = 2: one
    // item per CTA (the release count depends on the item's A tiles).
    constexpr bool kPersist = MT == 1;
    CtaTile ct = cta_tile(P, A, QT);
    if (!kPersist && ct.nq == 0) return;   // sub-block past the end of the tile's cell
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nsub = kPersist ? 1 : (int)((ct.nq + kM - 1) / kM);   // A tiles holding queries (1..MT)
    const int n_pad = P.n_pad;
    const double eps = P.eps;

    if (warp == 1) umma::tmem_alloc(&S.tmem_base, TCOLS);
    if (tid == 0) {
        for (int i = 0; i < ST; ++i) {
            umma::mbar_init(&S.full[i], 1);
            umma::mbar_init(&S.empty[i], 1);
        }
        for (int i = 0; i < NBAR; ++i) {
            umma::mbar_init(&S.accf[i], 1);
            umma::mbar_init(&S.acce[i], 4 * EPW * nsub);
        }
        umma::mbar_fence_init();
    }
    unsigned long long npairs = 0, queries = 0;
    uint32_t cnt = 0;   // blocks consumed so far (identical sequence in every role, across items)
    for (;;) {   // ------------------------------------------------------- items
    if (kPersist) {
        __syncthreads();   // everyone has read the previous item
        if (tid == 0) S.item = atomicAdd(work_counter, 1u);
        __syncthreads();
        const uint32_t item = S.item;
        if (item >= n_items) break;
        ct = cta_tile_at(P, A, QT, item);
        if (ct.nq == 0) continue;
    }
    const int part = ct.part, split = ct.split;
    const uint32_t g = ct.g, q0 = ct.q0, nq = ct.nq;
    if (tid == 0 && part == 0) queries += nq;
    for (int row = tid - 64; row >= 0 && row < QT; row += 32 * NE) {   // A tiles: thread = query row
        const int sub = row >> 7, rr = row & (kM - 1);
        const bool valid = row < (int)nq;
        unsigned char* a_raw = reinterpret_cast<unsigned char*>(S.a[sub]);
        for (int kc = 0; kc < KP / 8; ++kc) {
            union { uint4 u; __half h[8]; } c;
            c.u = valid ? *reinterpret_cast<const uint4*>(P.pts16 + g16(q0 + row, kc * 8, KP)) : make_uint4(0, 0, 0, 0);
            if (kc == KP / 8 - 1) {   // query-side augmented columns
                query_aug(P.thr16, valid ? P.norm16[q0 + row] : 0.0, valid, c.h[4], c.h[5]);
                c.h[6] = __float2half(1.f);
                c.h[7] = __float2half(1.f);
            }
            *reinterpret_cast<uint4*>(a_raw + umma::tile_off(rr, kc * 8, KP)) = c.u;
        }
    }
    if (SYM && part == 0 && tid < QT) {   // the self pair (q, q)
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

    const double u_lo = P.pts[(size_t)q0 * n_pad + P.u];
    const double u_hi = P.pts[(size_t)(q0 + nq - 1) * n_pad + P.u];
    const uint32_t nb0 = SYM ? P.nbr_self[g] : P.nbr_off[g], nb1 = P.nbr_off[g + 1];
    const int eidx = (warp - 2) >> 2;               // epilogue: (A tile, column part) of this warp
    const int esub = eidx % MT, ecol = eidx / MT;
    const int erow = kM * esub + 32 * (warp & 3) + lane;   // query row; TMEM lane = erow % 128
    for (uint32_t w0 = nb0; w0 < nb1; w0 += kMaxWin) {
        const int nwin = (int)min((uint32_t)kMaxWin, nb1 - w0);
        for (int i = tid; i < nwin; i += NT) {   // windows of this round (thread per adjacent cell)
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
            S.nbk[i] = (s > r ? (s - (r & ~7u) + BN - 1) / BN : 0u) | (diag ? 0x80000000u : 0u);
        }
        __syncthreads();
        if (warp == 0) {   // ---------------- producer
            if (lane == 0) {
                uint32_t c = cnt;
                for (int i = 0; i < nwin; ++i) {
                    const uint32_t nb = S.nbk[i] & 0x7fffffffu, rb = S.wr[i] & ~7u;
                    for (uint32_t bi = 0; bi < nb; ++bi, ++c) {
                        const uint32_t st = c % ST, ph = (c / ST) & 1u;
                        umma::mbar_wait(&S.empty[st], ph ^ 1u);
                        if (kExp & 2) {   // timing experiment: no candidate loads
                            umma::mbar_arrive(&S.full[st]);
                            continue;
                        }
                        umma::mbar_arrive_expect_tx(&S.full[st], kBlockBytes);
                        umma::bulk_g2s(umma::smem_u32(S.b[st]), P.pts16 + (size_t)(rb + bi * BN) * KP, kBlockBytes,
                                       &S.full[st]);
                    }
                }
            }
        } else if (warp == 1) {   // ---------------- MMA issuer
            if (lane == 0) {
                unsigned long long mp[5] = {0, 0, 0, 0, 0};   // wait acce, wait full, mma issue, commits, blocks
                uint32_t c = cnt;
                for (int i = 0; i < nwin; ++i) {
                    const uint32_t nb = S.nbk[i] & 0x7fffffffu;
                    for (uint32_t bi = 0; bi < nb; ++bi, ++c) {
                        const uint32_t st = c % ST, ph = (c / ST) & 1u, ab = c % NACC, aph = (c / NACC) & 1u;
                        const long long m0 = kProf ? clock64() : 0;
                        if (HS) {   // two N = 64 halves, each behind its own release
                            umma::mbar_wait(&S.full[st], ph);
                            const uint32_t b_s = umma::smem_u32(S.b[st]);
                            const uint32_t a_s = umma::smem_u32(S.a[0]);
#pragma unroll
                            for (int hf = 0; hf < 2; ++hf) {
                                umma::mbar_wait(&S.acce[hf], (c & 1u) ^ 1u);
                                umma::fence_after();
#pragma unroll
                                for (int ks = 0; ks < KS; ++ks)
                                    umma::mma_f16(tmem + (uint32_t)(hf * (BN / 2)),
                                                  umma::smem_desc(a_s + ks * 256, 128, kSBO),
                                                  umma::smem_desc(b_s + ks * 256 + hf * 8 * kSBO, 128, kSBO), kIdescH,
                                                  ks > 0 ? 1u : 0u);
                                umma::commit(&S.accf[hf]);
                            }
                            umma::commit(&S.empty[st]);
                            if (kProf) { mp[2] += clock64() - m0; mp[4] += 1; }
                            continue;
                        }
                        handoff_wait(&S.acce[ab], aph ^ 1u);
                        const long long m1 = kProf ? clock64() : 0;
                        umma::mbar_wait(&S.full[st], ph);
                        umma::fence_after();
                        const long long m2 = kProf ? clock64() : 0;
                        const uint32_t b_s = umma::smem_u32(S.b[st]);
#pragma unroll
                        for (int sub = 0; sub < MT; ++sub) {
                            if (sub >= nsub) break;
                            const uint32_t a_s = umma::smem_u32(S.a[sub]);
#pragma unroll
                            for (int ks = 0; ks < KS; ++ks)
                                umma::mma_f16(tmem + (uint32_t)((ab * MT + sub) * BN),
                                              umma::smem_desc(a_s + ks * 256, 128, kSBO),
                                              umma::smem_desc(b_s + ks * 256, 128, kSBO), kIdesc, ks > 0 ? 1u : 0u);
                        }
                        const long long m3 = kProf ? clock64() : 0;
                        // the accumulator's commit first: it is on the MMA -> epilogue
                        // critical path; the ring stage's commit is not
#ifndef GJ_UMMA_EMPTY_BY_EPILOGUE
                        umma::commit(&S.accf[ab]);
                        umma::commit(&S.empty[st]);
#else
                        umma::commit(&S.accf[ab]);
#endif
                        if (kProf) {
                            const long long m4 = clock64();
                            mp[0] += m1 - m0; mp[1] += m2 - m1; mp[2] += m3 - m2; mp[3] += m4 - m3; mp[4] += 1;
                        }
                    }
                }
                if (kProf) for (int k = 0; k < 5; ++k) atomicAdd(&g_umma_prof[8 + k], mp[k]);
            }
        } else if (esub < nsub) {   // ---------------- epilogue
            uint32_t c = cnt;
            const uint32_t qpos = q0 + erow;
            const bool rvalid = erow < (int)nq;
            const uint32_t lane_off = (uint32_t)(32 * (warp & 3)) << 16;
            const unsigned lt = (1u << lane) - 1u;
            // Survivors of the bound are staged per warp and decided 32 at a time
            // (one per lane), so a rare FP64 decision never holds the accumulator
            // pipeline for a full memory round trip per pair.
            uint2* sv = S.sv[warp - 2];
            uint32_t svn = 0;
            unsigned long long pr[4] = {0, 0, 0, 0};   // wait accf, reads -> release, after release, blocks
            unsigned long long rare_cyc = 0, rare_n = 0;
            for (int i = 0; i < nwin; ++i) {
                const uint32_t nbw = S.nbk[i], nb = nbw & 0x7fffffffu, rb = S.wr[i] & ~7u;
                const uint32_t wr = S.wr[i], wsd = S.ws[i];
                const bool diag = (nbw >> 31) != 0;
                for (uint32_t bi = 0; bi < nb; ++bi, ++c) {
                    const uint32_t ab = c % NACC, aph = (c / NACC) & 1u;
                    const long long p0 = kProf ? clock64() : 0;
                    if (!HS) {
                        handoff_wait(&S.accf[ab], aph);
                        umma::fence_after();
                    }
#ifdef GJ_UMMA_EMPTY_BY_EPILOGUE
                    // experiment: the accumulator is complete, so the MMA no longer reads
                    // the ring stage of this block -- free it from here
                    if (warp == 2 && lane == 0) umma::mbar_arrive(&S.empty[c % ST]);
#endif
                    long long p1 = kProf ? clock64() : 0;
                    if (kProf) pr[0] += p1 - p0;
                    const uint32_t tcol = tmem + lane_off + (uint32_t)((ab * MT + esub) * BN + ecol * CW);
                    if ((kExp & 1) && !HS) {   // timing experiment: no accumulator reads
                        __syncwarp();
                        if (lane == 0) umma::mbar_arrive(&S.acce[ab]);
                        continue;
                    }
                    // CW columns in chunks of NC x 32 (NC loads in flight, one wait); the
                    // accumulator is released right after the last wait.  Survivors:
                    // mask bit j of word w = column 64 w + j.
                    unsigned long long mask[NMW];
#pragma unroll
                    for (int w = 0; w < NMW; ++w) mask[w] = 0ull;
#pragma unroll
                    for (int h = 0; h < NL / NC; ++h) {
                        uint32_t v[NC][32];
                        if (HS) {   // half h of the accumulator
                            umma::mbar_wait(&S.accf[h], c & 1u);
                            umma::fence_after();
                        }
#pragma unroll
                        for (int x = 0; x < NC; ++x) umma::tmem_ld32_nowait(tcol + 32 * (NC * h + x), v[x]);
                        umma::tmem_wait_ld();
                        if (HS) {   // release this half at once
                            umma::fence_before();
                            __syncwarp();
                            if (lane == 0) umma::mbar_arrive(&S.acce[h]);
                            if (kProf && h == NL / NC - 1) { const long long t = clock64(); pr[1] += t - p1; p1 = t; }
                        } else if (h == NL / NC - 1) {
                            umma::fence_before();
                            __syncwarp();
                            if (lane == 0) umma::mbar_arrive(&S.acce[ab]);
                            if (kProf) { const long long t = clock64(); pr[1] += t - p1; p1 = t; }
                        }
                        if (kExp & 4) continue;   // timing experiment: reads only
                        // sign bits: balanced AND tree (short dependency chains)
                        uint32_t t[8 * NC];
#pragma unroll
                        for (int k = 0; k < 8 * NC; ++k) {
                            const int e0 = 4 * k;
                            t[k] = v[e0 / 32][e0 % 32] & v[(e0 + 1) / 32][(e0 + 1) % 32] &
                                   v[(e0 + 2) / 32][(e0 + 2) % 32] & v[(e0 + 3) / 32][(e0 + 3) % 32];
                        }
#pragma unroll
                        for (int w = 4 * NC; w >= 1; w >>= 1)
#pragma unroll
                            for (int k = 0; k < w; ++k) t[k] &= t[k + w];
                        if (rvalid && !(t[0] >> 31)) {   // rare: some accumulator > +0
#pragma unroll
                            for (int x = 0; x < NC; ++x)
#pragma unroll
                                for (int y = 0; y < 32; ++y)
                                    if (!(v[x][y] >> 31))
                                        mask[(NC * h + x) >> 1] |= 1ull << (32 * ((NC * h + x) & 1) + y);
                        }
                    }
                    unsigned long long anym = 0ull;
#pragma unroll
                    for (int w = 0; w < NMW; ++w) anym |= mask[w];
                    const bool rare_b = __any_sync(0xffffffffu, anym != 0ull);
                    if (kProf) {
                        pr[3] += 1;
                        if (!rare_b) pr[2] += clock64() - p1;
                    }
                    if (!rare_b) continue;
                    const uint32_t base = rb + bi * BN + ecol * CW;
#pragma unroll
                    for (int hh = 0; hh < NMW; ++hh) {
                        unsigned long long m = mask[hh];
                        while (__any_sync(0xffffffffu, m != 0ull)) {   // stage the survivors in [r, s)
                            uint32_t cpos = 0;
                            bool has = false;
                            if (m) {
                                const int bit = __ffsll((long long)m) - 1;
                                m &= m - 1;
                                cpos = base + 64 * hh + bit;
                                has = !(cpos < wr || cpos >= wsd || (diag && cpos <= qpos));
                            }
                            const unsigned hb = __ballot_sync(0xffffffffu, has);
                            if (has) sv[svn + __popc(hb & lt)] = make_uint2(qpos, cpos);
                            svn += __popc(hb);
                            if (svn >= 32) {   // a full batch: one FP64 decision per lane
                                __syncwarp();
                                npairs += decide_batch<MODE, SYM>(P, A, sv, 32, lane);
                                __syncwarp();
                                if ((uint32_t)lane < svn - 32) sv[lane] = sv[32 + lane];
                                svn -= 32;
                                __syncwarp();
                            }
                        }
                    }
                    if (kProf) { const long long t = clock64(); pr[2] += t - p1; rare_cyc += t - p1; ++rare_n; }
                }
            }
            if (svn) {   // the rest of this round's survivors
                __syncwarp();
                npairs += decide_batch<MODE, SYM>(P, A, sv, svn, lane);
            }
            if (kProf && lane == 0) {
                for (int k = 0; k < 4; ++k) atomicAdd(&g_umma_prof[k], pr[k]);
                atomicAdd(&g_umma_prof[4], rare_cyc);
                atomicAdd(&g_umma_prof[5], rare_n);
            }
        }
        // every role walked the same block sequence
        for (int i = 0; i < nwin; ++i) cnt += S.nbk[i] & 0x7fffffffu;
        __syncthreads();
    }
    if (!kPersist) break;
    }   // items
    umma::fence_before();
    __syncthreads();
    if (warp == 1) umma::tmem_dealloc(S.tmem_base, TCOLS);
    // executed accumulator entries (rows x columns of every block, padding included)
    if (A.mma_tests && tid == 0 && cnt) atomicAdd(A.mma_tests, (unsigned long long)cnt * (kM * nsub) * BN);

    if (MODE == kCount) {
        unsigned long long x = npairs;
#pragma unroll
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) S.red[warp] = x;
        __syncthreads();
        if (tid == 0) {
            unsigned long long t = 0;
            for (int w = 0; w < NW; ++w) t += S.red[w];
            if (t) atomicAdd((unsigned long long*)A.count, t);
            if (queries) atomicAdd((unsigned long long*)A.count + 1, queries);
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

template <int KP, int BN, int MT, int SL, int EPW, int MODE, bool SYM>
int launch_umma_k(const JoinParams& p, const JoinArgs& a, cudaStream_t s) {
    using Smem = WsSmem<KP, BN, MT, SL, EPW>;
    // two CTAs per SM (2 x 256 TMEM columns) or exactly one (512 columns),
    // forced by > 114 KB of shared memory
    constexpr int kCtas = ws_ctas_per_sm<KP, BN, MT, SL>();
    const size_t smem = std::max<size_t>(sizeof(Smem), kCtas == 4 ? 40 * 1024
                                                        : kCtas == 3 ? 58 * 1024
                                                        : (kCtas == 2 ? 80 * 1024 : 120 * 1024));
    static_assert(sizeof(Smem) <= 227 * 1024 / ws_ctas_per_sm<KP, BN, MT, SL>() - 1024, "shared memory");
    // the attribute is per device: one bit per device, set once
    static std::atomic<unsigned long long> attr_done{0};
    int dev = 0;
    GJ_CUDA(cudaGetDevice(&dev));
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(attr_done.load() & bit)) {
        GJ_CUDA(cudaFuncSetAttribute((const void*)k_join_umma<KP, BN, MT, SL, EPW, MODE, SYM>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_done.fetch_or(bit);
    }
    const unsigned total = grid_ctas(a, (int)p.tile_q, kM * MT);
    if (total == 0) return GJ_OK;
    uint32_t* counter = nullptr;
    unsigned grid = total;
    if (MT == 1) {   // persistent CTAs: as many as fit, items from an atomic counter
        static std::atomic<int> sms{0};   // SM count of this device (148 on B200); racing first calls agree
        int n_sm = sms.load();
        if (!n_sm) {
            GJ_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
            sms.store(n_sm);
        }
        grid = std::min<unsigned>(total, (unsigned)(n_sm * kCtas));
        GJ_CUDA(pool_malloc(&counter, sizeof(uint32_t), s));
        GJ_CUDA(cudaMemsetAsync(counter, 0, sizeof(uint32_t), s));
    }
    k_join_umma<KP, BN, MT, SL, EPW, MODE, SYM><<<grid, 32 * ws_warps<MT, EPW>(), smem, s>>>(p, a, counter, total);
    count_launch();
    GJ_CUDA(cudaGetLastError());
    if (counter) GJ_CUDA(cudaFreeAsync(counter, s));
    return GJ_OK;
}

template <int KP, int BN, int MT, int SL, int EPW>
int launch_umma(const JoinParams& p, JoinMode mode, const JoinArgs& a, bool sym, cudaStream_t s) {
    if (a.n_tiles <= 0) return GJ_OK;
    if (mode == kEmit) return sym ? launch_umma_k<KP, BN, MT, SL, EPW, kEmit, true>(p, a, s)
                                  : launch_umma_k<KP, BN, MT, SL, EPW, kEmit, false>(p, a, s);
    return sym ? launch_umma_k<KP, BN, MT, SL, EPW, kCount, true>(p, a, s)
               : launch_umma_k<KP, BN, MT, SL, EPW, kCount, false>(p, a, s);
}

// MMA depth dispatch; KMAX bounds the instantiated depths (a configuration
// whose shared memory cannot hold a deeper ring is not instantiated beyond it).
template <int BN, int MT, int SL, int EPW, int KMAX = 128>
int launch_umma_kp(const Index* ix, const JoinParams& p, JoinMode mode, const JoinArgs& a, bool sym, cudaStream_t s) {
    switch (ix->k16) {
        case 16: return launch_umma<16, BN, MT, SL, EPW>(p, mode, a, sym, s);
        case 32: return launch_umma<32, BN, MT, SL, EPW>(p, mode, a, sym, s);
        case 48: return launch_umma<48, BN, MT, SL, EPW>(p, mode, a, sym, s);
        case 64: if constexpr (KMAX >= 64) return launch_umma<64, BN, MT, SL, EPW>(p, mode, a, sym, s); break;
        case 80: if constexpr (KMAX >= 80) return launch_umma<80, BN, MT, SL, EPW>(p, mode, a, sym, s); break;
        case 96: if constexpr (KMAX >= 96) return launch_umma<96, BN, MT, SL, EPW>(p, mode, a, sym, s); break;
        case 112: if constexpr (KMAX >= 112) return launch_umma<112, BN, MT, SL, EPW>(p, mode, a, sym, s); break;
        case 128: if constexpr (KMAX >= 128) return launch_umma<128, BN, MT, SL, EPW>(p, mode, a, sym, s); break;
        default: break;
    }
    set_error("tcgen05 join: MMA depth " + std::to_string(ix->k16) + " not instantiated for this configuration");
    return GJ_ERR_INVALID;
}

}  // namespace

int launch_join_umma(const Index* ix, JoinMode mode, const JoinArgs& a, cudaStream_t s) {
    // GJ_UMMA_WS=1 selects the persistent kernel (gj_join_ws.cu; same pair set,
    // measured at parity with this one on expo32 / expo16, 5 % faster at K = 80,
    // 13 % slower on uniform16 -- DESIGN "Persistent tcgen05 join"); read once.
    static const bool persistent = [] {
        const char* e = getenv("GJ_UMMA_WS");
        return e && atoi(e) != 0;
    }();
    if (persistent && ix->tile_q == kM) return launch_join_ws(ix, mode, a, s);
    const JoinParams p = join_params(ix);
    const bool sym = ix->opt.symmetric != 0;
    // A tiles per CTA = tile_q / 128.  MT = 1 (default): 128-candidate blocks,
    // one 128-column accumulator per CTA and FOUR CTAs per SM (4 x 128 TMEM
    // columns): four independent MMA -> epilogue pipelines per SM, so one CTA's
    // epilogue (4 warps, 128 columns each) overlaps three others' MMAs.
    // Alternatives measured slower on expo32 (DESIGN "What bounds the tcgen05
    // join"): 256-candidate blocks with two CTAs per SM; two 128-column slots
    // per CTA with 8 epilogue warps and two CTAs per SM (round 2: 185-196 vs
    // 177-186 ms); 256-column slots, one CTA per SM, 16 epilogue warps.
    if (ix->tile_q / kM == 2) return launch_umma_kp<128, 2, 2, 1>(ix, p, mode, a, sym, s);
    // 128-candidate blocks with one accumulator per CTA: four CTAs per SM while
    // A + two ring stages fit a quarter of the SM's shared memory (K <= 48),
    // three up to K = 96 (3M x 64-d exponential, K = 80: 885 vs 899 ms with
    // 256-candidate blocks and two CTAs per SM); K = 112, 128: 256-candidate
    // blocks, two CTAs per SM
    // (four CTAs per SM with 8 epilogue warps of 64 columns each does not fit:
    // 48 registers per thread cannot hold a 32-column TMEM load, ptxas C7602)
    if (ix->k16 <= 48) return launch_umma_kp<128, 1, 1, 1, 48>(ix, p, mode, a, sym, s);
    if (ix->k16 <= 96) return launch_umma_kp<128, 1, 1, 1, 96>(ix, p, mode, a, sym, s);
    return launch_umma_kp<256, 1, 1, 2>(ix, p, mode, a, sym, s);
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
