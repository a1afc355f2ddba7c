// SelfJoinKernel on the tcgen05 tensor cores, persistent form (round 2,
// opt-in with GJ_UMMA_WS=1): one CTA per SM owns all 512 TMEM columns as four
// 128 x 128 fp32 accumulator slots and walks a dynamically scheduled list of
// (query tile, part) work items -- PAPER.md Alg. 1 l.596-607 with the
// certified tensor-core bound of gj_index.cu (tc_threshold_from) and the FP64
// decision of every surviving pair, so the pair set is the FP64 kernel's.
//
// Roles (24 warps = 6 warpgroups, 768 threads, 1 CTA per SM; setmaxnreg gives
// the two role warpgroups 48 registers and the four epilogue ones 96):
//   warp 0        producer: one cp.async.bulk per 128-candidate block into a
//                 ring of ST stages (full / empty mbarriers, transaction bytes)
//   warps 1..kIss MMA issuers: issuer w issues the blocks c = w (mod kIss),
//                 K/16 tcgen05.mma (M = N = 128) into slot c % 4, commits to
//                 empty[stage] and accf[slot].  Several issuers because a
//                 thread that touches shared memory (a barrier wait, even an
//                 LDS) stalls until its own MMAs drain (tools/micro/umma_rate.cu:
//                 one issuer with a per-block handshake reaches ~900 TFLOP/s,
//                 four ~1700-2100)
//   warp kIss+1   setup: item fetch (global atomic counter), A tile with the
//                 query-side augmented columns, SORTIDU windows of the
//                 adjacent cells, self pairs -- one item ahead (two buffers)
//   kDec warps    deciders: drain a survivor-pair queue in ticket order, FP64
//                 test of 64 pairs per pass (two per lane), emission
//   warps 8..23   epilogue: EG groups of 16 / EG warps; group g reads the
//                 blocks c = g (mod EG), warp w its TMEM lane quarter w % 4,
//                 32 EG columns: both 32-column loads in flight, slot released,
//                 then the sign-bit AND; a lane with a non-negative accumulator
//                 turns its 32 columns into a survivor mask (funnel shifts),
//                 applies the candidate window and queues the pairs
//                 (one atomicAdd per lane, one 64-bit store per pair).
// Measured (1 B200, expo32): 176-182 ms per join vs 171-181 for the per-tile
// kernel; the sign test and the slot handshake bound it (DESIGN "Persistent
// tcgen05 join").
#include <stdlib.h>

#include <algorithm>
#include <atomic>
#include <string>

#include "gj_internal.cuh"
#include "gj_umma.cuh"

namespace gj {
namespace {

constexpr int kM = 128;        // queries per work item (UMMA M, TMEM lanes)
constexpr int kBN = 128;       // candidates per block (UMMA N)
constexpr int kSlots = 4;      // accumulator slots: 4 x 128 = all 512 TMEM columns
constexpr int kCap = 512;      // adjacent-cell windows per item fill
#ifndef GJ_WS_ISS
#define GJ_WS_ISS 4
#endif
constexpr int kIss = GJ_WS_ISS;   // MMA issuer warps (warp 1 + w issues the blocks c = w mod kIss)
constexpr int kDec = 6 - kIss;    // decider warps (the role warps fill two warpgroups)
constexpr int kPQ = 4096 / kDec;  // survivor-pair queue entries per decider
constexpr int kEpi = 16;          // epilogue warps (four warpgroups)
constexpr int kWS = 1 + kIss;  // setup warp
constexpr int kWD = kWS + 1;   // first decider warp
constexpr int kW0 = kWD + kDec;  // first epilogue warp
#ifndef GJ_WS_NC
#define GJ_WS_NC 2
#endif
// 8 role warps drop to kRegLow, the 16 epilogue warps rise to kRegHigh (two
// 32-column TMEM loads in flight plus their survivor pushes need ~90; the
// launch allots 80 to each of 768 threads).  The increase draws on the CTA's
// own allocation, not the SM's: 2 x 128 x 48 + 4 x 128 x 96 = 768 x 80
// (a split that needs more never completes its setmaxnreg.inc).
constexpr int kRegLow = 48, kRegHigh = 96;
constexpr int kWarps = kW0 + kEpi;
constexpr int kThreads = 32 * kWarps;

struct ItemBuf {
    uint32_t nwin;   // windows in this fill; kEnd = no more work
    uint32_t q0, nq, pad_;
    uint32_t wr[kCap], ws[kCap], nbk[kCap];   // window [wr, ws), blocks (bit 31: own cell)
};
constexpr uint32_t kEnd = 0xffffffffu;

// A survivor pair in a decider queue: one 64-bit word (single-copy atomic in
// shared memory, so no fence is needed between writer and reader), query and
// candidate positions in the low 31 bits of each half, bit 31 of both = the
// round parity of the ticket (ticket / kPQ) & 1.  Entries start with parity 1,
// and a producer never runs a full round ahead of the decider, so an entry
// holds the expected ticket iff its parity bit matches.
__device__ __forceinline__ unsigned long long pair_word(uint32_t q, uint32_t c, uint32_t par) {
    return ((unsigned long long)(c | (par << 31)) << 32) | (q | (par << 31));
}

template <int KP>
constexpr int ps_stages() {
    // shared memory: 227 KB - A tiles - queues - item buffers - ~4 KB of barriers / flags / staging
    return std::min<int>(12, (232448 - 2 * kM * KP * 2 - kDec * kPQ * 8 - 2 * (int)sizeof(ItemBuf) - 4096) /
                                 (kBN * KP * 2));
}

template <int KP>
struct PsSmem {
    alignas(128) __half a[2][kM * KP];                    // query tiles (A), canonical K-major layout
    alignas(128) __half b[ps_stages<KP>()][kBN * KP];     // candidate ring (B)
    unsigned long long pq[kDec][kPQ];   // survivor pairs, one single-consumer queue per decider
    ItemBuf it[2];
    uint64_t full[ps_stages<KP>()], empty[ps_stages<KP>()], accf[kSlots], acce[kSlots], itf[2], ite[2];
    uint32_t q_tail[kDec], q_head[kDec];   // tickets allocated / consumed
    uint32_t epi_done, tmem_base;
};

// FP64 decision of one pair: the FP64 kernel's arithmetic (gj_join.cu).
__device__ __forceinline__ double dist2_fp64(const double* __restrict__ a, const double* __restrict__ b, int n_pad) {
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

// FP64 decision of up to two queued survivor pairs per lane and emission of
// the pairs inside eps (both orders when symmetric) with one warp-aggregated
// atomic.  Returns this lane's count contribution (kCount).
template <int MODE, bool SYM>
__device__ __forceinline__ unsigned long long decide2(const JoinParams& P, const JoinArgs& A, uint2 e0, bool h0, uint2 e1,
                                                      bool h1, int lane) {
    constexpr unsigned long long kMul = SYM ? 2ull : 1ull;
    const int n_pad = P.n_pad;
    const double d0 = h0 ? dist2_fp64(P.pts + (size_t)e0.x * n_pad, P.pts + (size_t)e0.y * n_pad, n_pad) : 0.0;
    const double d1 = h1 ? dist2_fp64(P.pts + (size_t)e1.x * n_pad, P.pts + (size_t)e1.y * n_pad, n_pad) : 0.0;
    const bool ok0 = h0 && d0 <= P.eps2, ok1 = h1 && d1 <= P.eps2;
    if (MODE != kEmit) return (ok0 ? kMul : 0ull) + (ok1 ? kMul : 0ull);
    const unsigned m0 = __ballot_sync(0xffffffffu, ok0), m1 = __ballot_sync(0xffffffffu, ok1);
    if (!(m0 | m1)) return 0ull;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd((unsigned long long*)A.count, kMul * (unsigned long long)(__popc(m0) + __popc(m1)));
    base = __shfl_sync(0xffffffffu, base, 0);
    const unsigned lt = (1u << lane) - 1u;
    uint2* out = reinterpret_cast<uint2*>(A.out);
    if (ok0) {
        const unsigned long long at = base + kMul * (unsigned long long)__popc(m0 & lt);
        if (at + kMul <= A.cap) {
            const uint32_t qi = P.orig[e0.x], ci = P.orig[e0.y];
            out[at] = make_uint2(qi, ci);
            if (SYM) out[at + 1] = make_uint2(ci, qi);
        }
    }
    if (ok1) {
        const unsigned long long at = base + kMul * (unsigned long long)(__popc(m0) + __popc(m1 & lt));
        if (at + kMul <= A.cap) {
            const uint32_t qi = P.orig[e1.x], ci = P.orig[e1.y];
            out[at] = make_uint2(qi, ci);
            if (SYM) out[at + 1] = make_uint2(ci, qi);
        }
    }
    return 0ull;
}

// Phase profile (timing experiment: -DGJ_WS_PROF=1, read by gj_debug_ws_prof,
// which only that build exports): clock64 cycles per role and phase, summed
// over all CTAs (slots listed at gj_debug_ws_prof).
#ifndef GJ_WS_PROF
#define GJ_WS_PROF 0
#endif
constexpr bool kProf = GJ_WS_PROF != 0;
// Timing experiments (-DGJ_WS_EXP=bits, A/B builds only; results are wrong):
// 1 = the epilogue releases each slot without reading it, 2 = no candidate
// loads (the producer arrives without a copy), 4 = no survivor-chunk pushes,
// 8 = the deciders consume the queue but make no FP64 decisions.
#ifndef GJ_WS_EXP
#define GJ_WS_EXP 0
#endif
constexpr int kExp = GJ_WS_EXP;
__device__ unsigned long long g_ws_prof[32];
struct Prof {
    unsigned long long p[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long t = 0;
    __device__ __forceinline__ void start() { if (kProf) t = clock64(); }
    __device__ __forceinline__ void mark(int k) {
        if (kProf) { const long long n = clock64(); p[k] += (unsigned long long)(n - t); t = n; }
    }
    __device__ __forceinline__ void add(int k, unsigned long long v) { if (kProf) p[k] += v; }
    __device__ __forceinline__ void flush(int base, int n) {
        if (kProf) for (int k = 0; k < n; ++k) if (p[k]) atomicAdd(&g_ws_prof[base + k], p[k]);
    }
};

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) { return *reinterpret_cast<const volatile uint32_t*>(p); }
__device__ __forceinline__ void st_volatile(uint32_t* p, uint32_t v) { *reinterpret_cast<volatile uint32_t*>(p) = v; }

// a & b & c as one LOP3 the compiler cannot re-associate (it turns a
// balanced C++ AND tree into a 16-deep dependent chain)
__device__ __forceinline__ uint32_t and3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0x80;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
// AND of the 32 accumulators' bits (sign bit set in the result iff all are
// negative): 16 LOP3 in a tree of depth 4.
__device__ __forceinline__ uint32_t and32(const uint32_t (&v)[32]) {
    uint32_t t[11];
#pragma unroll
    for (int k = 0; k < 10; ++k) t[k] = and3(v[3 * k], v[3 * k + 1], v[3 * k + 2]);
    t[10] = v[30] & v[31];
    const uint32_t x0 = and3(t[0], t[1], t[2]), x1 = and3(t[3], t[4], t[5]), x2 = and3(t[6], t[7], t[8]);
    return and3(x0, x1, x2) & and3(t[9], t[10], 0xffffffffu);
}

template <int KP, int EG, int MODE, bool SYM>
__global__ void __launch_bounds__(kThreads, 1)
    k_join_ws(JoinParams P, JoinArgs A, uint32_t* __restrict__ work_counter, uint32_t n_items) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    PsSmem<KP>& S = *reinterpret_cast<PsSmem<KP>*>(smem_raw);
    constexpr int ST = ps_stages<KP>();
    constexpr int KS = KP / 16;
    constexpr int WPG = kEpi / EG;          // epilogue warps per group
    constexpr int CW = 512 * EG / kEpi;     // accumulator columns per epilogue warp
    constexpr int NL = CW / 32;             // 32-column TMEM loads per warp and block
    constexpr int NC = GJ_WS_NC < NL ? GJ_WS_NC : NL;   // 32-column loads in flight per wait
    constexpr uint32_t kIdesc = umma::idesc_f16_f32(kM, kBN);
    constexpr uint32_t kSBO = KP * 16;
    constexpr uint32_t kBlockBytes = kBN * KP * 2;
    static_assert(ST >= 2, "candidate ring needs two stages");
    static_assert(sizeof(PsSmem<KP>) <= 232448, "shared memory");
    static_assert(kEpi % (4 * EG) == 0 && (EG == 1 || EG == 2 || EG == 4) && CW <= 256, "epilogue groups");

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n_pad = P.n_pad;
    if (warp == 1) umma::tmem_alloc(&S.tmem_base, 512);   // warp 1 also frees it
    if (tid == 0) {
        for (int i = 0; i < ST; ++i) {
            umma::mbar_init(&S.full[i], 1);
            umma::mbar_init(&S.empty[i], 1);
        }
        for (int i = 0; i < kSlots; ++i) {
            umma::mbar_init(&S.accf[i], 1);
            umma::mbar_init(&S.acce[i], WPG);
        }
        for (int i = 0; i < 2; ++i) {
            umma::mbar_init(&S.itf[i], 1);
            umma::mbar_init(&S.ite[i], kEpi + 1 + kIss);   // epilogue warps + producer + the issuers' commits
        }
        for (int d = 0; d < kDec; ++d) S.q_tail[d] = S.q_head[d] = 0;
        S.epi_done = 0;
        umma::mbar_fence_init();
    }
    for (int e = tid; e < kDec * kPQ; e += kThreads) S.pq[e / kPQ][e % kPQ] = pair_word(0u, 0u, 1u);
    umma::mbar_fence_init();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tmem = S.tmem_base;
    static_assert(kW0 == 8 && kPQ >= 64 + 32 && kThreads == 768 && 2 * 128 * kRegLow + 4 * 128 * kRegHigh <= 768 * 80,
                  "register split works on whole warpgroups");
    unsigned long long npairs = 0;
    Prof pf;
    const long long t_start = kProf ? clock64() : 0;
    pf.start();

    if (warp < kW0) {   // role warpgroups 0 and 1: give registers to the epilogue
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kRegLow));
        if (warp == kWS) {   // ---------------------------------------------- setup
            uint32_t it = 0;
            unsigned long long blocks = 0, queries = 0;
            for (;;) {
                uint32_t item = 0;
                if (lane == 0) item = atomicAdd(work_counter, 1u);
                item = __shfl_sync(0xffffffffu, item, 0);
                if (item >= n_items) {   // end marker
                    const uint32_t ib = it & 1u;
                    umma::mbar_wait(&S.ite[ib], ((it >> 1) & 1u) ^ 1u);
                    if (lane == 0) {
                        S.it[ib].nwin = kEnd;
                        umma::mbar_arrive(&S.itf[ib]);
                    }
                    break;
                }
                // item -> (tile position m, part of split)
                uint32_t m, part, split;
                if (A.part_off) {
                    uint32_t lo = 0, hi = (uint32_t)A.n_tiles;   // last m with part_off[m] <= item
                    while (hi - lo > 1) {
                        const uint32_t mid = (lo + hi) >> 1;
                        if (A.part_off[mid] <= item) lo = mid; else hi = mid;
                    }
                    m = lo;
                    part = item - A.part_off[m];
                    split = A.part_off[m + 1] - A.part_off[m];
                } else {
                    split = A.split > 1 ? (uint32_t)A.split : 1u;
                    part = item % split;
                    m = item / split;
                }
                const uint32_t tile = P.tile_order[tile_pos(A, (int64_t)m)];
                const uint32_t g = P.tile_cell[tile], q0 = P.tile_q0[tile];
                const uint32_t nq = min((uint32_t)kM, P.cell_start[g + 1] - q0);
                const double u_lo = P.pts[(size_t)q0 * n_pad + P.u];
                const double u_hi = P.pts[(size_t)(q0 + nq - 1) * n_pad + P.u];
                const uint32_t nb0 = SYM ? P.nbr_self[g] : P.nbr_off[g], nb1 = P.nbr_off[g + 1];
                if (part == 0) {
                    queries += nq;
                    if (SYM) {   // the self pairs (q, q)
                        if (MODE == kEmit) {
                            for (uint32_t r0 = 0; r0 < nq; r0 += 32) {
                                const bool active = r0 + lane < nq;
                                const unsigned mk = __ballot_sync(0xffffffffu, active);
                                unsigned long long base = 0;
                                if (lane == 0) base = atomicAdd((unsigned long long*)A.count, (unsigned long long)__popc(mk));
                                base = __shfl_sync(0xffffffffu, base, 0);
                                if (active) {
                                    const unsigned long long at = base + __popc(mk & ((1u << lane) - 1u));
                                    const uint32_t qid = P.orig[q0 + r0 + lane];
                                    if (at < A.cap) reinterpret_cast<uint2*>(A.out)[at] = make_uint2(qid, qid);
                                }
                            }
                        } else if (lane == 0) {
                            npairs += nq;
                        }
                    }
                }
                uint32_t w0 = nb0;
                do {   // one fill per kCap adjacent cells (at least one per item)
                    const uint32_t ib = it & 1u;
                    pf.mark(1);
                    umma::mbar_wait(&S.ite[ib], ((it >> 1) & 1u) ^ 1u);
                    pf.mark(0);
                    ItemBuf& B = S.it[ib];
                    // A tile: thread = query row; coordinates + (r_hi, r_lo, 1, 1)
                    unsigned char* a_raw = reinterpret_cast<unsigned char*>(S.a[ib]);
                    for (int row = lane; row < kM; row += 32) {
                        const bool valid = row < (int)nq;
                        const double nrm = valid ? P.norm16[q0 + row] : 0.0;
    #pragma unroll
                        for (int kc = 0; kc < KP / 8; ++kc) {
                            union { uint4 u; __half h[8]; } c;
                            c.u = valid ? *reinterpret_cast<const uint4*>(P.pts16 + g16(q0 + row, kc * 8, KP))
                                        : make_uint4(0, 0, 0, 0);
                            if (kc == KP / 8 - 1) {
                                query_aug(P.thr16, nrm, valid, c.h[4], c.h[5]);
                                c.h[6] = __float2half(1.f);
                                c.h[7] = __float2half(1.f);
                            }
                            *reinterpret_cast<uint4*>(a_raw + umma::tile_off(row, kc * 8, KP)) = c.u;
                        }
                    }
                    // SORTIDU windows of the adjacent cells (lane per cell)
                    const uint32_t nwin = min((uint32_t)kCap, nb1 > w0 ? nb1 - w0 : 0u);
                    for (uint32_t i = lane; i < nwin; i += 32) {
                        const uint32_t Bc = P.nbr[w0 + i];
                        uint32_t r = P.cell_start[Bc], s = P.cell_start[Bc + 1];
                        if (P.sortidu) {
                            uint32_t lo = r, hi = s;
                            while (lo < hi) {   // first r with u_lo - r(u) <= eps
                                const uint32_t mid = (lo + hi) >> 1;
                                if (u_lo - P.pts[(size_t)mid * n_pad + P.u] <= P.eps) hi = mid; else lo = mid + 1;
                            }
                            const uint32_t rr = lo;
                            hi = s;
                            while (lo < hi) {   // first s with s(u) - u_hi > eps
                                const uint32_t mid = (lo + hi) >> 1;
                                if (P.pts[(size_t)mid * n_pad + P.u] - u_hi > P.eps) hi = mid; else lo = mid + 1;
                            }
                            r = rr;
                            s = lo;
                        }
                        const bool diag = SYM && Bc == g;
                        if (diag) r = max(r, q0 + 1);
                        if (split > 1 && s > r) {
                            const uint64_t len = s - r;
                            s = r + (uint32_t)(len * (part + 1) / split);
                            r = r + (uint32_t)(len * part / split);
                        }
                        const uint32_t nb = s > r ? (s - (r & ~7u) + kBN - 1) / kBN : 0u;
                        B.wr[i] = r;
                        B.ws[i] = s;
                        B.nbk[i] = nb | (diag ? 0x80000000u : 0u);
                        blocks += nb;
                    }
                    if (lane == 0) {
                        B.nwin = nwin;
                        B.q0 = q0;
                        B.nq = nq;
                    }
                    umma::fence_proxy_async();   // A was written by the generic proxy, the MMA reads it
                    __syncwarp();
                    if (lane == 0) umma::mbar_arrive(&S.itf[ib]);
                    pf.add(2, 1);
                    pf.add(3, nwin);
                    ++it;
                    w0 += kCap;
                } while (w0 < nb1);
            }
            // executed accumulator entries (every block is 128 x 128) and processed queries
            for (int o = 16; o; o >>= 1) blocks += __shfl_xor_sync(0xffffffffu, blocks, o);
            if (lane == 0) {
                if (A.mma_tests && blocks) atomicAdd(A.mma_tests, blocks * (unsigned long long)(kM * kBN));
                if (MODE == kCount && queries) atomicAdd((unsigned long long*)A.count + 1, queries);
                pf.mark(1);
                pf.flush(8, 4);   // 8 wait ite, 9 busy, 10 fills, 11 windows
            }
        } else if (warp == 0) {   // ------------------------------------------ producer
            if (lane == 0) {
                uint32_t c = 0, it = 0;
                for (;; ++it) {
                    const uint32_t ib = it & 1u;
                    pf.mark(2);
                    umma::mbar_wait(&S.itf[ib], (it >> 1) & 1u);
                    pf.mark(1);
                    const ItemBuf& B = S.it[ib];
                    const uint32_t nwin = B.nwin;
                    if (nwin == kEnd) break;
                    for (uint32_t i = 0; i < nwin; ++i) {
                        const uint32_t nb = B.nbk[i] & 0x7fffffffu, rb = B.wr[i] & ~7u;
                        for (uint32_t bi = 0; bi < nb; ++bi, ++c) {
                            const uint32_t st = c % ST;
                            pf.mark(2);
                            umma::mbar_wait(&S.empty[st], ((c / ST) & 1u) ^ 1u);
                            pf.mark(0);
                            if (kExp & 2) {
                                umma::mbar_arrive(&S.full[st]);
                                continue;
                            }
                            umma::mbar_arrive_expect_tx(&S.full[st], kBlockBytes);
                            umma::bulk_g2s(umma::smem_u32(S.b[st]), P.pts16 + (size_t)(rb + bi * kBN) * KP, kBlockBytes,
                                           &S.full[st]);
                        }
                    }
                    umma::mbar_arrive(&S.ite[ib]);
                }
                pf.flush(6, 2);   // 6 wait empty, 7 wait itf
            }
        } else if (warp <= kIss) {   // --------------------------------------- MMA issuers
            // Issuer w = warp - 1 issues the blocks c = w (mod kIss), block c into
            // slot c % 4: a thread that waits on a barrier (or touches shared memory
            // at all) stalls until its own MMAs drain (tools/micro/umma_rate.cu), so
            // several issuers keep the tensor pipe busy while one of them waits.
            const uint32_t wi = (uint32_t)(warp - 1);
            if (lane == 0) {
                uint32_t c = 0, it = 0;
                for (;; ++it) {
                    const uint32_t ib = it & 1u;
                    pf.mark(3);
                    umma::mbar_wait(&S.itf[ib], (it >> 1) & 1u);
                    pf.mark(0);
                    const ItemBuf& B = S.it[ib];
                    const uint32_t nwin = B.nwin;
                    if (nwin == kEnd) break;
                    pf.add(5, 1);
                    umma::fence_after();
                    const uint32_t a_s = umma::smem_u32(S.a[ib]);
                    for (uint32_t i = 0; i < nwin; ++i) {
                        const uint32_t nb = B.nbk[i] & 0x7fffffffu;
                        for (uint32_t bi = (wi + kIss - c % kIss) % kIss; bi < nb; bi += kIss) {
                            const uint32_t cc = c + bi, st = cc % ST, slot = cc % kSlots;
                            pf.mark(3);
                            umma::mbar_wait(&S.acce[slot], ((cc / kSlots) & 1u) ^ 1u);
                            pf.mark(1);
                            umma::mbar_wait(&S.full[st], (cc / ST) & 1u);
                            pf.mark(2);
                            pf.add(4, 1);
                            umma::fence_after();
                            const uint32_t b_s = umma::smem_u32(S.b[st]);
    #pragma unroll
                            for (int ks = 0; ks < KS; ++ks)
                                umma::mma_f16(tmem + slot * kBN, umma::smem_desc(a_s + ks * 256, 128, kSBO),
                                              umma::smem_desc(b_s + ks * 256, 128, kSBO), kIdesc, ks > 0 ? 1u : 0u);
                            umma::commit(&S.accf[slot]);
                            umma::commit(&S.empty[st]);
                        }
                        c += nb;
                    }
                    umma::commit(&S.ite[ib]);   // arrives once every MMA reading A[ib] has completed
                }
                pf.mark(3);
                if (wi == 0) pf.flush(0, 6);   // 0 wait itf, 1 wait acce, 2 wait full, 3 issue + commits, 4 blocks / 4, 5 fills
            }
        } else {   // --------------------------------------------------------- deciders
            // Queue dq in ticket order, 64 pairs per pass (two per lane): FP64 test,
            // emission.  A pass waits for 64 queued pairs unless the epilogue is done.
            const int dq = warp - kWD;
            for (uint32_t hd = 0;;) {
                uint32_t avail = 0;
                pf.mark(2);
                if (lane == 0) {
                    for (;;) {
                        const uint32_t tl = ld_volatile(&S.q_tail[dq]);
                        if (tl - hd >= 64u) { avail = 64u; break; }
                        if (ld_volatile(&S.epi_done) == (uint32_t)kEpi) {
                            __threadfence_block();
                            avail = ld_volatile(&S.q_tail[dq]) - hd;
                            avail = avail > 64u ? 64u : avail;
                            break;
                        }
                        __nanosleep(64);
                    }
                    pf.mark(0);
                }
                avail = __shfl_sync(0xffffffffu, avail, 0);
                if (!avail) break;
                uint2 e[2];
                bool has[2];
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const uint32_t i = lane + 32u * k, t = hd + i;
                    has[k] = i < avail;
                    e[k] = make_uint2(0u, 0u);
                    if (has[k]) {   // allocated; wait until written (parity of its round)
                        const volatile unsigned long long* w = &S.pq[dq][t % kPQ];
                        const uint32_t par = (t / kPQ) & 1u;
                        unsigned long long x = *w;
                        while (((uint32_t)x >> 31) != par) x = *w;
                        e[k] = make_uint2((uint32_t)x & 0x7fffffffu, (uint32_t)(x >> 32) & 0x7fffffffu);
                    }
                }
                __syncwarp();   // every lane has read its entries
                hd += avail;
                if (lane == 0) st_volatile(&S.q_head[dq], hd);
                pf.mark(1);
                pf.add(4, avail);
                pf.add(5, 1);
                if (!(kExp & 8)) npairs += decide2<MODE, SYM>(P, A, e[0], has[0], e[1], has[1], lane);
                pf.mark(3);
            }
            pf.mark(2);
            if (lane == 0) pf.flush(20, 6);   // 20 idle, 21 read pairs, 22 -, 23 FP64 decisions, 24 pairs, 25 passes
        }
    } else {   // ----------------------------------------------------------------- epilogue
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kRegHigh));
        const int j = warp - kW0;
        const uint32_t grp = (uint32_t)(j / WPG);
        const int cpart = (j % WPG) / 4;
        const int quarter = warp & 3;
        const int erow = 32 * quarter + lane;
        const uint32_t lane_off = (uint32_t)(32 * quarter) << 16;
        const int dq = warp % kDec;   // survivor queue (decider) of this warp
        uint32_t c = 0;
        for (uint32_t it = 0;; ++it) {
            const uint32_t ib = it & 1u;
            pf.mark(3);
            umma::mbar_wait(&S.itf[ib], (it >> 1) & 1u);
            pf.mark(0);
            const ItemBuf& B = S.it[ib];
            const uint32_t nwin = B.nwin;
            if (nwin == kEnd) break;
            const uint32_t qpos = B.q0 + erow;
            const bool rvalid = erow < (int)B.nq;
            for (uint32_t i = 0; i < nwin; ++i) {
                const uint32_t nbw = B.nbk[i], nb = nbw & 0x7fffffffu;
                const uint32_t wr = B.wr[i], wsd = B.ws[i] | (nbw & 0x80000000u), rb = wr & ~7u;
                for (uint32_t bi = (grp + EG - c % EG) % EG; bi < nb; bi += EG) {
                    const uint32_t cc = c + bi, slot = cc % kSlots;
                    pf.mark(3);
                    umma::mbar_wait(&S.accf[slot], (cc / kSlots) & 1u);
                    pf.mark(1);
                    pf.add(6, 1);
                    umma::fence_after();
                    const uint32_t tcol = tmem + lane_off + slot * kBN + cpart * CW;
                    if (kExp & 1) {
                        umma::fence_before();
                        __syncwarp();
                        if (lane == 0) umma::mbar_arrive(&S.acce[slot]);
                        continue;
                    }
#pragma unroll
                    for (int h = 0; h < NL / NC; ++h) {
                        uint32_t v[NC][32];
#pragma unroll
                        for (int x = 0; x < NC; ++x) umma::tmem_ld32_nowait(tcol + 32 * (NC * h + x), v[x]);
                        umma::tmem_wait_ld();
                        if (h == NL / NC - 1) {   // slot fully read: release it to the MMA
                            umma::fence_before();
                            __syncwarp();
                            if (lane == 0) umma::mbar_arrive(&S.acce[slot]);
                            pf.mark(2);
                        }
                        bool rare[NC];
                        unsigned bal[NC];
                        unsigned anyr = 0;
#pragma unroll
                        for (int x = 0; x < NC; ++x) {
                            rare[x] = rvalid && !(and32(v[x]) >> 31);
                            bal[x] = __ballot_sync(0xffffffffu, rare[x]);
                            anyr |= bal[x];
                        }
                        if (anyr && !(kExp & 4)) {   // rare: queue the survivors for a decider
                            pf.mark(3);
#pragma unroll
                            for (int x = 0; x < NC; ++x) {
                                if (!rare[x]) continue;
                                // survivor mask of this lane's 32 columns (bit y = column y,
                                // accumulator sign bit clear; two independent shift chains),
                                // restricted to the candidate window [wr, ws) and, in the own
                                // cell, to candidates after the query
                                const uint32_t cb = rb + bi * kBN + cpart * CW + 32 * (NC * h + x);
                                uint32_t sl = 0, sh = 0;
#pragma unroll
                                for (int y = 15; y >= 0; --y) {
                                    sl = __funnelshift_l(v[x][y], sl, 1);
                                    sh = __funnelshift_l(v[x][y + 16], sh, 1);
                                }
                                const uint32_t lo0 = (wsd >> 31) ? max(wr, qpos + 1u) : wr, hi0 = wsd & 0x7fffffffu;
                                const uint32_t lo = lo0 > cb ? min(lo0 - cb, 32u) : 0u;
                                const uint32_t hi = hi0 > cb ? min(hi0 - cb, 32u) : 0u;
                                const uint32_t wm = (hi >= 32 ? 0xffffffffu : ((1u << hi) - 1u)) &
                                                    ~(lo >= 32 ? 0xffffffffu : ((1u << lo) - 1u));
                                uint32_t m = ~((sh << 16) | (sl & 0xffffu)) & wm;
                                const uint32_t n = __popc(m);
                                if (!n) continue;
                                pf.add(7, n);
                                // tickets [t, t + n) of queue dq; written once the decider has
                                // consumed all but kPQ - n of the earlier ones (kPQ >= 64 + 32:
                                // the decider's current 64 never wait on a later ticket)
                                uint32_t t = atomicAdd(&S.q_tail[dq], n);
                                while (t + n > ld_volatile(&S.q_head[dq]) + kPQ) __nanosleep(32);
                                while (m) {
                                    const uint32_t y = __ffs(m) - 1;
                                    m &= m - 1;
                                    *reinterpret_cast<volatile unsigned long long*>(&S.pq[dq][t % kPQ]) =
                                        pair_word(qpos, cb + y, (t / kPQ) & 1u);
                                    ++t;
                                }
                            }
                            pf.mark(4);
                        }
                    }
                }
                c += nb;
            }
            __syncwarp();
            if (lane == 0) umma::mbar_arrive(&S.ite[ib]);
        }
        __threadfence_block();
        if (lane == 0) atomicAdd(&S.epi_done, 1u);
        pf.mark(3);
        if (lane == 0) pf.flush(12, 8);   // 12 wait itf, 13 wait accf, 14 ld -> release, 15 sign test + rest, 16 queue pushes, 18 warp-blocks, 19 chunks pushed
    }
    umma::fence_before();
    __syncthreads();
    if (warp == 1) umma::tmem_dealloc(tmem, 512);
    if (kProf && tid == 0) {
        atomicAdd(&g_ws_prof[26], (unsigned long long)(clock64() - t_start));
        atomicAdd(&g_ws_prof[27], 1ull);
    }
    if (MODE == kCount) {
#pragma unroll
        for (int o = 16; o; o >>= 1) npairs += __shfl_xor_sync(0xffffffffu, npairs, o);
        if (lane == 0 && npairs) atomicAdd((unsigned long long*)A.count, npairs);
    }
}

int sm_count() {
    static std::atomic<int> n{0};
    int v = n.load();
    if (!v) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        n.store(v);
    }
    return v;
}

template <int KP, int EG, int MODE, bool SYM>
int launch_ws_k(const JoinParams& p, const JoinArgs& a, uint32_t n_items, cudaStream_t s) {
    const size_t smem = sizeof(PsSmem<KP>);
    static std::atomic<unsigned long long> attr_done{0};   // the attribute is per device
    int dev = 0;
    GJ_CUDA(cudaGetDevice(&dev));
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(attr_done.load() & bit)) {
        GJ_CUDA(cudaFuncSetAttribute((const void*)k_join_ws<KP, EG, MODE, SYM>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_done.fetch_or(bit);
    }
    uint32_t* counter = nullptr;
    GJ_CUDA(pool_malloc(&counter, sizeof(uint32_t), s));
    GJ_CUDA(cudaMemsetAsync(counter, 0, sizeof(uint32_t), s));
    const unsigned grid = (unsigned)std::min<int64_t>(sm_count(), n_items);
    k_join_ws<KP, EG, MODE, SYM><<<grid, kThreads, smem, s>>>(p, a, counter, n_items);
    count_launch();
    GJ_CUDA(cudaGetLastError());
    GJ_CUDA(cudaFreeAsync(counter, s));
    return GJ_OK;
}

template <int KP, int EG>
int launch_ws(const JoinParams& p, JoinMode mode, const JoinArgs& a, bool sym, uint32_t n_items, cudaStream_t s) {
    if (mode == kEmit) return sym ? launch_ws_k<KP, EG, kEmit, true>(p, a, n_items, s)
                                  : launch_ws_k<KP, EG, kEmit, false>(p, a, n_items, s);
    return sym ? launch_ws_k<KP, EG, kCount, true>(p, a, n_items, s)
               : launch_ws_k<KP, EG, kCount, false>(p, a, n_items, s);
}

// Epilogue groups (timing knob GJ_WS_EG = 1, 2 or 4; read once).
int ws_groups() {
    static int eg = [] {
        const char* e = getenv("GJ_WS_EG");
        const int v = e ? atoi(e) : 0;
        return (v == 1 || v == 2 || v == 4) ? v : 0;
    }();
    return eg;
}

constexpr int kEGmax = kEpi / 4;   // groups of four warps (one per TMEM lane quarter)

template <int KP>
int launch_ws_eg(const JoinParams& p, JoinMode mode, const JoinArgs& a, bool sym, uint32_t n_items, cudaStream_t s) {
    switch (ws_groups()) {
        case 1: return launch_ws<KP, 1>(p, mode, a, sym, n_items, s);
        case 2: return launch_ws<KP, 2>(p, mode, a, sym, n_items, s);
        default: return launch_ws<KP, kEGmax>(p, mode, a, sym, n_items, s);
    }
}

}  // namespace

int launch_join_ws(const Index* ix, JoinMode mode, const JoinArgs& a, cudaStream_t s) {
    if (a.n_tiles <= 0) return GJ_OK;
    if (ix->tile_q != kM) {
        set_error("persistent tcgen05 join: 128-query tiles only");
        return GJ_ERR_INVALID;
    }
    const JoinParams p = join_params(ix);
    const bool sym = ix->opt.symmetric != 0;
    const int64_t items = a.part_off ? a.total_parts : a.n_tiles * (a.split > 1 ? a.split : 1);
    if (items <= 0) return GJ_OK;
    const uint32_t n = (uint32_t)items;
    switch (ix->k16) {
        case 16: return launch_ws_eg<16>(p, mode, a, sym, n, s);
        case 32: return launch_ws_eg<32>(p, mode, a, sym, n, s);
        case 48: return launch_ws_eg<48>(p, mode, a, sym, n, s);
        case 64: return launch_ws<64, kEGmax>(p, mode, a, sym, n, s);
        case 80: return launch_ws<80, kEGmax>(p, mode, a, sym, n, s);
        case 96: return launch_ws<96, kEGmax>(p, mode, a, sym, n, s);
        case 112: return launch_ws<112, kEGmax>(p, mode, a, sym, n, s);
        case 128: return launch_ws<128, kEGmax>(p, mode, a, sym, n, s);
        default: break;
    }
    set_error("persistent tcgen05 join: MMA depth " + std::to_string(ix->k16) + " not instantiated");
    return GJ_ERR_INVALID;
}

}  // namespace gj

#if GJ_WS_PROF
// experiment build only: read and reset the phase counters
extern "C" __attribute__((visibility("default"))) int gj_debug_ws_prof(unsigned long long* out) {
    if (cudaMemcpyFromSymbol(out, gj::g_ws_prof, sizeof(gj::g_ws_prof)) != cudaSuccess) return -2;
    static const unsigned long long zero[32] = {};
    cudaMemcpyToSymbol(gj::g_ws_prof, zero, sizeof(zero));
    return 0;
}
#endif
