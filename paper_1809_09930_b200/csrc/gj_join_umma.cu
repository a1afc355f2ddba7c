// SelfJoinKernel on the 5th-generation tensor cores (tcgen05.mma, TMEM
// accumulators) with the certified distance bound of gj_join_tc.cu and the
// FP64 decision of every surviving pair (B200-first variant of PAPER.md
// Alg. 1 l.596-607; FP64 semantics unchanged).
//
// CTA = 6 warps = one 128-query tile of one cell (M = 128 TMEM lanes),
// candidates in blocks of N = 128 (see k_join_umma below for the roles).
// The fp16 operands carry augmented columns so that every accumulator is
// (T - ||q^ - c^||^2) / 2 (gj_index.cu tc_threshold_from): a pair survives the
// bound iff its accumulator is > +0, and survivors are decided in FP64.
#include <stdlib.h>

#include "gj_internal.cuh"
#include "gj_umma.cuh"

namespace gj {
namespace {

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

// Survivor of the bound: FP64 decision and emission (both orders when symmetric).
template <int MODE, bool SYM>
__device__ __noinline__ unsigned long long decide_and_emit(const JoinParams& P, const JoinArgs& A, uint32_t qpos,
                                                         uint32_t cpos) {
    constexpr unsigned long long kMul = SYM ? 2ull : 1ull;
    if (dist2_fp64(P.pts + (size_t)qpos * P.n_pad, P.pts + (size_t)cpos * P.n_pad, P.n_pad) > P.eps2) return 0;
    if (MODE == kEmit) {
        const uint32_t qi = P.orig[qpos], ci = P.orig[cpos];
        const unsigned long long at = atomicAdd((unsigned long long*)A.count, kMul);
        if (at + kMul <= A.cap) {
            uint2* out = reinterpret_cast<uint2*>(A.out);
            out[at] = make_uint2(qi, ci);
            if (SYM) out[at + 1] = make_uint2(ci, qi);
        }
        return 0;
    }
    return kMul;
}

constexpr int kWarpsWs = 6;             // 0 producer, 1 MMA issuer, 2..5 epilogue
constexpr int kThreadsWs = 32 * kWarpsWs;
constexpr int kMaxWin = 1024;            // adjacent cells handled per setup round
// Candidate block width BN (UMMA N) and accumulator slots: 256 TMEM columns
// per CTA (two CTAs per SM fill the 512), split into 256 / BN slots.
template <int KP, int BN>
constexpr int ws_stages2() { return (KP <= 64 ? 4 : 3) * (128 / BN); }

template <int KP, int BN>
struct WsSmem {
    alignas(128) __half a[kM * KP];                       // queries (A), canonical K-major layout
    alignas(128) __half b[ws_stages2<KP, BN>()][BN * KP]; // candidate ring (B)
    uint64_t full[ws_stages2<KP, BN>()], empty[ws_stages2<KP, BN>()], accf[256 / BN], acce[256 / BN];
    uint32_t tmem_base;
    uint32_t wr[kMaxWin], ws[kMaxWin], nbk[kMaxWin];      // window [r, s), blocks (bit 31: own cell)
    unsigned long long red[kWarpsWs];
};

// Warp-specialised tcgen05 join.  Per tile: the epilogue warps build the A
// tile (coordinates + augmented columns r_hi, r_lo, 1, 1); all warps compute
// the SORTIDU windows of the adjacent cells (thread per cell); then
//   producer  : per 128-candidate block, one cp.async.bulk of the contiguous
//               grouped-layout rows [8*floor(r/8) + 128 b, +128) into the ring
//               (full/empty mbarriers, transaction bytes);
//   MMA       : one thread, K/16 tcgen05.mma per block into one of two TMEM
//               accumulators, commits to empty[stage] and acc_full[acc];
//   epilogue  : 4 warps = 128 TMEM lanes = the tile's queries; tcgen05.ld,
//               AND of the sign bits (survivor iff acc > +0), release the
//               accumulator, then FP64 decision of the rare survivors whose
//               candidate lies in [r, s) (and after the query in its own cell).
template <int KP, int BN, int MODE, bool SYM>
__global__ void __launch_bounds__(kThreadsWs) k_join_umma(JoinParams P, JoinArgs A) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    WsSmem<KP, BN>& S = *reinterpret_cast<WsSmem<KP, BN>*>(smem_raw);
    constexpr int KS = KP / 16;
    constexpr int ST = ws_stages2<KP, BN>();
    constexpr int NACC = 256 / BN;
    constexpr int NL = BN / 32;   // 32-column TMEM loads per accumulator row
    constexpr uint32_t kIdesc = umma::idesc_f16_f32(kM, BN);
    constexpr uint32_t kSBO = KP * 16;
    constexpr uint32_t kBlockBytes = BN * KP * 2;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int split = A.split > 1 ? A.split : 1;
    const int part = (int)(blockIdx.x % split);
    const int64_t j = A.first + A.step * (int64_t)(blockIdx.x / split);
    const uint32_t tile = P.tile_order[j];
    const uint32_t g = P.tile_cell[tile];
    const uint32_t q0 = P.tile_q0[tile];
    const uint32_t nq = min((uint32_t)kM, P.cell_start[g + 1] - q0);
    const int n_pad = P.n_pad;
    const double eps = P.eps;

    if (warp == 1) umma::tmem_alloc(&S.tmem_base, 256);
    if (tid == 0) {
        for (int i = 0; i < ST; ++i) {
            umma::mbar_init(&S.full[i], 1);
            umma::mbar_init(&S.empty[i], 1);
        }
        for (int i = 0; i < NACC; ++i) {
            umma::mbar_init(&S.accf[i], 1);
            umma::mbar_init(&S.acce[i], 4);
        }
        umma::mbar_fence_init();
    }
    if (warp >= 2) {   // A tile: thread = query row
        const int row = tid - 64;
        const bool valid = row < (int)nq;
        unsigned char* a_raw = reinterpret_cast<unsigned char*>(S.a);
        for (int kc = 0; kc < KP / 8; ++kc) {
            union { uint4 u; __half h[8]; } c;
            c.u = valid ? *reinterpret_cast<const uint4*>(P.pts16 + g16(q0 + row, kc * 8, KP)) : make_uint4(0, 0, 0, 0);
            if (kc == KP / 8 - 1) {   // query-side augmented columns
                query_aug(P.thr16, valid ? P.norm16[q0 + row] : 0.0, valid, c.h[4], c.h[5]);
                c.h[6] = __float2half(1.f);
                c.h[7] = __float2half(1.f);
            }
            *reinterpret_cast<uint4*>(a_raw + umma::tile_off(row, kc * 8, KP)) = c.u;
        }
    }
    unsigned long long npairs = 0;
    if (SYM && part == 0 && tid < kM) {   // the self pair (q, q); warps 0..3 cover the 128 queries
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
    uint32_t cnt = 0;   // blocks consumed so far (identical sequence in every role)
    const int erow = 32 * (warp & 3) + lane;   // epilogue: TMEM lane = query row
    for (uint32_t w0 = nb0; w0 < nb1; w0 += kMaxWin) {
        const int nwin = (int)min((uint32_t)kMaxWin, nb1 - w0);
        for (int i = tid; i < nwin; i += kThreadsWs) {   // windows of this round (thread per adjacent cell)
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
                        umma::mbar_arrive_expect_tx(&S.full[st], kBlockBytes);
                        umma::bulk_g2s(umma::smem_u32(S.b[st]), P.pts16 + (size_t)(rb + bi * BN) * KP, kBlockBytes,
                                       &S.full[st]);
                    }
                }
            }
        } else if (warp == 1) {   // ---------------- MMA issuer
            if (lane == 0) {
                uint32_t c = cnt;
                const uint32_t a_s = umma::smem_u32(S.a);
                for (int i = 0; i < nwin; ++i) {
                    const uint32_t nb = S.nbk[i] & 0x7fffffffu;
                    for (uint32_t bi = 0; bi < nb; ++bi, ++c) {
                        const uint32_t st = c % ST, ph = (c / ST) & 1u, ab = c % NACC, aph = (c / NACC) & 1u;
                        umma::mbar_wait(&S.acce[ab], aph ^ 1u);
                        umma::mbar_wait(&S.full[st], ph);
                        umma::fence_after();
                        const uint32_t b_s = umma::smem_u32(S.b[st]);
#pragma unroll
                        for (int ks = 0; ks < KS; ++ks)
                            umma::mma_f16(tmem + ab * BN, umma::smem_desc(a_s + ks * 256, 128, kSBO),
                                          umma::smem_desc(b_s + ks * 256, 128, kSBO), kIdesc, ks > 0 ? 1u : 0u);
                        umma::commit(&S.empty[st]);
                        umma::commit(&S.accf[ab]);
                    }
                }
            }
        } else {   // ---------------- epilogue (warps 2..5)
            uint32_t c = cnt;
            const uint32_t qpos = q0 + erow;
            const bool rvalid = erow < (int)nq;
            const uint32_t lane_off = (uint32_t)(32 * (warp & 3)) << 16;
            for (int i = 0; i < nwin; ++i) {
                const uint32_t nbw = S.nbk[i], nb = nbw & 0x7fffffffu, rb = S.wr[i] & ~7u;
                const uint32_t wr = S.wr[i], wsd = S.ws[i];
                const bool diag = (nbw >> 31) != 0;
                for (uint32_t bi = 0; bi < nb; ++bi, ++c) {
                    const uint32_t ab = c % NACC, aph = (c / NACC) & 1u;
                    umma::mbar_wait(&S.accf[ab], aph);
                    umma::fence_after();
                    // all BN columns in flight at once, one wait, then release the accumulator
                    uint32_t v[NL][32];
#pragma unroll
                    for (int x = 0; x < NL; ++x) umma::tmem_ld32_nowait(tmem + lane_off + ab * BN + 32 * x, v[x]);
                    umma::tmem_wait_ld();
                    umma::fence_before();
                    __syncwarp();
                    if (lane == 0) umma::mbar_arrive(&S.acce[ab]);
                    uint32_t all = 0xffffffffu;
#pragma unroll
                    for (int x = 0; x < NL; ++x)
#pragma unroll
                        for (int y = 0; y < 32; ++y) all &= v[x][y];
                    unsigned long long mask[2] = {0, 0};
                    if (!(all >> 31)) {   // rare: some accumulator > +0
#pragma unroll
                        for (int x = 0; x < NL; ++x)
#pragma unroll
                            for (int y = 0; y < 32; ++y)
                                if (!(v[x][y] >> 31)) mask[x >> 1] |= 1ull << (32 * (x & 1) + y);
                    }
                    if (!rvalid) continue;
                    const uint32_t base = rb + bi * BN;
#pragma unroll
                    for (int hh = 0; hh < (NL + 1) / 2; ++hh) {
                        unsigned long long m = mask[hh];
                        while (m) {   // rare: FP64 decision of the survivors
                            const int bit = __ffsll((long long)m) - 1;
                            m &= m - 1;
                            const uint32_t cpos = base + 64 * hh + bit;
                            if (cpos < wr || cpos >= wsd || (diag && cpos <= qpos)) continue;
                            npairs += decide_and_emit<MODE, SYM>(P, A, qpos, cpos);
                        }
                    }
                }
            }
        }
        // every role walked the same block sequence
        for (int i = 0; i < nwin; ++i) cnt += S.nbk[i] & 0x7fffffffu;
        __syncthreads();
    }
    umma::fence_before();
    __syncthreads();
    if (warp == 1) umma::tmem_dealloc(tmem, 256);

    if (MODE == kCount) {
        unsigned long long x = npairs;
#pragma unroll
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) S.red[warp] = x;
        __syncthreads();
        if (tid == 0) {
            unsigned long long t = 0;
            for (int w = 0; w < kWarpsWs; ++w) t += S.red[w];
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

template <int KP, int BN>
int launch_umma(const JoinParams& p, JoinMode mode, const JoinArgs& a, bool sym, cudaStream_t s) {
    if (a.n_tiles <= 0) return GJ_OK;
    // at most two CTAs per SM: their 2 x 256 TMEM columns fill the SM's 512
    const size_t smem = std::max<size_t>(sizeof(WsSmem<KP, BN>), 80 * 1024);
    static_assert(sizeof(WsSmem<KP, BN>) <= 227 * 1024, "shared memory");
    static bool attr_done[2][2] = {{false, false}, {false, false}};
    auto setattr = [&](const void* f, int m, int y) -> int {
        if (!attr_done[m][y]) {
            GJ_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            attr_done[m][y] = true;
        }
        return GJ_OK;
    };
    dim3 grid((unsigned)(a.n_tiles * (a.split > 1 ? a.split : 1)));
    int rc = GJ_OK;
    if (mode == kEmit) {
        if (sym) {
            if ((rc = setattr((const void*)k_join_umma<KP, BN, kEmit, true>, 0, 1))) return rc;
            k_join_umma<KP, BN, kEmit, true><<<grid, kThreadsWs, smem, s>>>(p, a);
        } else {
            if ((rc = setattr((const void*)k_join_umma<KP, BN, kEmit, false>, 0, 0))) return rc;
            k_join_umma<KP, BN, kEmit, false><<<grid, kThreadsWs, smem, s>>>(p, a);
        }
    } else {
        if (sym) {
            if ((rc = setattr((const void*)k_join_umma<KP, BN, kCount, true>, 1, 1))) return rc;
            k_join_umma<KP, BN, kCount, true><<<grid, kThreadsWs, smem, s>>>(p, a);
        } else {
            if ((rc = setattr((const void*)k_join_umma<KP, BN, kCount, false>, 1, 0))) return rc;
            k_join_umma<KP, BN, kCount, false><<<grid, kThreadsWs, smem, s>>>(p, a);
        }
    }
    count_launch();
    GJ_CUDA(cudaGetLastError());
    return GJ_OK;
}

}  // namespace

int launch_join_umma(const Index* ix, JoinMode mode, const JoinArgs& a, cudaStream_t s) {
    const JoinParams p = join_params(ix);
    const bool sym = ix->opt.symmetric != 0;
    // block width: 64 candidates x 4 accumulator slots (default) or 128 x 2 (GJ_UMMA_BN=128)
    static const int bn = [] { const char* e = getenv("GJ_UMMA_BN"); return e && atoi(e) == 128 ? 128 : 64; }();
    if (bn == 128) {
        switch (ix->k16) {
            case 16: return launch_umma<16, 128>(p, mode, a, sym, s);
            case 32: return launch_umma<32, 128>(p, mode, a, sym, s);
            case 48: return launch_umma<48, 128>(p, mode, a, sym, s);
            case 64: return launch_umma<64, 128>(p, mode, a, sym, s);
            case 80: return launch_umma<80, 128>(p, mode, a, sym, s);
            case 96: return launch_umma<96, 128>(p, mode, a, sym, s);
            case 112: return launch_umma<112, 128>(p, mode, a, sym, s);
            default: return launch_umma<128, 128>(p, mode, a, sym, s);
        }
    }
    switch (ix->k16) {
        case 16: return launch_umma<16, 64>(p, mode, a, sym, s);
        case 32: return launch_umma<32, 64>(p, mode, a, sym, s);
        case 48: return launch_umma<48, 64>(p, mode, a, sym, s);
        case 64: return launch_umma<64, 64>(p, mode, a, sym, s);
        case 80: return launch_umma<80, 64>(p, mode, a, sym, s);
        case 96: return launch_umma<96, 64>(p, mode, a, sym, s);
        case 112: return launch_umma<112, 64>(p, mode, a, sym, s);
        default: return launch_umma<128, 64>(p, mode, a, sym, s);
    }
}

int selftest_umma(const void* A, const void* B, float* D, cudaStream_t s) {
    k_umma_selftest<<<1, 128, 0, s>>>(reinterpret_cast<const __half*>(A), reinterpret_cast<const __half*>(B), D);
    count_launch();
    GJ_CUDA(cudaGetLastError());
    GJ_CUDA(cudaStreamSynchronize(s));
    return GJ_OK;
}

}  // namespace gj
