// SelfJoinKernel with a certified FP32 prefilter (B200-first variant of
// PAPER.md Alg. 1 l.596-607; FP64 semantics unchanged).
//
// Same tiling as gj_join.cu (one CTA per 128-query tile of one cell, queries
// in registers, candidates of each adjacent cell streamed through shared
// memory, SORTIDU tile window, symmetric evaluation, warp-aggregated
// emission), but the SHORTC scan runs on float32 copies of the centred
// coordinates, fl32(x - min_j): the FP32 pipe has twice the FP64 pipe's lanes
// on B200 and the stage holds twice the candidates.  Each thread tests its
// query against two candidates at once with packed f32x2 adds / FMAs
// (sm_100 FADD2/FFMA2), candidates staged pairwise interleaved and negated.  A pair is rejected only
// when its running FP32 sum exceeds thr32, which PROVES dist > eps (1 + 1e-9)
// (derivation in gj_index.cu fp32_threshold and DESIGN.md); every pair that
// survives all n dims is decided by the FP64 test, with exactly the FP64
// kernel's arithmetic (FMA chain in dimension order).  The emitted pair set is
// therefore the FP64 kernel's pair set, bit for bit.
#include "gj_internal.cuh"

namespace gj {
namespace {

constexpr int kWinRound = 256;   // adjacent cells whose windows are computed per round

constexpr int kSmemFloats = 8192;   // 32 KB candidate stage

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

// CTAs per SM the register allocation must allow for n > 64 (GJ_J32_MINB):
// the 90-dim Songs-shaped query held in registers took 166 of them, leaving 3
// CTAs (12 warps, 18 % warps active, 42 % of stalls at CTA barriers) per SM;
// capped at 128 (4 CTAs, ~28 bytes of spills) the songs90 join went from 17.3
// to 13.4 ms, at 96 (5 CTAs, 128 bytes of spills) to 18.6
// (profiles/r2_ab_join32_registers.txt)
#ifndef GJ_J32_MINB
#define GJ_J32_MINB 4
#endif
template <int NPR, int MODE, bool SYM>
__global__ void __launch_bounds__(kTileQ, NPR >= 96 ? GJ_J32_MINB : 1) k_join32(JoinParams P, JoinArgs A) {
    constexpr int TC = (kSmemFloats / NPR) & ~1;   // candidates per stage (even: staged in pairs)
    __shared__ __align__(16) float Cs[kSmemFloats];
    __shared__ uint32_t Cid[TC];
    __shared__ uint32_t s_wr[kWinRound], s_ws[kWinRound];   // SORTIDU windows of one round of adjacent cells
    __shared__ unsigned char s_dg[kWinRound];
    __shared__ unsigned long long s_red[kTileQ / 32];

    const int tid = threadIdx.x, lane = tid & 31;
    const unsigned lt = (1u << lane) - 1u;
    // split-K over candidates: CTA (m, part) scans part `part` of every window
    const CtaTile ct = cta_tile(P, A, kTileQ);
    if (ct.nq == 0) return;   // sub-block past the end of the tile's cell
    const int part = ct.part, split = ct.split;
    const uint32_t g = ct.g, q0 = ct.q0, nq = ct.nq;
    const bool active = tid < (int)nq;
    const uint32_t qpos = q0 + (active ? tid : 0);
    const int n_pad = P.n_pad;

    // query coordinate d duplicated in both halves: operand of the packed
    // f32x2 ops that test one query against two candidates at once
    float2 q[NPR];
#pragma unroll
    for (int d = 0; d < NPR; d += 4) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (d < n_pad) v = *reinterpret_cast<const float4*>(P.pts32 + (size_t)qpos * n_pad + d);
        q[d] = make_float2(v.x, v.x);
        q[d + 1] = make_float2(v.y, v.y);
        q[d + 2] = make_float2(v.z, v.z);
        q[d + 3] = make_float2(v.w, v.w);
    }
    const double eps = P.eps, eps2 = P.eps2;
    const float thr = P.thr32, thr_in = P.thr32_in;
    const uint32_t qid = P.orig[qpos];
    const double u_lo = P.pts[(size_t)q0 * n_pad + P.u];
    const double u_hi = P.pts[(size_t)(q0 + nq - 1) * n_pad + P.u];
    const double* __restrict__ qrow64 = P.pts + (size_t)qpos * n_pad;
    constexpr unsigned long long kMul = SYM ? 2ull : 1ull;

    unsigned long long npairs = 0;
    if (SYM && part == 0) {   // the self pair (q, q)
        if (MODE == kEmit) {
            const unsigned m = __ballot_sync(0xffffffffu, active);
            unsigned long long base = 0;
            if (lane == 0 && m) base = atomicAdd((unsigned long long*)A.count, (unsigned long long)__popc(m));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (active) {
                const unsigned long long at = base + __popc(m & lt);
                if (at < A.cap) reinterpret_cast<uint2*>(A.out)[at] = make_uint2(qid, qid);
            }
        } else if (active) {
            npairs += 1;
        }
    }

    const uint32_t nb0 = SYM ? P.nbr_self[g] : P.nbr_off[g], nb1 = P.nbr_off[g + 1];
    // SORTIDU windows of up to kWinRound adjacent cells at a time, one thread per
    // cell (the binary searches run in parallel instead of one cell after another)
    for (uint32_t w0 = nb0; w0 < nb1; w0 += kWinRound) {
    const uint32_t nwin = min((uint32_t)kWinRound, nb1 - w0);
    __syncthreads();   // the previous round's windows are no longer read
    for (uint32_t i = tid; i < nwin; i += kTileQ) {
        const uint32_t B = P.nbr[w0 + i];
        uint32_t r = P.cell_start[B], s = P.cell_start[B + 1];
        if (P.sortidu) {   // tile-level SORTIDU window (exact predicates on the fp64 u-coordinates)
            uint32_t lo = r, hi = s;
            while (lo < hi) {   // first r with u_lo - r(u) <= eps
                const uint32_t mid = (lo + hi) >> 1;
                if (u_lo - P.pts[(size_t)mid * n_pad + P.u] <= eps) hi = mid; else lo = mid + 1;
            }
            const uint32_t rr = lo;
            lo = r;
            hi = s;
            while (lo < hi) {   // first s with s(u) - u_hi > eps
                const uint32_t mid = (lo + hi) >> 1;
                if (P.pts[(size_t)mid * n_pad + P.u] - u_hi > eps) hi = mid; else lo = mid + 1;
            }
            r = rr;
            s = max(lo, r);
        }
        const bool diag = SYM && B == g;
        if (diag) r = max(r, q0 + 1);
        if (split > 1 && s > r) {
            const uint64_t len = s - r;
            s = r + (uint32_t)(len * (part + 1) / split);
            r = r + (uint32_t)(len * part / split);
        }
        s_wr[i] = r;
        s_ws[i] = max(s, r);
        s_dg[i] = diag ? 1 : 0;
    }
    __syncthreads();
    for (uint32_t wi = 0; wi < nwin; ++wi) {
        const uint32_t r = s_wr[wi], s = s_ws[wi];
        const bool diag = s_dg[wi] != 0;
        for (uint32_t cb = r; cb < s; cb += TC) {
            const int cntc = (int)min((uint32_t)TC, s - cb);
            __syncthreads();
            {
                // stage candidate pairs (2p, 2p+1) interleaved and negated:
                // Cs[p][d] = (-c_2p[d], -c_2p+1[d]) so that q - c is one f32x2 add
                const float* src = P.pts32 + (size_t)cb * n_pad;
                const int q4 = n_pad / 4;                      // float4 chunks per row
                const int nv = ((cntc + 1) / 2) * q4;
                for (int i = tid; i < nv; i += kTileQ) {
                    const int pr = i / q4, d = (i - pr * q4) * 4;
                    const float4 a = *reinterpret_cast<const float4*>(src + (size_t)(2 * pr) * n_pad + d);
                    float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (2 * pr + 1 < cntc) b = *reinterpret_cast<const float4*>(src + (size_t)(2 * pr + 1) * n_pad + d);
                    float4* dst = reinterpret_cast<float4*>(Cs + (size_t)pr * 2 * n_pad + 2 * d);
                    dst[0] = make_float4(-a.x, -b.x, -a.y, -b.y);
                    dst[1] = make_float4(-a.z, -b.z, -a.w, -b.w);
                }
                for (int i = tid; i < cntc; i += kTileQ) Cid[i] = P.orig[cb + i];
            }
            __syncthreads();
            for (int c = 0; c < cntc; c += 2) {
                const bool two = c + 1 < cntc;
                const float* cp = Cs + (size_t)c * n_pad;     // pair c/2, interleaved
                const uint32_t p0 = cb + c;
                bool ok0 = active, ok1 = active && two;
                if (diag) {
                    ok0 = ok0 && p0 > qpos;
                    ok1 = ok1 && p0 + 1 > qpos;
                }
                // a.x / a.y: running sums of candidates c / c+1; a dead one starts at +inf
                float2 a = make_float2(ok0 ? 0.f : INFINITY, ok1 ? 0.f : INFINITY);
                if (ok0 || ok1) {
#pragma unroll
                    for (int d = 0; d < NPR; d += 4) {
                        if (d >= n_pad) break;
                        const float4 x = *reinterpret_cast<const float4*>(cp + 2 * d);
                        const float4 y = *reinterpret_cast<const float4*>(cp + 2 * d + 4);
                        float2 t;
                        t = __fadd2_rn(q[d], make_float2(x.x, x.y));     a = __ffma2_rn(t, t, a);
                        t = __fadd2_rn(q[d + 1], make_float2(x.z, x.w)); a = __ffma2_rn(t, t, a);
                        t = __fadd2_rn(q[d + 2], make_float2(y.x, y.y)); a = __ffma2_rn(t, t, a);
                        t = __fadd2_rn(q[d + 3], make_float2(y.z, y.w)); a = __ffma2_rn(t, t, a);
                        if ((d & 4) && P.shortc && a.x > thr && a.y > thr) break;   // SHORTC, every 8 dims
                    }
                }
                const float a0 = a.x, a1 = a.y;
                // survivors of the prefilter: decided in FP64
                // ... unless the bound also proves them inside (a <= thr_in): on dense
                // data almost every candidate is a pair and skips the FP64 row reads
                bool hit0 = ok0 && a0 <= thr, hit1 = ok1 && a1 <= thr;
                if (hit0 && !(a0 <= thr_in)) hit0 = dist2_fp64(qrow64, P.pts + (size_t)p0 * n_pad, n_pad) <= eps2;
                if (hit1 && !(a1 <= thr_in)) hit1 = dist2_fp64(qrow64, P.pts + (size_t)(p0 + 1) * n_pad, n_pad) <= eps2;
                if (MODE == kEmit) {
                    const unsigned m0 = __ballot_sync(0xffffffffu, hit0);
                    const unsigned m1 = __ballot_sync(0xffffffffu, hit1);
                    if (m0 | m1) {
                        const int leader = __ffs(m0 | m1) - 1;
                        unsigned long long base = 0;
                        if (lane == leader)
                            base = atomicAdd((unsigned long long*)A.count, kMul * (__popc(m0) + __popc(m1)));
                        base = __shfl_sync(0xffffffffu, base, leader);
                        uint2* out = reinterpret_cast<uint2*>(A.out);
                        if (hit0) {
                            const unsigned long long at = base + kMul * __popc(m0 & lt);
                            const uint32_t id = Cid[c];
                            if (at + kMul <= A.cap) {
                                out[at] = make_uint2(qid, id);
                                if (SYM) out[at + 1] = make_uint2(id, qid);
                            }
                        }
                        if (hit1) {
                            const unsigned long long at = base + kMul * (__popc(m0) + __popc(m1 & lt));
                            const uint32_t id = Cid[c + 1];
                            if (at + kMul <= A.cap) {
                                out[at] = make_uint2(qid, id);
                                if (SYM) out[at + 1] = make_uint2(id, qid);
                            }
                        }
                    }
                } else {
                    npairs += kMul * ((unsigned long long)hit0 + (unsigned long long)hit1);
                }
            }
        }
    }
    }
    if (MODE == kCount) {
        unsigned long long x = npairs;
#pragma unroll
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) s_red[tid >> 5] = x;
        __syncthreads();
        if (tid == 0) {
            unsigned long long t = 0;
            for (int w = 0; w < kTileQ / 32; ++w) t += s_red[w];
            if (t) atomicAdd((unsigned long long*)A.count, t);
            if (part == 0) atomicAdd((unsigned long long*)A.count + 1, (unsigned long long)nq);
        }
    }
}

template <int NPR>
int launch32(const JoinParams& p, JoinMode mode, const JoinArgs& a, bool sym, cudaStream_t s) {
    if (a.n_tiles <= 0) return GJ_OK;
    dim3 grid(grid_ctas(a, (int)p.tile_q, kTileQ));
    if (mode == kEmit) {
        if (sym) k_join32<NPR, kEmit, true><<<grid, kTileQ, 0, s>>>(p, a);
        else k_join32<NPR, kEmit, false><<<grid, kTileQ, 0, s>>>(p, a);
    } else {
        if (sym) k_join32<NPR, kCount, true><<<grid, kTileQ, 0, s>>>(p, a);
        else k_join32<NPR, kCount, false><<<grid, kTileQ, 0, s>>>(p, a);
    }
    count_launch();
    GJ_CUDA(cudaGetLastError());
    return GJ_OK;
}

}  // namespace

int launch_join32(const Index* ix, JoinMode mode, const JoinArgs& a, cudaStream_t s) {
    const JoinParams p = join_params(ix);
    const int np = ix->n_pad;
    const bool sym = ix->opt.symmetric != 0;
    if (np <= 8) return launch32<8>(p, mode, a, sym, s);
    if (np <= 16) return launch32<16>(p, mode, a, sym, s);
    if (np <= 24) return launch32<24>(p, mode, a, sym, s);
    if (np <= 32) return launch32<32>(p, mode, a, sym, s);
    if (np <= 48) return launch32<48>(p, mode, a, sym, s);
    if (np <= 64) return launch32<64>(p, mode, a, sym, s);
    if (np <= 96) return launch32<96>(p, mode, a, sym, s);
    return launch32<128>(p, mode, a, sym, s);
}

}  // namespace gj
