// SelfJoinKernel (Alg. 1 l.596-607) for sm_100a.
//
// Symmetric mode (default): dist(a,b) = dist(b,a) bit-for-bit (the per-dim
// squares are identical), so each unordered pair is evaluated once -- a tile
// of cell A visits only adjacent cells with index >= A, and in A itself only
// candidates after the query -- and both ordered pairs are emitted; the self
// pair is emitted directly.  Per-query mode (symmetric = 0) is Alg. 1 verbatim.
//
// One CTA = one query tile: up to 128 consecutive sorted points of ONE
// non-empty cell A (so the whole CTA shares getAdjCells' result, computed
// once per cell at index build).  One thread = one query point, its n
// coordinates held in registers.  For every adjacent non-empty cell B the CTA
// streams B's candidates through shared memory in coalesced double2 chunks;
// every thread tests its query against every staged candidate:
//   SORTIDU (§4.3): the staged range is the union of the tile's u-windows,
//     found by binary search in B's u-sorted run.  In emit / count mode every
//     thread tests every candidate of that union (a candidate outside its own
//     query's window is farther than eps on u alone, so the distance test
//     rejects it: same pairs); stats mode additionally applies each query's
//     own window |p(u) - q(u)| <= eps so the work counters are the paper's.
//   SHORTC (§4.4): the squared-distance sum is accumulated in dimension
//     order (highest variance first after REORDER) and abandoned as soon as
//     it exceeds eps^2 (checked every 4 dims; stats mode: every dim).
// Pairs are emitted with one warp-aggregated atomic per candidate that hit in
// at least one lane (ballot -> leader atomicAdd -> shfl -> per-lane store).
//
// This is filter 0, the FP64 reference scan of the north_star; the default
// (filter 2, gj_join_umma.cu) puts a certified tcgen05 bound in front of the
// same FP64 test because on the paper's workloads the gather is a contiguous
// range of a cell-sorted array, i.e. a dense block.
#include <stdlib.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "gj_internal.cuh"

namespace gj {
namespace {

constexpr int kWinRound = 256;   // adjacent cells whose windows are computed per round

using Params = JoinParams;

constexpr int kSmemDoubles = 4096;   // 32 KB candidate stage

// Stats mode: one candidate with the oracle's exact arithmetic (unfused,
// dimension order, SHORTC check after every dimension).  Returns dims used.
template <int NPR>
__device__ __forceinline__ int dims_exact(const double (&q)[NPR], const double* __restrict__ cp, int n,
                                          double eps2, double* acc_out) {
    double acc = 0.0;
    int used = 0;
#pragma unroll
    for (int d = 0; d < NPR; ++d) {
        if (d >= n) break;
        const double t = __dsub_rn(q[d], cp[d]);
        acc = __dadd_rn(acc, __dmul_rn(t, t));
        ++used;
        if (acc > eps2) break;
    }
    *acc_out = acc;
    return used;
}

// Counters (kCount/kStats): 0 pairs, 1 cells, 2 tests, 3 dims, 4 tests evaluated, 5 dims evaluated.
template <int NPR, int MODE, bool SYM>
__global__ void __launch_bounds__(kTileQ) k_join(Params P, JoinArgs A) {
    constexpr int TC = kSmemDoubles / NPR;   // candidates per shared-memory stage (even)
    __shared__ __align__(16) double Cs[kSmemDoubles];
    __shared__ uint32_t Cid[TC];
    __shared__ uint32_t s_wr[kWinRound], s_ws[kWinRound];   // SORTIDU windows of one round of adjacent cells
    __shared__ unsigned char s_dg[kWinRound];
    __shared__ unsigned long long s_red[6][kTileQ / 32];

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

    double q[NPR];
#pragma unroll
    for (int d = 0; d < NPR; d += 2) {
        double2 v = make_double2(0.0, 0.0);
        if (d < n_pad) v = *reinterpret_cast<const double2*>(P.pts + (size_t)qpos * n_pad + d);
        q[d] = v.x;
        q[d + 1] = v.y;
    }
    const double eps = P.eps, eps2 = P.eps2;
    const double qu = P.pts[(size_t)qpos * n_pad + P.u];
    const uint32_t qid = P.orig[qpos];
    const double u_lo = P.pts[(size_t)q0 * n_pad + P.u];
    const double u_hi = P.pts[(size_t)(q0 + nq - 1) * n_pad + P.u];
    constexpr unsigned long long kMul = SYM ? 2ull : 1ull;   // ordered pairs per evaluated pair

    unsigned long long cnt[6] = {0, 0, 0, 0, 0, 0};
    if (MODE == kStats && active && part == 0) cnt[1] += P.nbr_off[g + 1] - P.nbr_off[g];
    if (SYM && part == 0) {   // the self pair (q, q): d = 0 <= eps
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
            cnt[0] += 1;
            cnt[2] += 1;
            cnt[3] += P.n;
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
                const double2* src = reinterpret_cast<const double2*>(P.pts + (size_t)cb * n_pad);
                double2* dst = reinterpret_cast<double2*>(Cs);
                const int nv = cntc * n_pad / 2;
                for (int i = tid; i < nv; i += kTileQ) dst[i] = src[i];
                for (int i = tid; i < cntc; i += kTileQ) Cid[i] = P.orig[cb + i];
            }
            __syncthreads();
            for (int c = 0; c < cntc; c += 2) {
                const bool two = c + 1 < cntc;
                const double* cp0 = Cs + c * n_pad;
                const double* cp1 = two ? cp0 + n_pad : cp0;
                const uint32_t p0 = cb + c;
                bool ok0 = active, ok1 = active && two;
                if (diag) {
                    ok0 = ok0 && p0 > qpos;
                    ok1 = ok1 && p0 + 1 > qpos;
                }
                double a0, a1;
                if (MODE == kStats) {
                    if (P.sortidu) {   // the paper's per-query window |p(u) - q(u)| <= eps
                        const double c0u = cp0[P.u], c1u = cp1[P.u];
                        ok0 = ok0 && (qu - c0u <= eps) && (c0u - qu <= eps);
                        ok1 = ok1 && (qu - c1u <= eps) && (c1u - qu <= eps);
                    }
                    a0 = a1 = INFINITY;
                    if (ok0) {
                        const unsigned long long used = dims_exact<NPR>(q, cp0, P.n, eps2, &a0);
                        cnt[2] += kMul; cnt[3] += kMul * used; cnt[4] += 1; cnt[5] += used;
                    }
                    if (ok1) {
                        const unsigned long long used = dims_exact<NPR>(q, cp1, P.n, eps2, &a1);
                        cnt[2] += kMul; cnt[3] += kMul * used; cnt[4] += 1; cnt[5] += used;
                    }
                } else {
                    // two independent candidates per thread (two FMA chains in flight);
                    // a dead candidate starts at +inf so it never keeps the loop alive
                    a0 = ok0 ? 0.0 : INFINITY;
                    a1 = ok1 ? 0.0 : INFINITY;
                    if (ok0 || ok1) {
#pragma unroll
                        for (int d = 0; d < NPR; d += 4) {
                            if (d >= n_pad) break;
                            const double2 x0 = *reinterpret_cast<const double2*>(cp0 + d);
                            const double2 y0 = *reinterpret_cast<const double2*>(cp0 + d + 2);
                            const double2 x1 = *reinterpret_cast<const double2*>(cp1 + d);
                            const double2 y1 = *reinterpret_cast<const double2*>(cp1 + d + 2);
                            double t;
                            t = q[d] - x0.x;     a0 = fma(t, t, a0);
                            t = q[d] - x1.x;     a1 = fma(t, t, a1);
                            t = q[d + 1] - x0.y; a0 = fma(t, t, a0);
                            t = q[d + 1] - x1.y; a1 = fma(t, t, a1);
                            t = q[d + 2] - y0.x; a0 = fma(t, t, a0);
                            t = q[d + 2] - y1.x; a1 = fma(t, t, a1);
                            t = q[d + 3] - y0.y; a0 = fma(t, t, a0);
                            t = q[d + 3] - y1.y; a1 = fma(t, t, a1);
                            if (P.shortc && a0 > eps2 && a1 > eps2) break;   // SHORTC
                        }
                    }
                }
                const bool hit0 = ok0 && a0 <= eps2, hit1 = ok1 && a1 <= eps2;
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
                    cnt[0] += kMul * ((unsigned long long)hit0 + (unsigned long long)hit1);
                }
            }
        }
    }
    }
    if (MODE != kEmit) {
        if (MODE == kStats && !SYM) {
            cnt[4] = cnt[2];
            cnt[5] = cnt[3];
        }
        const int nv = MODE == kStats ? 6 : 1;
        for (int i = 0; i < nv; ++i) {
            unsigned long long x = cnt[i];
#pragma unroll
            for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
            if (lane == 0) s_red[i][tid >> 5] = x;
        }
        __syncthreads();
        if (tid < nv) {
            unsigned long long t = 0;
            for (int w = 0; w < kTileQ / 32; ++w) t += s_red[tid][w];
            if (t) atomicAdd((unsigned long long*)A.count + tid, t);
        }
        if (MODE == kCount && tid == 0 && part == 0)
            atomicAdd((unsigned long long*)A.count + 1, (unsigned long long)nq);
    }
}

// Work counters without the distance work (gj_join_counts): per query and
// adjacent cell, the paper's SORTIDU window [lo, hi) by binary search on the
// u-sorted run (the same predicates as the stats scan: q(u) - c(u) <= eps and
// not c(u) - q(u) > eps), the own cell restricted to candidates after the query
// when symmetric.  Counters: [0] cells, [1] paper tests, [2] tests evaluated.
__global__ void __launch_bounds__(kTileQ) k_count_tests(Params P, JoinArgs A, int sym, unsigned long long* out) {
    const CtaTile ct = cta_tile(P, A, kTileQ);
    const int tid = threadIdx.x;
    unsigned long long cells = 0, tests = 0, evald = 0;
    if (tid < (int)ct.nq) {
        const uint32_t g = ct.g, qpos = ct.q0 + tid;
        const int n_pad = P.n_pad;
        const double eps = P.eps;
        const double qu = P.pts[(size_t)qpos * n_pad + P.u];
        const uint32_t a0 = P.nbr_off[g], a1 = P.nbr_off[g + 1], self = P.nbr_self[g];
        cells = a1 - a0;
        for (uint32_t b = sym ? self : a0; b < a1; ++b) {
            const uint32_t B = P.nbr[b];
            uint32_t lo = P.cell_start[B], hi = P.cell_start[B + 1];
            if (P.sortidu) {
                uint32_t l = lo, h = hi;
                while (l < h) {   // first c with q(u) - c(u) <= eps
                    const uint32_t m = (l + h) >> 1;
                    if (qu - P.pts[(size_t)m * n_pad + P.u] <= eps) h = m; else l = m + 1;
                }
                const uint32_t lo2 = l;
                h = hi;
                while (l < h) {   // first c with c(u) - q(u) > eps
                    const uint32_t m = (l + h) >> 1;
                    if (P.pts[(size_t)m * n_pad + P.u] - qu > eps) h = m; else l = m + 1;
                }
                lo = lo2;
                hi = l;
            }
            if (sym && B == g) lo = max(lo, qpos + 1);
            if (hi > lo) evald += hi - lo;
        }
        tests = sym ? 2 * evald + 1 : evald;
    }
    unsigned long long v[3] = {cells, tests, evald};
    for (int i = 0; i < 3; ++i) {
        unsigned long long x = v[i];
#pragma unroll
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if ((tid & 31) == 0 && x) atomicAdd(out + i, x);
    }
}

template <int NPR, bool SYM>
void launch_mode(const Params& p, JoinMode mode, const JoinArgs& a, cudaStream_t s) {
    dim3 grid(grid_ctas(a, (int)p.tile_q, kTileQ));
    if (mode == kEmit) k_join<NPR, kEmit, SYM><<<grid, kTileQ, 0, s>>>(p, a);
    else if (mode == kCount) k_join<NPR, kCount, SYM><<<grid, kTileQ, 0, s>>>(p, a);
    else k_join<NPR, kStats, SYM><<<grid, kTileQ, 0, s>>>(p, a);
}

template <int NPR>
int launch_np(const Params& p, JoinMode mode, const JoinArgs& a, bool sym, cudaStream_t s) {
    if (a.n_tiles <= 0) return GJ_OK;
    if (sym) launch_mode<NPR, true>(p, mode, a, s);
    else launch_mode<NPR, false>(p, mode, a, s);
    count_launch();
    GJ_CUDA(cudaGetLastError());
    return GJ_OK;
}

}  // namespace

int count_tests(const Index* ix, const JoinArgs& a, unsigned long long* d_out, cudaStream_t s) {
    if (a.n_tiles <= 0) return GJ_OK;
    const Params p = join_params(ix);
    k_count_tests<<<grid_ctas(a, (int)p.tile_q, kTileQ), kTileQ, 0, s>>>(p, a, ix->opt.symmetric, d_out);
    count_launch();
    GJ_CUDA(cudaGetLastError());
    return GJ_OK;
}

JoinParams join_params(const Index* ix) {
    JoinParams p;
    p.pts = ix->pts;
    p.pts32 = ix->pts32;
    p.orig = ix->orig;
    p.cell_start = ix->cell_start;
    p.nbr_off = ix->nbr_off;
    p.nbr = ix->nbr;
    p.nbr_self = ix->nbr_self;
    p.tile_cell = ix->tile_cell;
    p.tile_q0 = ix->tile_q0;
    p.tile_order = ix->tile_order;
    p.n = ix->n;
    p.n_pad = ix->n_pad;
    p.u = ix->u;
    p.sortidu = ix->opt.sortidu;
    p.shortc = ix->opt.shortc;
    p.eps = ix->eps;
    p.eps2 = ix->eps2;
    p.thr32 = ix->thr32;
    p.thr32_in = ix->thr32_in;
    p.pts16 = ix->pts16;
    p.norm16 = ix->norm16;
    p.k16 = ix->k16;
    p.thr16 = ix->thr16;
    p.tile_q = (uint32_t)ix->tile_q;
    return p;
}

// Query sets of kDealBlock consecutive heaviest-first tiles (reading R12: one
// tile per set).  Larger sets keep spatially consecutive tiles in one launch
// (tiles of one cell have equal keys and keep their order); measured no
// faster: the expo32 join dealt into 24 launches took 215 ms with sets of 1 or
// 8 tiles, 209 with 32, vs 179 in 3 launches (profiles/r2_ab_deal_block.txt).
constexpr int kDealBlock = 1;
int deal_block() {
    static const int b = [] {
        const char* e = getenv("GJ_DEAL_BLOCK");
        const int v = e ? atoi(e) : 0;
        return v >= 1 ? v : kDealBlock;
    }();
    return b;
}

void query_sets(int64_t T, int64_t first, int64_t step, JoinArgs* a) {
    const int64_t B = deal_block();
    const int64_t U = (T + B - 1) / B;   // query sets
    a->blk = (int32_t)B;
    a->first = first;
    a->step = step;
    const int64_t nu = first < U ? (U - first + step - 1) / step : 0;
    a->n_tiles = nu * B;
    if (nu > 0 && first + step * (nu - 1) == U - 1) a->n_tiles -= U * B - T;   // the last set is partial
}

void batch_tiles(const Index* ix, int32_t batch, int32_t n_batches, int32_t rank, int32_t world, JoinArgs* a) {
    // entity partitioning (§6.2): query set l -> rank l mod |p|; batch (l div |p|) mod n_b
    query_sets(ix->T, (int64_t)rank + (int64_t)world * batch, (int64_t)world * n_batches, a);
}

// Work-balanced split plan of one launch: a tile whose estimated work
// (queries x candidates) exceeds W / (148 x 8) of the launch's total W is
// scanned by ceil(work / that) CTAs (each 1/parts of every candidate window),
// so a batch never waits on one heavy tile (clustered data: a few dense cells
// carry most of the work, and round-robin batching puts one in every batch).
// Returns false when every tile gets one CTA.
static bool plan_parts(const Index* ix, const JoinArgs& a, std::vector<uint32_t>* off) {
    if (a.n_tiles <= 0 || a.split > 1 || ix->h_work_by_pos.size() != (size_t)ix->T) return false;
    double W = 0.0, wmax = 0.0;
    for (int64_t m = 0; m < a.n_tiles; ++m) {
        const double w = (double)ix->h_work_by_pos[(size_t)tile_pos(a, m)];
        W += w;
        wmax = w > wmax ? w : wmax;
    }
    // parts of about 1 / (148 x div) of the launch's work: div = 4 for the
    // tcgen05 kernels, whose persistent CTAs take items from a counter (coarse
    // first parts, the guided sizing below refines the tail; expo32 8-rank
    // projection 0.84-0.85 vs 0.83-0.84 with 8), div = 8 for the SIMT kernels
    // whose CTAs are dispatched once per item (songs90 FP32 join 13.4 ms vs 17.9
    // with 4; profiles/r2_ab_plan_div_persistent.txt).  GJ_PLAN_DIV overrides
    // both (timing experiments, read once).
    static const double env_div = [] {
        const char* e = getenv("GJ_PLAN_DIV");
        const double v = e ? atof(e) : 0.0;
        return v > 0.0 ? v : 0.0;
    }();
    const double div = env_div > 0.0 ? env_div : (ix->filter == 2 ? 4.0 : 8.0);
    const double target = W / (148.0 * div);
    if (!(target > 0.0) || wmax <= target) return false;
    // Guided self-scheduling (items are taken in order: the persistent tcgen05
    // kernels pull them from a counter, the others are dispatched in CTA
    // order): a tile's parts are sized by the work still to come,
    // target_m = max(R_m / (148 x div), target / 16), so the last items of a
    // launch are small and the CTAs finish together (expo32 dealt into 24
    // launches: 8.2 vs 8.6 ms per launch; GJ_PLAN_GUIDED=0 turns it off).
    static const bool guided = [] {
        const char* e = getenv("GJ_PLAN_GUIDED");
        return !e || atoi(e) != 0;
    }();
    off->resize((size_t)a.n_tiles + 1);
    uint64_t acc = 0;
    double R = W;   // work of tiles m.. of this launch
    for (int64_t m = 0; m < a.n_tiles; ++m) {
        (*off)[(size_t)m] = (uint32_t)acc;
        const double w = (double)ix->h_work_by_pos[(size_t)tile_pos(a, m)];
        const double t = guided ? std::max(R / (148.0 * div), target / 16.0) : target;
        acc += (uint64_t)std::min(512.0, std::max(1.0, std::ceil(w / t)));
        R -= w;
    }
    (*off)[(size_t)a.n_tiles] = (uint32_t)acc;
    return true;
}

static int launch_join_planned(const Index* ix, JoinMode mode, const JoinArgs& a, cudaStream_t s);

int launch_join(const Index* ix, JoinMode mode, const JoinArgs& a0, cudaStream_t s) {
    std::vector<uint32_t> off;
    if (mode == kStats || a0.part_off || !plan_parts(ix, a0, &off)) return launch_join_planned(ix, mode, a0, s);
    JoinArgs a = a0;
    uint32_t* d_off = nullptr;
    GJ_CUDA(pool_malloc(&d_off, off.size() * sizeof(uint32_t), s));
    // pageable source: the copy is staged before the call returns
    GJ_CUDA(cudaMemcpyAsync(d_off, off.data(), off.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    a.part_off = d_off;
    a.total_parts = (int64_t)off.back();
    const int rc = launch_join_planned(ix, mode, a, s);
    GJ_CUDA(cudaFreeAsync(d_off, s));
    return rc;
}

static int launch_join_planned(const Index* ix, JoinMode mode, const JoinArgs& a, cudaStream_t s) {
    if (ix->filter == 2 && mode != kStats) return launch_join_umma(ix, mode, a, s);
    if (ix->filter == 1 && mode != kStats) return launch_join32(ix, mode, a, s);
    const Params p = join_params(ix);
    const int np = ix->n_pad;
    const bool sym = ix->opt.symmetric != 0;
    if (np <= 8) return launch_np<8>(p, mode, a, sym, s);
    if (np <= 16) return launch_np<16>(p, mode, a, sym, s);
    if (np <= 24) return launch_np<24>(p, mode, a, sym, s);
    if (np <= 32) return launch_np<32>(p, mode, a, sym, s);
    if (np <= 48) return launch_np<48>(p, mode, a, sym, s);
    if (np <= 64) return launch_np<64>(p, mode, a, sym, s);
    if (np <= 96) return launch_np<96>(p, mode, a, sym, s);
    return launch_np<128>(p, mode, a, sym, s);
}

}  // namespace gj
