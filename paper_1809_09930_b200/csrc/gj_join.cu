// SelfJoinKernel (Alg. 1 l.596-607) for sm_100a.
//
// One CTA = one query tile: up to 128 consecutive sorted points of ONE
// non-empty cell A (so the whole CTA shares getAdjCells' result, computed
// once per cell at index build).  One thread = one query point, its n
// coordinates held in registers.  For every adjacent non-empty cell B the CTA
// streams B's candidates through shared memory in coalesced double2 chunks;
// every thread tests its query against every staged candidate:
//   SORTIDU (§4.3): the staged range is the union of the tile's u-windows,
//     found by binary search in B's u-sorted run; each thread then applies
//     its own window |p(u) - q(u)| <= eps exactly.
//   SHORTC (§4.4): the squared-distance sum is accumulated in dimension
//     order (highest variance first after REORDER) and abandoned as soon as
//     it exceeds eps^2 (checked every 4 dims; stats mode: every dim).
// Pairs are emitted with one warp-aggregated atomic per candidate that hit in
// at least one lane (ballot -> leader atomicAdd -> shfl -> per-lane store).
//
// No tensor cores: the candidate work is a filtered gather with a
// data-dependent early exit, not a dense contraction (north_star).
#include "gj_internal.cuh"

namespace gj {
namespace {

struct Params {
    const double* __restrict__ pts;
    const uint32_t* __restrict__ orig;
    const uint32_t* __restrict__ cell_start;
    const uint32_t* __restrict__ nbr_off;
    const uint32_t* __restrict__ nbr;
    const uint32_t* __restrict__ tile_cell;
    const uint32_t* __restrict__ tile_q0;
    const uint32_t* __restrict__ tile_order;
    int n, n_pad, u, sortidu, shortc;
    double eps, eps2;
};

constexpr int kSmemDoubles = 4096;   // 32 KB candidate stage

template <int NPR, int MODE>
__global__ void __launch_bounds__(kTileQ) k_join(Params P, JoinArgs A) {
    constexpr int TC = kSmemDoubles / NPR;
    __shared__ __align__(16) double Cs[kSmemDoubles];
    __shared__ uint32_t Cid[TC];
    __shared__ uint32_t s_win[2];
    __shared__ unsigned long long s_red[4][kTileQ / 32];

    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t j = A.first + A.step * (int64_t)blockIdx.x;
    const uint32_t tile = P.tile_order[j];
    const uint32_t g = P.tile_cell[tile];
    const uint32_t q0 = P.tile_q0[tile];
    const uint32_t nq = min((uint32_t)kTileQ, P.cell_start[g + 1] - q0);
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

    uint64_t c_cells = 0, c_tests = 0, c_dims = 0, c_pairs = 0;
    const uint32_t nb0 = P.nbr_off[g], nb1 = P.nbr_off[g + 1];
    for (uint32_t b = nb0; b < nb1; ++b) {
        const uint32_t B = P.nbr[b];
        uint32_t r = P.cell_start[B], s = P.cell_start[B + 1];
        if (P.sortidu) {
            __syncthreads();
            if (tid < 2) {   // lane 0: first r with u_lo - r(u) <= eps; lane 1: first s with s(u) - u_hi > eps
                uint32_t lo = r, hi = s;
                while (lo < hi) {
                    uint32_t mid = (lo + hi) >> 1;
                    double cu = P.pts[(size_t)mid * n_pad + P.u];
                    bool pred = tid == 0 ? (u_lo - cu <= eps) : (cu - u_hi > eps);
                    if (pred) hi = mid; else lo = mid + 1;
                }
                s_win[tid] = lo;
            }
            __syncthreads();
            r = s_win[0];
            s = max(s_win[1], r);
        }
        if (MODE == kStats && active) ++c_cells;
        for (uint32_t cb = r; cb < s; cb += TC) {
            const int cnt = (int)min((uint32_t)TC, s - cb);
            __syncthreads();
            {
                const double2* src = reinterpret_cast<const double2*>(P.pts + (size_t)cb * n_pad);
                double2* dst = reinterpret_cast<double2*>(Cs);
                const int nv = cnt * n_pad / 2;
                for (int i = tid; i < nv; i += kTileQ) dst[i] = src[i];
                for (int i = tid; i < cnt; i += kTileQ) Cid[i] = P.orig[cb + i];
            }
            __syncthreads();
            for (int c = 0; c < cnt; ++c) {
                const double* cp = Cs + c * n_pad;
                bool ok = active;
                if (P.sortidu) {
                    const double cu = cp[P.u];
                    ok = ok && (qu - cu <= eps) && (cu - qu <= eps);
                }
                double acc = 0.0;
                if (ok) {
                    if (MODE == kStats) {
                        ++c_tests;
                        int used = 0;
#pragma unroll
                        for (int d = 0; d < NPR; ++d) {
                            if (d >= P.n) break;
                            // unfused, in dimension order: the oracle's arithmetic
                            const double t = __dsub_rn(q[d], cp[d]);
                            acc = __dadd_rn(acc, __dmul_rn(t, t));
                            ++used;
                            if (acc > eps2) break;
                        }
                        c_dims += used;
                    } else {
#pragma unroll
                        for (int d = 0; d < NPR; d += 4) {
                            if (d >= n_pad) break;
                            const double2 a = *reinterpret_cast<const double2*>(cp + d);
                            const double2 b2 = *reinterpret_cast<const double2*>(cp + d + 2);
                            double t0 = q[d] - a.x, t1 = q[d + 1] - a.y, t2 = q[d + 2] - b2.x, t3 = q[d + 3] - b2.y;
                            acc = fma(t0, t0, acc);
                            acc = fma(t1, t1, acc);
                            acc = fma(t2, t2, acc);
                            acc = fma(t3, t3, acc);
                            if (P.shortc && acc > eps2) break;
                        }
                    }
                }
                const bool hit = ok && acc <= eps2;
                if (MODE == kEmit) {
                    const unsigned m = __ballot_sync(0xffffffffu, hit);
                    if (m) {
                        const int leader = __ffs(m) - 1;
                        unsigned long long base = 0;
                        if (lane == leader) base = atomicAdd((unsigned long long*)A.count, (unsigned long long)__popc(m));
                        base = __shfl_sync(0xffffffffu, base, leader);
                        if (hit) {
                            const unsigned long long at = base + __popc(m & ((1u << lane) - 1u));
                            if (at < A.cap) reinterpret_cast<uint2*>(A.out)[at] = make_uint2(qid, Cid[c]);
                        }
                    }
                } else {
                    c_pairs += hit;
                }
            }
        }
    }
    if (MODE != kEmit) {
        unsigned long long v[4] = {c_pairs, c_cells, c_tests, c_dims};
        const int nv = MODE == kStats ? 4 : 1;
        for (int i = 0; i < nv; ++i) {
            unsigned long long x = v[i];
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
        if (MODE == kCount && tid == 0) atomicAdd((unsigned long long*)A.count + 1, (unsigned long long)nq);
    }
}

template <int NPR>
int launch_np(const Params& p, JoinMode mode, const JoinArgs& a, cudaStream_t s) {
    if (a.n_tiles <= 0) return GJ_OK;
    dim3 grid((unsigned)a.n_tiles);
    if (mode == kEmit) k_join<NPR, kEmit><<<grid, kTileQ, 0, s>>>(p, a);
    else if (mode == kCount) k_join<NPR, kCount><<<grid, kTileQ, 0, s>>>(p, a);
    else k_join<NPR, kStats><<<grid, kTileQ, 0, s>>>(p, a);
    count_launch();
    GJ_CUDA(cudaGetLastError());
    return GJ_OK;
}

}  // namespace

void batch_tiles(const Index* ix, int32_t batch, int32_t n_batches, int32_t rank, int32_t world, JoinArgs* a) {
    // entity partitioning (§6.2): position j -> rank j mod |p|; batch (j div |p|) mod n_b
    a->first = (int64_t)rank + (int64_t)world * batch;
    a->step = (int64_t)world * n_batches;
    a->n_tiles = a->first < ix->T ? (ix->T - a->first + a->step - 1) / a->step : 0;
}

int launch_join(const Index* ix, JoinMode mode, const JoinArgs& a, cudaStream_t s) {
    Params p;
    p.pts = ix->pts;
    p.orig = ix->orig;
    p.cell_start = ix->cell_start;
    p.nbr_off = ix->nbr_off;
    p.nbr = ix->nbr;
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
    const int np = ix->n_pad;
    if (np <= 8) return launch_np<8>(p, mode, a, s);
    if (np <= 16) return launch_np<16>(p, mode, a, s);
    if (np <= 24) return launch_np<24>(p, mode, a, s);
    if (np <= 32) return launch_np<32>(p, mode, a, s);
    if (np <= 48) return launch_np<48>(p, mode, a, s);
    if (np <= 64) return launch_np<64>(p, mode, a, s);
    if (np <= 96) return launch_np<96>(p, mode, a, s);
    return launch_np<128>(p, mode, a, s);
}

}  // namespace gj
