// constructIndex on the device (Alg. 1 l.581-582).
//
//  1. per-dim min/max over D and variance over the 1% sample (§4.2 l.498)
//  2. REORDER permutation by non-increasing variance, grid geometry over the
//     first k reordered dims (§4.1 l.252), overflow check of the linear id
//  3. per point: linearised cell id (§3.2.1 l.122, row-major) and the SORTIDU
//     key of the un-indexed dim u (§4.3 l.514)
//  4. stable device radix sort by u, then by cell id -> points grouped by cell,
//     u-sorted within each cell (§3.2.1 "lookup array"; §4.3 sort)
//  5. gather of the reordered, sorted point array (row stride n_pad)
//  6. non-empty cell array (ids + starts), |G| (§3.2.1 l.119, l.122)
//  7. adjacent non-empty cells of every cell: 3^k offsets located by binary
//     search (§3.2.1 l.185, §5.6 l.896), CSR
//  8. query tiles (<= 128 queries of one cell) with their candidate count,
//     ordered heaviest first for load balance (§6.2 entity partitioning).
//
// Readings: R2 cell_j = floor(x_j/eps) - floor(min_j/eps);
// R6 sample = every round(1/f)-th point, unbiased variance, ties -> lower dim;
// R7 u = position k if k < n else 0; R9 first indexed dim most significant.
#include <math.h>
#include <string.h>

#include <cmath>

#include <algorithm>
#include <mutex>
#include <vector>

#include "gj_internal.cuh"

namespace gj {
namespace {

enum ColMode { kMinMax = 0, kSum = 1, kSqDev = 2 };

// Column reduction over rows r = i * rstride, i in [0, m).  Block size is a
// multiple of n so each thread owns one column; partials are [block][n]
// (and [block][n] for the max in kMinMax mode at part2).
__global__ void k_col_reduce(const double* __restrict__ X, int64_t m, int64_t rstride, int n, int mode,
                             const double* __restrict__ mean, double* __restrict__ part,
                             double* __restrict__ part2) {
    extern __shared__ double sh[];
    const int rpb = blockDim.x / n;
    const int j = threadIdx.x % n, rl = threadIdx.x / n;
    double a = mode == kMinMax ? INFINITY : 0.0, b = -INFINITY;
    const double mu = mode == kSqDev ? mean[j] : 0.0;
    for (int64_t i = (int64_t)blockIdx.x * rpb + rl; i < m; i += (int64_t)gridDim.x * rpb) {
        double x = X[i * rstride * n + j];
        if (mode == kMinMax) {
            a = fmin(a, x);
            b = fmax(b, x);
        } else if (mode == kSum) {
            a += x;
        } else {
            double d = x - mu;
            a += d * d;
        }
    }
    double* sa = sh;
    double* sb = sh + blockDim.x;
    sa[threadIdx.x] = a;
    sb[threadIdx.x] = b;
    __syncthreads();
    if (rl == 0) {
        for (int r = 1; r < rpb; ++r) {
            if (mode == kMinMax) {
                a = fmin(a, sa[r * n + j]);
                b = fmax(b, sb[r * n + j]);
            } else {
                a += sa[r * n + j];
            }
        }
        part[(int64_t)blockIdx.x * n + j] = a;
        if (mode == kMinMax) part2[(int64_t)blockIdx.x * n + j] = b;
    }
}

// Deterministic reduction of the block partials: one CTA per column, each
// thread folds a fixed strided subset, then a fixed-shape tree (the result
// does not depend on scheduling).
__global__ void __launch_bounds__(256) k_col_final(const double* __restrict__ part, const double* __restrict__ part2,
                                                  int nb, int n, int mode, int64_t m, double* __restrict__ outa,
                                                  double* __restrict__ outb) {
    __shared__ double sa[256], sb[256];
    const int j = blockIdx.x, t = threadIdx.x;
    double a = mode == kMinMax ? INFINITY : 0.0, b = -INFINITY;
    for (int i = t; i < nb; i += 256) {
        if (mode == kMinMax) {
            a = fmin(a, part[(int64_t)i * n + j]);
            b = fmax(b, part2[(int64_t)i * n + j]);
        } else {
            a += part[(int64_t)i * n + j];
        }
    }
    sa[t] = a;
    sb[t] = b;
    __syncthreads();
    for (int w = 128; w >= 1; w >>= 1) {
        if (t < w) {
            if (mode == kMinMax) {
                sa[t] = fmin(sa[t], sa[t + w]);
                sb[t] = fmax(sb[t], sb[t + w]);
            } else {
                sa[t] += sa[t + w];
            }
        }
        __syncthreads();
    }
    if (t != 0) return;
    a = sa[0];
    b = sb[0];
    if (mode == kMinMax) {
        outa[j] = a;
        outb[j] = b;
    } else if (mode == kSum) {
        outa[j] = a / (double)m;          // sample mean
    } else {
        outa[j] = m > 1 ? a / (double)(m - 1) : 0.0;   // unbiased sample variance
    }
}

// REORDER permutation + grid geometry (single block).
__global__ void k_meta(Meta* meta, int n, int k, double eps, int reorder) {
    const int t = threadIdx.x;
    if (t < n) {
        int rank = t;
        if (reorder) {
            double v = meta->var[t];
            rank = 0;
            for (int i = 0; i < n; ++i) {
                double w = meta->var[i];
                rank += (w > v) || (w == v && i < t);
            }
        }
        meta->order[rank] = t;
    }
    __syncthreads();
    if (t == 0) {
        int overflow = 0;
        double prod = 1.0;
        for (int d = 0; d < k; ++d) {
            int o = meta->order[d];
            double fb = floor(meta->mins[o] / eps), fm = floor(meta->maxs[o] / eps);
            if (!(fabs(fb) < 4.0e18) || !(fabs(fm) < 4.0e18)) overflow = 1;
            int64_t b = overflow ? 0 : (int64_t)fb;
            int64_t w = overflow ? 1 : (int64_t)fm - b + 1;
            meta->base[d] = b;
            meta->width[d] = w;
            prod *= (double)w;
        }
        if (prod >= 9.2e18) overflow = 1;
        uint64_t s = 1;
        for (int d = k - 1; d >= 0; --d) {
            meta->stride[d] = s;
            s *= (uint64_t)meta->width[d];
        }
        meta->overflow = overflow;
    }
}

__device__ __forceinline__ uint64_t order_key(double x) {
    uint64_t b = (uint64_t)__double_as_longlong(x + 0.0);   // -0.0 -> +0.0
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void k_cell_keys(const double* __restrict__ X, int64_t N, int n, int k, int u, double eps,
                            const Meta* __restrict__ meta, uint64_t* __restrict__ cellkey,
                            uint64_t* __restrict__ ukey, uint32_t* __restrict__ idx) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const double* x = X + i * n;
    uint64_t lin = 0;
    for (int d = 0; d < k; ++d) {
        int o = meta->order[d];
        int64_t c = (int64_t)floor(x[o] / eps) - meta->base[d];
        lin += (uint64_t)c * meta->stride[d];
    }
    cellkey[i] = lin;
    ukey[i] = order_key(x[meta->order[u]]);
    idx[i] = (uint32_t)i;
}

__global__ void k_gather_u64(const uint64_t* __restrict__ src, const uint32_t* __restrict__ idx, int64_t N,
                             uint64_t* __restrict__ dst) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < N) dst[i] = src[idx[i]];
}

// pts[p][t] = X[idx[p]][order[t]] (0 for t >= n); one thread per output element.
// pts32 (optional): the same coordinate centred on the dimension minimum and
// rounded to float32, fl32(x - min) -- input of the certified FP32 prefilter.
// pts[p][t] = X[idx[p]][order[t]] (0 in the padding columns): one warp per
// sorted row, lane t writes dims t, t + 32, ... (coalesced 256-byte rows, no
// per-element 64-bit division).
__global__ void k_gather_points(const double* __restrict__ X, const uint32_t* __restrict__ idx, int64_t N,
                                int n, int n_pad, const Meta* __restrict__ meta, double* __restrict__ pts,
                                float* __restrict__ pts32) {
    __shared__ int ord[kMaxDim];
    __shared__ double mn[kMaxDim];
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
        ord[t] = meta->order[t];
        mn[t] = meta->mins[ord[t]];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t p = w0; p < N; p += nw) {
        const double* src = X + (int64_t)idx[p] * n;
        double* dst = pts + p * n_pad;
        for (int t = lane; t < n_pad; t += 32) {
            const double x = t < n ? src[ord[t]] : 0.0;
            dst[t] = x;
            if (pts32) pts32[p * n_pad + t] = t < n ? __double2float_rn(x - mn[t]) : 0.0f;
        }
    }
}

// pts32[p][t] = fl32(pts[p][t] - min_t) (reordered dims), 0 in the padding columns.
__global__ void k_make32(const double* __restrict__ pts, int64_t N, int n, int n_pad, const Meta* __restrict__ meta,
                         float* __restrict__ pts32) {
    __shared__ double mn[kMaxDim];
    for (int t = threadIdx.x; t < n; t += blockDim.x) mn[t] = meta->mins[meta->order[t]];
    __syncthreads();
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= N * n_pad) return;
    const int t = (int)(e % n_pad);
    pts32[e] = t < n ? __double2float_rn(pts[e] - mn[t]) : 0.0f;
}

__global__ void k_heads(const uint64_t* __restrict__ key, int64_t N, uint32_t* __restrict__ head) {
    int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p < N) head[p] = (p == 0 || key[p] != key[p - 1]) ? 1u : 0u;
}

__global__ void k_cells(const uint64_t* __restrict__ key, const uint32_t* __restrict__ head,
                        const uint32_t* __restrict__ pos, int64_t N, uint64_t* __restrict__ cell_id,
                        uint32_t* __restrict__ cell_start, int64_t G) {
    int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p < N && head[p]) {
        cell_id[pos[p]] = key[p];
        cell_start[pos[p]] = (uint32_t)p;
    }
    if (p == 0) cell_start[G] = (uint32_t)N;
}

// Adjacent non-empty cells (getAdjCells, Alg. 1 l.600; §5.6 l.896 "perform a
// binary search to find the non-empty cells that exist in the index").
//
// The linear ids are row-major with the first indexed dimension most
// significant (R9), so the non-empty cells sharing a coordinate prefix form a
// contiguous range of the sorted id array.  One warp per cell: lane l takes
// the l-th of the 3^m (m = min(k, 3)) offsets of the first m dimensions and
// locates its prefix range by binary search; it then walks the remaining
// offsets depth first, each child range found by binary search INSIDE its
// parent's range, and an empty range prunes the whole subtree.  On sparse
// grids (Songs-shaped data at k = 8: 3^8 = 6561 offsets per cell, few
// non-empty) almost every subtree is pruned near the root, where the flat
// enumeration paid one full-array binary search per offset; the results (and
// their order) are the same.  FILL=false: counts + candidate sums (all
// adjacent cells; and only cells with a larger index, for symmetric
// evaluation); FILL=true: CSR in increasing cell index (lanes in prefix
// order, each lane's walk in increasing id order) + the position of the cell
// itself in its own list.
__device__ __forceinline__ uint32_t lower_bound_u64(const uint64_t* __restrict__ a, uint32_t lo, uint32_t hi,
                                                    uint64_t key) {
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// Depth-first walk of lane's prefix subtree; calls f(hit index) in increasing id order.
template <typename F>
__device__ __forceinline__ void adj_walk(const uint64_t* __restrict__ cell_id, uint32_t lo0, uint32_t hi0,
                                         uint64_t base0, int m, int k, const int64_t* c, const int64_t* w,
                                         const uint64_t* st, F&& f) {
    uint32_t lo_s[kMaxK + 1], hi_s[kMaxK + 1];
    uint64_t base_s[kMaxK + 1];
    int64_t nx[kMaxK + 1];
    int depth = m;
    lo_s[m] = lo0;
    hi_s[m] = hi0;
    base_s[m] = base0;
    if (m < k) nx[m] = c[m] - 1;
    while (depth >= m) {
        if (depth == k) {   // a leaf: the range holds exactly the one cell with this id
            if (lo_s[k] < hi_s[k]) f(lo_s[k]);
            --depth;
            continue;
        }
        if (nx[depth] > c[depth] + 1) {
            --depth;
            continue;
        }
        const int64_t x = nx[depth]++;
        if (x < 0 || x >= w[depth]) continue;
        const uint64_t cb = base_s[depth] + (uint64_t)x * st[depth];
        const uint32_t clo = lower_bound_u64(cell_id, lo_s[depth], hi_s[depth], cb);
        const uint32_t chi = lower_bound_u64(cell_id, clo, hi_s[depth], cb + st[depth]);
        if (clo == chi) continue;   // no non-empty cell below: prune the subtree
        ++depth;
        lo_s[depth] = clo;
        hi_s[depth] = chi;
        base_s[depth] = cb;
        if (depth < k) nx[depth] = c[depth] - 1;
    }
}

template <bool FILL>
__global__ void k_adjacent(const uint64_t* __restrict__ cell_id, const uint32_t* __restrict__ cell_start,
                           int64_t G, int k, const Meta* __restrict__ meta, uint32_t* __restrict__ cnt,
                           uint64_t* __restrict__ cand, uint64_t* __restrict__ cand_after,
                           const uint32_t* __restrict__ off, uint32_t* __restrict__ nbr,
                           uint32_t* __restrict__ nbr_self) {
    __shared__ int64_t s_w[kMaxK];
    __shared__ uint64_t s_s[kMaxK];
    if (threadIdx.x < k) {
        s_w[threadIdx.x] = meta->width[threadIdx.x];
        s_s[threadIdx.x] = meta->stride[threadIdx.x];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (g >= G) return;
    const uint64_t lin = cell_id[g];
    int64_t c[kMaxK], w[kMaxK];
    uint64_t st[kMaxK];
    for (int d = 0; d < k; ++d) {
        w[d] = s_w[d];
        st[d] = s_s[d];
        c[d] = (int64_t)((lin / st[d]) % (uint64_t)w[d]);
    }
    // lane's prefix: offsets of the first m dims from the lane id, base 3, first dim most significant
    const int m = k < 3 ? k : 3;
    int np = 1;
    for (int d = 0; d < m; ++d) np *= 3;
    bool ok = lane < np;
    uint64_t base = 0;
    {
        int r = lane, div = np / 3;
        for (int d = 0; d < m; ++d) {
            const int64_t x = c[d] + (ok ? (r / div) : 1) - 1;
            r %= div;
            div /= 3;
            if (x < 0 || x >= w[d]) ok = false;
            base += (uint64_t)(ok ? x : 0) * st[d];
        }
    }
    uint32_t plo = 0, phi = 0;
    if (ok) {
        plo = lower_bound_u64(cell_id, 0, (uint32_t)G, base);
        phi = lower_bound_u64(cell_id, plo, (uint32_t)G, base + st[m - 1]);
    }
    uint32_t found = 0;
    uint64_t csum = 0, casum = 0;
    if (plo < phi)
        adj_walk(cell_id, plo, phi, base, m, k, c, w, st, [&](uint32_t hit) {
            ++found;
            if (!FILL) {
                const uint64_t sz = cell_start[hit + 1] - cell_start[hit];
                csum += sz;
                if ((int64_t)hit > g) casum += sz;
            }
        });
    if (!FILL) {
#pragma unroll
        for (int s = 16; s; s >>= 1) {
            found += __shfl_xor_sync(0xffffffffu, found, s);
            csum += __shfl_xor_sync(0xffffffffu, csum, s);
            casum += __shfl_xor_sync(0xffffffffu, casum, s);
        }
        if (lane == 0) {
            cnt[g] = found;
            cand[g] = csum;
            cand_after[g] = casum;
        }
        return;
    }
    // exclusive scan of the lanes' counts: lane order = prefix order = id order
    uint32_t incl = found;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, s);
        if (lane >= s) incl += y;
    }
    uint32_t wpos = off[g] + incl - found;
    if (plo < phi)
        adj_walk(cell_id, plo, phi, base, m, k, c, w, st, [&](uint32_t hit) {
            nbr[wpos] = hit;
            if ((int64_t)hit == g) nbr_self[g] = wpos;
            ++wpos;
        });
}

__global__ void k_tile_count(const uint32_t* __restrict__ cell_start, int64_t G, uint32_t tq, uint32_t* __restrict__ nt) {
    int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g < G) nt[g] = (cell_start[g + 1] - cell_start[g] + tq - 1) / tq;
}

// One thread per TILE (a cell's tiles are consecutive from toff[g]; every
// non-empty cell has at least one, so toff is strictly increasing): the few
// huge cells of skewed data no longer serialise thousands of tiles on one thread.
__global__ void k_tile_fill(const uint32_t* __restrict__ cell_start, const uint32_t* __restrict__ toff,
                            const uint64_t* __restrict__ cand, const uint64_t* __restrict__ cand_after, int sym,
                            int64_t G, int64_t T, uint32_t tq, uint32_t* __restrict__ tile_cell,
                            uint32_t* __restrict__ tile_q0, uint64_t* __restrict__ tile_work,
                            uint64_t* __restrict__ sort_key, uint32_t* __restrict__ sort_val,
                            unsigned long long* __restrict__ total) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long tot = 0;
    if (t < T) {
        int64_t lo = 0, hi = G;   // last g with toff[g] <= t
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if ((int64_t)toff[mid] <= t) lo = mid; else hi = mid;
        }
        const int64_t g = lo;
        const uint32_t a = cell_start[g], b = cell_start[g + 1];
        const uint32_t q = a + (uint32_t)(t - (int64_t)toff[g]) * tq;
        const uint32_t nq = min(tq, b - q);
        // candidate tests of the tile: all adjacent points per query, or (symmetric)
        // points of later cells plus the later points of the own cell
        const uint64_t w = sym ? (uint64_t)nq * (cand_after[g] + (b - q)) - (uint64_t)nq * (nq + 1) / 2
                               : (uint64_t)nq * cand[g];
        tile_cell[t] = (uint32_t)g;
        tile_q0[t] = q;
        tile_work[t] = w;
        sort_key[t] = ~w;   // descending work
        sort_val[t] = (uint32_t)t;
        tot = (unsigned long long)nq * cand[g];   // queries x candidates (pre-SORTIDU) of the tile
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if ((threadIdx.x & 31) == 0 && tot) atomicAdd(total, tot);
}

int col_reduce(const double* X, int64_t m, int64_t rstride, int n, int mode, const double* mean, double* outa,
               double* outb, cudaStream_t s) {
    int rpb = std::max(1, 256 / n);
    int bs = rpb * n;
    int64_t need = (m + rpb - 1) / rpb;
    int nb = (int)std::max<int64_t>(1, std::min<int64_t>(need, 592));
    double* part = nullptr;
    GJ_CUDA(pool_malloc(&part, 2 * (size_t)nb * n * sizeof(double), s));
    k_col_reduce<<<nb, bs, 2 * bs * sizeof(double), s>>>(X, m, rstride, n, mode, mean, part, part + (size_t)nb * n); count_launch();
    k_col_final<<<n, 256, 0, s>>>(part, part + (size_t)nb * n, nb, n, mode, m, outa, outb); count_launch();
    GJ_CUDA(cudaGetLastError());
    GJ_CUDA(cudaFreeAsync(part, s));
    return GJ_OK;
}

inline unsigned blocks_for(int64_t n, int bs) { return (unsigned)((n + bs - 1) / bs); }

// Threshold of the certified FP32 prefilter (DESIGN.md §"FP32 prefilter").
// With x' = fl32(x - min_j), s_j = max_j - min_j, u = 2^-24:
//   |fl32(q'_j - c'_j) - (q_j - c_j)| <= a_j = 4.001 u s_j          (per dim)
//   ||delta~|| >= ||delta|| - A,  A = ||a|| (+ a subnormal slack)
//   fp32 recursive FMA sum S~_k of k <= n squares: S~_k <= (1 + gamma_n) sum_all delta~^2
// so S~_k > T = (1 + gamma_n) (eps (1 + 1e-9) + A)^2 proves ||delta|| > eps (1 + 1e-9):
// the pair is outside eps and outside the 1e-12 ambiguity band.  Every pair the
// filter does not reject is decided by the FP64 test.  The filter is switched
// off when it could not reject much (A > 1e-3 eps) or fp32 could overflow.
}  // namespace

int fp32_threshold_from_spans(double eps, int n, const double* spans, float* thr, double* margin) {
    double ss = 0.0, smax = 0.0;
    for (int t = 0; t < n; ++t) {
        ss += spans[t] * spans[t];
        smax = std::max(smax, spans[t]);
    }
    const double u = std::ldexp(1.0, -24);
    const double A = 4.001 * u * std::sqrt(ss) * (1.0 + 1e-12) + std::sqrt((double)n) * std::ldexp(1.0, -147);
    const double gamma = n * u / (1.0 - n * u);
    const double T = (1.0 + gamma) * (eps * (1.0 + 1e-9) + A) * (eps * (1.0 + 1e-9) + A);
    float T32 = (float)T;
    if ((double)T32 < T) T32 = std::nextafter(T32, INFINITY);
    *margin = T / (eps * eps) - 1.0;
    *thr = T32;
    return (smax < 1e30) && (T32 < 1e30f) && !(A > 1e-3 * eps);
}

float fp32_accept_threshold_from_spans(double eps, int n, const double* spans) {
    // Certain-inside side of the same analysis: the float32 running sum is
    // >= (1 - gamma_n) ||t||^2 and ||q - c|| <= ||t|| + A, so a final sum
    // <= (1 - gamma_n)(eps (1 - 1e-9) - A)^2 proves dist <= eps (1 - 1e-9): the
    // FP64 test would accept it too.  Rounded down; -1 (never) if A >= eps.
    double ss = 0.0;
    for (int t = 0; t < n; ++t) ss += spans[t] * spans[t];
    const double u = std::ldexp(1.0, -24);
    const double A = 4.001 * u * std::sqrt(ss) * (1.0 + 1e-12) + std::sqrt((double)n) * std::ldexp(1.0, -147);
    const double gamma = n * u / (1.0 - n * u);
    const double r = eps * (1.0 - 1e-9) - A;
    if (!(r > 0.0) || !std::isfinite(r)) return -1.0f;
    const double T = (1.0 - gamma) * r * r;
    float T32 = (float)T;
    if ((double)T32 > T) T32 = std::nextafter(T32, -INFINITY);
    return T32;
}

static bool fp32_threshold(Index* ix) {
    const Meta& m = ix->h_meta;
    double spans[kMaxDim];
    for (int t = 0; t < ix->n; ++t) spans[t] = m.maxs[m.order[t]] - m.mins[m.order[t]];
    ix->thr32_in = fp32_accept_threshold_from_spans(ix->eps, ix->n, spans);
    return fp32_threshold_from_spans(ix->eps, ix->n, spans, &ix->thr32, &ix->filter_margin) != 0;
}

// Threshold of the certified tensor-core bound (gj_join_umma.cu;
// DESIGN.md §"Tensor-core bound").  Operands: x^ = fp16(S (x - min)) for the
// n coordinates, R2 = max ||x^||^2, K = padded MMA depth (n + 4 augmented
// columns, rounded up to 16).  A query row carries (r_hi, r_lo, 1, 1) and a
// candidate row (1, 1, h_hi, h_lo) in the augmented columns, with
// r = (T - ||q^||^2)/2 and h = -||c^||^2/2 split into fp16 hi + lo, so the
// tensor core accumulates acc = q^.c^ + r + h = (T - ||q^ - c^||^2)/2 (+ err).
//   err   <= a + b T,  a = kappa (2.001 R2) + 2^-22 R2 + 2^-23 + 2^-51 R2,
//                      b = 0.5005 kappa + 2^-23 + 2^-51,
//            kappa = (K + 2) 2^-21 (4x a truncating fp32 adder, products exact),
//            2^-22 |r|, 2^-22 |h| from the hi/lo splits
//   delta : | ||q^ - c^|| - S ||q - c|| | <= 2^-11 (||q'|| + ||c'||) + sqrt(n) 2^-24
// A pair is rejected iff acc <= 0 (sign bit set), which implies
// ||q^ - c^||^2 >= T - 2 err, hence S||q - c|| >= sqrt(T - 2 err) - delta, so with
//   T = ((S eps (1 + 1e-9) + delta)^2 + 2a) / (1 - 2b)
// every rejected pair has ||q - c|| >= eps (1 + 1e-9).  Enabled when the
// relative slack T / (S eps)^2 - 1 < 0.25.
int tc_threshold_from(double eps, int n, int K, double S, double R2, double* thr, double* margin) {
    const double u11 = std::ldexp(1.0, -11);
    const double R = std::sqrt(R2);
    const double Rp = (R + std::sqrt((double)n) * std::ldexp(1.0, -25)) / (1.0 - u11);
    const double delta = u11 * 2.0 * Rp + std::sqrt((double)n) * std::ldexp(1.0, -24);
    const double kappa = (K + 2) * std::ldexp(1.0, -21);
    const double a = kappa * 2.001 * R2 + std::ldexp(1.0, -22) * R2 + std::ldexp(1.0, -23) + std::ldexp(1.0, -51) * R2;
    const double b = 0.5005 * kappa + std::ldexp(1.0, -23) + std::ldexp(1.0, -51);
    const double epsS = S * eps * (1.0 + 1e-9);
    const double T = ((epsS + delta) * (epsS + delta) + 2.0 * a) / (1.0 - 2.0 * b) * (1.0 + 1e-12);
    *thr = T;
    *margin = T / ((S * eps) * (S * eps)) - 1.0;
    // fp16 range: r, h, R2 and the padding sentinel must stay well inside 65504
    return std::isfinite(T) && *margin < 0.25 && T < 40000.0 && R2 < 40000.0;
}

namespace {
// pts16[p][t] = fp16(S (pts[p][t] - min_t)) for t < n, 0 beyond: one thread per
// (row, 8-column chunk), i.e. one 16-byte core-matrix row segment of the
// grouped layout (g16), written with a single vector store.
// One thread per point: pts16[p][t] = fp16(S (pts[p][t] - min_t)) for t < n
// (0 up to K - 4), norm16[p] = ||x^_p||^2 exactly in fp64 from the rounded
// halves, the candidate-side augmented columns (1, 1, h_hi, h_lo) with
// h = -||x^_p||^2 / 2, and R2 = max_p norm16[p].  Chunks of 8 halves go out as
// 16-byte core-matrix rows (g16); the last chunk, which holds the augmented
// columns, is written once the norm is known.
template <int KP>
__global__ void k_make16(const double* __restrict__ pts, int64_t N, int n, int n_pad, double S,
                         const Meta* __restrict__ meta, __half* __restrict__ pts16, double* __restrict__ norm16,
                         unsigned long long* __restrict__ r2max) {
    __shared__ double mn[kMaxDim];
    for (int t = threadIdx.x; t < n; t += blockDim.x) mn[t] = meta->mins[meta->order[t]];
    __syncthreads();
    constexpr int NCH = KP / 8;
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double nrm = 0.0;
    if (p < N) {
        const double* row = pts + p * n_pad;
        union { uint4 u; __half h[8]; } v;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int t = 8 * c + i;
                v.h[i] = t < n ? __double2half(S * (row[t] - mn[t])) : __float2half(0.f);
                const double hd = (double)__half2float(v.h[i]);
                nrm += hd * hd;
            }
            if (c < NCH - 1) *reinterpret_cast<uint4*>(pts16 + g16(p, 8 * c, KP)) = v.u;
        }
        const double h = -0.5 * nrm;
        const __half hh = __double2half(h);
        v.h[4] = __float2half(1.f);
        v.h[5] = __float2half(1.f);
        v.h[6] = hh;
        v.h[7] = __double2half(h - (double)__half2float(hh));
        *reinterpret_cast<uint4*>(pts16 + g16(p, KP - 8, KP)) = v.u;
        norm16[p] = nrm;
    }
    unsigned long long bits = (unsigned long long)__double_as_longlong(nrm);
#pragma unroll
    for (int o = 16; o; o >>= 1) bits = max(bits, __shfl_xor_sync(0xffffffffu, bits, o));
    if ((threadIdx.x & 31) == 0) atomicMax(r2max, bits);
}

}  // namespace

// Builds the fp16 operands; *ok = true if the tensor-core bound is certified.
static int make_fp16(Index* ix, unsigned long long* d_r2, bool* ok) {
    cudaStream_t s = ix->stream;
    const Meta& m = ix->h_meta;
    // dims carried by the MMA: the first n_mma of the REORDER order (all n by
    // default; GJ_MMA_DIMS=<d> keeps only the d highest-variance dims, a timing
    // experiment -- the bound then proves ||q - c|| over those dims > eps, which
    // still implies the full distance does)
    static const int env_dims = [] { const char* e = getenv("GJ_MMA_DIMS"); return e ? atoi(e) : 0; }();
    const int n_mma = env_dims > 0 ? std::min(env_dims, ix->n) : ix->n;
    ix->n_mma = n_mma;
    double ss = 0.0;
    for (int t = 0; t < n_mma; ++t) {
        const double sj = m.maxs[m.order[t]] - m.mins[m.order[t]];
        ss += sj * sj;
    }
    *ok = false;
    const double span = std::max(std::sqrt(ss), ix->eps);   // >= every ||x - min|| and eps
    if (!(span < 1e300) || !(span > 0.0)) return GJ_OK;
    // S: power of two with S * span in [90, 180]: r, h, R2 and the sentinel fit fp16
    ix->tc_scale = std::ldexp(1.0, (int)std::floor(std::log2(180.0 / span)));
    ix->k16 = (n_mma + 4 + 15) & ~15;
    if (ix->k16 > 128) return GJ_OK;   // n > 124: no MMA depth instantiated; fall back to the SIMT filters
    const int64_t N = ix->N;
    // rows padded to a multiple of 8 plus one 256-row block of zeros: block loads
    // (<= 256 rows) that start at a row multiple of 8 never read past the allocation
    const size_t rows16 = (size_t)((N + 7) & ~7ll) + 256;
    GJ_CUDA(pool_malloc(&ix->pts16, rows16 * ix->k16 * sizeof(__half), s));
    {   // zero only the last (partial) 8-row group and the padding block: k_make16
        // writes every element of the groups holding rows < N
        const size_t z0 = (size_t)(N & ~7ll) * ix->k16;
        GJ_CUDA(cudaMemsetAsync(ix->pts16 + z0, 0, (rows16 * ix->k16 - z0) * sizeof(__half), s));
    }
    GJ_CUDA(pool_malloc(&ix->norm16, (size_t)N * sizeof(double), s));
    GJ_CUDA(cudaMemsetAsync(d_r2, 0, sizeof(*d_r2), s));
    switch (ix->k16) {
#define GJ_MAKE16(KP)                                                                                            \
    case KP:                                                                                                     \
        k_make16<KP><<<blocks_for(N, 128), 128, 0, s>>>(ix->pts, N, n_mma, ix->n_pad, ix->tc_scale, ix->meta,   \
                                                       ix->pts16, ix->norm16, d_r2);                             \
        break;
        GJ_MAKE16(16) GJ_MAKE16(32) GJ_MAKE16(48) GJ_MAKE16(64) GJ_MAKE16(80) GJ_MAKE16(96) GJ_MAKE16(112)
        GJ_MAKE16(128)
#undef GJ_MAKE16
        default: set_error("fp16 operands: unsupported MMA depth"); return GJ_ERR_INVALID;
    }
    count_launch();
    GJ_CUDA(cudaGetLastError());
    *ok = true;   // launched; make_fp16_finish decides once R2 is on the host
    return GJ_OK;
}

// The certified threshold from R2 = max ||x^||^2 (read back by the caller
// together with its next count); frees the operands when it is not useful.
static int make_fp16_finish(Index* ix, unsigned long long h_r2, bool* ok) {
    cudaStream_t s = ix->stream;
    double R2;
    memcpy(&R2, &h_r2, sizeof(R2));
    *ok = tc_threshold_from(ix->eps, ix->n_mma, ix->k16, ix->tc_scale, R2, &ix->thr16, &ix->margin16) != 0;
    if (!*ok) {
        GJ_CUDA(cudaFreeAsync(ix->pts16, s));
        GJ_CUDA(cudaFreeAsync(ix->norm16, s));
        ix->pts16 = nullptr;
        ix->norm16 = nullptr;
    }
    return GJ_OK;
}


// Small pinned host blocks for the build's read-backs (a pageable
// cudaMemcpyAsync device -> host waits for the stream, i.e. is one more
// synchronisation), reused across builds and threads.
namespace {
struct Staging {
    Meta meta;
    unsigned long long r2;
    uint32_t count;
};
std::mutex g_stage_mu;
std::vector<Staging*> g_stage_free;
struct StagingLease {
    Staging* p = nullptr;
    cudaError_t get() {
        std::lock_guard<std::mutex> l(g_stage_mu);
        if (!g_stage_free.empty()) {
            p = g_stage_free.back();
            g_stage_free.pop_back();
            return cudaSuccess;
        }
        return cudaMallocHost(reinterpret_cast<void**>(&p), sizeof(Staging));
    }
    ~StagingLease() {
        if (!p) return;
        std::lock_guard<std::mutex> l(g_stage_mu);
        g_stage_free.push_back(p);
    }
};
}  // namespace

int build_index(Index* ix, const double* X) {
    cudaStream_t s = ix->stream;
    const int64_t N = ix->N;
    const int n = ix->n, k = ix->k;
    int rc;
    cudaEvent_t ev0, ev1;
    GJ_CUDA(cudaEventCreate(&ev0));
    GJ_CUDA(cudaEventCreate(&ev1));
    GJ_CUDA(cudaEventRecord(ev0, s));

    GJ_CUDA(pool_malloc(&ix->meta, sizeof(Meta), s));
    GJ_CUDA(cudaMemsetAsync(ix->meta, 0, sizeof(Meta), s));
    Meta* M = ix->meta;
    // 1. min/max over D, variance over the sample
    if ((rc = col_reduce(X, N, 1, n, kMinMax, nullptr, M->mins, M->maxs, s))) return rc;
    const int64_t step = std::max<int64_t>(1, (int64_t)llround(1.0 / ix->opt.sample_frac));
    const int64_t m = (N + step - 1) / step;
    double* mean = nullptr;
    GJ_CUDA(pool_malloc(&mean, n * sizeof(double), s));
    if ((rc = col_reduce(X, m, step, n, kSum, nullptr, mean, nullptr, s))) return rc;
    if ((rc = col_reduce(X, m, step, n, kSqDev, mean, M->var, nullptr, s))) return rc;
    GJ_CUDA(cudaFreeAsync(mean, s));
    // 2. permutation + geometry (read back with the cell count, step 6: nothing
    // before needs it on the host)
    k_meta<<<1, 128, 0, s>>>(M, n, k, ix->eps, ix->opt.reorder); count_launch();
    GJ_CUDA(cudaGetLastError());
    StagingLease stage;
    GJ_CUDA(stage.get());
    // 3. keys
    uint64_t *cellkey = nullptr, *ukey = nullptr, *tmp64 = nullptr;
    uint32_t* idx = nullptr;
    GJ_CUDA(pool_malloc(&cellkey, N * sizeof(uint64_t), s));
    GJ_CUDA(pool_malloc(&ukey, N * sizeof(uint64_t), s));
    GJ_CUDA(pool_malloc(&tmp64, N * sizeof(uint64_t), s));
    GJ_CUDA(pool_malloc(&idx, N * sizeof(uint32_t), s));
    k_cell_keys<<<blocks_for(N, 256), 256, 0, s>>>(X, N, n, k, ix->u, ix->eps, M, cellkey, ukey, idx); count_launch();
    GJ_CUDA(cudaGetLastError());
    // 4. stable sort by u, then by cell id
    uint64_t vb = 0;
    if (ix->opt.sortidu) {
        if ((rc = varying_bits_u64(ukey, N, &vb, s))) return rc;
        if ((rc = radix_sort_u64(ukey, idx, N, vb, s))) return rc;
    }
    k_gather_u64<<<blocks_for(N, 256), 256, 0, s>>>(cellkey, idx, N, tmp64); count_launch();
    GJ_CUDA(cudaGetLastError());
    if ((rc = varying_bits_u64(tmp64, N, &vb, s))) return rc;
    if ((rc = radix_sort_u64(tmp64, idx, N, vb, s))) return rc;
    // 5. sorted, reordered point array
    GJ_CUDA(pool_malloc(&ix->pts, (size_t)N * ix->n_pad * sizeof(double), s));
    GJ_CUDA(pool_malloc(&ix->orig, N * sizeof(uint32_t), s));
    k_gather_points<<<(unsigned)std::min<int64_t>(blocks_for(N * 32, 256), 148 * 16), 256, 0, s>>>(X, idx, N, n, ix->n_pad, M,
                                                                                             ix->pts, nullptr); count_launch();
    GJ_CUDA(cudaMemcpyAsync(ix->orig, idx, N * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
    // 6. non-empty cells
    uint32_t *head = nullptr, *pos = nullptr, *d_tot = nullptr;
    GJ_CUDA(pool_malloc(&head, N * sizeof(uint32_t), s));
    GJ_CUDA(pool_malloc(&pos, N * sizeof(uint32_t), s));
    GJ_CUDA(pool_malloc(&d_tot, 4 * sizeof(uint32_t), s));
    k_heads<<<blocks_for(N, 256), 256, 0, s>>>(tmp64, N, head); count_launch();
    if ((rc = scan_u32(head, pos, N, d_tot, s))) return rc;
    GJ_CUDA(cudaMemcpyAsync(&stage.p->meta, M, sizeof(Meta), cudaMemcpyDeviceToHost, s));
    GJ_CUDA(cudaMemcpyAsync(&stage.p->count, d_tot, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    GJ_CUDA(cudaStreamSynchronize(s));
    ix->h_meta = stage.p->meta;
    uint32_t h_tot = stage.p->count;
    if (ix->h_meta.overflow) {
        set_error("linearized cell id needs >= 2^63 cells (prod of per-dim widths); choose a smaller k");
        return GJ_ERR_OVERFLOW;
    }
    const bool fp32_ok = fp32_threshold(ix);
    const bool want32 = ix->filter >= 1 && fp32_ok;
    // certified tensor-core operands (filter 2): launched here, R2 read back
    // with the adjacency count below
    unsigned long long* d_r2 = nullptr;
    bool tc_launched = false;
    if (ix->filter >= 2) {
        GJ_CUDA(pool_malloc(&d_r2, sizeof(*d_r2), s));
        if ((rc = make_fp16(ix, d_r2, &tc_launched))) return rc;
    }
    const int64_t G = h_tot;
    ix->G = G;
    GJ_CUDA(pool_malloc(&ix->cell_id, G * sizeof(uint64_t), s));
    GJ_CUDA(pool_malloc(&ix->cell_start, (G + 1) * sizeof(uint32_t), s));
    k_cells<<<blocks_for(N, 256), 256, 0, s>>>(tmp64, head, pos, N, ix->cell_id, ix->cell_start, G); count_launch();
    GJ_CUDA(cudaGetLastError());
    // 7. adjacent non-empty cells
    uint32_t* cnt = head;               // reuse (G <= N)
    uint64_t* cand = tmp64;             // reuse: tmp64 no longer needed
    uint64_t* cand_after = cellkey;     // reuse: cell keys no longer needed
    GJ_CUDA(pool_malloc(&ix->nbr_off, (G + 1) * sizeof(uint32_t), s));
    GJ_CUDA(pool_malloc(&ix->nbr_self, G * sizeof(uint32_t), s));
    k_adjacent<false><<<blocks_for(G * 32, 256), 256, 0, s>>>(ix->cell_id, ix->cell_start, G, k, M, cnt, cand,
                                                             cand_after, nullptr, nullptr, nullptr); count_launch();
    GJ_CUDA(cudaGetLastError());
    if ((rc = scan_u32(cnt, ix->nbr_off, G, d_tot, s))) return rc;
    GJ_CUDA(cudaMemcpyAsync(ix->nbr_off + G, d_tot, sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
    GJ_CUDA(cudaMemcpyAsync(&stage.p->count, d_tot, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    if (d_r2) GJ_CUDA(cudaMemcpyAsync(&stage.p->r2, d_r2, sizeof(*d_r2), cudaMemcpyDeviceToHost, s));
    GJ_CUDA(cudaStreamSynchronize(s));
    ix->A = stage.p->count;
    if (ix->filter >= 2) {   // certified tensor-core bound, else fall back to the FP32 / FP64 scan
        bool tc_ok = false;
        if (tc_launched && (rc = make_fp16_finish(ix, stage.p->r2, &tc_ok))) return rc;
        if (d_r2) GJ_CUDA(cudaFreeAsync(d_r2, s));
        if (!tc_ok) ix->filter = want32 ? 1 : 0;
    } else if (ix->filter == 1 && !want32) {
        ix->filter = 0;
    }
    if (ix->filter == 1) {   // the FP32 filter's operands fl32(x - min), only when it runs
        GJ_CUDA(pool_malloc(&ix->pts32, (size_t)N * ix->n_pad * sizeof(float), s));
        k_make32<<<blocks_for(N * ix->n_pad, 256), 256, 0, s>>>(ix->pts, N, n, ix->n_pad, M, ix->pts32); count_launch();
        GJ_CUDA(cudaGetLastError());
    }
    GJ_CUDA(pool_malloc(&ix->nbr, std::max<int64_t>(1, ix->A) * sizeof(uint32_t), s));
    k_adjacent<true><<<blocks_for(G * 32, 256), 256, 0, s>>>(ix->cell_id, ix->cell_start, G, k, M, nullptr,
                                                            nullptr, nullptr, ix->nbr_off, ix->nbr, ix->nbr_self); count_launch();
    GJ_CUDA(cudaGetLastError());
    // 8. tiles, heaviest first (256 queries for the two-accumulator-tile tcgen05 kernel)
    ix->tile_q = ix->filter == 2 ? 128 * (ix->opt.mma_tiles == 2 ? 2 : 1) : kTileQ;
    k_tile_count<<<blocks_for(G, 256), 256, 0, s>>>(ix->cell_start, G, (uint32_t)ix->tile_q, pos); count_launch();
    if ((rc = scan_u32(pos, pos, G, d_tot, s))) return rc;
    GJ_CUDA(cudaMemcpyAsync(&stage.p->count, d_tot, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    GJ_CUDA(cudaStreamSynchronize(s));
    const int64_t T = stage.p->count;
    ix->T = T;
    GJ_CUDA(pool_malloc(&ix->tile_cell, T * sizeof(uint32_t), s));
    GJ_CUDA(pool_malloc(&ix->tile_q0, T * sizeof(uint32_t), s));
    GJ_CUDA(pool_malloc(&ix->tile_order, T * sizeof(uint32_t), s));
    GJ_CUDA(pool_malloc(&ix->tile_work, T * sizeof(uint64_t), s));
    uint64_t* skey = ukey;              // reuse (T <= N)
    unsigned long long* d_total = nullptr;
    GJ_CUDA(pool_malloc(&d_total, sizeof(*d_total), s));
    GJ_CUDA(cudaMemsetAsync(d_total, 0, sizeof(*d_total), s));
    k_tile_fill<<<blocks_for(T, 256), 256, 0, s>>>(ix->cell_start, pos, cand, cand_after, ix->opt.symmetric, G, T,
                                                   (uint32_t)ix->tile_q,
                                                   ix->tile_cell, ix->tile_q0,
                                                   ix->tile_work, skey, ix->tile_order, d_total); count_launch();
    GJ_CUDA(cudaGetLastError());
    if ((rc = varying_bits_u64(skey, T, &vb, s))) return rc;
    if ((rc = radix_sort_u64(skey, ix->tile_order, T, vb, s))) return rc;
    // host copy of the heaviest-first work (keys are ~work) for work-balanced split plans
    ix->h_work_by_pos.resize((size_t)T);
    if (T > 0) {
        GJ_CUDA(cudaMemcpyAsync(ix->h_work_by_pos.data(), skey, (size_t)T * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
        GJ_CUDA(cudaStreamSynchronize(s));
        for (auto& w : ix->h_work_by_pos) w = ~w;
    }
    unsigned long long h_total = 0;
    GJ_CUDA(cudaMemcpyAsync(&h_total, d_total, sizeof(h_total), cudaMemcpyDeviceToHost, s));
    GJ_CUDA(pool_malloc(&ix->scratch_count, 8 * sizeof(uint64_t), s));
    GJ_CUDA(cudaFreeAsync(d_total, s));
    GJ_CUDA(cudaFreeAsync(cellkey, s));
    GJ_CUDA(cudaFreeAsync(ukey, s));
    GJ_CUDA(cudaFreeAsync(tmp64, s));
    GJ_CUDA(cudaFreeAsync(idx, s));
    GJ_CUDA(cudaFreeAsync(head, s));
    GJ_CUDA(cudaFreeAsync(pos, s));
    GJ_CUDA(cudaFreeAsync(d_tot, s));
    GJ_CUDA(cudaEventRecord(ev1, s));
    GJ_CUDA(cudaStreamSynchronize(s));
    float ms = 0;
    GJ_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    ix->build_ms = ms;
    ix->est_candidates = (double)h_total;
    return GJ_OK;
}

}  // namespace gj
