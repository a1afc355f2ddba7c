// Internal declarations shared by the CUDA translation units of libgpujoin.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <vector>

#include "../../include/gpujoin.h"

namespace gj {

constexpr int kTileQ = 128;          // queries per tile = threads per join CTA
constexpr int kMaxDim = 128;         // largest supported n (query dims live in registers)

void set_error(const std::string& msg);

// Device memory: every allocation of the library comes from one private
// stream-ordered pool per device whose release threshold is unbounded, so
// memory freed by one join (index arrays, result batches) is reused by the
// next without returning to the driver (no page-table remapping per step).
// gj_release_cached_memory() trims it.
cudaError_t pool_malloc_raw(void** p, size_t bytes, cudaStream_t s);
template <typename T>
inline cudaError_t pool_malloc(T** p, size_t bytes, cudaStream_t s) {
    return pool_malloc_raw(reinterpret_cast<void**>(p), bytes, s);
}
cudaError_t pool_trim();

// Kernels launched by this library (bench.py reports it as gpu_launches).
extern std::atomic<long long> g_launches;
inline void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

#define GJ_CUDA(call)                                                                        \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess) {                                                             \
            ::gj::set_error(std::string(#call) + ": " + cudaGetErrorString(e_));           \
            return GJ_ERR_CUDA;                                                              \
        }                                                                                    \
    } while (0)

// Device-resident metadata written by the index-build kernels.
struct Meta {
    int32_t order[kMaxDim];      // REORDER permutation: position t <- original dim
    double mins[kMaxDim];
    double maxs[kMaxDim];
    double var[kMaxDim];
    int64_t base[16];                // per indexed dim: floor(min/eps)
    int64_t width[16];               // cells per indexed dim
    uint64_t stride[16];             // row-major strides of the linear id
    int32_t overflow;                // 1 if prod(width) >= 2^63
    int32_t pad_;
};
constexpr int kMaxK = 16;

struct Index {
    int64_t N = 0;
    int32_t n = 0, n_pad = 0, k = 0, u = 0;
    double eps = 0, eps2 = 0;
    gj_options opt{};
    cudaStream_t stream = 0;
    // device arrays
    double* pts = nullptr;           // [N][n_pad] reordered dims, sorted by (cell, u)
    float* pts32 = nullptr;          // [N][n_pad] fl32(x - min_j): input of the certified FP32 prefilter
    int filter = 0;                  // 0 FP64 scan, 1 FP32 prefilter, 2 tcgen05 bound (+ FP64 decision)
    float thr32 = 0.f;               // FP32 prefilter rejection threshold (> eps^2, see fp32_threshold)
    float thr32_in = -1.f;           // FP32 certain-inside threshold (< eps^2): accepted without the FP64 test
    double filter_margin = 0;        // thr32 / eps^2 - 1
    __half* pts16 = nullptr;         // [N][k16] fp16(S (x - min_j)) + candidate-side augmented columns
    double* norm16 = nullptr;        // [N] ||fp16 coordinates||^2 (exact, fp64)
    int k16 = 0;                     // MMA depth: n_mma + 4 augmented columns, rounded up to 16
    int n_mma = 0;                   // leading (REORDER-order) dims carried by the MMA bound
    int tile_q = kTileQ;             // queries per tile: 128, or 256 for the M = 2 x 128 tcgen05 kernel
    double tc_scale = 1.0;           // S, a power of two
    double thr16 = 0.0;              // tensor-core bound threshold T (scaled units)
    double margin16 = 0;             // thr16 / (S eps)^2 - 1
    uint32_t* orig = nullptr;        // [N] sorted position -> original id
    uint64_t* cell_id = nullptr;     // [G] sorted non-empty linear ids
    uint32_t* cell_start = nullptr;  // [G+1]
    uint32_t* nbr_off = nullptr;     // [G+1]
    uint32_t* nbr = nullptr;         // [A] adjacent non-empty cells (offset order)
    uint32_t* nbr_self = nullptr;    // [G] position of cell g inside its own adjacency list
    uint32_t* tile_cell = nullptr;   // [T]
    uint32_t* tile_q0 = nullptr;     // [T]
    uint32_t* tile_order = nullptr;  // [T] tiles, heaviest estimated work first
    uint64_t* tile_work = nullptr;   // [T] queries * candidates (pre-SORTIDU)
    std::vector<uint64_t> h_work_by_pos;   // host: tile_work of tile_order[j] (work-balanced split plans)
    Meta* meta = nullptr;            // device
    uint64_t* scratch_count = nullptr;   // [4] device counters
    Meta h_meta{};                   // host copy
    int64_t G = 0, A = 0, T = 0;
    double est_candidates = 0, build_ms = 0;
    // result pipeline resources (lazily created)
    cudaStream_t pipe_stream[3] = {0, 0, 0};
    cudaEvent_t pipe_event[3] = {0, 0, 0};
};

// ---- radix sort / scan (gj_radix.cu) ----
// Exclusive scan of n uint32 -> uint32 (out may alias in); total returned via d_total (device).
int scan_u32(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* d_total, cudaStream_t s);
// Stable LSD radix sort of (key, val) pairs on the key bits set in `bits_mask`.
// keys/vals are sorted in place (double-buffered internally).
int radix_sort_u64(uint64_t* keys, uint32_t* vals, int64_t n, uint64_t bits_mask, cudaStream_t s);
// OR over i of (keys[i] ^ keys[0]) -> host.
int varying_bits_u64(const uint64_t* keys, int64_t n, uint64_t* h_out, cudaStream_t s);

// ---- index build (gj_index.cu) ----
// Certified FP32 prefilter threshold from the per-dim spans (max - min);
// returns 0 when the filter cannot be certified usefully.
int fp32_threshold_from_spans(double eps, int n, const double* spans, float* thr, double* margin);
float fp32_accept_threshold_from_spans(double eps, int n, const double* spans);
// Certified tensor-core bound threshold (scaled units); returns 0 if not useful.
int tc_threshold_from(double eps, int n, int K, double S, double R2, double* thr, double* margin);
int build_index(Index* ix, const double* d_points);

// ---- join (gj_join.cu) ----
enum JoinMode { kEmit = 0, kCount = 1, kStats = 2 };
struct JoinArgs {
    uint32_t* out;            // [cap][2]
    uint64_t cap;
    uint64_t* count;          // device counter(s); kStats: [4] = cells, tests, dims, pairs
    int64_t first;            // first query set (unit of blk tile positions)
    int64_t step;             // query sets first + step * k of this launch
    int64_t n_tiles;          // number of tile positions m (tile_pos below)
    int32_t blk;              // tile positions per query set (0 / 1: one)
    int32_t split;            // CTAs per tile, each scanning 1/split of every candidate window (0/1 = none)
    // Work-balanced split (optional, overrides split): tile m of the launch gets
    // part_off[m+1] - part_off[m] CTAs; part_off[n_tiles] = total parts.
    const uint32_t* part_off;
    int64_t total_parts;
    // optional (tcgen05 join): += MMA tests executed (rows x columns of every
    // accumulator block, padding included) -- the executed-vs-useful ratio
    unsigned long long* mma_tests;
};
struct JoinParams {
    const double* __restrict__ pts;
    const float* __restrict__ pts32;
    const uint32_t* __restrict__ orig;
    const uint32_t* __restrict__ cell_start;
    const uint32_t* __restrict__ nbr_off;
    const uint32_t* __restrict__ nbr;
    const uint32_t* __restrict__ nbr_self;
    const uint32_t* __restrict__ tile_cell;
    const uint32_t* __restrict__ tile_q0;
    const uint32_t* __restrict__ tile_order;
    int n, n_pad, u, sortidu, shortc;
    double eps, eps2;
    float thr32, thr32_in;
    const __half* __restrict__ pts16;
    const double* __restrict__ norm16;
    int k16;
    double thr16;
    uint32_t tile_q;                 // queries per index tile (128 or 256)
};

// Query sets (§6.2 l.1013, reading R12): blk consecutive positions
// of the heaviest-first tile order form one set Q_l; the sets of a launch are
// l = first + step * k.  Launch-local tile m sits at position
//   (first + step * (m / blk)) * blk + m % blk.
__host__ __device__ __forceinline__ int64_t tile_pos(const JoinArgs& a, int64_t m) {
    if (a.blk <= 1) return a.first + a.step * m;
    return (a.first + a.step * (m / a.blk)) * a.blk + m % a.blk;
}
// Tile positions per query set of the entity partitioning and result
// batching (kDealBlock; GJ_DEAL_BLOCK overrides it for timing experiments).
int deal_block();

// The query block of one CTA.  A CTA handles `qper` queries (128, or 256 in
// the two-accumulator tcgen05 kernel); an index tile of tile_q queries is
// covered by tile_q / qper CTAs, and each of those by A.split candidate parts:
//   blockIdx.x = (m * (tile_q / qper) + sub) * split + part.
// nq = 0 marks an empty sub-block (the tile's cell ended earlier).
struct CtaTile {
    uint32_t g, q0, nq;
    int part, split;
};
__device__ __forceinline__ CtaTile cta_tile_at(const JoinParams& P, const JoinArgs& A, uint32_t qper, uint32_t b) {
    const uint32_t subs = P.tile_q > qper ? P.tile_q / qper : 1u;
    CtaTile t;
    uint32_t m, sub;
    if (A.part_off) {   // item b: (unit r = b / subs, sub = b % subs), unit r -> (tile m, part)
        sub = b % subs;
        const uint32_t r = b / subs;
        uint32_t lo = 0, hi = (uint32_t)A.n_tiles;   // last m with part_off[m] <= r
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (A.part_off[mid] <= r) lo = mid; else hi = mid;
        }
        m = lo;
        t.part = (int)(r - A.part_off[m]);
        t.split = (int)(A.part_off[m + 1] - A.part_off[m]);
    } else {
        const uint32_t split = A.split > 1 ? (uint32_t)A.split : 1u;
        t.part = (int)(b % split);
        t.split = (int)split;
        const uint32_t mm = b / split;
        sub = mm % subs;
        m = mm / subs;
    }
    const int64_t j = tile_pos(A, (int64_t)m);
    const uint32_t tile = P.tile_order[j];
    t.g = P.tile_cell[tile];
    t.q0 = P.tile_q0[tile] + sub * qper;
    const uint32_t end = P.cell_start[t.g + 1];
    t.nq = t.q0 < end ? min(qper, end - t.q0) : 0u;
    return t;
}
__device__ __forceinline__ CtaTile cta_tile(const JoinParams& P, const JoinArgs& A, uint32_t qper) {
    return cta_tile_at(P, A, qper, blockIdx.x);
}
// CTAs of a launch over a.n_tiles index tiles with `qper` queries per CTA.
inline unsigned grid_ctas(const JoinArgs& a, int tile_q, int qper) {
    const int64_t subs = tile_q > qper ? tile_q / qper : 1;
    if (a.part_off) return (unsigned)(a.total_parts * subs);
    return (unsigned)(a.n_tiles * subs * (a.split > 1 ? a.split : 1));
}
JoinParams join_params(const Index* ix);

// Grouped core-matrix layout of the fp16 operand array (Index::pts16): element
// (p, k) of the logical [N][K] matrix sits at halves offset
//   (p / 8) * 8K + (k / 8) * 64 + (p % 8) * 8 + (k % 8)
// i.e. every 8-row group is K/8 consecutive 8x8 "core matrices" of 128 B -- the
// canonical K-major SWIZZLE_NONE UMMA layout -- so 128 consecutive rows starting
// at a multiple of 8 are one contiguous 128*K*2-byte block (one bulk copy).
__host__ __device__ __forceinline__ size_t g16(size_t p, int k, int K) {
    return (p >> 3) * (size_t)(8 * K) + (size_t)((k >> 3) * 64 + (int)(p & 7) * 8 + (k & 7));
}

// Query-side augmented MMA columns (r_hi, r_lo) of the tensor-core bound:
// r = (T - ||q^||^2) / 2 split into fp16 hi + lo; invalid rows get the
// sentinel -65504 so that every accumulator of the row is negative.
__device__ __forceinline__ void query_aug(double T, double nq, bool valid, __half& rhi, __half& rlo) {
    if (!valid) {
        rhi = __float2half(-65504.f);
        rlo = __float2half(0.f);
        return;
    }
    const double r = 0.5 * (T - nq);
    rhi = __double2half(r);
    rlo = __double2half(r - (double)__half2float(rhi));
}
int launch_join(const Index* ix, JoinMode mode, const JoinArgs& a, cudaStream_t s);
// cells / paper tests / tests evaluated of the tiles in a (no distance work); adds to d_out[0..2].
int count_tests(const Index* ix, const JoinArgs& a, unsigned long long* d_out, cudaStream_t s);
// FP32-prefilter variant (gj_join32.cu); kEmit / kCount only.
int launch_join32(const Index* ix, JoinMode mode, const JoinArgs& a, cudaStream_t s);
// Tensor-core bound variants; kEmit / kCount only.
int launch_join_umma(const Index* ix, JoinMode mode, const JoinArgs& a, cudaStream_t s);  // tcgen05 (gj_join_umma.cu)
int selftest_umma(const void* A, const void* B, float* D, cudaStream_t s);
// Persistent tcgen05 join (gj_join_ws.cu): one CTA per SM, four accumulator slots.
int launch_join_ws(const Index* ix, JoinMode mode, const JoinArgs& a, cudaStream_t s);
// Query sets first + step * k of T tiles (blk, first, step, n_tiles of a).
void query_sets(int64_t T, int64_t first, int64_t step, JoinArgs* a);
// Number of tile positions for (rank, world, batch, n_batches); sets first/step.
void batch_tiles(const Index* ix, int32_t batch, int32_t n_batches, int32_t rank, int32_t world,
                 JoinArgs* a);

}  // namespace gj
