/*
 * gpujoin.h -- C ABI of the B200 epsilon self-join (arxiv 1809.09930).
 *
 * The library computes the distance-similarity self-join of PAPER.md §3.1
 * (l.104-110): every ORDERED pair (a, b) of points of D with
 * dist(a, b) = sqrt(sum_j (a(x_j) - b(x_j))^2) <= eps, the self pair (a, a)
 * included (§5.2 l.800-802 counts it in |R|).  The test is evaluated in
 * float64 as sum_j (a_j - b_j)^2 <= eps^2.
 *
 * The hot path is Algorithm 1 (§4.5 l.573-612): reorderVariance (§4.2),
 * constructIndex over k < n dimensions (§3.2.1, §4.1), computeNumBatches
 * (§3.2.2), SelfJoinKernel with SORTIDU (§4.3) and SHORTC (§4.4), and the
 * entity partitioning of query points over GPUs (§6.2).
 *
 * Conventions for every entry point
 *  - Return value: GJ_OK (0) on success, a negative GJ_ERR_* code otherwise;
 *    gj_last_error() then returns a thread-local human-readable message.
 *    No entry point aborts the process.
 *  - "device pointer" = memory from cudaMalloc / torch CUDA tensors on the
 *    current device; "host pointer" = ordinary or pinned host memory.
 *  - All GPU work of an index is issued on the CUDA stream given in
 *    gj_options.stream at build time (0 = legacy default stream).  Calls
 *    marked [async] only enqueue work; others synchronise that stream.
 *  - Point ids in results are the row numbers of the ORIGINAL input array
 *    (0-based, uint32), independent of any internal reordering.
 *  - Ownership: the caller owns every buffer it passes; the index owns its
 *    own device memory until gj_free_index().
 */
#ifndef GPUJOIN_H
#define GPUJOIN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define GJ_API __attribute__((visibility("default")))
#else
#define GJ_API
#endif

#define GJ_OK 0
#define GJ_ERR_INVALID -1   /* bad argument (null, size, k outside [1,n], eps <= 0 ...) */
#define GJ_ERR_CUDA -2      /* a CUDA runtime call failed (message has the CUDA error) */
#define GJ_ERR_OVERFLOW -3  /* linearised cell id needs >= 2^63: choose a smaller k (§4.1) */
#define GJ_ERR_CAPACITY -4  /* result buffer too small; *n_pairs holds the required count */
#define GJ_ERR_NOMEM -5     /* device or pinned allocation failed */

typedef struct gj_index gj_index; /* opaque handle */

/* Options of Algorithm 1.  Zero-initialise then set fields; gj_default_options fills them
 * (reorder = sortidu = shortc = symmetric = 1, filter = 2, sample_frac = 0.01, stream = 0). */
typedef struct {
    int32_t reorder;     /* 1: REORDER dims by variance (§4.2); 0: index the first k dims */
    int32_t sortidu;     /* 1: SORTIDU prune on the un-indexed dim u (§4.3)               */
    int32_t shortc;      /* 1: SHORTC short-circuit of the distance sum (§4.4)            */
    int32_t symmetric;   /* 1: evaluate each unordered pair once, emit both orders (default);
                            0: one full neighbour search per query (Alg. 1 verbatim).
                            With 1, the output of ONE batch or ONE rank is not the
                            neighbour sets of that share's queries: a pair (a, b) is found
                            by the share owning the tile of a or of b (whichever comes
                            first in the symmetric order) and both orders are emitted
                            there.  Only the union over all batches and ranks is the
                            self-join.  Use 0 when each share must be query-complete.   */
    double sample_frac;  /* variance sample fraction (§4.2 "1% of |D|"), in (0,1]        */
    uint64_t stream;     /* cudaStream_t the index issues its work on                     */
    int32_t filter;      /* candidate filter of the join kernel; every pair it cannot reject is
                            decided by the FP64 test, so the pair set is the same for all:
                            0 = FP64 SHORTC scan (Alg. 1 verbatim arithmetic)
                            1 = certified FP32 SHORTC prefilter (SIMT, packed f32x2)
                            2 = certified tensor-core bound on dense cell-pair blocks with
                                tcgen05.mma (fp16 operands, fp32 accumulators in TMEM) (default)
                            2 falls back to 1, then 0, when the data's spread makes the
                            bound uncertifiable.  (Round 1's legacy mma.sync variant,
                            filter 3, was removed: GJ_ERR_INVALID.)
                            gj_join_stats always runs the FP64 scan.                          */
    int32_t mma_tiles;   /* filter 2 only: queries per index tile, in units of 128:
                            1 (or 0, default) = tiles of 128 queries: one tcgen05 CTA per
                            tile part holds one 128-query A tile (UMMA M = 128) and one
                            128-column TMEM accumulator, streams 128-candidate B blocks, and
                            runs four per SM (three for MMA depth 64..96; 256-candidate
                            blocks, two per SM, beyond); 2 = tiles of 256 queries, two A
                            tiles per CTA sharing every candidate block, one CTA per SM.
                            (Environment GJ_UMMA_WS=1 selects the persistent kernel: one CTA
                            per SM, four accumulator slots.)  The pair set does not depend
                            on any of these.                                                  */
} gj_options;

/* Read-only description of a built index. */
typedef struct {
    int64_t n_points;     /* |D|                                                   */
    int32_t dim;          /* n                                                     */
    int32_t dim_pad;      /* n rounded up to a multiple of 4 (row stride, doubles) */
    int32_t k;            /* indexed dims                                          */
    int32_t u;            /* position (in reordered dims) of the SORTIDU dim       */
    double eps;
    int64_t n_cells;      /* |G|: non-empty cells (§5.6)                           */
    int64_t n_adjacent;   /* sum over cells of non-empty adjacent cells            */
    int64_t n_tiles;      /* query tiles (<= tile_queries queries of one cell each) */
    double est_candidates;/* sum over queries of candidates before SORTIDU         */
    double build_ms;      /* device time of gj_build_index (CUDA events)           */
    int32_t filter;       /* filter the join kernel actually runs (0..2, see gj_options) */
    float filter_threshold;  /* its rejection threshold (filter 2: in scaled units)      */
    double filter_margin; /* threshold / eps^2 - 1 (relative slack of the bound)          */
    int32_t tile_queries; /* queries per tile: 128, or 256 (filter 2 with mma_tiles = 2)  */
    int32_t mma_depth;    /* filters 2/3: MMA depth K (n + 4 augmented columns rounded up to
                             16), 0 when the tensor-core operands were not built       */
} gj_info;

/* Work counters of one join (gj_join_stats).  cells/tests/dims/pairs are the
 * paper's per-query counts (Alg. 1 run once per query point), identical for
 * symmetric and per-query evaluation; *_evaluated is what the kernel ran. */
typedef struct {
    int64_t cells;           /* (query, adjacent non-empty cell) visits                        */
    int64_t tests;           /* candidate distance tests after SORTIDU                         */
    int64_t dims;            /* dims evaluated with a per-dimension SHORTC check (algorithmic) */
    int64_t pairs;           /* result pairs (ordered, self pairs included)                    */
    int64_t tests_evaluated; /* distance tests the kernel evaluated (symmetric: unordered)     */
    int64_t dims_evaluated;  /* per-dimension-SHORTC dims of those tests                        */
} gj_stats;

GJ_API void gj_default_options(gj_options* opt);

/* constructIndex (Alg. 1 l.581-582; §3.2.1, §4.1-4.3).
 *  points : n_points x dim row-major float64, host OR device pointer (host
 *           input is staged to the device inside the call).
 *  eps    : > 0, search radius and grid cell edge length (§3.2.1 l.121).
 *  k      : 1 <= k <= dim indexed dimensions (§4.1; the paper uses 2 <= k < n).
 *  opt    : may be NULL (defaults: reorder=sortidu=shortc=1, sample_frac=0.01).
 *  out    : receives the handle; free with gj_free_index.
 * Errors: GJ_ERR_INVALID, GJ_ERR_OVERFLOW, GJ_ERR_CUDA, GJ_ERR_NOMEM.
 * n_points must be < 2^32 - 1 (ids are uint32).  Synchronises the stream. */
GJ_API int gj_build_index(const double* points, int64_t n_points, int32_t dim, double eps, int32_t k,
                   const gj_options* opt, gj_index** out);

GJ_API int gj_index_info(const gj_index* idx, gj_info* info);

/* Dimension order chosen by REORDER: order[t] = original dim at position t. */
GJ_API int gj_dim_order(const gj_index* idx, int32_t* order, int32_t cap);

/* Device pointer to the index's reordered, cell-sorted point array
 * (n_points x dim_pad float64) and its sorted-position -> original-id map. */
GJ_API int gj_device_arrays(const gj_index* idx, const double** points_sorted, const uint32_t** orig_id);

/* Result-size estimator (§3.2.2 l.199): runs the join in count-only mode on
 * every round(1/frac)-th query tile of this rank's share and scales by the
 * sampled query fraction.  Returns estimated pairs of this rank's share. */
GJ_API int gj_estimate(gj_index* idx, double frac, int32_t rank, int32_t world, int64_t* est_pairs);

/* Host only: rejection threshold of the certified FP32 prefilter for radius
 * eps and per-dimension spans s_j = max_j - min_j (n values).  A pair whose
 * float32 running sum of fl32(fl32(q_j - min_j) - fl32(c_j - min_j))^2 (FMA
 * accumulation, any prefix of the dims) exceeds *thr is provably farther than
 * eps (1 + 1e-9).  *margin = thr / eps^2 - 1 (from the exact double value).
 * Returns 1 if the filter is enabled for such data, 0 if not, <0 on error. */
GJ_API int gj_fp32_threshold(double eps, int32_t n, const double* spans, float* thr, double* margin);

/* Certain-inside side of the same FP32 analysis (host only): a float32 running sum
 * <= *thr_in proves dist(a, b) <= eps (1 - 1e-9), so filter 1 accepts such a pair
 * without the FP64 test (the FP64 test would accept it too).  *thr_in = -1 when the
 * spread leaves no such region.  GJ_OK or GJ_ERR_INVALID. */
GJ_API int gj_fp32_accept_threshold(double eps, int32_t n, const double* spans, float* thr_in);

/* Host only: threshold T of the certified tensor-core bound (filter 2/3) for
 * radius eps, n coordinates, MMA depth K (>= n + 4), power-of-two scale S and
 * R2 = max squared norm of the fp16 operand rows.  The kernel rejects a pair
 * iff its accumulator q^.c^ + (T - ||q^||^2)/2 - ||c^||^2/2 is <= 0, which
 * implies dist > eps (1 + 1e-9).  Returns 1 if usable, 0 if not, <0 on error. */
GJ_API int gj_tc_threshold(double eps, int32_t n, int32_t K, double S, double R2, double* thr, double* margin);

/* Diagnostic: D[128][128] = A[128][32] . B[128][32]^T (fp16 row-major device
 * inputs, fp32 row-major device output) through the join kernel's tcgen05 /
 * TMEM path (shared-memory layout, descriptors, TMEM load).  Synchronous. */
GJ_API int gj_selftest_umma(const void* A, const void* B, float* D, uint64_t stream);

/* computeNumBatches (§3.2.2 l.199-200): n_b = max(3, ceil(est / batch_size)).
 * batch_size <= 0 selects the device-memory-sized b_s (reading R15): a quarter of
 * the current device's free HBM (sampled at the first such call in the process)
 * split over the 3 pipeline result slots, 8 bytes per pair (~1.9e9 pairs on an
 * idle 180 GB B200), at least the paper's 1e8. */
GJ_API int64_t gj_num_batches(int64_t est_pairs, int64_t batch_size);

/* Entity partitioning arithmetic (§6.2 l.1013), host only.  The query sets
 * Q_l are runs of `block` consecutive positions of the index's heaviest-first
 * tile order (positions l*block .. l*block + block - 1, the last run partial;
 * reading R12); rank `rank` of `world` processes, in batch `batch` of
 * `n_batches`, the sets l = first + step * k (l mod world = rank,
 * (l div world) mod n_batches = batch): `count` tile positions in all,
 *   position of tile m = (first + step * (m / block)) * block + m % block.
 * block is the library's constant (1; GJ_DEAL_BLOCK overrides it).  Errors:
 * GJ_ERR_INVALID for null outputs, n_tiles < 0, rank / batch out of range. */
GJ_API int gj_partition(int64_t n_tiles, int32_t rank, int32_t world, int32_t batch, int32_t n_batches,
                        int64_t* first, int64_t* step, int64_t* count, int32_t* block);

/* selfJoinKernel for one batch (Alg. 1 l.586) [async].
 *  Processes batch `batch` of `n_batches` of rank `rank`'s share of the
 *  query tiles (entity partitioning §6.2: query set l -- `block` consecutive
 *  positions of the index's heaviest-first tile order, gj_partition -- belongs
 *  to rank l mod world; batch = (l div world) mod n_batches).  Appends ordered pairs (query_id, neighbour_id) as uint32
 *  pairs to out_pairs (device, capacity pairs) at positions obtained from the
 *  device counter *d_count (uint64, device pointer; caller zeroes it before
 *  the first batch that shares the buffer).  Pairs past capacity are counted
 *  but not written: after the stream completes, *d_count > capacity means the
 *  batch must be re-run with a larger buffer.  Pair order is unspecified. */
GJ_API int gj_self_join_async(gj_index* idx, uint32_t* out_pairs, int64_t capacity, uint64_t* d_count,
                       int32_t batch, int32_t n_batches, int32_t rank, int32_t world);

/* gj_self_join_async on a caller-chosen CUDA stream (0 = the index's stream)
 * [async]: batches on different streams run concurrently (Fig. 4 uses three),
 * so one batch's tail overlaps the next.  The caller orders `stream` after the
 * index build (e.g. an event recorded on the index stream) and after the zeroing
 * of *d_count; concurrent batches may share out_pairs and d_count. */
GJ_API int gj_self_join_async_stream(gj_index* idx, uint32_t* out_pairs, int64_t capacity, uint64_t* d_count,
                                     int32_t batch, int32_t n_batches, int32_t rank, int32_t world,
                                     uint64_t stream);

/* Same, count only (no pair payload written) [async]. */
GJ_API int gj_self_join_count_async(gj_index* idx, uint64_t* d_count, int32_t batch, int32_t n_batches,
                             int32_t rank, int32_t world);

/* Convenience: whole share of `rank` into a device buffer, synchronous.
 * On GJ_ERR_CAPACITY *n_pairs holds the required capacity. */
GJ_API int gj_self_join(gj_index* idx, uint32_t* out_pairs, int64_t capacity, int32_t rank, int32_t world,
                 int64_t* n_pairs);

/* The full GPU-Join pipeline of Alg. 1 with Fig. 4's overlap: estimator,
 * n_b = max(3, ceil(est/batch_size)) batches on 3 streams with 3 device
 * result buffers, device->host drains of each batch overlapping the next
 * batch's kernel, into the HOST buffer out_pairs (capacity pairs).  If
 * out_pairs is pinned the drains land in it directly, otherwise through 3
 * pinned staging buffers.  batch_size <= 0 selects the HBM-sized b_s of
 * gj_num_batches (reading R15), never below the paper's 1e8 (§3.2.2 l.199).
 * On GJ_ERR_CAPACITY *n_pairs holds the required capacity. */
GJ_API int gj_self_join_host(gj_index* idx, uint32_t* out_pairs, int64_t capacity, int32_t rank,
                      int32_t world, int64_t batch_size, int64_t* n_pairs, int32_t* n_batches_out);

/* The work counters cells, tests and tests_evaluated of gj_join_stats (same
 * definitions, equal values) for the tiles of (rank, world), WITHOUT the
 * distance work: per query and adjacent cell the SORTIDU window is found by
 * binary search (§4.3).  dims, pairs and dims_evaluated are set to -1.
 * Cheap (milliseconds at |D| = 2e6): the roofline denominator of the
 * tensor-core filters, whose unit of work is the evaluated test. */
GJ_API int gj_join_counts(gj_index* idx, int32_t rank, int32_t world, gj_stats* st);

/* Executed tensor-core work of rank's share (filter 2): the number of
 * accumulator entries (query row x candidate column of every 128 x 128 MMA
 * block, padding rows and columns included) the tcgen05 join computes --
 * divided by gj_stats.tests_evaluated it is the MMA waste ratio.  Runs the
 * join once in count-only mode (no pairs written).  *mma_tests = -1 when the
 * index does not run filter 2.  Synchronous. */
GJ_API int gj_join_mma_tests(gj_index* idx, int32_t rank, int32_t world, int64_t* mma_tests);

/* Work counters of rank's share (cells visited, SORTIDU-window tests,
 * algorithmic SHORTC dims, pairs).  Synchronous; slower than the join. */
GJ_API int gj_join_stats(gj_index* idx, int32_t rank, int32_t world, gj_stats* st);

/* constructNeighborTable (Alg. 1 l.587): sort n_pairs device pairs by
 * (query, neighbour) in place and write the CSR offsets (n_points + 1
 * uint64, device) of each query's neighbour run.  Synchronous.
 * n_pairs must be < 2^32 (32-bit radix-sort offsets): GJ_ERR_INVALID otherwise;
 * sort larger results per batch. */
GJ_API int gj_neighbor_table(gj_index* idx, uint32_t* pairs, int64_t n_pairs, uint64_t* offsets);

/* Frees the index.  Synchronises the whole current device first, so joins still
 * running on caller streams (gj_self_join_async_stream) finish before the
 * index arrays return to the library pool. */
GJ_API void gj_free_index(gj_index* idx);
GJ_API const char* gj_last_error(void);
GJ_API int32_t gj_abi_version(void);
/* Number of CUDA kernels this library has launched in this process. */
/* Device memory of every index and join comes from a library-private, stream-ordered
 * memory pool per device that keeps freed memory cached for the next build / join
 * (no driver remapping per step).  This returns the cached, unused part to the driver;
 * it synchronises the current device.  GJ_OK, or GJ_ERR_CUDA. */
GJ_API int gj_release_cached_memory(void);

GJ_API int64_t gj_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* GPUJOIN_H */
