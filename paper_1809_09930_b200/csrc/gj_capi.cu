// C ABI (include/gpujoin.h): argument checking, handle lifetime, batching and
// the Fig. 4 result pipeline.  All arithmetic of the method runs in the
// kernels of gj_index.cu / gj_join.cu / gj_radix.cu.
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <mutex>
#include <string>

#include "gj_internal.cuh"

struct gj_index {
    gj::Index ix;
};

namespace gj {

static thread_local std::string g_err;
std::atomic<long long> g_launches{0};
void set_error(const std::string& msg) { g_err = msg; }

namespace {
cudaMemPool_t g_pool[64] = {};
std::mutex g_pool_mu;
cudaError_t device_pool(cudaMemPool_t* out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lock(g_pool_mu);
    if (!g_pool[dev]) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        if ((e = cudaMemPoolCreate(&g_pool[dev], &props)) != cudaSuccess) return e;
        uint64_t keep = ~0ull;
        if ((e = cudaMemPoolSetAttribute(g_pool[dev], cudaMemPoolAttrReleaseThreshold, &keep)) != cudaSuccess) return e;
        // warm the pool with one large reservation (1/16 of the free memory, at
        // most 8 GB): later requests are carved from memory that is already
        // mapped, instead of the pool growing (and the host stalling) mid-join
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
            const size_t want = std::min<size_t>(8ull << 30, free_b / 16);
            void* tmp = nullptr;
            if (want > 0 && cudaMallocFromPoolAsync(&tmp, want, g_pool[dev], 0) == cudaSuccess) {
                cudaFreeAsync(tmp, 0);
                cudaStreamSynchronize(0);
            }
            cudaGetLastError();
        }
    }
    *out = g_pool[dev];
    return cudaSuccess;
}
}  // namespace

cudaError_t pool_malloc_raw(void** p, size_t bytes, cudaStream_t s) {
    cudaMemPool_t pool;
    cudaError_t e = device_pool(&pool);
    if (e != cudaSuccess) return e;
    // large requests in 32 MB granules: a freed block then fits the next step's
    // request of a slightly different size (estimate-sized result batches)
    // instead of fragmenting the cache and making the pool map new memory
    constexpr size_t kGranule = 32ull << 20;
    if (bytes > kGranule / 2) bytes = (bytes + kGranule - 1) / kGranule * kGranule;
    return cudaMallocFromPoolAsync(p, bytes, pool, s);
}

cudaError_t pool_trim() {
    cudaMemPool_t pool;
    cudaError_t e = device_pool(&pool);
    if (e != cudaSuccess) return e;
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return e;
    return cudaMemPoolTrimTo(pool, 0);
}

namespace {

__global__ void k_share_queries(const uint32_t* __restrict__ tile_order, const uint32_t* __restrict__ tile_cell,
                                const uint32_t* __restrict__ tile_q0, const uint32_t* __restrict__ cell_start,
                                uint32_t tq, JoinArgs a, unsigned long long* out) {
    unsigned long long acc = 0;
    for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < a.n_tiles; m += (int64_t)gridDim.x * blockDim.x) {
        uint32_t t = tile_order[tile_pos(a, m)];
        uint32_t g = tile_cell[t];
        acc += min(tq, cell_start[g + 1] - tile_q0[t]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

__global__ void k_pairs_to_keys(const uint2* __restrict__ p, int64_t n, uint64_t* __restrict__ key) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) key[i] = ((uint64_t)p[i].x << 32) | p[i].y;
}

__global__ void k_keys_to_pairs(const uint64_t* __restrict__ key, int64_t n, uint2* __restrict__ p) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = make_uint2((uint32_t)(key[i] >> 32), (uint32_t)key[i]);
}

__global__ void k_offsets(const uint64_t* __restrict__ key, int64_t n, int64_t npts, uint64_t* __restrict__ off) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > npts) return;
    uint64_t target = (uint64_t)i << 32;
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (key[mid] < target) lo = mid + 1; else hi = mid;
    }
    off[i] = (uint64_t)lo;
}

bool is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

bool is_pinned_host(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

int check_rank(int32_t rank, int32_t world) {
    if (world < 1 || rank < 0 || rank >= world) {
        set_error("need 0 <= rank < world");
        return GJ_ERR_INVALID;
    }
    return GJ_OK;
}

}  // namespace
}  // namespace gj

using namespace gj;

extern "C" {

int32_t gj_abi_version(void) { return 3; }

int64_t gj_launch_count(void) { return (int64_t)g_launches.load(); }

int gj_release_cached_memory(void) {
    GJ_CUDA(pool_trim());
    return GJ_OK;
}

const char* gj_last_error(void) { return g_err.c_str(); }

void gj_default_options(gj_options* opt) {
    if (!opt) return;
    memset(opt, 0, sizeof(*opt));
    opt->reorder = 1;
    opt->sortidu = 1;
    opt->shortc = 1;
    opt->symmetric = 1;
    opt->filter = 2;
    opt->sample_frac = 0.01;
}

int gj_build_index(const double* points, int64_t n_points, int32_t dim, double eps, int32_t k,
                   const gj_options* opt, gj_index** out) {
    if (!out || !points) { set_error("null argument"); return GJ_ERR_INVALID; }
    *out = nullptr;
    if (n_points < 1 || n_points >= 0xFFFFFFFFll) { set_error("n_points must be in [1, 2^32-1)"); return GJ_ERR_INVALID; }
    if (dim < 1 || dim > kMaxDim) { set_error("dim must be in [1, 128]"); return GJ_ERR_INVALID; }
    if (k < 1 || k > dim || k > kMaxK) { set_error("k must be in [1, min(dim, 16)]"); return GJ_ERR_INVALID; }
    if (!(eps > 0.0) || !std::isfinite(eps)) { set_error("eps must be finite and > 0"); return GJ_ERR_INVALID; }
    gj_options o;
    gj_default_options(&o);
    if (opt) o = *opt;
    if (!(o.sample_frac > 0.0 && o.sample_frac <= 1.0)) { set_error("sample_frac must be in (0,1]"); return GJ_ERR_INVALID; }
    gj_index* h = new gj_index();
    Index& ix = h->ix;
    ix.N = n_points;
    ix.n = dim;
    ix.n_pad = (dim + 3) & ~3;
    ix.k = k;
    ix.u = k < dim ? k : 0;
    ix.eps = eps;
    ix.eps2 = eps * eps;
    ix.opt = o;
    ix.stream = (cudaStream_t)o.stream;
    if (o.filter < 0 || o.filter > 2) { set_error("filter must be 0, 1 or 2"); delete h; return GJ_ERR_INVALID; }
    if (o.mma_tiles < 0 || o.mma_tiles > 2) { set_error("mma_tiles must be 0, 1 or 2"); delete h; return GJ_ERR_INVALID; }
    ix.filter = o.filter;
    const double* dX = points;
    double* staged = nullptr;
    int rc = GJ_OK;
    static const bool trace = getenv("GJ_TRACE") != nullptr;   // host-side phase times (diagnostics)
    const auto ta = std::chrono::steady_clock::now();
    auto ms_since = [](std::chrono::steady_clock::time_point t) {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
    };
    const bool on_device = is_device_ptr(points);
    if (trace) fprintf(stderr, "[gj] build_index: pointer query %.1f ms\n", ms_since(ta));
    if (!on_device) {
        size_t bytes = (size_t)n_points * dim * sizeof(double);
        const auto tp = std::chrono::steady_clock::now();
        const cudaError_t ea = pool_malloc(&staged, bytes, ix.stream);
        if (trace) fprintf(stderr, "[gj] build_index: staging alloc %.1f ms\n", ms_since(tp));
        if (ea != cudaSuccess) {
            cudaGetLastError();
            set_error("device allocation for staged points failed");
            delete h;
            return GJ_ERR_NOMEM;
        }
        const auto tc = std::chrono::steady_clock::now();
        cudaMemcpyAsync(staged, points, bytes, cudaMemcpyHostToDevice, ix.stream);
        if (trace) fprintf(stderr, "[gj] build_index: H2D enqueue %.1f ms\n", ms_since(tc));
        dX = staged;
    }
    if (trace) {
        const auto t0 = std::chrono::steady_clock::now();
        cudaStreamSynchronize(ix.stream);
        const auto t1 = std::chrono::steady_clock::now();
        fprintf(stderr, "[gj] build_index: staging + H2D %.1f ms\n", std::chrono::duration<double, std::milli>(t1 - t0).count());
    }
    const auto tb = std::chrono::steady_clock::now();
    rc = build_index(&ix, dX);
    if (trace)
        fprintf(stderr, "[gj] build_index: build %.1f ms\n",
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tb).count());
    if (staged) cudaFreeAsync(staged, ix.stream);
    if (rc != GJ_OK) {
        gj_free_index(h);
        return rc;
    }
    *out = h;
    return GJ_OK;
}

int gj_index_info(const gj_index* h, gj_info* info) {
    if (!h || !info) { set_error("null argument"); return GJ_ERR_INVALID; }
    const Index& ix = h->ix;
    info->n_points = ix.N;
    info->dim = ix.n;
    info->dim_pad = ix.n_pad;
    info->k = ix.k;
    info->u = ix.u;
    info->eps = ix.eps;
    info->n_cells = ix.G;
    info->n_adjacent = ix.A;
    info->n_tiles = ix.T;
    info->est_candidates = ix.est_candidates;
    info->build_ms = ix.build_ms;
    info->filter = ix.filter;
    info->filter_threshold = ix.filter >= 2 ? (float)ix.thr16 : ix.thr32;
    info->filter_margin = ix.filter >= 2 ? ix.margin16 : ix.filter_margin;
    info->tile_queries = ix.tile_q;
    info->mma_depth = ix.pts16 ? ix.k16 : 0;
    return GJ_OK;
}

int gj_dim_order(const gj_index* h, int32_t* order, int32_t cap) {
    if (!h || !order) { set_error("null argument"); return GJ_ERR_INVALID; }
    for (int t = 0; t < std::min(cap, h->ix.n); ++t) order[t] = h->ix.h_meta.order[t];
    return h->ix.n;
}

int gj_device_arrays(const gj_index* h, const double** pts, const uint32_t** orig) {
    if (!h) { set_error("null argument"); return GJ_ERR_INVALID; }
    if (pts) *pts = h->ix.pts;
    if (orig) *orig = h->ix.orig;
    return GJ_OK;
}

int gj_partition(int64_t n_tiles, int32_t rank, int32_t world, int32_t batch, int32_t n_batches, int64_t* first,
                 int64_t* step, int64_t* count, int32_t* block) {
    if (!first || !step || !count || !block || n_tiles < 0) { set_error("bad argument"); return GJ_ERR_INVALID; }
    if (int rc = check_rank(rank, world)) return rc;
    if (n_batches < 1 || batch < 0 || batch >= n_batches) { set_error("need 0 <= batch < n_batches"); return GJ_ERR_INVALID; }
    Index tmp;
    tmp.T = n_tiles;
    JoinArgs a{};
    batch_tiles(&tmp, batch, n_batches, rank, world, &a);
    *first = a.first;
    *step = a.step;
    *count = a.n_tiles;
    *block = a.blk;
    return GJ_OK;
}

int gj_fp32_threshold(double eps, int32_t n, const double* spans, float* thr, double* margin) {
    if (!spans || !thr || !margin || n < 1 || n > kMaxDim || !(eps > 0.0)) { set_error("bad argument"); return GJ_ERR_INVALID; }
    return fp32_threshold_from_spans(eps, n, spans, thr, margin);
}

int gj_fp32_accept_threshold(double eps, int32_t n, const double* spans, float* thr_in) {
    if (!spans || !thr_in || n < 1 || n > kMaxDim || !(eps > 0.0)) { set_error("bad argument"); return GJ_ERR_INVALID; }
    *thr_in = fp32_accept_threshold_from_spans(eps, n, spans);
    return GJ_OK;
}

int gj_tc_threshold(double eps, int32_t n, int32_t K, double S, double R2, double* thr, double* margin) {
    if (!thr || !margin || n < 1 || K < n + 4 || !(eps > 0.0) || !(S > 0.0) || !(R2 >= 0.0)) {
        set_error("bad argument");
        return GJ_ERR_INVALID;
    }
    return tc_threshold_from(eps, n, K, S, R2, thr, margin);
}

int gj_selftest_umma(const void* A, const void* B, float* D, uint64_t stream) {
    if (!A || !B || !D) { set_error("null argument"); return GJ_ERR_INVALID; }
    return selftest_umma(A, B, D, (cudaStream_t)stream);
}

// b_s sized against device memory (reading R15): the paper's 1e8 pairs was
// sized for 2018 GPUs; a B200 holds ~2e10 pairs.
// Sized once per device and process (cudaMemGetInfo is a driver round trip
// that can stall the host for milliseconds; the join path calls this per step).
static int64_t auto_batch_size() {
    static int64_t cached[64] = {};
    static std::mutex mu;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
        cudaGetLastError();
        return 100000000ll;
    }
    std::lock_guard<std::mutex> lock(mu);
    if (!cached[dev]) {
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
            cudaGetLastError();
            return 100000000ll;
        }
        cached[dev] = std::max<int64_t>(100000000ll, (int64_t)(free_b / 4 / 3 / 8));
    }
    return cached[dev];
}

int64_t gj_num_batches(int64_t est_pairs, int64_t batch_size) {
    if (batch_size <= 0) batch_size = auto_batch_size();
    int64_t nb = (std::max<int64_t>(est_pairs, 0) + batch_size - 1) / batch_size;
    return std::max<int64_t>(3, nb);
}

int gj_self_join_async(gj_index* h, uint32_t* out_pairs, int64_t capacity, uint64_t* d_count, int32_t batch,
                       int32_t n_batches, int32_t rank, int32_t world) {
    if (!h || !d_count || (capacity > 0 && !out_pairs) || capacity < 0) { set_error("bad argument"); return GJ_ERR_INVALID; }
    if (int rc = check_rank(rank, world)) return rc;
    if (n_batches < 1 || batch < 0 || batch >= n_batches) { set_error("need 0 <= batch < n_batches"); return GJ_ERR_INVALID; }
    JoinArgs a{};
    a.out = out_pairs;
    a.cap = (uint64_t)capacity;
    a.count = d_count;
    batch_tiles(&h->ix, batch, n_batches, rank, world, &a);
    return launch_join(&h->ix, kEmit, a, h->ix.stream);
}

int gj_self_join_async_stream(gj_index* h, uint32_t* out_pairs, int64_t capacity, uint64_t* d_count, int32_t batch,
                              int32_t n_batches, int32_t rank, int32_t world, uint64_t stream) {
    if (!h || !d_count || (capacity > 0 && !out_pairs) || capacity < 0) { set_error("bad argument"); return GJ_ERR_INVALID; }
    if (int rc = check_rank(rank, world)) return rc;
    if (n_batches < 1 || batch < 0 || batch >= n_batches) { set_error("need 0 <= batch < n_batches"); return GJ_ERR_INVALID; }
    JoinArgs a{};
    a.out = out_pairs;
    a.cap = (uint64_t)capacity;
    a.count = d_count;
    batch_tiles(&h->ix, batch, n_batches, rank, world, &a);
    return launch_join(&h->ix, kEmit, a, stream ? (cudaStream_t)stream : h->ix.stream);
}

int gj_self_join_count_async(gj_index* h, uint64_t* d_count, int32_t batch, int32_t n_batches, int32_t rank,
                             int32_t world) {
    if (!h || !d_count) { set_error("bad argument"); return GJ_ERR_INVALID; }
    if (int rc = check_rank(rank, world)) return rc;
    if (n_batches < 1 || batch < 0 || batch >= n_batches) { set_error("need 0 <= batch < n_batches"); return GJ_ERR_INVALID; }
    JoinArgs a{};
    a.count = d_count;   // [0] pairs, [1] queries of the processed tiles
    batch_tiles(&h->ix, batch, n_batches, rank, world, &a);
    return launch_join(&h->ix, kCount, a, h->ix.stream);
}

int gj_estimate(gj_index* h, double frac, int32_t rank, int32_t world, int64_t* est_pairs) {
    if (!h || !est_pairs || !(frac > 0.0 && frac <= 1.0)) { set_error("bad argument"); return GJ_ERR_INVALID; }
    if (int rc = check_rank(rank, world)) return rc;
    Index& ix = h->ix;
    cudaStream_t s = ix.stream;
    const int64_t stepf = std::max<int64_t>(1, llround(1.0 / frac));
    JoinArgs a{};
    a.count = ix.scratch_count;
    query_sets(ix.T, rank, (int64_t)world * stepf, &a);   // every stepf-th query set of the rank's share
    // a 1% sample of tiles is too few CTAs to fill 148 SMs when its tiles are
    // heavy.  Fewer sampled tiles than SMs (a rank's share on several GPUs):
    // every sampled tile's candidate scan is split over ~8 waves of 148 CTAs;
    // otherwise the work-balanced plan of launch_join splits only the heavy
    // ones (a uniform split repeats the window set-up of light tiles: songs90
    // estimate 2.8 -> 0.4 ms, profiles/r2_ab_estimator_split.txt).
    // GJ_EST_UNIFORM=0 / 1 forces either.
    static const int force = [] {
        const char* e = getenv("GJ_EST_UNIFORM");
        return e ? atoi(e) : -1;
    }();
    if (force == 1 || (force < 0 && a.n_tiles < 148))
        a.split = (int32_t)std::max<int64_t>(1, std::min<int64_t>(64, (8 * 148 + a.n_tiles - 1) / std::max<int64_t>(1, a.n_tiles)));
    GJ_CUDA(cudaMemsetAsync(ix.scratch_count, 0, 8 * sizeof(uint64_t), s));
    if (int rc = launch_join(&ix, kCount, a, s)) return rc;
    // queries of the whole share
    JoinArgs sh{};
    query_sets(ix.T, rank, world, &sh);
    if (sh.n_tiles > 0) {
        k_share_queries<<<(unsigned)std::min<int64_t>(592, (sh.n_tiles + 255) / 256), 256, 0, s>>>(
            ix.tile_order, ix.tile_cell, ix.tile_q0, ix.cell_start, (uint32_t)ix.tile_q, sh,
            (unsigned long long*)ix.scratch_count + 2); count_launch();
    }
    GJ_CUDA(cudaGetLastError());
    uint64_t c[3];
    GJ_CUDA(cudaMemcpyAsync(c, ix.scratch_count, sizeof(c), cudaMemcpyDeviceToHost, s));
    GJ_CUDA(cudaStreamSynchronize(s));
    *est_pairs = c[1] ? (int64_t)std::ceil((double)c[0] * (double)c[2] / (double)c[1]) : 0;
    return GJ_OK;
}

int gj_self_join(gj_index* h, uint32_t* out_pairs, int64_t capacity, int32_t rank, int32_t world, int64_t* n_pairs) {
    if (!h || !n_pairs) { set_error("null argument"); return GJ_ERR_INVALID; }
    Index& ix = h->ix;
    GJ_CUDA(cudaMemsetAsync(ix.scratch_count, 0, sizeof(uint64_t), ix.stream));
    if (int rc = gj_self_join_async(h, out_pairs, capacity, ix.scratch_count, 0, 1, rank, world)) return rc;
    uint64_t c = 0;
    GJ_CUDA(cudaMemcpyAsync(&c, ix.scratch_count, sizeof(c), cudaMemcpyDeviceToHost, ix.stream));
    GJ_CUDA(cudaStreamSynchronize(ix.stream));
    *n_pairs = (int64_t)c;
    if ((int64_t)c > capacity) {
        set_error("result buffer too small");
        return GJ_ERR_CAPACITY;
    }
    return GJ_OK;
}

int gj_self_join_host(gj_index* h, uint32_t* out_pairs, int64_t capacity, int32_t rank, int32_t world,
                      int64_t batch_size, int64_t* n_pairs, int32_t* n_batches_out) {
    if (!h || !n_pairs || (capacity > 0 && !out_pairs) || capacity < 0) { set_error("bad argument"); return GJ_ERR_INVALID; }
    if (int rc = check_rank(rank, world)) return rc;
    Index& ix = h->ix;
    if (batch_size <= 0) batch_size = auto_batch_size();
    int64_t est = 0;
    if (int rc = gj_estimate(h, 0.01, rank, world, &est)) return rc;
    const int64_t nb = gj_num_batches(est, batch_size);
    if (n_batches_out) *n_batches_out = (int32_t)nb;
    // per-stream device buffers sized for one batch (+25% headroom over the estimate);
    // a slot whose batch overflows is regrown on its own (cap_of[i])
    // (GJ_BATCH_HEADROOM overrides the 1.25 factor: tests force the regrow path with it)
    static const double headroom = [] { const char* e = getenv("GJ_BATCH_HEADROOM"); return e ? atof(e) : 1.25; }();
    const int64_t per = std::max<int64_t>(1024, (int64_t)(headroom * (double)est / (double)nb) + 1024);
    int64_t cap_of[3] = {per, per, per};
    const bool direct = out_pairs && is_pinned_host(out_pairs);
    uint32_t* dbuf[3] = {nullptr, nullptr, nullptr};
    uint32_t* hbuf[3] = {nullptr, nullptr, nullptr};
    uint64_t* dcnt = nullptr;
    uint64_t* hcnt = nullptr;
    int rc = GJ_OK;
    int64_t written = 0;
    bool overflow = false;
    auto cleanup = [&]() {
        for (int i = 0; i < 3; ++i) {
            if (dbuf[i]) cudaFreeAsync(dbuf[i], ix.stream);
            if (hbuf[i]) cudaFreeHost(hbuf[i]);
        }
        if (dcnt) cudaFreeAsync(dcnt, ix.stream);
        cudaStreamSynchronize(ix.stream);
        if (hcnt) cudaFreeHost(hcnt);
    };
    // a CUDA error anywhere below records the message and rc, and falls through
    // to cleanup() (no early return leaks the slot buffers)
    auto cu = [&](cudaError_t e, const char* what) -> bool {
        if (e == cudaSuccess) return true;
        set_error(std::string("gj_self_join_host: ") + what + ": " + cudaGetErrorString(e));
        if (rc == GJ_OK) rc = GJ_ERR_CUDA;
        return false;
    };
    for (int i = 0; i < 3; ++i) {
        if (!ix.pipe_stream[i]) {
            if (!cu(cudaStreamCreateWithFlags(&ix.pipe_stream[i], cudaStreamNonBlocking), "stream") ||
                !cu(cudaEventCreateWithFlags(&ix.pipe_event[i], cudaEventDisableTiming), "event")) {
                cleanup();
                return rc;
            }
        }
        if (pool_malloc(&dbuf[i], (size_t)per * 2 * sizeof(uint32_t), ix.stream) != cudaSuccess ||
            (!direct && cudaMallocHost(&hbuf[i], (size_t)per * 2 * sizeof(uint32_t)) != cudaSuccess)) {
            cudaGetLastError();
            cleanup();
            set_error("result buffer allocation failed");
            return GJ_ERR_NOMEM;
        }
    }
    if (pool_malloc(&dcnt, 3 * sizeof(uint64_t), ix.stream) != cudaSuccess || cudaMallocHost(&hcnt, 3 * sizeof(uint64_t)) != cudaSuccess) {
        cudaGetLastError();
        cleanup();
        set_error("counter allocation failed");
        return GJ_ERR_NOMEM;
    }
    // the pipeline streams wait for the index build on the index stream
    cudaEvent_t ready = nullptr;
    if (cu(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming), "event") && cu(cudaEventRecord(ready, ix.stream), "record"))
        for (int i = 0; i < 3 && rc == GJ_OK; ++i) cu(cudaStreamWaitEvent(ix.pipe_stream[i], ready, 0), "wait");
    if (ready) cudaEventDestroy(ready);

    int64_t pending_n[3] = {0, 0, 0};
    int64_t pending_at[3] = {-1, -1, -1};
    auto drain = [&](int i) -> int {   // host side of batch in slot i ("Table" stage)
        if (pending_at[i] < 0) return GJ_OK;
        if (!cu(cudaEventSynchronize(ix.pipe_event[i]), "drain")) return rc;
        if (!direct && pending_n[i] > 0 && pending_at[i] + pending_n[i] <= capacity)
            memcpy(out_pairs + 2 * pending_at[i], hbuf[i], (size_t)pending_n[i] * 2 * sizeof(uint32_t));
        pending_at[i] = -1;
        return GJ_OK;
    };
    for (int64_t b = 0; b < nb && rc == GJ_OK; ++b) {
        const int i = (int)(b % 3);
        cudaStream_t st = ix.pipe_stream[i];
        if (drain(i) != GJ_OK) break;
        // kernel (retry with a larger buffer if the estimate was low)
        for (;;) {
            if (!cu(cudaMemsetAsync(dcnt + i, 0, sizeof(uint64_t), st), "memset")) break;
            JoinArgs a{};
            a.out = dbuf[i];
            a.cap = (uint64_t)cap_of[i];
            a.count = dcnt + i;
            batch_tiles(&ix, (int32_t)b, (int32_t)nb, rank, world, &a);
            if ((rc = launch_join(&ix, kEmit, a, st))) break;
            if (!cu(cudaMemcpyAsync(hcnt + i, dcnt + i, sizeof(uint64_t), cudaMemcpyDeviceToHost, st), "count D2H") ||
                !cu(cudaStreamSynchronize(st), "batch"))
                break;
            if ((int64_t)hcnt[i] <= cap_of[i]) break;
            // re-plan: grow this slot's buffers and rerun the batch (§3.2.2 estimate was low)
            cap_of[i] = (int64_t)hcnt[i] + 1024;
            cudaFreeAsync(dbuf[i], st);
            dbuf[i] = nullptr;
            if (pool_malloc(&dbuf[i], (size_t)cap_of[i] * 2 * sizeof(uint32_t), st) != cudaSuccess) { cudaGetLastError(); rc = GJ_ERR_NOMEM; break; }
            if (!direct) {
                cudaFreeHost(hbuf[i]);
                hbuf[i] = nullptr;
                if (cudaMallocHost(&hbuf[i], (size_t)cap_of[i] * 2 * sizeof(uint32_t)) != cudaSuccess) { cudaGetLastError(); rc = GJ_ERR_NOMEM; break; }
            }
        }
        if (rc) break;
        const int64_t cnt = (int64_t)hcnt[i];
        if (written + cnt > capacity) overflow = true;
        if (cnt > 0 && !overflow) {
            void* dst = direct ? (void*)(out_pairs + 2 * written) : (void*)hbuf[i];
            if (!cu(cudaMemcpyAsync(dst, dbuf[i], (size_t)cnt * 2 * sizeof(uint32_t), cudaMemcpyDeviceToHost, st), "pairs D2H")) break;
        }
        if (!cu(cudaEventRecord(ix.pipe_event[i], st), "record")) break;
        pending_at[i] = overflow ? -2 : written;
        pending_n[i] = cnt;
        if (overflow) pending_at[i] = -1;
        written += cnt;
    }
    for (int i = 0; i < 3 && rc == GJ_OK; ++i) drain(i);
    for (int i = 0; i < 3; ++i) cudaStreamSynchronize(ix.pipe_stream[i]);
    cleanup();
    *n_pairs = written;
    if (rc) return rc;
    if (overflow) {
        set_error("host result buffer too small");
        return GJ_ERR_CAPACITY;
    }
    return GJ_OK;
}

int gj_join_counts(gj_index* h, int32_t rank, int32_t world, gj_stats* st) {
    if (!h || !st) { set_error("null argument"); return GJ_ERR_INVALID; }
    if (int rc = check_rank(rank, world)) return rc;
    Index& ix = h->ix;
    JoinArgs a{};
    batch_tiles(&ix, 0, 1, rank, world, &a);
    GJ_CUDA(cudaMemsetAsync(ix.scratch_count, 0, 8 * sizeof(uint64_t), ix.stream));
    if (int rc = count_tests(&ix, a, (unsigned long long*)ix.scratch_count, ix.stream)) return rc;
    uint64_t c[3];
    GJ_CUDA(cudaMemcpyAsync(c, ix.scratch_count, sizeof(c), cudaMemcpyDeviceToHost, ix.stream));
    GJ_CUDA(cudaStreamSynchronize(ix.stream));
    st->cells = (int64_t)c[0];
    st->tests = (int64_t)c[1];
    st->tests_evaluated = (int64_t)c[2];
    st->dims = st->pairs = st->dims_evaluated = -1;
    return GJ_OK;
}

int gj_join_mma_tests(gj_index* h, int32_t rank, int32_t world, int64_t* mma_tests) {
    if (!h || !mma_tests) { set_error("null argument"); return GJ_ERR_INVALID; }
    if (int rc = check_rank(rank, world)) return rc;
    Index& ix = h->ix;
    *mma_tests = -1;
    if (ix.filter != 2) return GJ_OK;
    JoinArgs a{};
    a.count = ix.scratch_count;
    a.mma_tests = (unsigned long long*)ix.scratch_count + 4;
    batch_tiles(&ix, 0, 1, rank, world, &a);
    GJ_CUDA(cudaMemsetAsync(ix.scratch_count, 0, 8 * sizeof(uint64_t), ix.stream));
    if (int rc = launch_join(&ix, kCount, a, ix.stream)) return rc;
    uint64_t c = 0;
    GJ_CUDA(cudaMemcpyAsync(&c, ix.scratch_count + 4, sizeof(c), cudaMemcpyDeviceToHost, ix.stream));
    GJ_CUDA(cudaStreamSynchronize(ix.stream));
    *mma_tests = (int64_t)c;
    return GJ_OK;
}

int gj_join_stats(gj_index* h, int32_t rank, int32_t world, gj_stats* st) {
    if (!h || !st) { set_error("null argument"); return GJ_ERR_INVALID; }
    if (int rc = check_rank(rank, world)) return rc;
    Index& ix = h->ix;
    JoinArgs a{};
    a.count = ix.scratch_count;
    batch_tiles(&ix, 0, 1, rank, world, &a);
    GJ_CUDA(cudaMemsetAsync(ix.scratch_count, 0, 8 * sizeof(uint64_t), ix.stream));
    if (int rc = launch_join(&ix, kStats, a, ix.stream)) return rc;
    uint64_t c[6];
    GJ_CUDA(cudaMemcpyAsync(c, ix.scratch_count, sizeof(c), cudaMemcpyDeviceToHost, ix.stream));
    GJ_CUDA(cudaStreamSynchronize(ix.stream));
    st->pairs = (int64_t)c[0];
    st->cells = (int64_t)c[1];
    st->tests = (int64_t)c[2];
    st->dims = (int64_t)c[3];
    st->tests_evaluated = (int64_t)c[4];
    st->dims_evaluated = (int64_t)c[5];
    return GJ_OK;
}

int gj_neighbor_table(gj_index* h, uint32_t* pairs, int64_t n_pairs, uint64_t* offsets) {
    if (!h || (n_pairs > 0 && !pairs) || !offsets || n_pairs < 0) { set_error("bad argument"); return GJ_ERR_INVALID; }
    // the radix sort's histogram scan and scatter offsets are 32-bit
    if (n_pairs > (int64_t)UINT32_MAX) { set_error("gj_neighbor_table: n_pairs > 2^32-1"); return GJ_ERR_INVALID; }
    Index& ix = h->ix;
    cudaStream_t s = ix.stream;
    uint64_t* keys = nullptr;
    uint32_t* vals = nullptr;
    const int64_t n = std::max<int64_t>(n_pairs, 1);
    GJ_CUDA(pool_malloc(&keys, n * sizeof(uint64_t), s));
    GJ_CUDA(pool_malloc(&vals, n * sizeof(uint32_t), s));
    unsigned blocks = (unsigned)((n + 255) / 256);
    if (n_pairs > 0) {
        k_pairs_to_keys<<<blocks, 256, 0, s>>>(reinterpret_cast<const uint2*>(pairs), n_pairs, keys); count_launch();
        GJ_CUDA(cudaGetLastError());
        uint64_t vb = 0;
        if (int rc = varying_bits_u64(keys, n_pairs, &vb, s)) return rc;
        if (int rc = radix_sort_u64(keys, vals, n_pairs, vb, s)) return rc;
        k_keys_to_pairs<<<blocks, 256, 0, s>>>(keys, n_pairs, reinterpret_cast<uint2*>(pairs)); count_launch();
    }
    k_offsets<<<(unsigned)((ix.N + 1 + 255) / 256), 256, 0, s>>>(keys, n_pairs, ix.N, offsets); count_launch();
    GJ_CUDA(cudaGetLastError());
    GJ_CUDA(cudaFreeAsync(keys, s));
    GJ_CUDA(cudaFreeAsync(vals, s));
    GJ_CUDA(cudaStreamSynchronize(s));
    return GJ_OK;
}

void gj_free_index(gj_index* h) {
    if (!h) return;
    Index& ix = h->ix;
    // joins launched with gj_self_join_async_stream on caller streams may still
    // read pts / pts16 / nbr: wait for all work on the device before the arrays
    // go back to the pool (which reuses them at once)
    cudaDeviceSynchronize();
    cudaGetLastError();
    void* ptrs[] = {ix.pts, ix.pts32, ix.pts16, ix.norm16, ix.orig, ix.cell_id, ix.cell_start, ix.nbr_off, ix.nbr, ix.nbr_self, ix.tile_cell, ix.tile_q0,
                    ix.tile_order, ix.tile_work, ix.meta, ix.scratch_count};
    for (void* p : ptrs)   // back to the library pool (stream-ordered)
        if (p) cudaFreeAsync(p, ix.stream);
    cudaStreamSynchronize(ix.stream);
    for (int i = 0; i < 3; ++i) {
        if (ix.pipe_stream[i]) cudaStreamDestroy(ix.pipe_stream[i]);
        if (ix.pipe_event[i]) cudaEventDestroy(ix.pipe_event[i]);
    }
    delete h;
}

}  // extern "C"
