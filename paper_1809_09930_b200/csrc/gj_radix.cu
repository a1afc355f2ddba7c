// Device-wide exclusive scan and stable LSD radix sort (uint64 keys, uint32
// values) used by constructIndex: the "device radix sort of points by cell id"
// of the north_star (§3.2.1 l.121: points sorted so that points close
// in space are close in memory), and by the heaviest-first tile ordering.
//
// Radix pass = 3 kernels: per-tile digit histogram, exclusive scan of the
// digit-major histogram, stable scatter.  Tile = 256 threads x 8 keys; the
// scatter ranks keys with __match_any_sync per warp-round so equal digits keep
// their input order (stability is what makes the (cell, u) two-key sort work).
#include <algorithm>
#include <vector>

#include "gj_internal.cuh"

namespace gj {
namespace {

constexpr int kThreads = 256;
constexpr int kItems = 8;
constexpr int kTile = kThreads * kItems;   // 2048 keys per block
constexpr int kWarps = kThreads / 32;

// ---------------------------------------------------------------- scan
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* total, uint32_t* sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        sh[lane] = w;   // inclusive warp totals
    }
    __syncthreads();
    uint32_t warp_off = warp ? sh[warp - 1] : 0;
    *total = sh[(blockDim.x >> 5) - 1];
    __syncthreads();
    return warp_off + x - v;
}

__global__ void k_scan_reduce(const uint32_t* __restrict__ in, int64_t n, uint32_t* __restrict__ sums) {
    __shared__ uint32_t sh[32];
    int64_t base = (int64_t)blockIdx.x * kScanTile;
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        int64_t e = base + (int64_t)i * kScanThreads + threadIdx.x;
        if (e < n) s += in[e];
    }
    uint32_t tot;
    block_exclusive_scan(s, &tot, sh);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// Single block: exclusive scan of the per-block sums in place (serial chunks).
__global__ void k_scan_sums(uint32_t* sums, int64_t nb, uint32_t* d_total) {
    __shared__ uint32_t sh[32];
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t c = 0; c < nb; c += blockDim.x) {
        int64_t e = c + threadIdx.x;
        uint32_t v = e < nb ? sums[e] : 0;
        uint32_t tot;
        uint32_t ex = block_exclusive_scan(v, &tot, sh);
        if (e < nb) sums[e] = carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0 && d_total) *d_total = carry;
}

__global__ void k_scan_down(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, int64_t n,
                            const uint32_t* __restrict__ sums) {
    __shared__ uint32_t sh[32];
    int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    uint32_t v[kScanItems];
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        int64_t e = base + i;
        v[i] = e < n ? in[e] : 0;
        s += v[i];
    }
    uint32_t tot;
    uint32_t ex = block_exclusive_scan(s, &tot, sh) + sums[blockIdx.x];
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        int64_t e = base + i;
        if (e < n) out[e] = ex;
        ex += v[i];
    }
}

// ---------------------------------------------------------------- radix
__global__ void k_radix_hist(const uint64_t* __restrict__ keys, int64_t n, int shift,
                             uint32_t* __restrict__ hist, int64_t nblocks) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    int64_t base = (int64_t)blockIdx.x * kTile;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        int64_t e = base + (int64_t)i * kThreads + threadIdx.x;
        if (e < n) atomicAdd(&h[(keys[e] >> shift) & 0xFF], 1u);
    }
    __syncthreads();
    hist[(int64_t)threadIdx.x * nblocks + blockIdx.x] = h[threadIdx.x];   // digit-major
}

__global__ void k_radix_scatter(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                                uint64_t* __restrict__ okeys, uint32_t* __restrict__ ovals, int64_t n,
                                int shift, const uint32_t* __restrict__ offs, int64_t nblocks) {
    __shared__ uint32_t wh[kWarps][256];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kWarps * 256; i += kThreads) (&wh[0][0])[i] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kTile + (int64_t)warp * (32 * kItems);
    const unsigned lt = (1u << lane) - 1u;
    uint64_t k[kItems];
    uint32_t v[kItems], local[kItems];
    int dg[kItems];
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        int64_t e = base + r * 32 + lane;
        bool valid = e < n;
        k[r] = valid ? keys[e] : 0;
        v[r] = valid ? vals[e] : 0;
        int d = valid ? (int)((k[r] >> shift) & 0xFF) : 256 + lane;
        dg[r] = d;
        unsigned peers = __match_any_sync(0xffffffffu, d);
        uint32_t before = valid ? wh[warp][d] : 0;
        local[r] = before + __popc(peers & lt);
        __syncwarp();
        if (valid && (__ffs(peers) - 1) == lane) wh[warp][d] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // exclusive prefix over warps for every digit
    {
        int d = threadIdx.x;   // kThreads == 256 digits
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            uint32_t t = wh[w][d];
            wh[w][d] = run;
            run += t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        int64_t e = base + r * 32 + lane;
        if (e < n) {
            int d = dg[r];
            uint64_t pos = (uint64_t)offs[(int64_t)d * nblocks + blockIdx.x] + wh[warp][d] + local[r];
            okeys[pos] = k[r];
            ovals[pos] = v[r];
        }
    }
}

__global__ void k_or_xor(const uint64_t* __restrict__ keys, int64_t n, unsigned long long* out) {
    __shared__ unsigned long long sh[32];
    uint64_t k0 = keys[0], acc = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        acc |= keys[i] ^ k0;
#pragma unroll
    for (int o = 16; o; o >>= 1) acc |= __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) acc |= sh[w];
        atomicOr(out, (unsigned long long)acc);
    }
}

}  // namespace

int scan_u32(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* d_total, cudaStream_t s) {
    if (n <= 0) {
        if (d_total) GJ_CUDA(cudaMemsetAsync(d_total, 0, sizeof(uint32_t), s));
        return GJ_OK;
    }
    int64_t nb = (n + kScanTile - 1) / kScanTile;
    uint32_t* sums = nullptr;
    GJ_CUDA(pool_malloc(&sums, nb * sizeof(uint32_t), s));
    k_scan_reduce<<<(unsigned)nb, kScanThreads, 0, s>>>(in, n, sums); count_launch();
    k_scan_sums<<<1, 1024, 0, s>>>(sums, nb, d_total); count_launch();
    k_scan_down<<<(unsigned)nb, kScanThreads, 0, s>>>(in, out, n, sums); count_launch();
    GJ_CUDA(cudaGetLastError());
    GJ_CUDA(cudaFreeAsync(sums, s));
    return GJ_OK;
}

int varying_bits_u64(const uint64_t* keys, int64_t n, uint64_t* h_out, cudaStream_t s) {
    *h_out = 0;
    if (n <= 1) return GJ_OK;
    unsigned long long* d = nullptr;
    GJ_CUDA(pool_malloc(&d, sizeof(*d), s));
    GJ_CUDA(cudaMemsetAsync(d, 0, sizeof(*d), s));
    int blocks = (int)std::min<int64_t>(1184, (n + 255) / 256);
    k_or_xor<<<blocks, 256, 0, s>>>(keys, n, d); count_launch();
    GJ_CUDA(cudaGetLastError());
    GJ_CUDA(cudaMemcpyAsync(h_out, d, sizeof(*d), cudaMemcpyDeviceToHost, s));
    GJ_CUDA(cudaFreeAsync(d, s));
    GJ_CUDA(cudaStreamSynchronize(s));
    return GJ_OK;
}

int radix_sort_u64(uint64_t* keys, uint32_t* vals, int64_t n, uint64_t bits_mask, cudaStream_t s) {
    if (n <= 1 || bits_mask == 0) return GJ_OK;
    const int64_t nb = (n + kTile - 1) / kTile;
    uint64_t* k2 = nullptr;
    uint32_t *v2 = nullptr, *hist = nullptr;
    GJ_CUDA(pool_malloc(&k2, n * sizeof(uint64_t), s));
    GJ_CUDA(pool_malloc(&v2, n * sizeof(uint32_t), s));
    GJ_CUDA(pool_malloc(&hist, 256 * nb * sizeof(uint32_t), s));
    uint64_t *ka = keys, *kb = k2;
    uint32_t *va = vals, *vb = v2;
    int rc = GJ_OK;
    for (int shift = 0; shift < 64; shift += 8) {
        if (((bits_mask >> shift) & 0xFFull) == 0) continue;
        k_radix_hist<<<(unsigned)nb, kThreads, 0, s>>>(ka, n, shift, hist, nb); count_launch();
        rc = scan_u32(hist, hist, 256 * nb, nullptr, s);
        if (rc) return rc;
        k_radix_scatter<<<(unsigned)nb, kThreads, 0, s>>>(ka, va, kb, vb, n, shift, hist, nb); count_launch();
        GJ_CUDA(cudaGetLastError());
        std::swap(ka, kb);
        std::swap(va, vb);
    }
    if (ka != keys) {
        GJ_CUDA(cudaMemcpyAsync(keys, ka, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
        GJ_CUDA(cudaMemcpyAsync(vals, va, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
    }
    GJ_CUDA(cudaFreeAsync(k2, s));
    GJ_CUDA(cudaFreeAsync(v2, s));
    GJ_CUDA(cudaFreeAsync(hist, s));
    return GJ_OK;
}

}  // namespace gj
