// SelfJoinKernel on the 5th-generation tensor cores (tcgen05.mma, TMEM
// accumulators) with the certified distance bound of gj_join_tc.cu and the
// FP64 decision of every surviving pair (B200-first variant of PAPER.md
// Alg. 1 l.596-607; FP64 semantics unchanged).
//
// CTA = 256 threads = one 128-query tile of one cell.  The tile's fp16
// operand rows (A, M = 128) sit in shared memory in the canonical K-major
// UMMA layout for the whole CTA lifetime.  The candidates of every adjacent
// cell's SORTIDU window stream through a 3-buffer cp.async ring of
// 128-candidate blocks (B, N = 128).  Thread 0 issues, per block, K/16
// tcgen05.mma into one of two 128-column TMEM accumulators and commits to an
// mbarrier; while the tensor core works on block kb, all 8 warps run the
// epilogue of block kb-1: tcgen05.ld (warp w reads TMEM lanes 32(w%4).. and
// columns 64(w/4)..), v = ||c^||^2 - 2 acc, survivor iff v <= thr - ||q^||^2,
// and the rare survivors are decided in FP64 and emitted.
#include "gj_internal.cuh"
#include "gj_umma.cuh"

namespace gj {
namespace {

constexpr int kM = 128;         // queries per tile (UMMA M)
constexpr int kN = 128;         // candidates per block (UMMA N)
constexpr int kThreads = 256;   // 8 warps
// B ring depth: as many 128-candidate stages as fit next to the A tile in
// ~100 KB (two CTAs per SM), at least 3; prefetch distance = stages - 1.
template <int KP>
constexpr int stages() {
    return (100 * 1024 - kM * KP * 2) / (kN * KP * 2) < 3 ? 3 : ((100 * 1024 - kM * KP * 2) / (kN * KP * 2) > 8 ? 8 : (100 * 1024 - kM * KP * 2) / (kN * KP * 2));
}

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

template <int KP>
struct Smem {
    alignas(128) __half a[kM * KP];
    alignas(128) __half b[stages<KP>()][kN * KP];
    uint64_t mbar[2];
    uint32_t tmem_base;
    uint32_t win[2];
    unsigned long long red[kThreads / 32];
};

template <int KP, int MODE, bool SYM>
__global__ void __launch_bounds__(kThreads) k_join_umma(JoinParams P, JoinArgs A) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem<KP>& S = *reinterpret_cast<Smem<KP>*>(smem_raw);
    constexpr int KS = KP / 16;
    constexpr int kBufs = stages<KP>();
    constexpr uint32_t kIdesc = umma::idesc_f16_f32(kM, kN);
    constexpr uint32_t kSBO = KP * 16;   // bytes between 8-row groups

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

    // ---- setup: TMEM (warp 0), mbarriers (thread 0), the A tile (all)
    if (warp == 0) umma::tmem_alloc(&S.tmem_base, 2 * kN);
    if (tid == 0) {
        umma::mbar_init(&S.mbar[0], 1);
        umma::mbar_init(&S.mbar[1], 1);
        umma::mbar_fence_init();
    }
    const uint32_t a_s = umma::smem_u32(S.a);
    unsigned char* a_raw = reinterpret_cast<unsigned char*>(S.a);
    for (int i = tid; i < kM * (KP / 8); i += kThreads) {
        const int row = i / (KP / 8), kc = i % (KP / 8);
        const uint32_t off = umma::tile_off(row, kc * 8, KP);
        const bool valid = row < (int)nq;
        if (kc < KP / 8 - 1) {
            if (valid) umma::cp_async16(a_s + off, P.pts16 + (size_t)(q0 + row) * KP + kc * 8);
            else *reinterpret_cast<uint4*>(a_raw + off) = make_uint4(0, 0, 0, 0);
        } else {   // last chunk: coordinates (if any) + query-side augmented columns (r_hi, r_lo, 1, 1)
            union { uint4 u; __half h[8]; } c;
            c.u = valid ? *reinterpret_cast<const uint4*>(P.pts16 + (size_t)(q0 + row) * KP + kc * 8) : make_uint4(0, 0, 0, 0);
            query_aug(P.thr16, valid ? P.norm16[q0 + row] : 0.0, valid, c.h[4], c.h[5]);
            c.h[6] = __float2half(1.f);
            c.h[7] = __float2half(1.f);
            *reinterpret_cast<uint4*>(a_raw + off) = c.u;
        }
    }
    umma::cp_async_commit();
    // this thread's epilogue row (TMEM lane) and column half
    const int erow = 32 * (warp & 3) + lane;
    const int ecol0 = 64 * (warp >> 2);
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tmem = S.tmem_base;

    unsigned long long npairs = 0;
    if (SYM && part == 0) {   // the self pair (q, q)
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

    uint32_t phase[2] = {0, 0};
    const double u_lo = P.pts[(size_t)q0 * n_pad + P.u];
    const double u_hi = P.pts[(size_t)(q0 + nq - 1) * n_pad + P.u];
    const uint32_t nb0 = SYM ? P.nbr_self[g] : P.nbr_off[g], nb1 = P.nbr_off[g + 1];
    for (uint32_t nbi = nb0; nbi < nb1; ++nbi) {
        const uint32_t B = P.nbr[nbi];
        uint32_t r = P.cell_start[B], s = P.cell_start[B + 1];
        __syncthreads();   // previous window fully consumed (buffers, S.win)
        if (P.sortidu) {   // tile-level SORTIDU window (exact predicates on the fp64 u-coordinates)
            if (tid < 2) {
                uint32_t lo = r, hi = s;
                while (lo < hi) {
                    uint32_t mid = (lo + hi) >> 1;
                    double cu = P.pts[(size_t)mid * n_pad + P.u];
                    bool pred = tid == 0 ? (u_lo - cu <= eps) : (cu - u_hi > eps);
                    if (pred) hi = mid; else lo = mid + 1;
                }
                S.win[tid] = lo;
            }
            __syncthreads();
            r = S.win[0];
            s = max(S.win[1], r);
        }
        const bool diag = SYM && B == g;
        if (diag) r = max(r, q0 + 1);
        if (split > 1 && s > r) {
            const uint64_t len = s - r;
            s = r + (uint32_t)(len * (part + 1) / split);
            r = r + (uint32_t)(len * part / split);
        }
        if (s <= r) continue;
        const int nblk = (int)((s - r + kN - 1) / kN);

        auto load_block = [&](int kb) {
            const int buf = kb % kBufs;
            const uint32_t start = r + (uint32_t)kb * kN;
            const int cnt = (int)min((uint32_t)kN, s - start);
            const uint32_t b_s = umma::smem_u32(S.b[buf]);
            for (int i = tid; i < kN * (KP / 8); i += kThreads) {
                const int row = i / (KP / 8), kc = i % (KP / 8);
                const uint32_t off = umma::tile_off(row, kc * 8, KP);
                if (row < cnt) {
                    umma::cp_async16(b_s + off, P.pts16 + (size_t)(start + row) * KP + kc * 8);
                } else {   // padding candidate: zeros, h_hi = -65504 -> every accumulator < 0
                    union { uint4 u; __half h[8]; } c;
                    c.u = make_uint4(0, 0, 0, 0);
                    if (kc == KP / 8 - 1) c.h[6] = __float2half(-65504.f);
                    *reinterpret_cast<uint4*>(reinterpret_cast<unsigned char*>(S.b[buf]) + off) = c.u;
                }
            }
        };
        auto epilogue = [&](int kb) {
            const int ab = kb & 1;
            umma::mbar_wait(&S.mbar[ab], phase[ab]);
            phase[ab] ^= 1u;
            umma::fence_after();
            const uint32_t cbase = r + (uint32_t)kb * kN;
            // acc = (T - ||q^ - c^||^2) / 2 + err: a pair survives iff acc > +0 (sign bit clear)
            float v[2][32];
#pragma unroll
            for (int h = 0; h < 2; ++h)
                umma::tmem_ld32(tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(ab * kN + ecol0 + 32 * h), v[h]);
            uint32_t all = 0xffffffffu;
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int i = 0; i < 32; ++i) all &= __float_as_uint(v[h][i]);
            unsigned long long mask = 0;
            if (!(all >> 31)) {   // rare: some accumulator non-negative
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (!(__float_as_uint(v[h][i]) >> 31)) mask |= 1ull << (32 * h + i);
            }
            umma::fence_before();
            while (mask) {   // rare: FP64 decision of the survivors
                const int bit = __ffsll((long long)mask) - 1;
                mask &= mask - 1;
                const uint32_t qpos = q0 + erow, cpos = cbase + ecol0 + bit;
                if (diag && cpos <= qpos) continue;
                npairs += decide_and_emit<MODE, SYM>(P, A, qpos, cpos);
            }
        };

#pragma unroll
        for (int p = 0; p < kBufs - 1; ++p) {   // prologue: prefetch kBufs-1 blocks
            if (p < nblk) load_block(p);
            umma::cp_async_commit();
        }
        for (int kb = 0; kb < nblk; ++kb) {
            umma::cp_async_wait<kBufs - 2>();   // block kb (and the A tile) landed; later ones may be in flight
            umma::fence_proxy_async();
            __syncthreads();
            if (tid == 0) {
                umma::fence_after();
                const uint32_t a0 = a_s, b0 = umma::smem_u32(S.b[kb % kBufs]);
                const uint32_t d = tmem + (uint32_t)((kb & 1) * kN);
#pragma unroll
                for (int ks = 0; ks < KS; ++ks)
                    umma::mma_f16(d, umma::smem_desc(a0 + ks * 256, 128, kSBO), umma::smem_desc(b0 + ks * 256, 128, kSBO),
                                  kIdesc, ks > 0 ? 1u : 0u);
                umma::commit(&S.mbar[kb & 1]);
            }
            if (kb >= 1) epilogue(kb - 1);   // overlaps MMA(kb)
            if (kb + kBufs - 1 < nblk) load_block(kb + kBufs - 1);   // buffer of block kb-1 (its MMA completed)
            umma::cp_async_commit();
        }
        epilogue(nblk - 1);
    }
    umma::cp_async_wait<0>();
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc(tmem, 2 * kN);

    if (MODE == kCount) {
        unsigned long long x = npairs;
#pragma unroll
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) S.red[warp] = x;
        __syncthreads();
        if (tid == 0) {
            unsigned long long t = 0;
            for (int w = 0; w < kThreads / 32; ++w) t += S.red[w];
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

template <int KP>
int launch_umma(const JoinParams& p, JoinMode mode, const JoinArgs& a, bool sym, cudaStream_t s) {
    if (a.n_tiles <= 0) return GJ_OK;
    // request enough dynamic smem that at most 2 CTAs share an SM: the two
    // CTAs' 2 x 256 TMEM columns fill the SM's 512
    const size_t smem = std::max<size_t>(sizeof(Smem<KP>), 80 * 1024);
    static_assert(sizeof(Smem<KP>) <= 227 * 1024, "shared memory");
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
            if ((rc = setattr((const void*)k_join_umma<KP, kEmit, true>, 0, 1))) return rc;
            k_join_umma<KP, kEmit, true><<<grid, kThreads, smem, s>>>(p, a);
        } else {
            if ((rc = setattr((const void*)k_join_umma<KP, kEmit, false>, 0, 0))) return rc;
            k_join_umma<KP, kEmit, false><<<grid, kThreads, smem, s>>>(p, a);
        }
    } else {
        if (sym) {
            if ((rc = setattr((const void*)k_join_umma<KP, kCount, true>, 1, 1))) return rc;
            k_join_umma<KP, kCount, true><<<grid, kThreads, smem, s>>>(p, a);
        } else {
            if ((rc = setattr((const void*)k_join_umma<KP, kCount, false>, 1, 0))) return rc;
            k_join_umma<KP, kCount, false><<<grid, kThreads, smem, s>>>(p, a);
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
    switch (ix->k16) {
        case 16: return launch_umma<16>(p, mode, a, sym, s);
        case 32: return launch_umma<32>(p, mode, a, sym, s);
        case 48: return launch_umma<48>(p, mode, a, sym, s);
        case 64: return launch_umma<64>(p, mode, a, sym, s);
        case 80: return launch_umma<80>(p, mode, a, sym, s);
        case 96: return launch_umma<96>(p, mode, a, sym, s);
        case 112: return launch_umma<112>(p, mode, a, sym, s);
        default: return launch_umma<128>(p, mode, a, sym, s);
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
