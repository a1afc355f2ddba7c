// SelfJoinKernel with a certified tensor-core distance bound (B200-first
// variant of PAPER.md Alg. 1 l.596-607; FP64 semantics unchanged).
//
// On the worst-case data of §5.5 (exponential, low variance) the grid cells
// are huge and the candidate work of a query tile against an adjacent cell is
// a dense all-pairs block.  Over such blocks ||q - c||^2 = ||q||^2 + ||c||^2
// - 2 q.c, and q.c for a 128-query x 64-candidate block is a small GEMM:
// the tensor cores evaluate it (fp16 operands fp16(S (x - min)), fp32
// accumulation, mma.sync m16n8k16) and the epilogue rejects every pair whose
// bound v = ||c^||^2 - 2 acc exceeds thr - ||q^||^2 -- which PROVES
// dist > eps (1 + 1e-9) (gj_index.cu tc_threshold_from).  The rare
// pairs the bound cannot reject are decided by the FP64 test with exactly the
// FP64 kernel's arithmetic, so the emitted pair set is the FP64 kernel's.
//
// CTA = 4 warps = one 128-query tile of one cell (as in gj_join.cu), warp w
// owns queries 32w..32w+31 as two m16 MMA row tiles held in registers (A
// fragments).  Candidates of every adjacent cell's SORTIDU window stream
// through a 2-stage cp.async pipeline of 64-candidate blocks (B operand,
// padded rows -> conflict-free ldmatrix), shared by the 4 warps.  Symmetric
// evaluation and split-K as in the SIMT kernels.  SHORTC has no role here:
// the MMA evaluates all dims of a block at once.
#include <cuda_fp16.h>

#include "gj_internal.cuh"

namespace gj {
namespace {

constexpr int kBN = 64;   // candidates per pipeline block

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];\n" : "=r"(r0), "=r"(r1) : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

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

// Survivor of the bound: FP64 decision and emission (both orders when
// symmetric).  Out of line: it runs for a tiny fraction of the pairs.
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

template <int KP, int MODE, bool SYM>
__global__ void __launch_bounds__(kTileQ) k_join_tc(JoinParams P, JoinArgs A) {
    constexpr int KS = KP / 16;        // MMA k-steps
    constexpr int RS = KP + 8;         // smem row stride in halves (16 B pad: conflict-free ldmatrix)
    constexpr int CH = KP / 8;         // 16-byte chunks per candidate row
    __shared__ __align__(16) __half Bs[2][kBN * RS];
    __shared__ uint32_t s_win[2];
    __shared__ unsigned long long s_red[kTileQ / 32];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gq = lane >> 2, tq = lane & 3;
    const CtaTile ct = cta_tile(P, A, kTileQ);
    if (ct.nq == 0) return;   // sub-block past the end of the tile's cell
    const int part = ct.part, split = ct.split;
    const uint32_t g = ct.g, q0 = ct.q0, nq = ct.nq;
    const int n_pad = P.n_pad;
    const double eps = P.eps;

    // A fragments (rows = this warp's queries); the augmented columns K-4..K-1
    // (lane tq = 2: r_hi, r_lo; tq = 3: 1, 1) turn every accumulator into
    // (T - ||q^ - c^||^2) / 2 (see tc_threshold_from)
    uint32_t af[2][KS][4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int row = 32 * warp + 16 * mt + gq + 8 * h;
            const bool valid = row < (int)nq;
            const uint32_t prow = q0 + (valid ? row : 0);
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                af[mt][ks][h] = *reinterpret_cast<const uint32_t*>(P.pts16 + g16(prow, 16 * ks + 2 * tq, KP));
                af[mt][ks][2 + h] = *reinterpret_cast<const uint32_t*>(P.pts16 + g16(prow, 16 * ks + 8 + 2 * tq, KP));
            }
            if (tq >= 2) {
                __half2 aug;
                if (tq == 2) {
                    __half rhi, rlo;
                    query_aug(P.thr16, P.norm16[prow], valid, rhi, rlo);
                    aug = __halves2half2(rhi, rlo);
                } else {
                    aug = __halves2half2(__float2half(1.f), __float2half(1.f));
                }
                af[mt][KS - 1][2 + h] = *reinterpret_cast<uint32_t*>(&aug);
            }
        }
    }

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

    const double u_lo = P.pts[(size_t)q0 * n_pad + P.u];
    const double u_hi = P.pts[(size_t)(q0 + nq - 1) * n_pad + P.u];
    const uint32_t nb0 = SYM ? P.nbr_self[g] : P.nbr_off[g], nb1 = P.nbr_off[g + 1];
    for (uint32_t b = nb0; b < nb1; ++b) {
        const uint32_t B = P.nbr[b];
        uint32_t r = P.cell_start[B], s = P.cell_start[B + 1];
        if (P.sortidu) {   // tile-level SORTIDU window (exact predicates on the fp64 u-coordinates)
            __syncthreads();
            if (tid < 2) {
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
        const bool diag = SYM && B == g;
        if (diag) r = max(r, q0 + 1);
        if (split > 1 && s > r) {
            const uint64_t len = s - r;
            s = r + (uint32_t)(len * (part + 1) / split);
            r = r + (uint32_t)(len * part / split);
        }
        if (s <= r) continue;
        const int nblk = (int)((s - r + kBN - 1) / kBN);

        auto load_block = [&](int buf, uint32_t start) {
            const int cnt = (int)min((uint32_t)kBN, s - start);
            for (int i = tid; i < kBN * CH; i += kTileQ) {
                const int row = i / CH, ch = i - row * CH;
                __half* dst = &Bs[buf][row * RS + ch * 8];
                if (row < cnt) {
                    cp_async16(dst, P.pts16 + g16(start + row, ch * 8, KP));
                } else {   // padding candidate: zeros, h_hi = -65504 -> every accumulator < 0
                    union { uint4 u; __half h[8]; } c;
                    c.u = make_uint4(0, 0, 0, 0);
                    if (ch == CH - 1) c.h[6] = __float2half(-65504.f);
                    *reinterpret_cast<uint4*>(dst) = c.u;
                }
            }
            cp_async_commit();
        };

        __syncthreads();   // previous window's last block fully consumed
        load_block(0, r);
        for (int kb = 0; kb < nblk; ++kb) {
            const uint32_t cbase = r + (uint32_t)kb * kBN;
            if (kb + 1 < nblk) {
                load_block((kb + 1) & 1, cbase + kBN);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncthreads();
            const int buf = kb & 1;
            if (32 * warp >= (int)nq) {   // warp has no queries in this tile (small cell)
                __syncthreads();
                continue;
            }
            float acc[2][8][4];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int nt = 0; nt < 8; ++nt)
#pragma unroll
                    for (int e = 0; e < 4; ++e) acc[mt][nt][e] = 0.f;
            const uint32_t bbase = smem_u32(&Bs[buf][0]);
#pragma unroll
            for (int nt = 0; nt < 8; ++nt) {
                uint32_t bf[KS][2];
                const uint32_t rowaddr = bbase + (uint32_t)((8 * nt + (lane & 7)) * RS) * 2u;
#pragma unroll
                for (int k2 = 0; k2 + 1 < KS; k2 += 2)
                    ldsm_x4(rowaddr + (uint32_t)(32 * (k2 / 2) + 8 * (lane >> 3)) * 2u, bf[k2][0], bf[k2][1],
                            bf[k2 + 1][0], bf[k2 + 1][1]);
                if (KS & 1)
                    ldsm_x2(rowaddr + (uint32_t)(16 * (KS - 1) + 8 * ((lane >> 3) & 1)) * 2u, bf[KS - 1][0],
                            bf[KS - 1][1]);
#pragma unroll
                for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                    for (int ks = 0; ks < KS; ++ks) mma16816(acc[mt][nt], af[mt][ks], bf[ks][0], bf[ks][1]);
            }
            // epilogue: acc = (T - ||q^ - c^||^2) / 2 + err; survivor iff acc > +0
            uint32_t all = 0xffffffffu;
#pragma unroll
            for (int nt = 0; nt < 8; ++nt)
#pragma unroll
                for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                    for (int e = 0; e < 4; ++e) all &= __float_as_uint(acc[mt][nt][e]);
            if (!(all >> 31)) {   // rare: decide the survivors in FP64
                unsigned long long mask = 0;
#pragma unroll
                for (int nt = 0; nt < 8; ++nt)
#pragma unroll
                    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            if (!(__float_as_uint(acc[mt][nt][e]) >> 31)) mask |= 1ull << (nt * 8 + mt * 4 + e);
                while (mask) {
                    const int bit = __ffsll((long long)mask) - 1;
                    mask &= mask - 1;
                    const int nt = bit >> 3, mt = (bit >> 2) & 1, e = bit & 3;
                    const uint32_t qpos = q0 + 32 * warp + 16 * mt + gq + 8 * (e >> 1);
                    const uint32_t cpos = cbase + 8 * nt + 2 * tq + (e & 1);
                    if (diag && cpos <= qpos) continue;
                    npairs += decide_and_emit<MODE, SYM>(P, A, qpos, cpos);
                }
            }
            __syncthreads();   // buffer kb&1 is refilled by the load issued in the next iteration
        }
    }
    if (MODE == kCount) {
        unsigned long long x = npairs;
#pragma unroll
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) s_red[warp] = x;
        __syncthreads();
        if (tid == 0) {
            unsigned long long t = 0;
            for (int w = 0; w < kTileQ / 32; ++w) t += s_red[w];
            if (t) atomicAdd((unsigned long long*)A.count, t);
            if (part == 0) atomicAdd((unsigned long long*)A.count + 1, (unsigned long long)nq);
        }
    }
}

template <int KP>
int launch_tc(const JoinParams& p, JoinMode mode, const JoinArgs& a, bool sym, cudaStream_t s) {
    if (a.n_tiles <= 0) return GJ_OK;
    dim3 grid(grid_ctas(a, (int)p.tile_q, kTileQ));
    if (mode == kEmit) {
        if (sym) k_join_tc<KP, kEmit, true><<<grid, kTileQ, 0, s>>>(p, a);
        else k_join_tc<KP, kEmit, false><<<grid, kTileQ, 0, s>>>(p, a);
    } else {
        if (sym) k_join_tc<KP, kCount, true><<<grid, kTileQ, 0, s>>>(p, a);
        else k_join_tc<KP, kCount, false><<<grid, kTileQ, 0, s>>>(p, a);
    }
    count_launch();
    GJ_CUDA(cudaGetLastError());
    return GJ_OK;
}

}  // namespace

int launch_join_tc(const Index* ix, JoinMode mode, const JoinArgs& a, cudaStream_t s) {
    const JoinParams p = join_params(ix);
    const bool sym = ix->opt.symmetric != 0;
    switch (ix->k16) {
        case 16: return launch_tc<16>(p, mode, a, sym, s);
        case 32: return launch_tc<32>(p, mode, a, sym, s);
        case 48: return launch_tc<48>(p, mode, a, sym, s);
        case 64: return launch_tc<64>(p, mode, a, sym, s);
        case 80: return launch_tc<80>(p, mode, a, sym, s);
        case 96: return launch_tc<96>(p, mode, a, sym, s);
        case 112: return launch_tc<112>(p, mode, a, sym, s);
        default: return launch_tc<128>(p, mode, a, sym, s);
    }
}

}  // namespace gj
