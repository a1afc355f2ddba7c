// Round 2 experiment (rejected, not built): warp-per-32-query-tile variant of
// the certified FP32 filter for small cells (gj_join32.cu).  Parity-green,
// but 35-44 ms vs 12-17 ms for the 128-query CTA kernel on songs90 k = 4..8:
// each warp streams candidate rows straight from global memory one at a time
// (the SHORTC break keeps the compiler from issuing the next rows' loads
// early) at 12 resident warps per SM (168 registers), so it is latency-bound;
// the CTA kernel's shared-memory staging of candidate pairs wins even with
// three of its four warps idle.
// ---------------------------------------------------------------------------
// Warp-per-tile variant for indexes whose cells are small (tiles of 32
// queries, gj_index.cu: mean cell size < 64, e.g. the Songs-shaped data at
// k >= 6 where cells average ~30 points, so a 128-query CTA ran 3/4 idle).
// A CTA holds four independent warps; warp w takes unit 4 blockIdx + w of the
// launch (a (tile, part) of the work-balanced plan, 32 queries of one cell).
// Each lane keeps its query as float2 pairs of consecutive dims; a candidate
// row is read straight from global memory (every lane reads the same row:
// one broadcast transaction per float4) and tested with packed f32x2 ops on
// two dims at a time -- two partial FMA chains (even / odd dims) whose sum is
// the running sum (tests/test_fp32_bound_cpu.py emulates this order).  Same
// certified thresholds, FP64 decisions and emission as k_join32.
constexpr int kWarpQ = 32;
constexpr int kWWin = 128;   // adjacent cells whose windows one warp holds per round

__device__ __forceinline__ CtaTile warp_unit(const JoinParams& P, const JoinArgs& A, uint32_t u) {
    CtaTile t;
    uint32_t m;
    if (A.part_off) {   // unit u -> (tile m, part): last m with part_off[m] <= u
        uint32_t lo = 0, hi = (uint32_t)A.n_tiles;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (A.part_off[mid] <= u) lo = mid; else hi = mid;
        }
        m = lo;
        t.part = (int)(u - A.part_off[m]);
        t.split = (int)(A.part_off[m + 1] - A.part_off[m]);
    } else {
        const uint32_t split = A.split > 1 ? (uint32_t)A.split : 1u;
        t.part = (int)(u % split);
        t.split = (int)split;
        m = u / split;
    }
    t.nq = 0;
    if ((int64_t)m >= A.n_tiles) return t;
    const int64_t j = A.first + A.step * (int64_t)m;
    const uint32_t tile = P.tile_order[j];
    t.g = P.tile_cell[tile];
    t.q0 = P.tile_q0[tile];
    const uint32_t end = P.cell_start[t.g + 1];
    t.nq = t.q0 < end ? min((uint32_t)kWarpQ, end - t.q0) : 0u;
    return t;
}

template <int NPR, int MODE, bool SYM>
__global__ void __launch_bounds__(128) k_join32w(JoinParams P, JoinArgs A) {
    __shared__ uint32_t s_wr[4][kWWin], s_ws[4][kWWin];
    __shared__ unsigned char s_dg[4][kWWin];
    __shared__ unsigned long long s_red[4];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const CtaTile ct = warp_unit(P, A, blockIdx.x * 4u + (uint32_t)w);
    unsigned long long npairs = 0;
    if (ct.nq > 0) {
        const int part = ct.part, split = ct.split;
        const uint32_t g = ct.g, q0 = ct.q0, nq = ct.nq;
        const bool active = lane < (int)nq;
        const uint32_t qpos = q0 + (active ? lane : 0);
        const int n_pad = P.n_pad;
        // -q as float2 pairs of consecutive dims (t = c - q, squared)
        float2 nqv[NPR / 2];
#pragma unroll
        for (int d = 0; d < NPR; d += 4) {
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (d < n_pad) v = *reinterpret_cast<const float4*>(P.pts32 + (size_t)qpos * n_pad + d);
            nqv[d / 2] = make_float2(-v.x, -v.y);
            nqv[d / 2 + 1] = make_float2(-v.z, -v.w);
        }
        const double eps = P.eps, eps2 = P.eps2;
        const float thr = P.thr32, thr_in = P.thr32_in;
        const uint32_t qid = P.orig[qpos];
        const double u_lo = P.pts[(size_t)q0 * n_pad + P.u];
        const double u_hi = P.pts[(size_t)(q0 + nq - 1) * n_pad + P.u];
        const double* __restrict__ qrow64 = P.pts + (size_t)qpos * n_pad;
        constexpr unsigned long long kMul = SYM ? 2ull : 1ull;
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
        for (uint32_t w0 = nb0; w0 < nb1; w0 += kWWin) {
            const uint32_t nwin = min((uint32_t)kWWin, nb1 - w0);
            __syncwarp();
            for (uint32_t i = lane; i < nwin; i += 32) {   // tile-level SORTIDU windows, lane per adjacent cell
                const uint32_t B = P.nbr[w0 + i];
                uint32_t r = P.cell_start[B], s = P.cell_start[B + 1];
                if (P.sortidu) {
                    uint32_t lo = r, hi = s;
                    while (lo < hi) {   // first r with u_lo - r(u) <= eps
                        const uint32_t mid = (lo + hi) >> 1;
                        if (u_lo - P.pts[(size_t)mid * n_pad + P.u] <= eps) hi = mid; else lo = mid + 1;
                    }
                    const uint32_t rr = lo;
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
                s_wr[w][i] = r;
                s_ws[w][i] = max(s, r);
                s_dg[w][i] = diag ? 1 : 0;
            }
            __syncwarp();
            for (uint32_t wi = 0; wi < nwin; ++wi) {
                const uint32_t r = s_wr[w][wi], s = s_ws[w][wi];
                const bool diag = s_dg[w][wi] != 0;
                for (uint32_t p = r; p < s; ++p) {
                    const bool ok = active && (!diag || p > qpos);
                    float2 a = make_float2(0.f, ok ? 0.f : INFINITY);
                    if (ok) {
                        const float* cp = P.pts32 + (size_t)p * n_pad;
#pragma unroll
                        for (int d = 0; d < NPR; d += 8) {
                            if (d >= n_pad) break;
                            const float4 x = __ldg(reinterpret_cast<const float4*>(cp + d));
                            float2 t;
                            t = __fadd2_rn(make_float2(x.x, x.y), nqv[d / 2]);     a = __ffma2_rn(t, t, a);
                            t = __fadd2_rn(make_float2(x.z, x.w), nqv[d / 2 + 1]); a = __ffma2_rn(t, t, a);
                            if (d + 4 < n_pad) {
                                const float4 y = __ldg(reinterpret_cast<const float4*>(cp + d + 4));
                                t = __fadd2_rn(make_float2(y.x, y.y), nqv[d / 2 + 2]); a = __ffma2_rn(t, t, a);
                                t = __fadd2_rn(make_float2(y.z, y.w), nqv[d / 2 + 3]); a = __ffma2_rn(t, t, a);
                            }
                            if (P.shortc && a.x + a.y > thr) break;   // SHORTC, every 8 dims
                        }
                    }
                    const float sum = a.x + a.y;
                    // survivors of the prefilter: decided in FP64 unless the bound
                    // also proves them inside (sum <= thr_in)
                    bool hit = ok && sum <= thr;
                    if (hit && !(sum <= thr_in)) hit = dist2_fp64(qrow64, P.pts + (size_t)p * n_pad, n_pad) <= eps2;
                    if (MODE == kEmit) {
                        const unsigned m = __ballot_sync(0xffffffffu, hit);
                        if (m) {
                            const int leader = __ffs(m) - 1;
                            unsigned long long base = 0;
                            if (lane == leader) base = atomicAdd((unsigned long long*)A.count, kMul * __popc(m));
                            base = __shfl_sync(0xffffffffu, base, leader);
                            if (hit) {
                                const unsigned long long at = base + kMul * __popc(m & lt);
                                const uint32_t id = P.orig[p];
                                if (at + kMul <= A.cap) {
                                    uint2* out = reinterpret_cast<uint2*>(A.out);
                                    out[at] = make_uint2(qid, id);
                                    if (SYM) out[at + 1] = make_uint2(id, qid);
                                }
                            }
                        }
                    } else {
                        npairs += kMul * (unsigned long long)hit;
                    }
                }
            }
        }
    }
    if (MODE == kCount) {
        unsigned long long x = npairs;
#pragma unroll
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) s_red[w] = x;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long t = 0, q = 0;
            for (int i = 0; i < 4; ++i) t += s_red[i];
            if (t) atomicAdd((unsigned long long*)A.count, t);
            for (int i = 0; i < 4; ++i) {
                const CtaTile c = warp_unit(P, A, blockIdx.x * 4u + (uint32_t)i);
                if (c.nq > 0 && c.part == 0) q += c.nq;
            }
            if (q) atomicAdd((unsigned long long*)A.count + 1, q);
        }
    }
}

template <int NPR>
int launch32w(const JoinParams& p, JoinMode mode, const JoinArgs& a, bool sym, cudaStream_t s) {
    if (a.n_tiles <= 0) return GJ_OK;
    const int64_t units = a.part_off ? a.total_parts : a.n_tiles * (a.split > 1 ? a.split : 1);
    dim3 grid((unsigned)((units + 3) / 4));
    if (mode == kEmit) {
        if (sym) k_join32w<NPR, kEmit, true><<<grid, 128, 0, s>>>(p, a);
        else k_join32w<NPR, kEmit, false><<<grid, 128, 0, s>>>(p, a);
    } else {
        if (sym) k_join32w<NPR, kCount, true><<<grid, 128, 0, s>>>(p, a);
        else k_join32w<NPR, kCount, false><<<grid, 128, 0, s>>>(p, a);
    }
    count_launch();
    GJ_CUDA(cudaGetLastError());
    return GJ_OK;
}

