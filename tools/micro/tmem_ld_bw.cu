// Microbenchmark: tcgen05.ld (TMEM -> registers) throughput per SM on B200.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_ld_bw tmem_ld_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int NX>   // x32 loads in flight per wait
__global__ void k_tmem(int reps, unsigned* out, long long* cycles) {
    __shared__ uint32_t base;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t t = base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(((warp >> 2) * 128) & 511);
    unsigned acc = threadIdx.x * 7u + 1u;
    long long c0 = clock64();
    for (int r = 0; r < reps; ++r) {
        uint32_t v[NX][32];
#pragma unroll
        for (int x = 0; x < NX; ++x) {
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
                "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
                : "=r"(v[x][0]), "=r"(v[x][1]), "=r"(v[x][2]), "=r"(v[x][3]), "=r"(v[x][4]), "=r"(v[x][5]),
                  "=r"(v[x][6]), "=r"(v[x][7]), "=r"(v[x][8]), "=r"(v[x][9]), "=r"(v[x][10]), "=r"(v[x][11]),
                  "=r"(v[x][12]), "=r"(v[x][13]), "=r"(v[x][14]), "=r"(v[x][15]), "=r"(v[x][16]), "=r"(v[x][17]),
                  "=r"(v[x][18]), "=r"(v[x][19]), "=r"(v[x][20]), "=r"(v[x][21]), "=r"(v[x][22]), "=r"(v[x][23]),
                  "=r"(v[x][24]), "=r"(v[x][25]), "=r"(v[x][26]), "=r"(v[x][27]), "=r"(v[x][28]), "=r"(v[x][29]),
                  "=r"(v[x][30]), "=r"(v[x][31])
                : "r"(t + (uint32_t)((32 * x) & 127)));
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
        for (int x = 0; x < NX; ++x)
#pragma unroll
            for (int y = 0; y < 32; ++y) acc &= v[x][y];
        acc ^= (unsigned)r;
    }
    long long c1 = clock64();
    if (acc == 0x12345678u) out[threadIdx.x] = acc;
    if (threadIdx.x == 0) cycles[blockIdx.x] = c1 - c0;
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(base));
}

template <int NX>
void run(int warps) {
    unsigned* out; long long* cyc;
    cudaMalloc(&out, 4096); cudaMalloc(&cyc, 148 * 8);
    const int reps = 20000;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k_tmem<NX><<<148, 32 * warps>>>(100, out, cyc);
    cudaEventRecord(e0);
    k_tmem<NX><<<148, 32 * warps>>>(reps, out, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    double bytes_sm = (double)reps * warps * NX * 32 * 32 * 4;
    printf("warps=%2d x32-loads/wait=%d : %.1f B/cycle/SM (clock64), %.2f TB/s chip, err=%s\n", warps, NX,
           bytes_sm / c, bytes_sm * 148 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    cudaFree(out); cudaFree(cyc);
}

int main() {
    for (int w : {4, 8, 12, 16, 24, 32}) { run<2>(w); run<4>(w); }
    return 0;
}
