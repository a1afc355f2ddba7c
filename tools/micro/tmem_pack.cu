// What does tcgen05.ld ... .pack::16b return for 32-bit TMEM data?  Writes known
// fp32 values with tcgen05.st, reads them back with and without .pack::16b.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "gj_umma.cuh"
using namespace gj;

__global__ void k(uint32_t* out) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) umma::tmem_alloc(&tbase, 32);
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t t = tbase;
    if (warp == 0) {
        uint32_t v[16];
        for (int j = 0; j < 16; ++j) {   // column j, lane i: float (j + 1) * (lane even ? -1 : 1) + tag
            float f = (float)(j + 1) * ((lane & 1) ? 1.f : -1.f) + 0.001f * lane;
            v[j] = __float_as_uint(f);
        }
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
                     :: "r"(t), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        uint32_t r[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(t));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        for (int j = 0; j < 8; ++j) out[lane * 32 + j] = r[j];
        for (int j = 0; j < 16; ++j) out[lane * 32 + 16 + j] = v[j];
    }
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc(t, 32);
}

int main() {
    uint32_t* d; cudaMalloc(&d, 32 * 32 * 4);
    k<<<1, 128>>>(d);
    uint32_t h[32 * 32];
    cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%s\n", cudaGetErrorString(e));
    for (int lane = 0; lane < 2; ++lane) {
        printf("lane %d stored:", lane);
        for (int j = 0; j < 16; ++j) printf(" %08x", h[lane * 32 + 16 + j]);
        printf("\nlane %d packed:", lane);
        for (int j = 0; j < 8; ++j) printf(" %08x", h[lane * 32 + j]);
        printf("\n");
    }
    return 0;
}
