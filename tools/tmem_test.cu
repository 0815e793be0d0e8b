// TMEM as per-thread accumulator storage: 2 CTAs/SM x 512 threads, 256 columns each.
// Every thread stores 64 words, reads them back, adds, stores, reads again.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void tst16(uint32_t addr, const uint32_t (&v)[16]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 :: "r"(addr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                    "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
}
__device__ __forceinline__ void tld16(uint32_t addr, uint32_t (&v)[16]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(addr));
}

__global__ void __launch_bounds__(512, 2) k(int *bad, int reps) {
    __shared__ uint32_t taddr_s;
    const int warp = threadIdx.x / 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" :: "r"((uint32_t)__cvta_generic_to_shared(&taddr_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = taddr_s + ((uint32_t)(32 * (warp % 4)) << 16) + (uint32_t)((warp / 4) * 64);
    int errs = 0;
    for (int r = 0; r < reps; ++r) {
        for (int c = 0; c < 4; ++c) {
            uint32_t v[16];
            for (int i = 0; i < 16; ++i) v[i] = (blockIdx.x * 512 + threadIdx.x) * 1000u + c * 16 + i + r;
            tst16(base + c * 16, v);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;");
        for (int c = 0; c < 4; ++c) {
            uint32_t v[16];
            tld16(base + c * 16, v);
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            for (int i = 0; i < 16; ++i) errs += v[i] != (blockIdx.x * 512 + threadIdx.x) * 1000u + c * 16 + i + r;
        }
    }
    if (errs) atomicAdd(bad, errs);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" :: "r"(taddr_s));
}

int main() {
    int *bad;
    cudaMalloc(&bad, 4);
    cudaMemset(bad, 0, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<<<2960, 512>>>(bad, 1);
    cudaEventRecord(a);
    k<<<2960, 512>>>(bad, 64);
    cudaEventRecord(b);
    cudaError_t e = cudaDeviceSynchronize();
    int h = -1;
    cudaMemcpy(&h, bad, 4, cudaMemcpyDeviceToHost);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    // bytes: 2960 CTAs * 512 thr * 64 reps * (256 B st + 256 B ld)
    double bytes = 2960.0 * 512 * 64 * 512;
    printf("err=%s mismatches=%d  %.3f ms  %.1f TB/s (ld+st)\n", cudaGetErrorString(e), h, ms, bytes / ms / 1e9);
    return 0;
}
