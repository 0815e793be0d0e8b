// pipes_bench.cu -- measured throughput of the integer/FP64 primitives the
// CKKS kernels are built from (IMAD.WIDE, IMAD, IMAD.HI, DFMA, Shoup, 128-bit MAC).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipes_bench tools/pipes_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

typedef uint64_t u64;
typedef uint32_t u32;

#define ITERS 2048
#define CH 8

__global__ void k_wide(u64 *sink, u32 m) {
    u64 x[CH];
    for (int i = 0; i < CH; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            u64 r;
            asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"((u32)x[i]), "r"(m), "l"(x[i]));
            x[i] = r;
        }
    u64 s = 0;
    for (int i = 0; i < CH; ++i) s ^= x[i];
    if (s == 42) sink[0] = s;
}

__global__ void k_lo(u64 *sink, u32 m) {
    u32 x[CH];
    for (int i = 0; i < CH; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(x[i]) : "r"(m));
    u32 s = 0;
    for (int i = 0; i < CH; ++i) s ^= x[i];
    if (s == 42) sink[0] = s;
}

__global__ void k_hi(u64 *sink, u32 m) {
    u32 x[CH];
    for (int i = 0; i < CH; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) asm volatile("mad.hi.u32 %0, %0, %1, %0;" : "+r"(x[i]) : "r"(m));
    u32 s = 0;
    for (int i = 0; i < CH; ++i) s ^= x[i];
    if (s == 42) sink[0] = s;
}

__global__ void k_dfma(u64 *sink, double m) {
    double x[CH];
    for (int i = 0; i < CH; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) x[i] = fma(x[i], m, 0.5);
    double s = 0;
    for (int i = 0; i < CH; ++i) s += x[i];
    if (s == 42) sink[0] = (u64)s;
}

__global__ void k_mul64hi(u64 *sink, u64 m) {
    u64 x[CH];
    for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 77 + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) x[i] = __umul64hi(x[i], m) + x[i];
    u64 s = 0;
    for (int i = 0; i < CH; ++i) s ^= x[i];
    if (s == 42) sink[0] = s;
}

__device__ __forceinline__ u64 shoup_lazy(u64 x, u64 w, u64 ws, u64 p) {
    u64 q = __umul64hi(x, ws);
    return x * w - q * p;
}
__global__ void k_shoup(u64 *sink, u64 p, u64 w, u64 ws) {
    u64 x[CH];
    for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 77 + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) x[i] = shoup_lazy(x[i], w, ws, p);
    u64 s = 0;
    for (int i = 0; i < CH; ++i) s ^= x[i];
    if (s == 42) sink[0] = s;
}

// 128-bit MAC: lo/umulhi form
__global__ void k_mac_c(u64 *sink, u64 b) {
    u64 lo[4] = {0, 0, 0, 0}, hi[4] = {0, 0, 0, 0};
    u64 a = threadIdx.x * 0x9e3779b97f4a7c15ull;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            u64 x = a + it * 4 + i;
            u64 l = x * b, h = __umul64hi(x, b);
            u64 s = lo[i] + l;
            hi[i] += h + (s < l);
            lo[i] = s;
        }
    u64 s = 0;
    for (int i = 0; i < 4; ++i) s ^= lo[i] ^ hi[i];
    if (s == 42) sink[0] = s;
}

// 128-bit MAC: 32-bit limb multiply-add chains (4 x mad.wide equivalents)
__global__ void k_mac_ptx(u64 *sink, u64 b) {
    u32 acc[4][4] = {};
    u64 a = threadIdx.x * 0x9e3779b97f4a7c15ull;
    const u32 b0 = (u32)b, b1 = (u32)(b >> 32);
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            u64 x = a + it * 4 + i;
            u32 a0 = (u32)x, a1 = (u32)(x >> 32);
            asm volatile(
                "mad.lo.cc.u32  %0, %4, %6, %0;\n\t"
                "madc.hi.cc.u32 %1, %4, %6, %1;\n\t"
                "madc.lo.cc.u32 %2, %5, %7, %2;\n\t"
                "madc.hi.u32    %3, %5, %7, %3;\n\t"
                "mad.lo.cc.u32  %1, %4, %7, %1;\n\t"
                "madc.hi.cc.u32 %2, %4, %7, %2;\n\t"
                "addc.u32       %3, %3, 0;\n\t"
                "mad.lo.cc.u32  %1, %5, %6, %1;\n\t"
                "madc.hi.cc.u32 %2, %5, %6, %2;\n\t"
                "addc.u32       %3, %3, 0;\n\t"
                : "+r"(acc[i][0]), "+r"(acc[i][1]), "+r"(acc[i][2]), "+r"(acc[i][3])
                : "r"(a0), "r"(a1), "r"(b0), "r"(b1));
        }
    u32 s = 0;
    for (int i = 0; i < 4; ++i) s ^= acc[i][0] ^ acc[i][1] ^ acc[i][2] ^ acc[i][3];
    if (s == 42) sink[0] = s;
}

// FP64 modmul for p < 2^50: r = a*w mod p via h = a*w, l = fma(a,w,-h), q = floor(h*pinv)
__global__ void k_fpmod(u64 *sink, double p, double pinv, double w) {
    double x[CH];
    for (int i = 0; i < CH; ++i) x[i] = (double)(threadIdx.x * 977 + i);
    const double magic = 6755399441055744.0;  // 1.5 * 2^52
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            double h = x[i] * w;
            double l = fma(x[i], w, -h);
            double q = __dadd_rd(h * pinv, magic) - magic;
            double r = fma(-q, p, h) + l;
            r = r < 0 ? r + p : r;
            x[i] = r >= p ? r - p : r;
        }
    double s = 0;
    for (int i = 0; i < CH; ++i) s += x[i];
    if (s == 42) sink[0] = (u64)s;
}

template <class F>
static void timeit(const char *name, F launch, double ops_per_thread) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int blocks = 148 * 8, threads = 256;
    launch(blocks, threads);
    cudaEventRecord(a);
    launch(blocks, threads);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double total = (double)blocks * threads * ops_per_thread;
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double per_sm_clk = total / (ms * 1e-3) / (148.0 * clk * 1e3);
    printf("%-12s %8.3f ms  %10.2f Gop/s  %6.2f op/clk/SM  (%.2f warp-cycles/op/SMSP)\n", name, ms,
           total / (ms * 1e-3) / 1e9, per_sm_clk, 32.0 * 4 / per_sm_clk / 4);
}

int main() {
    u64 *sink;
    cudaMalloc(&sink, 8);
    const u64 p = 1099511480321ull, w = 123456789012ull;
    const u64 ws = (u64)(((unsigned __int128)w << 64) / p);
    timeit("imad.wide", [&](int b, int t) { k_wide<<<b, t>>>(sink, 12345); }, ITERS * CH);
    timeit("imad.lo32", [&](int b, int t) { k_lo<<<b, t>>>(sink, 12345); }, ITERS * CH);
    timeit("imad.hi32", [&](int b, int t) { k_hi<<<b, t>>>(sink, 12345); }, ITERS * CH);
    timeit("dfma", [&](int b, int t) { k_dfma<<<b, t>>>(sink, 1.0000001); }, ITERS * CH);
    timeit("umul64hi", [&](int b, int t) { k_mul64hi<<<b, t>>>(sink, 0x123456789abcdefull); }, ITERS * CH);
    timeit("shoup", [&](int b, int t) { k_shoup<<<b, t>>>(sink, p, w, ws); }, ITERS * CH);
    timeit("mac128_c", [&](int b, int t) { k_mac_c<<<b, t>>>(sink, 0x0fedcba987654321ull); }, ITERS * 4);
    timeit("mac128_ptx", [&](int b, int t) { k_mac_ptx<<<b, t>>>(sink, 0x0fedcba987654321ull); }, ITERS * 4);
    timeit("fp64_modmul", [&](int b, int t) { k_fpmod<<<b, t>>>(sink, (double)p, 1.0 / (double)p, (double)w); },
           ITERS * CH);
    cudaError_t e = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
