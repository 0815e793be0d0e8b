// conv.cu -- fused tensor-and-accumulate for an encrypted convolution layer.
//
// For every output cell (f, i, j) of a valid, strided, multi-channel convolution the
// layer needs the degree-2 raw product
//     raw = sum_{c,p,q} x[c][i*s+p][j*s+q] (x) w[f][c][p][q]
// (reference conv2d_enc, layers.py:92-127: one mul_ct_ct_raw + raw_add per tap).
// The tensor is pointwise in (row, position), so each (row r, position x) is an
// independent small convolution.  A CTA owns one row and XC consecutive positions:
//   * the weights of FG filters (all taps, both components) for those positions are
//     staged once in shared memory and reused by every output cell;
//   * SW warps-worth of workers stride over the output cells; each thread keeps FG
//     filters' three 128-bit accumulators in registers, so every input tap is loaded
//     once per cell and reused across the FG filters;
//   * products are summed lazily in 128 bits (Karatsuba: a0b0, a1b1,
//     (a0+a1)(b0+b1)) and reduced once per cell with Montgomery REDC, giving the
//     reference's canonical Montgomery residues exactly.
#include "common.cuh"

namespace {
constexpr int XC = 32;  // positions per CTA (one warp-width)
constexpr int SW = 8;   // workers per position  -> 256 threads
constexpr int FG = 5;   // filters per CTA group
}  // namespace

template <bool FLUSH>
__global__ void __launch_bounds__(XC *SW, 2) k_conv_tensor(Ctx K, heb_ct A, heb_ct B, heb_ct D, int C, int m, int n,
                                                            int F, int P, int Q, int s, int om, int on, int logn,
                                                            int flush) {
    extern __shared__ u64 wsm[];  // [tap][fl][comp][XC]
    const int xl = threadIdx.x % XC, w = threadIdx.x / XC;
    const int x = blockIdx.x * XC + xl;
    const int r = blockIdx.y;
    const int f0 = blockIdx.z * FG;
    const int nf = min(FG, F - f0);
    const int taps = C * P * Q;
    const PrimeInfo Pr = K.pi[r];
    const u64 p = Pr.p;
    const int64_t roff = ((int64_t)r << logn) + x;

    // stage weights of filters f0 .. f0+nf-1 for positions [x0, x0+XC)
    for (int e = w; e < taps * nf; e += SW) {
        const int tap = e / nf, fl = e % nf;
        const int64_t widx = (int64_t)(f0 + fl) * taps + tap;
        const u64 *src = B.data + widx * B.ct_stride + roff;
        u64 *dst = wsm + ((size_t)(tap * FG + fl) * 2) * XC + xl;
        if (Pr.use_fp) {  // FP64 rows: stage the weights as doubles
            dst[0] = (u64)__double_as_longlong(ntt::u2d(src[0]));
            dst[XC] = (u64)__double_as_longlong(ntt::u2d(src[B.comp_stride]));
        } else {
            dst[0] = src[0];
            dst[XC] = src[B.comp_stride];
        }
    }
    __syncthreads();

    const int cells = om * on;
    if (Pr.use_fp) {
        // Rows with p < 2^42: every product reduced exactly on the FP64 pipe (6 ops),
        // sums exact below 2^47; one R^-1 product per output restores the Montgomery
        // factor of the reference's mont_mul accumulation.
        const double pd = Pr.pd, pinvd = Pr.pinvd, rinv = (double)Pr.rinv;
        const double *wd = reinterpret_cast<const double *>(wsm);
        for (int cell = w; cell < cells; cell += SW) {
            const int i = cell / on, j = cell % on;
            double s0[FG], s1[FG], s2[FG];
#pragma unroll
            for (int fl = 0; fl < FG; ++fl) s0[fl] = s1[fl] = s2[fl] = 0.0;
            for (int c = 0; c < C; ++c) {
                for (int pp = 0; pp < P; ++pp) {
                    const int64_t rowcell = (int64_t)c * m * n + (int64_t)(i * s + pp) * n + j * s;
                    for (int qq = 0; qq < Q; ++qq) {
                        const int tap = (c * P + pp) * Q + qq;
                        const u64 *ap = A.data + (rowcell + qq) * A.ct_stride + roff;
                        const double a0 = ntt::u2d(__ldg(ap)), a1 = ntt::u2d(__ldg(ap + A.comp_stride));
                        const double sa = a0 + a1;
                        const double *wt = wd + (size_t)(tap * FG) * 2 * XC + xl;
#pragma unroll
                        for (int fl = 0; fl < FG; ++fl) {
                            if (fl < nf) {
                                const double b0 = wt[(2 * fl) * XC], b1 = wt[(2 * fl + 1) * XC];
                                s0[fl] += ntt::fmul(a0, b0, pd, pinvd);
                                s2[fl] += ntt::fmul(a1, b1, pd, pinvd);
                                s1[fl] += ntt::fmul(sa, b0 + b1, pd, pinvd);
                            }
                        }
                    }
                }
            }
#pragma unroll
            for (int fl = 0; fl < FG; ++fl) {
                if (fl < nf) {
                    const double e0 = ntt::fmul(s0[fl], rinv, pd, pinvd);
                    const double e2 = ntt::fmul(s2[fl], rinv, pd, pinvd);
                    const double e1 = ntt::fmul(s1[fl], rinv, pd, pinvd) - e0 - e2;
                    u64 *dp = D.data + ((int64_t)(f0 + fl) * cells + cell) * D.ct_stride + roff;
                    dp[0] = ntt::fcanon(e0, pd, pinvd);
                    dp[D.comp_stride] = ntt::fcanon(e1, pd, pinvd);
                    dp[2 * D.comp_stride] = ntt::fcanon(e2, pd, pinvd);
                }
            }
        }
        return;
    }
    for (int cell = w; cell < cells; cell += SW) {
        const int i = cell / on, j = cell % on;
        acc4 s0[FG], s1[FG], s2[FG];
        u64 t0[FG], t1[FG], t2[FG];
#pragma unroll
        for (int fl = 0; fl < FG; ++fl) {
            s0[fl] = s1[fl] = s2[fl] = acc4{0, 0, 0, 0};
            t0[fl] = t1[fl] = t2[fl] = 0;
        }
        int since = 0;
        for (int c = 0; c < C; ++c) {
            for (int pp = 0; pp < P; ++pp) {
                const int64_t rowcell = (int64_t)c * m * n + (int64_t)(i * s + pp) * n + j * s;
                for (int qq = 0; qq < Q; ++qq) {
                    const int tap = (c * P + pp) * Q + qq;
                    const u64 *ap = A.data + (rowcell + qq) * A.ct_stride + roff;
                    const u64 a0 = __ldg(ap), a1 = __ldg(ap + A.comp_stride);
                    const u64 sa = add_mod(a0, a1, p);
                    const u64 *wt = wsm + (size_t)(tap * FG) * 2 * XC + xl;
#pragma unroll
                    for (int fl = 0; fl < FG; ++fl) {
                        if (fl < nf) {
                            const u64 b0 = wt[(2 * fl) * XC], b1 = wt[(2 * fl + 1) * XC];
                            mac4(s0[fl], a0, b0);
                            mac4(s2[fl], a1, b1);
                            mac4(s1[fl], sa, add_mod(b0, b1, p));
                        }
                    }
                    if (FLUSH && ++since == flush) {
#pragma unroll
                        for (int fl = 0; fl < FG; ++fl) {
                            t0[fl] = add_mod(t0[fl], redc128(to128(s0[fl]), p, Pr.pinv, Pr.r1s), p);
                            t1[fl] = add_mod(t1[fl], redc128(to128(s1[fl]), p, Pr.pinv, Pr.r1s), p);
                            t2[fl] = add_mod(t2[fl], redc128(to128(s2[fl]), p, Pr.pinv, Pr.r1s), p);
                            s0[fl] = s1[fl] = s2[fl] = acc4{0, 0, 0, 0};
                        }
                        since = 0;
                    }
                }
            }
        }
#pragma unroll
        for (int fl = 0; fl < FG; ++fl) {
            if (fl < nf) {
                const u64 d0 = add_mod(t0[fl], redc128(to128(s0[fl]), p, Pr.pinv, Pr.r1s), p);
                const u64 d2 = add_mod(t2[fl], redc128(to128(s2[fl]), p, Pr.pinv, Pr.r1s), p);
                const u64 e1 = add_mod(t1[fl], redc128(to128(s1[fl]), p, Pr.pinv, Pr.r1s), p);
                u64 *dp = D.data + ((int64_t)(f0 + fl) * cells + cell) * D.ct_stride + roff;
                dp[0] = d0;
                dp[D.comp_stride] = sub_mod(sub_mod(e1, d0, p), d2, p);
                dp[2 * D.comp_stride] = d2;
            }
        }
    }
}

extern "C" int heb_conv_tensor(heb_ctx *c, heb_ct a, heb_ct b, heb_ct d, int channels, int m, int n, int filters,
                               int kp, int kq, int stride, int k, void *stream) {
    if (!c || channels < 1 || filters < 1 || kp < 1 || kq < 1 || stride < 1 || kp > m || kq > n || k < 1 ||
        k > c->num_rows || c->n % XC)
        return fail(HEB_EINVAL, "heb_conv_tensor: bad args");
    const int om = (m - kp) / stride + 1, on = (n - kq) / stride + 1;
    const int taps = channels * kp * kq;
    const size_t sm = sizeof(u64) * (size_t)taps * FG * 2 * XC;
    if (sm > 220 * 1024) return fail(HEB_EUNSUP, "heb_conv_tensor: %d taps exceed the shared-memory stage", taps);
    cudaStream_t st = (cudaStream_t)stream;
    const bool need_flush = taps > c->flush;
    CUDA_TRY(prep_kernel(k_conv_tensor<true>, sm));
    CUDA_TRY(prep_kernel(k_conv_tensor<false>, sm));
    dim3 grid(c->n / XC, k, (filters + FG - 1) / FG);
    const double nout = (double)filters * om * on;
    {
        PROF("k_conv_tensor", st,
             8.0 * c->n * k * (2.0 * channels * m * n + 2.0 * filters * taps + 3.0 * nout));
        if (need_flush)
            k_conv_tensor<true><<<grid, XC * SW, sm, st>>>(kctx(c), a, b, d, channels, m, n, filters, kp, kq, stride,
                                                           om, on, c->log_n, c->flush);
        else
            k_conv_tensor<false><<<grid, XC * SW, sm, st>>>(kctx(c), a, b, d, channels, m, n, filters, kp, kq, stride,
                                                            om, on, c->log_n, c->flush);
    }
    LAUNCH_CHECK();
    return HEB_OK;
}
