// pointwise.cu -- HBM-bound pointwise kernels and the batched layer evaluator.
#include "common.cuh"

__global__ void k_add(Ctx K, heb_ct a, heb_ct b, heb_ct o, int64_t lines, int comps, int k, int logn) {
    const int n = 1 << logn;
    for (int64_t line = blockIdx.y; line < lines; line += gridDim.y) {
        LineIdx L = line_of(line, comps, k);
        const u64 p = K.pi[L.r].p;
        const u64 *x = at(a, L.b, L.c, L.r, logn), *y = at(b, L.b, L.c, L.r, logn);
        u64 *z = at(o, L.b, L.c, L.r, logn);
        const ulonglong2 *x2 = reinterpret_cast<const ulonglong2 *>(x), *y2 = reinterpret_cast<const ulonglong2 *>(y);
        ulonglong2 *z2 = reinterpret_cast<ulonglong2 *>(z);
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n / 2; i += gridDim.x * blockDim.x) {
            const ulonglong2 u = x2[i], v = y2[i];
            z2[i] = make_ulonglong2(add_mod(u.x, v.x, p), add_mod(u.y, v.y, p));
        }
    }
}

__global__ void k_add_plain(Ctx K, heb_ct a, const u64 *pt, int64_t pstride, heb_ct o, int64_t lines, int k,
                            int logn, int copy_c1) {
    const int n = 1 << logn;
    for (int64_t line = blockIdx.y; line < lines; line += gridDim.y) {
        LineIdx L = line_of(line, 2, k);
        const u64 p = K.pi[L.r].p;
        const u64 *x = at(a, L.b, L.c, L.r, logn);
        u64 *z = at(o, L.b, L.c, L.r, logn);
        const u64 *y = pt + L.b * pstride + ((int64_t)L.r << logn);
        if (L.c != 0 && !copy_c1) continue;
        const ulonglong2 *x2 = reinterpret_cast<const ulonglong2 *>(x), *y2 = reinterpret_cast<const ulonglong2 *>(y);
        ulonglong2 *z2 = reinterpret_cast<ulonglong2 *>(z);
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n / 2; i += gridDim.x * blockDim.x) {
            const ulonglong2 u = x2[i];
            if (L.c == 0) {
                const ulonglong2 v = y2[i];
                z2[i] = make_ulonglong2(add_mod(u.x, v.x, p), add_mod(u.y, v.y, p));
            } else {
                z2[i] = u;
            }
        }
    }
}

// (d0, d1, d2) (+)= (a0 b0, a0 b1 + a1 b0, a1 b1); d1 via Karatsuba (3 products).
// Two adjacent positions per thread (16-byte loads and stores).
__device__ __forceinline__ void tensor_one(u64 x0, u64 x1, u64 y0, u64 y1, const PrimeInfo &P, unsigned long long &e0, unsigned long long &e1,
                                           unsigned long long &e2) {
    e0 = mont_mul(x0, y0, P.p, P.pinv);
    e2 = mont_mul(x1, y1, P.p, P.pinv);
    const u64 s = mont_mul(add_mod(x0, x1, P.p), add_mod(y0, y1, P.p), P.p, P.pinv);
    e1 = sub_mod(sub_mod(s, e0, P.p), e2, P.p);
}
__global__ void k_tensor(Ctx K, heb_ct a, heb_ct b, heb_ct d, int64_t lines, int k, int logn, int acc) {
    const int n = 1 << logn;
    for (int64_t line = blockIdx.y; line < lines; line += gridDim.y) {
        const int r = (int)(line % k);
        const int64_t it = line / k;
        const PrimeInfo P = K.pi[r];
        const ulonglong2 *a0 = reinterpret_cast<const ulonglong2 *>(at(a, it, 0, r, logn));
        const ulonglong2 *a1 = reinterpret_cast<const ulonglong2 *>(at(a, it, 1, r, logn));
        const ulonglong2 *b0 = reinterpret_cast<const ulonglong2 *>(at(b, it, 0, r, logn));
        const ulonglong2 *b1 = reinterpret_cast<const ulonglong2 *>(at(b, it, 1, r, logn));
        ulonglong2 *d0 = reinterpret_cast<ulonglong2 *>(at(d, it, 0, r, logn));
        ulonglong2 *d1 = reinterpret_cast<ulonglong2 *>(at(d, it, 1, r, logn));
        ulonglong2 *d2 = reinterpret_cast<ulonglong2 *>(at(d, it, 2, r, logn));
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n / 2; i += gridDim.x * blockDim.x) {
            const ulonglong2 x0 = a0[i], x1 = a1[i], y0 = b0[i], y1 = b1[i];
            ulonglong2 e0, e1, e2;
            tensor_one(x0.x, x1.x, y0.x, y1.x, P, e0.x, e1.x, e2.x);
            tensor_one(x0.y, x1.y, y0.y, y1.y, P, e0.y, e1.y, e2.y);
            if (acc) {
                const ulonglong2 o0 = d0[i], o1 = d1[i], o2 = d2[i];
                e0 = make_ulonglong2(add_mod(o0.x, e0.x, P.p), add_mod(o0.y, e0.y, P.p));
                e1 = make_ulonglong2(add_mod(o1.x, e1.x, P.p), add_mod(o1.y, e1.y, P.p));
                e2 = make_ulonglong2(add_mod(o2.x, e2.x, P.p), add_mod(o2.y, e2.y, P.p));
            }
            d0[i] = e0;
            d1[i] = e1;
            d2[i] = e2;
        }
    }
}

__global__ void k_mul_rows(Ctx K, const u64 *a, const u64 *b, u64 *o, int rows, int logn) {
    const int n = 1 << logn;
    for (int r = blockIdx.y; r < rows; r += gridDim.y) {
        const PrimeInfo P = K.pi[r];
        const size_t off = (size_t)r << logn;
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
            o[off + i] = mont_mul(a[off + i], b[off + i], P.p, P.pinv);
    }
}

// evaluation-domain automorphism X -> X^g: out[i] = in[j], 2 brv(j)+1 = (2 brv(i)+1) g mod 2n
__global__ void k_galois(const u64 *in, u64 *out, int64_t lines, int64_t bstride, int rows, int logn, u64 g) {
    const int n = 1 << logn;
    const u64 mask2n = 2ull * n - 1;
    for (int64_t line = blockIdx.y; line < lines; line += gridDim.y) {
        const int r = (int)(line % rows);
        const int64_t b = line / rows;
        const u64 *src = in + b * bstride + ((int64_t)r << logn);
        u64 *dst = out + b * bstride + ((int64_t)r << logn);
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
            const u64 e = 2ull * (__brev((unsigned)i) >> (32 - logn)) + 1;
            const u64 e2 = (e * g) & mask2n;
            const unsigned j = __brev((unsigned)((e2 - 1) >> 1)) >> (32 - logn);
            dst[i] = src[j];
        }
    }
}



extern "C" int heb_add(heb_ctx *c, heb_ct a, heb_ct b, heb_ct o, int64_t count, int comps, int k, void *stream) {
    if (!c || k < 1 || k > c->num_rows || comps < 1) return fail(HEB_EINVAL, "heb_add: bad args");
    if ((a.ct_stride | a.comp_stride | b.ct_stride | b.comp_stride | o.ct_stride | o.comp_stride) & 1)
        return fail(HEB_EINVAL, "heb_add: strides must be even (16-byte position pairs)");
    if (count <= 0) return HEB_OK;
    const int64_t lines = count * comps * k;
    { PROF("k_add", (cudaStream_t)stream, 24.0 * c->n * lines); k_add<<<pw_grid(c->n / 2, lines), 256, 0, (cudaStream_t)stream>>>(kctx(c), a, b, o, lines, comps, k, c->log_n); }
    LAUNCH_CHECK();
    return HEB_OK;
}

extern "C" int heb_add_plain(heb_ctx *c, heb_ct a, const uint64_t *pt, int64_t pstride, heb_ct o, int64_t count,
                             int k, void *stream) {
    if (!c || !pt || k < 1 || k > c->num_rows) return fail(HEB_EINVAL, "heb_add_plain: bad args");
    if ((a.ct_stride | a.comp_stride | o.ct_stride | o.comp_stride | pstride) & 1)
        return fail(HEB_EINVAL, "heb_add_plain: strides must be even (16-byte position pairs)");
    if (count <= 0) return HEB_OK;
    const int64_t lines = count * 2 * k;
    const int copy_c1 = (o.data != a.data) || (o.comp_stride != a.comp_stride) || (o.ct_stride != a.ct_stride);
    { PROF("k_add_plain", (cudaStream_t)stream, 8.0 * c->n * (2.0 * lines + k * (pstride ? count : 1))); k_add_plain<<<pw_grid(c->n / 2, lines), 256, 0, (cudaStream_t)stream>>>(kctx(c), a, pt, pstride, o, lines, k,
                                                                         c->log_n, copy_c1); }
    LAUNCH_CHECK();
    return HEB_OK;
}

extern "C" int heb_tensor(heb_ctx *c, heb_ct a, heb_ct b, heb_ct d, int64_t count, int k, int accumulate,
                          void *stream) {
    if (!c || k < 1 || k > c->num_rows) return fail(HEB_EINVAL, "heb_tensor: bad args");
    if ((a.ct_stride | a.comp_stride | b.ct_stride | b.comp_stride | d.ct_stride | d.comp_stride) & 1)
        return fail(HEB_EINVAL, "heb_tensor: strides must be even (16-byte position pairs)");
    if (count <= 0) return HEB_OK;
    const int64_t lines = count * k;
    { PROF("k_tensor", (cudaStream_t)stream, 8.0 * c->n * lines * (accumulate ? 10.0 : 7.0)); k_tensor<<<pw_grid(c->n / 2, lines), 256, 0, (cudaStream_t)stream>>>(kctx(c), a, b, d, lines, k, c->log_n,
                                                                      accumulate); }
    LAUNCH_CHECK();
    return HEB_OK;
}

extern "C" int heb_mul_rows(heb_ctx *c, const uint64_t *a, const uint64_t *b, uint64_t *o, int rows, void *stream) {
    if (!c || rows < 1 || rows > c->num_rows) return fail(HEB_EINVAL, "heb_mul_rows: bad args");
    { PROF("k_mul_rows", (cudaStream_t)stream, 24.0 * c->n * rows); k_mul_rows<<<pw_grid(c->n, rows), 256, 0, (cudaStream_t)stream>>>(kctx(c), a, b, o, rows, c->log_n); }
    LAUNCH_CHECK();
    return HEB_OK;
}

extern "C" int heb_galois(heb_ctx *c, const uint64_t *in, uint64_t *out, int64_t count, int rows, int64_t bstride,
                          uint64_t galois, void *stream) {
    if (!c || !(galois & 1) || in == out || rows < 1 || rows > c->num_rows) return fail(HEB_EINVAL, "heb_galois: bad args");
    if (count <= 0) return HEB_OK;
    const int64_t lines = count * rows;
    { PROF("k_galois", (cudaStream_t)stream, 16.0 * c->n * lines); k_galois<<<pw_grid(c->n, lines), 256, 0, (cudaStream_t)stream>>>(in, out, lines, bstride, rows, c->log_n,
                                                                      galois % (2ull * c->n)); }
    LAUNCH_CHECK();
    return HEB_OK;
}


__global__ void k_galois_ct(heb_ct in, heb_ct out, int64_t lines, int k, int logn, u64 g) {
    const int n = 1 << logn;
    const u64 mask2n = 2ull * n - 1;
    for (int64_t line = blockIdx.y; line < lines; line += gridDim.y) {
        LineIdx L = line_of(line, 2, k);
        const u64 *src = at(in, L.b, L.c, L.r, logn);
        u64 *dst = at(out, L.b, L.c, L.r, logn);
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
            const u64 e = 2ull * (__brev((unsigned)i) >> (32 - logn)) + 1;
            const u64 e2 = (e * g) & mask2n;
            dst[i] = src[__brev((unsigned)((e2 - 1) >> 1)) >> (32 - logn)];
        }
    }
}

// =============================================================================
// batched layer evaluator
// =============================================================================
// raw_o (row r, position x) = sum_t A[ia] (x) B[ib]; lazy 128-bit sums, Karatsuba d1
__global__ void k_dot_tensor(Ctx K, heb_ct A, heb_ct B, const int32_t *ia, const int32_t *ib, int taps, heb_ct D,
                             int64_t n_out, int k, int logn, int flush) {
    const int n = 1 << logn;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= n) return;
    const int r = blockIdx.z;
    const PrimeInfo P = K.pi[r];
    for (int64_t o = blockIdx.y; o < n_out; o += gridDim.y) {
        acc4 s0 = {0, 0, 0, 0}, s1 = {0, 0, 0, 0}, s2 = {0, 0, 0, 0};
        u64 t0 = 0, t1 = 0, t2 = 0;
        int since = 0;
        for (int t = 0; t < taps; ++t) {
            const int64_t a = ia[o * taps + t], b = ib[o * taps + t];
            const u64 *ap = A.data + a * A.ct_stride + ((int64_t)r << logn) + x;
            const u64 *bp = B.data + b * B.ct_stride + ((int64_t)r << logn) + x;
            const u64 a0 = __ldg(ap), a1 = __ldg(ap + A.comp_stride);
            const u64 b0 = __ldg(bp), b1 = __ldg(bp + B.comp_stride);
            mac4(s0, a0, b0);
            mac4(s2, a1, b1);
            mac4(s1, add_mod(a0, a1, P.p), add_mod(b0, b1, P.p));
            if (++since == flush) {
                t0 = add_mod(t0, redc128(to128(s0), P.p, P.pinv, P.r1s), P.p);
                t1 = add_mod(t1, redc128(to128(s1), P.p, P.pinv, P.r1s), P.p);
                t2 = add_mod(t2, redc128(to128(s2), P.p, P.pinv, P.r1s), P.p);
                s0 = s1 = s2 = acc4{0, 0, 0, 0};
                since = 0;
            }
        }
        t0 = add_mod(t0, redc128(to128(s0), P.p, P.pinv, P.r1s), P.p);
        t1 = add_mod(t1, redc128(to128(s1), P.p, P.pinv, P.r1s), P.p);
        t2 = add_mod(t2, redc128(to128(s2), P.p, P.pinv, P.r1s), P.p);
        u64 *dp = D.data + o * D.ct_stride + ((int64_t)r << logn) + x;
        dp[0] = t0;
        dp[D.comp_stride] = sub_mod(sub_mod(t1, t0, P.p), t2, P.p);
        dp[2 * D.comp_stride] = t2;
    }
}

extern "C" int heb_dot_tensor(heb_ctx *c, heb_ct a, heb_ct b, const int32_t *ia, const int32_t *ib, int taps,
                              heb_ct d, int64_t n_out, int k, void *stream) {
    if (!c || !ia || !ib || taps < 1 || k < 1 || k > c->num_rows) return fail(HEB_EINVAL, "heb_dot_tensor: bad args");
    if (n_out <= 0) return HEB_OK;
    dim3 grid((c->n + 127) / 128, gdim(n_out), k);
    { PROF("k_dot_tensor", (cudaStream_t)stream, 24.0 * c->n * n_out * k); k_dot_tensor<<<grid, 128, 0, (cudaStream_t)stream>>>(kctx(c), a, b, ia, ib, taps, d, n_out, k, c->log_n, c->flush); }
    LAUNCH_CHECK();
    return HEB_OK;
}

__global__ void k_sum_gather(Ctx K, heb_ct A, const int32_t *idx, int terms, heb_ct O, int64_t lines, int comps,
                             int k, int logn) {
    const int n = 1 << logn;
    for (int64_t line = blockIdx.y; line < lines; line += gridDim.y) {
        LineIdx L = line_of(line, comps, k);
        const u64 p = K.pi[L.r].p;
        const int32_t *ix = idx + L.b * terms;
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
            u64 s = 0;
            for (int t = 0; t < terms; ++t) s = add_mod(s, at(A, ix[t], L.c, L.r, logn)[i], p);
            at(O, L.b, L.c, L.r, logn)[i] = s;
        }
    }
}

extern "C" int heb_sum_gather(heb_ctx *c, heb_ct a, const int32_t *idx, int terms, heb_ct o, int64_t n_out,
                              int comps, int k, void *stream) {
    if (!c || !idx || terms < 1 || k < 1 || k > c->num_rows || comps < 1) return fail(HEB_EINVAL, "heb_sum_gather: bad args");
    if (n_out <= 0) return HEB_OK;
    const int64_t lines = n_out * comps * k;
    { PROF("k_sum_gather", (cudaStream_t)stream, 8.0 * c->n * lines * (terms + 1.0)); k_sum_gather<<<pw_grid(c->n, lines), 256, 0, (cudaStream_t)stream>>>(kctx(c), a, idx, terms, o, lines, comps, k,
                                                                          c->log_n); }
    LAUNCH_CHECK();
    return HEB_OK;
}

extern "C" int heb_gather(heb_ctx *c, heb_ct a, const int32_t *idx, heb_ct o, int64_t n_out, int comps, int k,
                          void *stream) {
    return heb_sum_gather(c, a, idx, 1, o, n_out, comps, k, stream);
}

