/*
 * heoracle.c -- CPU oracle for the CKKS evaluation path (TEST INFRASTRUCTURE).
 *
 * This file is a plain-C restatement of the reference's numba kernels in
 * /root/reference/pkg/src/hecnn/backends/kernels.py.  It exists only to
 * CHECK the CUDA product path: tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load it; the product
 * package never does.  It is pinned against golden vectors produced by the
 * reference itself (tests/golden/make_golden.py).
 *
 * Conventions (kernels.py:1-13): every residue array holds x*2^64 mod p in
 * [0, p) ("Montgomery form"), primes < 2^62, one row per prime, row-major
 * (rows, n) uint64 arrays.  Each function below cites the reference
 * function whose semantics it restates.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;
typedef uint64_t u64;
typedef int64_t i64;

/* kernels.py:38-49 -- Montgomery REDC of x*y, canonical output. */
static inline u64 mont_mul(u64 x, u64 y, u64 p, u64 pinv) {
    u128 t = (u128)x * y;
    u64 lo = (u64)t, hi = (u64)(t >> 64);
    u64 m = lo * pinv;
    u64 r = hi + (u64)(((u128)m * p) >> 64) + (lo != 0);
    return r >= p ? r - p : r;
}
static inline u64 add_mod(u64 x, u64 y, u64 p) { u64 s = x + y; return s >= p ? s - p : s; }
static inline u64 sub_mod(u64 x, u64 y, u64 p) { u64 d = x + p - y; return d >= p ? d - p : d; }

/* kernels.py:68-88 -- in-place forward negacyclic NTT, natural in, bit-reversed out. */
void or_ntt_fwd_rows(u64 *f, int rows, int n, const u64 *tw, int tw_stride,
                     const u64 *p, const u64 *pinv) {
    for (int r = 0; r < rows; r++) {
        u64 *a = f + (size_t)r * n;
        const u64 *w = tw + (size_t)r * tw_stride;
        u64 pr = p[r], pi = pinv[r];
        int wi = 0;
        for (int half = n >> 1; half > 0; half >>= 1) {
            for (int base = 0; base < n; base += 2 * half) {
                u64 z = w[++wi];
                for (int j = base; j < base + half; j++) {
                    u64 x = a[j], y = mont_mul(a[j + half], z, pr, pi);
                    a[j] = add_mod(x, y, pr);
                    a[j + half] = sub_mod(x, y, pr);
                }
            }
        }
    }
}

/* kernels.py:91-114 -- in-place inverse (GS, table walked backwards) then * n^-1. */
void or_ntt_inv_rows(u64 *f, int rows, int n, const u64 *tw, int tw_stride,
                     const u64 *ninv, const u64 *p, const u64 *pinv) {
    for (int r = 0; r < rows; r++) {
        u64 *a = f + (size_t)r * n;
        const u64 *w = tw + (size_t)r * tw_stride;
        u64 pr = p[r], pi = pinv[r];
        int wi = n;
        for (int half = 1; half < n; half <<= 1) {
            for (int base = 0; base < n; base += 2 * half) {
                u64 z = w[--wi];
                for (int j = base; j < base + half; j++) {
                    u64 x = a[j], y = a[j + half];
                    a[j] = add_mod(x, y, pr);
                    a[j + half] = mont_mul(sub_mod(y, x, pr), z, pr, pi);
                }
            }
        }
        for (int j = 0; j < n; j++) a[j] = mont_mul(a[j], ninv[r], pr, pi);
    }
}

/* kernels.py:117-123 / 135-142 / 145-152 / 166-175 / 178-197 -- pointwise rows. */
void or_add_rows(const u64 *a, const u64 *b, int rows, int n, const u64 *p, u64 *out) {
    for (int r = 0; r < rows; r++)
        for (int j = 0; j < n; j++) {
            size_t i = (size_t)r * n + j;
            out[i] = add_mod(a[i], b[i], p[r]);
        }
}
void or_neg_rows(const u64 *a, int rows, int n, const u64 *p, u64 *out) {
    for (int r = 0; r < rows; r++)
        for (int j = 0; j < n; j++) {
            size_t i = (size_t)r * n + j;
            out[i] = a[i] ? p[r] - a[i] : 0;
        }
}
void or_mul_rows(const u64 *a, const u64 *b, int rows, int n, const u64 *p, const u64 *pinv, u64 *out) {
    for (int r = 0; r < rows; r++)
        for (int j = 0; j < n; j++) {
            size_t i = (size_t)r * n + j;
            out[i] = mont_mul(a[i], b[i], p[r], pinv[r]);
        }
}
void or_scalar_mul_rows(const u64 *a, const u64 *c, int rows, int n, const u64 *p,
                        const u64 *pinv, u64 *out) {
    for (int r = 0; r < rows; r++)
        for (int j = 0; j < n; j++) {
            size_t i = (size_t)r * n + j;
            out[i] = mont_mul(a[i], c[r], p[r], pinv[r]);
        }
}
void or_from_mont_rows(u64 *a, int rows, int n, const u64 *p, const u64 *pinv) {
    for (int r = 0; r < rows; r++)
        for (int j = 0; j < n; j++) {
            size_t i = (size_t)r * n + j;
            a[i] = mont_mul(a[i], 1, p[r], pinv[r]);
        }
}

/* kernels.py:200-212 -- standard-form residue -> centered signed value. */
void or_centered_rows(const u64 *a, int rows, int n, const u64 *p, i64 *out) {
    for (int r = 0; r < rows; r++) {
        u64 half = p[r] >> 1;
        for (int j = 0; j < n; j++) {
            size_t i = (size_t)r * n + j;
            out[i] = a[i] > half ? (i64)a[i] - (i64)p[r] : (i64)a[i];
        }
    }
}

/* Python-semantics v mod p for signed v (kernels.py:226). */
static inline u64 pymod(i64 v, u64 p) {
    i64 m = v % (i64)p;
    return (u64)(m < 0 ? m + (i64)p : m);
}

/* kernels.py:215-227 -- centered int64 coefficients -> Montgomery rows per prime. */
void or_spread_centered(const i64 *coeffs, int n, int rows, const u64 *p, const u64 *r2,
                        const u64 *pinv, u64 *out) {
    for (int r = 0; r < rows; r++)
        for (int j = 0; j < n; j++)
            out[(size_t)r * n + j] = mont_mul(pymod(coeffs[j], p[r]), r2[r], p[r], pinv[r]);
}

/* kernels.py:230-246 -- degree-2 tensor product. */
void or_ctct_products(const u64 *a0, const u64 *a1, const u64 *b0, const u64 *b1, int rows, int n,
                      const u64 *p, const u64 *pinv, u64 *d0, u64 *d1, u64 *d2) {
    for (int r = 0; r < rows; r++)
        for (int j = 0; j < n; j++) {
            size_t i = (size_t)r * n + j;
            u64 pr = p[r], pi = pinv[r];
            d0[i] = mont_mul(a0[i], b0[i], pr, pi);
            d1[i] = add_mod(mont_mul(a0[i], b1[i], pr, pi), mont_mul(a1[i], b0[i], pr, pi), pr);
            d2[i] = mont_mul(a1[i], b1[i], pr, pi);
        }
}

/* kernels.py:270-294 -- rescale: divide by the last row's prime and drop it.
 * tw/ninv/p/pinv/r2 cover the k rows of comp; drop_inv holds q_last^-1 (Mont)
 * for the k-1 surviving rows. */
void or_divide_drop_last(const u64 *comp, int k, int n, const u64 *tw, int tw_stride,
                         const u64 *ninv, const u64 *p, const u64 *pinv, const u64 *r2,
                         const u64 *drop_inv, u64 *out) {
    u64 *last = malloc(sizeof(u64) * n);
    i64 *cent = malloc(sizeof(i64) * n);
    u64 *tmp = malloc(sizeof(u64) * (size_t)(k - 1) * n);
    memcpy(last, comp + (size_t)(k - 1) * n, sizeof(u64) * n);
    or_ntt_inv_rows(last, 1, n, tw + (size_t)(k - 1) * tw_stride, tw_stride, ninv + k - 1, p + k - 1, pinv + k - 1);
    or_from_mont_rows(last, 1, n, p + k - 1, pinv + k - 1);
    or_centered_rows(last, 1, n, p + k - 1, cent);
    or_spread_centered(cent, n, k - 1, p, r2, pinv, tmp);
    or_ntt_fwd_rows(tmp, k - 1, n, tw, tw_stride, p, pinv);
    for (int r = 0; r < k - 1; r++)
        for (int j = 0; j < n; j++) {
            size_t i = (size_t)r * n + j;
            out[i] = mont_mul(sub_mod(comp[i], tmp[i], p[r]), drop_inv[r], p[r], pinv[r]);
        }
    free(last); free(cent); free(tmp);
}

/* kernels.py:297-340 -- ModUp + key inner product.
 * d2_eval/d2_cent: (k, n); evk_b/evk_a: (digits, grows, n); acc0/acc1: (k+1, n).
 * Global per-prime tables tw_all (grows, tw_stride), p_all, pinv_all, r2_all. */
void or_relin_accumulate(const u64 *d2_eval, const i64 *d2_cent, int k, int n,
                         const u64 *evk_b, const u64 *evk_a, int grows, int sp_row,
                         const u64 *tw_all, int tw_stride, const u64 *p_all,
                         const u64 *pinv_all, const u64 *r2_all, u64 *acc0, u64 *acc1) {
    u64 *dig = malloc(sizeof(u64) * n);
    for (int j = 0; j < k; j++) {
        for (int t = 0; t <= k; t++) {
            int gt = t < k ? t : sp_row;
            u64 pt = p_all[gt], pit = pinv_all[gt];
            if (t == j) {
                memcpy(dig, d2_eval + (size_t)j * n, sizeof(u64) * n);
            } else {
                for (int x = 0; x < n; x++)
                    dig[x] = mont_mul(pymod(d2_cent[(size_t)j * n + x], pt), r2_all[gt], pt, pit);
                or_ntt_fwd_rows(dig, 1, n, tw_all + (size_t)gt * tw_stride, tw_stride, p_all + gt, pinv_all + gt);
            }
            const u64 *eb = evk_b + ((size_t)j * grows + gt) * n;
            const u64 *ea = evk_a + ((size_t)j * grows + gt) * n;
            for (int x = 0; x < n; x++) {
                size_t i = (size_t)t * n + x;
                acc0[i] = add_mod(acc0[i], mont_mul(dig[x], eb[x], pt, pit), pt);
                acc1[i] = add_mod(acc1[i], mont_mul(dig[x], ea[x], pt, pit), pt);
            }
        }
    }
    free(dig);
}

/* kernels.py:343-371 -- ModDown: rounded division by the special prime. */
void or_moddown_special(const u64 *acc, int k, int n, int sp_row, const u64 *tw_all, int tw_stride,
                        const u64 *ninv_all, const u64 *p_all, const u64 *pinv_all,
                        const u64 *r2_all, const u64 *sp_inv, u64 *out) {
    u64 *last = malloc(sizeof(u64) * n);
    i64 *cent = malloc(sizeof(i64) * n);
    u64 *tmp = malloc(sizeof(u64) * (size_t)k * n);
    memcpy(last, acc + (size_t)k * n, sizeof(u64) * n);
    or_ntt_inv_rows(last, 1, n, tw_all + (size_t)sp_row * tw_stride, tw_stride, ninv_all + sp_row,
                    p_all + sp_row, pinv_all + sp_row);
    or_from_mont_rows(last, 1, n, p_all + sp_row, pinv_all + sp_row);
    or_centered_rows(last, 1, n, p_all + sp_row, cent);
    or_spread_centered(cent, n, k, p_all, r2_all, pinv_all, tmp);
    or_ntt_fwd_rows(tmp, k, n, tw_all, tw_stride, p_all, pinv_all);
    for (int r = 0; r < k; r++)
        for (int j = 0; j < n; j++) {
            size_t i = (size_t)r * n + j;
            out[i] = mont_mul(sub_mod(acc[i], tmp[i], p_all[r]), sp_inv[r], p_all[r], pinv_all[r]);
        }
    free(last); free(cent); free(tmp);
}

/* kernels.py:374-383 -- decrypt guard: count coefficients whose residue disagrees. */
long or_residue_check(const i64 *coeffs, int n, u64 q, const u64 *expect) {
    long bad = 0;
    for (int j = 0; j < n; j++)
        if (pymod(coeffs[j], q) != expect[j]) bad++;
    return bad;
}

/* Evaluation-domain Galois automorphism X -> X^g (no reference counterpart:
 * rotation is absent there).  Slot i of the NTT output holds a(psi^(2*brv(i)+1));
 * sigma_g(a) at psi^e equals a(psi^(e*g)), so out[i] = in[j] with
 * 2*brv(j)+1 = (2*brv(i)+1)*g mod 2n.  Pure permutation: Montgomery form kept. */
static u64 brv(u64 x, int bits) {
    u64 y = 0;
    for (int i = 0; i < bits; i++) y |= ((x >> i) & 1) << (bits - 1 - i);
    return y;
}
void or_galois_eval(const u64 *in, int rows, int n, u64 galois, u64 *out) {
    int logn = 0;
    while ((1 << logn) < n) logn++;
    u64 two_n = 2 * (u64)n;
    for (int i = 0; i < n; i++) {
        u64 e = (2 * brv(i, logn) + 1) % two_n;
        u64 e2 = (u64)(((u128)e * galois) % two_n);
        u64 j = brv((e2 - 1) / 2, logn);
        for (int r = 0; r < rows; r++) out[(size_t)r * n + i] = in[(size_t)r * n + j];
    }
}
