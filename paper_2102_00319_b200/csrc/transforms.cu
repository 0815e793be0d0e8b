// transforms.cu -- NTT entry points and the client-side kernels (encrypt/decrypt/keygen).
#include "common.cuh"

// =============================================================================
// transforms
// =============================================================================
#ifndef PLAIN_E
#define PLAIN_E 16
#endif
template <int LOGN>
__global__ void __launch_bounds__((KT<LOGN, PLAIN_E>), NTT_MINB_T((KT<LOGN, PLAIN_E>)))
    k_ntt_fwd(Ctx K, u64 *data, int64_t count, int row0, int64_t bstride, int mont) {
    constexpr int E = PLAIN_E;
    extern __shared__ u64 sm[];
    const int r = lbx<LOGN>(), prime = row0 + r;
    const PrimeInfo P = K.pi[prime];
    for (int64_t b = blockIdx.y; b < count; b += gridDim.y) {
        u64 *row = data + b * bstride + ((int64_t)r << LOGN);
        u64 y[E];
        // mont: standard-form coefficients in, Montgomery evaluation rows out (to_mont + NTT)
        fwd_any<LOGN, E>(K, prime, P, sm, [&](int i) {
            const u64 v = __ldcg(row + i);
            return mont ? shoup(v, P.rmod, P.rmod_s, P.p) : v;
        }, y);
        // all reads of `row` (by both CTAs of a split row) done before in-place writes
        if constexpr (Row<LOGN>::SPLIT) cooperative_groups::this_cluster().sync();
        else __syncthreads();
        storev<LOGN, E>(row + tpos<LOGN, E>(), y);
    }
}

template <int LOGN>
__global__ void __launch_bounds__((KT<LOGN, PLAIN_E>), NTT_MINB_T((KT<LOGN, PLAIN_E>)))
    k_ntt_inv(Ctx K, u64 *data, int64_t count, int row0, int64_t bstride, int mont) {
    constexpr int E = PLAIN_E;
    extern __shared__ u64 sm[];
    const int r = lbx<LOGN>(), prime = row0 + r;
    const PrimeInfo P = K.pi[prime];
    for (int64_t b = blockIdx.y; b < count; b += gridDim.y) {
        u64 *row = data + b * bstride + ((int64_t)r << LOGN);
        u64 x[E];
        loadv<LOGN, E>(row + tpos<LOGN, E>(), x);
        // mont: Montgomery evaluation rows in, standard-form coefficients out (INTT + from_mont)
        inv_any<LOGN, E>(K, prime, P, sm, x, [&](int i, u64 v) { row[i] = v; }, mont != 0);
    }
}

template <int LOGN>
static int launch_ntt(heb_ctx *c, uint64_t *data, int64_t count, int rows, int row0, int64_t bstride,
                      cudaStream_t st, bool inverse, int mont) {
    constexpr int T = KT<LOGN>;
    constexpr size_t sm = smem_bytes<LOGN>();
    dim3 grid(rows, gdim(count));
    if (inverse) {
        CUDA_TRY(prep_kernel(k_ntt_inv<LOGN>, sm));
        { PROF("k_ntt_inv", st, 16.0 * c->n * rows * count); CUDA_TRY(launch_rows<LOGN>(k_ntt_inv<LOGN>, dim3(grid), KT<LOGN, PLAIN_E>, sm, st, kctx(c), data, count, row0, bstride, mont)); }
    } else {
        CUDA_TRY(prep_kernel(k_ntt_fwd<LOGN>, sm));
        { PROF("k_ntt_fwd", st, 16.0 * c->n * rows * count); CUDA_TRY(launch_rows<LOGN>(k_ntt_fwd<LOGN>, dim3(grid), KT<LOGN, PLAIN_E>, sm, st, kctx(c), data, count, row0, bstride, mont)); }
    }
    LAUNCH_CHECK();
    return HEB_OK;
}

extern "C" int heb_ntt_fwd(heb_ctx *c, uint64_t *data, int64_t count, int rows, int row0, int64_t bstride,
                           void *stream) {
    if (!c || !data || rows < 1 || row0 < 0 || row0 + rows > c->num_rows) return fail(HEB_EINVAL, "heb_ntt_fwd: bad rows");
    if (count <= 0) return HEB_OK;
    DISPATCH_LOGN(c, launch_ntt, c, data, count, rows, row0, bstride, (cudaStream_t)stream, false, 0);
}
extern "C" int heb_ntt_inv(heb_ctx *c, uint64_t *data, int64_t count, int rows, int row0, int64_t bstride,
                           void *stream) {
    if (!c || !data || rows < 1 || row0 < 0 || row0 + rows > c->num_rows) return fail(HEB_EINVAL, "heb_ntt_inv: bad rows");
    if (count <= 0) return HEB_OK;
    DISPATCH_LOGN(c, launch_ntt, c, data, count, rows, row0, bstride, (cudaStream_t)stream, true, 0);
}
extern "C" int heb_coeff_to_eval(heb_ctx *c, uint64_t *data, int64_t count, int rows, int64_t bstride, void *stream) {
    if (!c || !data || rows < 1 || rows > c->num_rows) return fail(HEB_EINVAL, "heb_coeff_to_eval: bad rows");
    if (count <= 0) return HEB_OK;
    DISPATCH_LOGN(c, launch_ntt, c, data, count, rows, 0, bstride, (cudaStream_t)stream, false, 1);
}
extern "C" int heb_eval_to_coeff(heb_ctx *c, uint64_t *data, int64_t count, int rows, int64_t bstride, void *stream) {
    if (!c || !data || rows < 1 || rows > c->num_rows) return fail(HEB_EINVAL, "heb_eval_to_coeff: bad rows");
    if (count <= 0) return HEB_OK;
    DISPATCH_LOGN(c, launch_ntt, c, data, count, rows, 0, bstride, (cudaStream_t)stream, true, 1);
}

// spread_centered + ntt_fwd_rows (ckks.py:120-126): signed coefficient -> (v mod p) * R, NTT
template <int LOGN>
__global__ void ROW_BOUNDS(LOGN) k_spread_ntt(Ctx K, const i64 *coeffs, int64_t count,
                                                                      u64 *out, int64_t ostride) {
    extern __shared__ u64 sm[];
    const int r = lbx<LOGN>();
    const PrimeInfo P = K.pi[r];
    for (int64_t b = blockIdx.y; b < count; b += gridDim.y) {
        const i64 *src = coeffs + (b << LOGN);
        u64 y[16];
        fwd_any<LOGN>(K, r, P, sm,
                           [&](int i) { return signed_mul_const(__ldcg(src + i), P.rmod, P.rmod_s, P.p); }, y);
        store16<LOGN>(out + b * ostride + ((int64_t)r << LOGN) + tpos<LOGN>(), y);
    }
}

template <int LOGN>
static int launch_spread(heb_ctx *c, const int64_t *coeffs, int64_t count, uint64_t *out, int rows,
                         int64_t ostride, cudaStream_t st) {
    constexpr size_t sm = smem_bytes<LOGN>();
    CUDA_TRY(prep_kernel(k_spread_ntt<LOGN>, sm));
    { PROF("k_spread_ntt", st, 8.0 * c->n * count * (1.0 + rows)); CUDA_TRY(launch_rows<LOGN>(k_spread_ntt<LOGN>, dim3(dim3(rows, gdim(count))), KT<LOGN>, sm, st, kctx(c), coeffs, count, out, ostride)); }
    LAUNCH_CHECK();
    return HEB_OK;
}

extern "C" int heb_spread_ntt(heb_ctx *c, const int64_t *coeffs, int64_t count, uint64_t *out, int rows,
                              int64_t ostride, void *stream) {
    if (!c || !coeffs || !out || rows < 1 || rows > c->num_rows) return fail(HEB_EINVAL, "heb_spread_ntt: bad args");
    if (count <= 0) return HEB_OK;
    DISPATCH_LOGN(c, launch_spread, c, coeffs, count, out, rows, ostride, (cudaStream_t)stream);
}

// =============================================================================
// client side: encrypt / decrypt / key generation (ckks.py:135-273)
// =============================================================================
template <int LOGN>
__global__ void ROW_BOUNDS(LOGN) k_encrypt(Ctx K, const i64 *v, const i64 *e0m, const i64 *e1,
                                                                   const u64 *pkb, const u64 *pka, heb_ct out,
                                                                   int64_t count) {
    extern __shared__ u64 sm[];
    const int r = lbx<LOGN>();
    const PrimeInfo P = K.pi[r];
    const int n = 1 << LOGN, pos = tpos<LOGN>();
    const ulonglong2 *tw = tw_row<LOGN>(K, r);
    for (int64_t b = blockIdx.y; b < count; b += gridDim.y) {
        auto spread = [&](const i64 *src) { return [=](int i) { return signed_mul_const(__ldcg(src + i), P.rmod, P.rmod_s, P.p); }; };
        u64 V[16], E[16], pk[16], o[16];
        fwd_any<LOGN>(K, r, P, sm, spread(v + b * n), V);
        fwd_any<LOGN>(K, r, P, sm, spread(e0m + b * n), E);
        load16<LOGN>(pkb + ((size_t)r << LOGN) + pos, pk);
#pragma unroll
        for (int m = 0; m < 16; ++m) o[m] = add_mod(mont_mul(V[m], pk[m], P.p, P.pinv), E[m], P.p);
        store16<LOGN>(at(out, b, 0, r, LOGN) + pos, o);
        fwd_any<LOGN>(K, r, P, sm, spread(e1 + b * n), E);
        load16<LOGN>(pka + ((size_t)r << LOGN) + pos, pk);
#pragma unroll
        for (int m = 0; m < 16; ++m) o[m] = add_mod(mont_mul(V[m], pk[m], P.p, P.pinv), E[m], P.p);
        store16<LOGN>(at(out, b, 1, r, LOGN) + pos, o);
    }
}

template <int LOGN>
static int launch_encrypt(heb_ctx *c, const i64 *v, const i64 *e0m, const i64 *e1, const u64 *pkb, const u64 *pka,
                          heb_ct out, int64_t count, int k, cudaStream_t st) {
    constexpr size_t sm = smem_bytes<LOGN>();
    CUDA_TRY(prep_kernel(k_encrypt<LOGN>, sm));
    { PROF("k_encrypt", st, 8.0 * c->n * (3.0 * count + 2.0 * k + 2.0 * count * k)); CUDA_TRY(launch_rows<LOGN>(k_encrypt<LOGN>, dim3(dim3(k, gdim(count))), KT<LOGN>, sm, st, kctx(c), v, e0m, e1, pkb, pka, out, count)); }
    LAUNCH_CHECK();
    return HEB_OK;
}

extern "C" int heb_encrypt(heb_ctx *c, const int64_t *v, const int64_t *e0m, const int64_t *e1, const uint64_t *pk_b,
                           const uint64_t *pk_a, heb_ct out, int64_t count, int k, void *stream) {
    if (!c || !v || !e0m || !e1 || !pk_b || !pk_a || k < 1 || k > c->num_rows - 1)
        return fail(HEB_EINVAL, "heb_encrypt: bad args");
    if (count <= 0) return HEB_OK;
    DISPATCH_LOGN(c, launch_encrypt, c, v, e0m, e1, pk_b, pk_a, out, count, k, (cudaStream_t)stream);
}

// decrypt rows 0/1: m = c1*s + c0 -> INTT -> std form
template <int LOGN>
__global__ void ROW_BOUNDS(LOGN) k_decrypt_rows(Ctx K, heb_ct ct, const u64 *s, u64 *tmp,
                                                                        int rows, int64_t count) {
    extern __shared__ u64 sm[];
    const int r = lbx<LOGN>();
    const PrimeInfo P = K.pi[r];
    const LastConst lc = K.last[r];
    const int n = 1 << LOGN, pos = tpos<LOGN>();
    for (int64_t b = blockIdx.y; b < count; b += gridDim.y) {
        u64 x[16], y[16], z[16];
        load16<LOGN>(at(ct, b, 1, r, LOGN) + pos, x);
        load16<LOGN>(s + ((size_t)r << LOGN) + pos, y);
        load16<LOGN>(at(ct, b, 0, r, LOGN) + pos, z);
#pragma unroll
        for (int m = 0; m < 16; ++m) x[m] = add_mod(mont_mul(x[m], y[m], P.p, P.pinv), z[m], P.p);
        u64 *dst = tmp + (b * rows + r) * n;
        inv_any<LOGN>(K, r, P, sm, x, [&](int i, u64 v) { dst[i] = v; }, true);
    }
}

__global__ void k_decrypt_finish(Ctx K, const u64 *tmp, i64 *coeffs, unsigned long long *bad, int rows, int64_t count, int logn) {
    const int n = 1 << logn;
    const u64 q0 = K.pi[0].p;
    const u64 q1 = rows > 1 ? K.pi[1].p : 1;
    for (int64_t b = blockIdx.y; b < count; b += gridDim.y) {
        int local = 0;
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
            const i64 v = center(tmp[(b * rows) * n + i], q0);
            coeffs[b * n + i] = v;
            if (rows > 1) {
                i64 m = v % (i64)q1;
                if (m < 0) m += (i64)q1;
                local += ((u64)m != tmp[(b * rows + 1) * n + i]);
            } else {
                local += ((double)(v < 0 ? -v : v) >= (double)q0 / 4.0);
            }
        }
        if (local) atomicAdd(bad + b, (unsigned long long)local);
    }
}

template <int LOGN>
static int launch_decrypt(heb_ctx *c, heb_ct ct, const u64 *s, i64 *coeffs, i64 *bad, int64_t count, int k,
                          cudaStream_t st) {
    constexpr size_t sm = smem_bytes<LOGN>();
    CUDA_TRY(prep_kernel(k_decrypt_rows<LOGN>, sm));
    const int rows = k >= 2 ? 2 : 1;
    Scratch tmp(c, st);
    CUDA_TRY(tmp.get(sizeof(u64) * (size_t)count * rows * c->n));
    CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(i64) * count, st));
    { PROF("k_decrypt_rows", st, 8.0 * c->n * (3.0 * count * rows + rows)); CUDA_TRY(launch_rows<LOGN>(k_decrypt_rows<LOGN>, dim3(dim3(rows, gdim(count))), KT<LOGN>, sm, st, kctx(c), ct, s, (u64 *)tmp.p, rows,
                                                                                    count)); }
    LAUNCH_CHECK();
    { PROF("k_decrypt_finish", st, 8.0 * c->n * count * (rows + 1.0)); k_decrypt_finish<<<pw_grid(c->n, count), 256, 0, st>>>(kctx(c), (const u64 *)tmp.p, coeffs, (unsigned long long *)bad,
                                                            rows, count, c->log_n); }
    LAUNCH_CHECK();
    return HEB_OK;
}

extern "C" int heb_decrypt(heb_ctx *c, heb_ct ct, const uint64_t *s_eval, int64_t *coeffs, int64_t *bad,
                           int64_t count, int k, void *stream) {
    if (!c || !s_eval || !coeffs || !bad || k < 1 || k > c->num_rows - 1) return fail(HEB_EINVAL, "heb_decrypt: bad args");
    if (count <= 0) return HEB_OK;
    DISPATCH_LOGN(c, launch_decrypt, c, ct, s_eval, coeffs, bad, count, k, (cudaStream_t)stream);
}

// pk_b = e - a*s   (row r)
template <int LOGN>
__global__ void ROW_BOUNDS(LOGN) k_make_pk(Ctx K, const u64 *s, const u64 *a, const i64 *e,
                                                                   u64 *pkb) {
    extern __shared__ u64 sm[];
    const int r = lbx<LOGN>();
    const PrimeInfo P = K.pi[r];
    const int pos = tpos<LOGN>();
    u64 E[16], x[16], y[16];
    fwd_any<LOGN>(K, r, P, sm,
                       [&](int i) { return signed_mul_const(__ldcg(e + i), P.rmod, P.rmod_s, P.p); }, E);
    const size_t off = ((size_t)r << LOGN) + pos;
    load16<LOGN>(a + off, x);
    load16<LOGN>(s + off, y);
#pragma unroll
    for (int m = 0; m < 16; ++m) E[m] = sub_mod(E[m], mont_mul(x[m], y[m], P.p, P.pinv), P.p);
    store16<LOGN>(pkb + off, E);
}

// kb[j][r] = e_j - a_j,r s_r  (+ (P mod q_j) R * target_j on r == j, applied with mont_mul)
template <int LOGN>
__global__ void ROW_BOUNDS(LOGN) k_make_swk(Ctx K, const u64 *s, const u64 *target,
                                                                    const u64 *a, const i64 *e, u64 *kb) {
    extern __shared__ u64 sm[];
    const int r = lbx<LOGN>(), j = blockIdx.y;
    const int R = K.num_rows;
    const PrimeInfo P = K.pi[r];
    const int pos = tpos<LOGN>();
    const i64 *ej = e + ((size_t)j << LOGN);
    u64 E[16], x[16], y[16];
    fwd_any<LOGN>(K, r, P, sm,
                       [&](int i) { return signed_mul_const(__ldcg(ej + i), P.rmod, P.rmod_s, P.p); }, E);
    const size_t off = (((size_t)j * R + r) << LOGN) + pos;
    load16<LOGN>(a + off, x);
    load16<LOGN>(s + ((size_t)r << LOGN) + pos, y);
#pragma unroll
    for (int m = 0; m < 16; ++m) E[m] = sub_mod(E[m], mont_mul(x[m], y[m], P.p, P.pinv), P.p);
    if (r == j) {
        // factor = (P mod q_j) * R mod q_j (Montgomery); mont_mul(target, factor) = target * P
        const LevelConst C = K.lc[(size_t)(R - 2) * R + j];  // P mod q_j
        load16<LOGN>(target + ((size_t)r << LOGN) + pos, x);
#pragma unroll
        for (int m = 0; m < 16; ++m) E[m] = add_mod(E[m], shoup(x[m], C.pmod.x, C.pmod.y, P.p), P.p);
    }
    store16<LOGN>(kb + off, E);
}

template <int LOGN>
static int launch_pk(heb_ctx *c, const u64 *s, const u64 *a, const i64 *e, u64 *pkb, int rows, cudaStream_t st) {
    constexpr size_t sm = smem_bytes<LOGN>();
    CUDA_TRY(prep_kernel(k_make_pk<LOGN>, sm));
    { PROF("k_make_pk", st, 8.0 * c->n * (1.0 + 3.0 * rows)); CUDA_TRY(launch_rows<LOGN>(k_make_pk<LOGN>, dim3(rows), KT<LOGN>, sm, st, kctx(c), s, a, e, pkb)); }
    LAUNCH_CHECK();
    return HEB_OK;
}
template <int LOGN>
static int launch_swk(heb_ctx *c, const u64 *s, const u64 *t, const u64 *a, const i64 *e, u64 *kb, int digits,
                      cudaStream_t st) {
    constexpr size_t sm = smem_bytes<LOGN>();
    CUDA_TRY(prep_kernel(k_make_swk<LOGN>, sm));
    { PROF("k_make_swk", st, 8.0 * c->n * (digits + 4.0 * digits * c->num_rows)); CUDA_TRY(launch_rows<LOGN>(k_make_swk<LOGN>, dim3(dim3(c->num_rows, digits)), KT<LOGN>, sm, st, kctx(c), s, t, a, e, kb)); }
    LAUNCH_CHECK();
    return HEB_OK;
}

extern "C" int heb_make_public_key(heb_ctx *c, const uint64_t *s, const uint64_t *a, const int64_t *e, uint64_t *pkb,
                                   int rows, void *stream) {
    if (!c || !s || !a || !e || !pkb || rows < 1 || rows > c->num_rows) return fail(HEB_EINVAL, "heb_make_public_key: bad args");
    DISPATCH_LOGN(c, launch_pk, c, s, a, e, pkb, rows, (cudaStream_t)stream);
}
extern "C" int heb_make_switch_key(heb_ctx *c, const uint64_t *s, const uint64_t *target, const uint64_t *a,
                                   const int64_t *e, uint64_t *kb, int digits, void *stream) {
    if (!c || !s || !target || !a || !e || !kb || digits < 1 || digits > c->num_rows - 1)
        return fail(HEB_EINVAL, "heb_make_switch_key: bad args");
    DISPATCH_LOGN(c, launch_swk, c, s, target, a, e, kb, digits, (cudaStream_t)stream);
}

