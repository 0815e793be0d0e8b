// layers.cu -- encrypted-CNN layer entry points of the C ABI.
//
// Each entry point evaluates one whole layer of the reference's layer API
// (/root/reference/pkg/src/hecnn/layers.py:92-294) over every independent ciphertext of
// the layer: the tensor / gather kernels of conv.cu and pointwise.cu, then one batched
// key switch + rescale (keyswitch.cu), with the raw degree-2 intermediates in the
// stream's scratch arena.  The host keeps the level / exact-scale / noise ledger
// (layers.py in this package); these calls only move residues.
#include "common.cuh"

extern "C" int heb_conv_tensor(heb_ctx *, heb_ct, heb_ct, heb_ct, int, int, int, int, int, int, int, int, void *);
extern "C" int heb_dot_tensor(heb_ctx *, heb_ct, heb_ct, const int32_t *, const int32_t *, int, heb_ct, int64_t,
                              int, void *);
extern "C" int heb_relin_rescale(heb_ctx *, heb_ct, const uint64_t *, heb_ct, int64_t, int, void *);
extern "C" int heb_tensor(heb_ctx *, heb_ct, heb_ct, heb_ct, int64_t, int, int, void *);
extern "C" int heb_rescale(heb_ctx *, heb_ct, const uint64_t *, int64_t, heb_ct, int64_t, int, int, void *);
extern "C" int heb_add(heb_ctx *, heb_ct, heb_ct, heb_ct, int64_t, int, int, void *);
extern "C" int heb_add_plain(heb_ctx *, heb_ct, const uint64_t *, int64_t, heb_ct, int64_t, int, void *);

int conv_tensor_max_taps();  // conv.cu

#define HEB_TRY(expr)                 \
    do {                              \
        const int _s = (expr);        \
        if (_s != HEB_OK) return _s;  \
    } while (0)

static inline heb_ct compact(void *p, int comps, int k, int n) {
    return heb_ct{(u64 *)p, (int64_t)comps * k * n, (int64_t)k * n};
}

// conv windows as (input item, weight item) index lists, for layers whose taps exceed
// the fused kernel's shared-memory stage: o = (f, i, j), t = (c, p, q)
__global__ void k_conv_index(int32_t *ia, int32_t *ib, int channels, int m, int n, int filters, int kp, int kq,
                             int stride, int om, int on) {
    const int taps = channels * kp * kq;
    const int64_t total = (int64_t)filters * om * on * taps;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
        const int t = (int)(x % taps);
        const int64_t o = x / taps;
        const int j = (int)(o % on), i = (int)((o / on) % om), f = (int)(o / ((int64_t)om * on));
        const int q = t % kq, p = (t / kq) % kp, c = t / (kp * kq);
        ia[x] = c * m * n + (i * stride + p) * n + (j * stride + q);
        ib[x] = ((f * channels + c) * kp + p) * kq + q;
    }
}

// y_item += bias[item / per] over 2 components of k rows (per-filter broadcast bias)
__global__ void k_add_bias(Ctx K, heb_ct y, heb_ct bias, int64_t per, int64_t lines, int k, int logn) {
    const int n = 1 << logn;
    for (int64_t line = blockIdx.y; line < lines; line += gridDim.y) {
        LineIdx L = line_of(line, 2, k);
        const u64 p = K.pi[L.r].p;
        u64 *z = at(y, L.b, L.c, L.r, logn);
        const u64 *b = at(bias, L.b / per, L.c, L.r, logn);
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
            z[i] = add_mod(z[i], b[i], p);
    }
}

// 2x2 sum pool: out (c, i, j) = sum of the window at (2i, 2j) -- every residue add is
// exact mod p, so the sum equals the reference's WINDOW_ORDER chain (layers.py:26,189-204)
// bit for bit.  Two adjacent positions per thread (16-byte accesses).
__global__ void k_sumpool(Ctx K, heb_ct y, heb_ct o, int m, int n, int om, int on, int64_t lines, int k, int logn) {
    const int nn = 1 << logn;
    for (int64_t line = blockIdx.y; line < lines; line += gridDim.y) {
        LineIdx L = line_of(line, 2, k);
        const u64 p = K.pi[L.r].p;
        const int64_t cell = L.b % ((int64_t)om * on), ch = L.b / ((int64_t)om * on);
        const int i = (int)(cell / on), j = (int)(cell % on);
        const int64_t base = ch * m * n + (2 * i) * n + 2 * j;
        const ulonglong2 *w00 = reinterpret_cast<const ulonglong2 *>(at(y, base, L.c, L.r, logn));
        const ulonglong2 *w01 = reinterpret_cast<const ulonglong2 *>(at(y, base + 1, L.c, L.r, logn));
        const ulonglong2 *w10 = reinterpret_cast<const ulonglong2 *>(at(y, base + n, L.c, L.r, logn));
        const ulonglong2 *w11 = reinterpret_cast<const ulonglong2 *>(at(y, base + n + 1, L.c, L.r, logn));
        ulonglong2 *z = reinterpret_cast<ulonglong2 *>(at(o, L.b, L.c, L.r, logn));
        for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < nn / 2; x += gridDim.x * blockDim.x) {
            const ulonglong2 a = __ldcs(w00 + x), b = __ldcs(w01 + x), c = __ldcs(w10 + x), d = __ldcs(w11 + x);
            z[x] = make_ulonglong2(add_mod(add_mod(a.x, b.x, p), add_mod(c.x, d.x, p), p),
                                   add_mod(add_mod(a.y, b.y, p), add_mod(c.y, d.y, p), p));
        }
    }
}

static int add_bias(heb_ctx *c, heb_ct y, heb_ct bias, int64_t count, int64_t per, int k, cudaStream_t st) {
    if (!bias.data || count <= 0) return HEB_OK;
    const int64_t lines = count * 2 * k;
    { PROF("k_add_bias", st, 8.0 * c->n * lines * 2.0 + 16.0 * c->n * k * (count / per)); k_add_bias<<<pw_grid(c->n, lines), 256, 0, st>>>(kctx(c), y, bias, per, lines, k, c->log_n); }
    LAUNCH_CHECK();
    return HEB_OK;
}

// mul_ct_pt (ckks.py:320-331): product with the plaintext rows fused into the rescale
extern "C" int heb_mul_plain_rescale(heb_ctx *c, heb_ct ct, const uint64_t *pt, int64_t pt_stride, heb_ct out,
                                     int64_t count, int level, void *stream) {
    if (!pt) return fail(HEB_EINVAL, "heb_mul_plain_rescale: null plaintext");
    return heb_rescale(c, ct, pt, pt_stride, out, count, 2, level, stream);
}

extern "C" int heb_conv(heb_ctx *c, heb_ct x, heb_ct w, heb_ct bias, heb_ct out, int channels, int m, int n,
                        int filters, int kp, int kq, int stride, int level, const uint64_t *evk, void *stream) {
    if (!c || !evk || channels < 1 || filters < 1 || kp < 1 || kq < 1 || stride < 1 || kp > m || kq > n ||
        level < 1 || level > c->num_rows - 2)
        return fail(HEB_EINVAL, "heb_conv: bad args");
    cudaStream_t st = (cudaStream_t)stream;
    const int k = level + 1, om = (m - kp) / stride + 1, on = (n - kq) / stride + 1, taps = channels * kp * kq;
    const int64_t n_out = (int64_t)filters * om * on;
    Scratch sraw(c, st);
    CUDA_TRY(sraw.get(sizeof(u64) * (size_t)n_out * 3 * k * c->n));
    const heb_ct raw = compact(sraw.p, 3, k, c->n);
    // fused kernel (weights staged in shared memory) unless the taps overflow its stage
    if (taps <= conv_tensor_max_taps()) {
        HEB_TRY(heb_conv_tensor(c, x, w, raw, channels, m, n, filters, kp, kq, stride, k, stream));
    } else {
        Scratch sidx(c, st);
        CUDA_TRY(sidx.get(sizeof(int32_t) * 2 * (size_t)n_out * taps));
        int32_t *ia = (int32_t *)sidx.p, *ib = ia + n_out * taps;
        k_conv_index<<<1184, 256, 0, st>>>(ia, ib, channels, m, n, filters, kp, kq, stride, om, on);
        LAUNCH_CHECK();
        HEB_TRY(heb_dot_tensor(c, x, w, ia, ib, taps, raw, n_out, k, stream));
    }
    HEB_TRY(heb_relin_rescale(c, raw, evk, out, n_out, level, stream));
    return add_bias(c, out, bias, n_out, (int64_t)om * on, k - 1, st);
}

extern "C" int heb_square(heb_ctx *c, heb_ct y, heb_ct out, int64_t count, int level, const uint64_t *evk,
                          void *stream) {
    if (!c || !evk || level < 1 || level > c->num_rows - 2) return fail(HEB_EINVAL, "heb_square: bad args");
    if (count <= 0) return HEB_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int k = level + 1;
    Scratch sraw(c, st);
    CUDA_TRY(sraw.get(sizeof(u64) * (size_t)count * 3 * k * c->n));
    const heb_ct raw = compact(sraw.p, 3, k, c->n);
    HEB_TRY(heb_tensor(c, y, y, raw, count, k, 0, stream));
    return heb_relin_rescale(c, raw, evk, out, count, level, stream);
}

extern "C" int heb_poly_act(heb_ctx *c, heb_ct y, const uint64_t *pt_quad, const uint64_t *pt_lin,
                            const uint64_t *pt_const, heb_ct out, int64_t count, int level, const uint64_t *evk,
                            void *stream) {
    if (!c || !evk || !pt_quad || !pt_lin || !pt_const || level < 2 || level > c->num_rows - 2)
        return fail(HEB_EINVAL, "heb_poly_act: bad args");
    if (count <= 0) return HEB_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int k = level + 1;
    // approx_relu_cell (layers.py:164-186): c2 (y^2) + c1 y + c0, coefficients folded
    // into the three plaintexts; y^2 at level-1, both products rescaled, sum at level-2
    Scratch st_sq(c, st), st_q(c, st), st_l(c, st);
    CUDA_TRY(st_sq.get(sizeof(u64) * (size_t)count * 2 * (k - 1) * c->n));
    CUDA_TRY(st_q.get(sizeof(u64) * (size_t)count * 2 * (k - 2) * c->n));
    CUDA_TRY(st_l.get(sizeof(u64) * (size_t)count * 2 * (k - 1) * c->n));
    const heb_ct sq = compact(st_sq.p, 2, k - 1, c->n), quad = compact(st_q.p, 2, k - 2, c->n),
                 lin = compact(st_l.p, 2, k - 1, c->n);
    HEB_TRY(heb_square(c, y, sq, count, level, evk, stream));
    HEB_TRY(heb_rescale(c, sq, pt_quad, 0, quad, count, 2, level - 1, stream));
    HEB_TRY(heb_rescale(c, y, pt_lin, 0, lin, count, 2, level, stream));
    HEB_TRY(heb_add(c, quad, lin, out, count, 2, k - 2, stream));
    return heb_add_plain(c, out, pt_const, 0, out, count, k - 2, stream);
}

extern "C" int heb_sumpool(heb_ctx *c, heb_ct y, heb_ct out, int channels, int m, int n, int level, void *stream) {
    if (!c || channels < 1 || m < 2 || n < 2 || level < 0 || level > c->num_rows - 2)
        return fail(HEB_EINVAL, "heb_sumpool: bad args");
    cudaStream_t st = (cudaStream_t)stream;
    const int k = level + 1, om = m / 2, on = n / 2;
    const int64_t lines = (int64_t)channels * om * on * 2 * k;
    { PROF("k_sumpool", st, 8.0 * c->n * lines * 5.0); k_sumpool<<<pw_grid(c->n / 2, lines), 256, 0, st>>>(kctx(c), y, out, m, n, om, on, lines, k, c->log_n); }
    LAUNCH_CHECK();
    return HEB_OK;
}

extern "C" int heb_fc(heb_ctx *c, heb_ct x, heb_ct w, const int32_t *x_idx, const int32_t *w_idx, int taps,
                      heb_ct bias, heb_ct out, int64_t n_out, int level, const uint64_t *evk, void *stream) {
    if (!c || !evk || !x_idx || !w_idx || taps < 1 || level < 1 || level > c->num_rows - 2)
        return fail(HEB_EINVAL, "heb_fc: bad args");
    if (n_out <= 0) return HEB_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int k = level + 1;
    Scratch sraw(c, st);
    CUDA_TRY(sraw.get(sizeof(u64) * (size_t)n_out * 3 * k * c->n));
    const heb_ct raw = compact(sraw.p, 3, k, c->n);
    HEB_TRY(heb_dot_tensor(c, x, w, x_idx, w_idx, taps, raw, n_out, k, stream));
    HEB_TRY(heb_relin_rescale(c, raw, evk, out, n_out, level, stream));
    return add_bias(c, out, bias, n_out, 1, k - 1, st);
}
