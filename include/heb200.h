/*
 * heb200.h -- C ABI of the B200 CKKS evaluation engine (libheb200.so).
 *
 * The drop-in boundary for the reference's HE backend plugin
 * (/root/reference/pkg/src/hecnn/backends/base.py:190-602, hooks :554-602).
 * Plain pointers and sizes only; every call returns 0 on success or a
 * negative HEB_E* status, with a message in heb_last_error() (thread-local).
 *
 * Data layout (device memory, u64 words):
 *   a "row" is N residues of one prime; residues are x*2^64 mod p in [0,p)
 *   ("Montgomery form", reference kernels.py:1-13), evaluation (NTT) domain,
 *   position i = a(psi^(2*brv(i)+1)).
 *   A ciphertext batch operand heb_ct points at component 0 / row 0 of item 0;
 *   item b, component c, row r lives at data + b*ct_stride + c*comp_stride + r*N.
 *   Rows are the prefix 0..level of the context's primes (row 0 = base prime).
 *   Raw products (degree 2) use the same descriptor with three components.
 * All work is enqueued on `stream` (a cudaStream_t, may be NULL); temporary
 * device memory comes from a per-stream scratch arena owned by the context (LIFO bump
 * allocation over device blocks that only grow during the first calls of a shape), so
 * independent calls may use independent streams and CUDA-graph replays touch no
 * allocator.  One host thread at a time per stream (a lock per arena serialises).
 */
#ifndef HEB200_H
#define HEB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HEB_OK 0
#define HEB_EINVAL (-1)   /* bad argument (maps to ValueError) */
#define HEB_ECUDA (-2)    /* CUDA runtime/launch failure (DeviceError) */
#define HEB_ENOMEM (-3)   /* device allocation failed (DeviceError) */
#define HEB_EUNSUP (-4)   /* ring degree / shape not supported (ConfigurationError) */

typedef struct heb_ctx heb_ctx;

typedef struct heb_ct {
    uint64_t *data;
    int64_t ct_stride;    /* words between batch items */
    int64_t comp_stride;  /* words between components (c0/c1 or d0/d1/d2) */
} heb_ct;

/* --- library / context ---------------------------------------------------- */
int heb_version(void);
const char *heb_last_error(void);
int heb_device_count(int *count);

/* Build the device tables for one modulus chain.  primes[num_rows] in chain row
 * order (base, levels..., special) -- reference chain.py:26-31; psi[] holds each
 * prime's 2N-th root from find_2n_root (kernels.py:439-446) or NULL to derive it.
 * Replaces the per-backend precomputation in ckks.py:81-93 / chain.py:97-147. */
int heb_ctx_create(heb_ctx **out, int device, int log_n, int num_rows, const uint64_t *primes,
                   const uint64_t *psi);
int heb_ctx_destroy(heb_ctx *ctx);
int heb_ctx_ring_degree(const heb_ctx *ctx);
/* Key-switch / rescale batches are processed in chunks of this many items
 * (default 1024), bounding the scratch arena. */
int heb_ctx_set_chunk(heb_ctx *ctx, int items);
/* Free the scratch arena of `stream` (after synchronising it); the next call on that
 * stream grows a new one.  For one-off evaluations on streams that will not be reused.
 * Refused (HEB_EINVAL) while CUDA graphs captured on `stream` may replay into the arena:
 * destroy them first, then heb_ctx_clear_captured. */
int heb_ctx_release_scratch(heb_ctx *ctx, void *stream);
/* Declare that no CUDA graph captured on `stream` is alive any more. */
int heb_ctx_clear_captured(heb_ctx *ctx, void *stream);

/* --- memory ----------------------------------------------------------------- */
int heb_alloc(size_t bytes, void **out, void *stream);
int heb_free(void *ptr, void *stream);
int heb_h2d(void *dst, const void *src, size_t bytes, void *stream);
int heb_d2h(void *dst, const void *src, size_t bytes, void *stream);
int heb_sync(void *stream);

/* --- transforms (kernels.py:68-114) ------------------------------------------ */
/* In place over `count` blocks of `rows` rows starting at chain row `row0`. */
int heb_ntt_fwd(heb_ctx *ctx, uint64_t *data, int64_t count, int rows, int row0, int64_t block_stride,
                void *stream);
int heb_ntt_inv(heb_ctx *ctx, uint64_t *data, int64_t count, int rows, int row0, int64_t block_stride,
                void *stream);
/* Serialization transforms (ckks.py:393-408), in place over rows 0..rows-1:
 * eval_to_coeff = ntt_inv_rows + from_mont_rows (Montgomery eval rows -> standard-form
 * coefficients, the reference's payload format); coeff_to_eval = to_mont_rows + ntt_fwd_rows. */
int heb_eval_to_coeff(heb_ctx *ctx, uint64_t *data, int64_t count, int rows, int64_t block_stride, void *stream);
int heb_coeff_to_eval(heb_ctx *ctx, uint64_t *data, int64_t count, int rows, int64_t block_stride, void *stream);
/* Centered int64 coefficients (count, N) -> evaluation rows 0..rows-1 (Montgomery).
 * Restates spread_centered + ntt_fwd_rows (ckks.py:120-126); rows = num_rows gives
 * every chain row including the special prime (keygen, ckks.py:128-129). */
int heb_spread_ntt(heb_ctx *ctx, const int64_t *coeffs, int64_t count, uint64_t *out, int rows,
                   int64_t out_stride, void *stream);

/* --- arithmetic (ckks.py:279-387) --------------------------------------------- */
/* out = a + b over `comps` components of k rows (add_ct_ct / raw_add). */
int heb_add(heb_ctx *ctx, heb_ct a, heb_ct b, heb_ct out, int64_t count, int comps, int k, void *stream);
/* out.c0 = ct.c0 + pt (pt: k rows, item stride pt_stride; 0 = broadcast); c1 copied
 * unless out aliases ct (add_ct_pt, ckks.py:295-302). */
int heb_add_plain(heb_ctx *ctx, heb_ct ct, const uint64_t *pt, int64_t pt_stride, heb_ct out, int64_t count,
                  int k, void *stream);
/* raw (d0,d1,d2) (+)= (a0b0, a0b1+a1b0, a1b1)  (ctct_products, kernels.py:230-246). */
int heb_tensor(heb_ctx *ctx, heb_ct a, heb_ct b, heb_ct raw, int64_t count, int k, int accumulate,
               void *stream);
/* Rescale `comps` components at `level` (k = level+1 rows -> k-1): divide_drop_last,
 * kernels.py:270-294.  If pt != NULL each component is first multiplied by the
 * plaintext rows (mul_ct_pt = mul_rows + rescale, ckks.py:320-331). */
int heb_rescale(heb_ctx *ctx, heb_ct in, const uint64_t *pt, int64_t pt_stride, heb_ct out, int64_t count,
                int comps, int level, void *stream);
/* mul_ct_pt (ckks.py:320-331, base.py:427-445): both components times the plaintext
 * rows (pt: level+1 rows, item stride pt_stride; 0 = broadcast), then rescale to
 * level-1.  Same as heb_rescale with pt != NULL and comps = 2. */
int heb_mul_plain_rescale(heb_ctx *ctx, heb_ct ct, const uint64_t *pt, int64_t pt_stride, heb_ct out, int64_t count,
                          int level, void *stream);
/* Prepare a switching key for the device key switch: from the reference layout
 * (EvalKeyPayload b/a arrays, (digits, num_rows, N) Montgomery residues, ckks.py:72-75)
 * to (digits, num_rows, 2, N) pairs (w, floor(w*2^64/p)) with w = residue * R^-1, so
 * each key product is a single Shoup multiplication.  out holds digits*num_rows*4*N words. */
int heb_prepare_switch_key(heb_ctx *ctx, const uint64_t *kb, const uint64_t *ka, int digits, uint64_t *out,
                           void *stream);
/* raw_finalize (ckks.py:359-387): key switch of d2 with the relinearisation key
 * (relin_accumulate + moddown_special), add d0/d1, rescale.  evk = prepared key
 * (heb_prepare_switch_key).  Output level = level-1. */
int heb_relin_rescale(heb_ctx *ctx, heb_ct raw, const uint64_t *evk, heb_ct out, int64_t count, int level,
                      void *stream);
/* Galois automorphism X -> X^galois on both components followed by a key switch
 * with the matching prepared switching key; level kept.  No reference
 * counterpart (rotation is a non-goal there). */
int heb_rotate(heb_ctx *ctx, heb_ct ct, const uint64_t *gk, heb_ct out, int64_t count, int level,
               uint64_t galois, void *stream);
/* Evaluation-domain permutation only (rows 0..rows-1 of `count` blocks). */
int heb_galois(heb_ctx *ctx, const uint64_t *in, uint64_t *out, int64_t count, int rows, int64_t block_stride,
               uint64_t galois, void *stream);
/* out = a (*) b pointwise Montgomery product over `rows` rows (mul_rows). */
int heb_mul_rows(heb_ctx *ctx, const uint64_t *a, const uint64_t *b, uint64_t *out, int rows, void *stream);

/* --- client side (ckks.py:135-273) ------------------------------------------------ */
/* Encrypt `count` messages: c0 = v*pk_b + (e0+m), c1 = v*pk_a + e1 over k rows.
 * v, e0m, e1: int64 coefficient vectors (count, N) sampled on the host. */
int heb_encrypt(heb_ctx *ctx, const int64_t *v, const int64_t *e0m, const int64_t *e1, const uint64_t *pk_b,
                const uint64_t *pk_a, heb_ct out, int64_t count, int k, void *stream);
/* Decrypt to centered int64 coefficients of row 0 with the cross-residue guard
 * (ckks.py:237-269): bad[b] = number of coefficients whose residue mod q_1 differs
 * from row 1 (k >= 2), or of coefficients >= q_0/4 in magnitude (k == 1). */
int heb_decrypt(heb_ctx *ctx, heb_ct ct, const uint64_t *s_eval, int64_t *coeffs, int64_t *bad, int64_t count,
                int k, void *stream);
/* pk_b = e - a*s over `rows` rows (keygen, ckks.py:143-149). */
int heb_make_public_key(heb_ctx *ctx, const uint64_t *s_eval, const uint64_t *a, const int64_t *e,
                        uint64_t *pk_b, int rows, void *stream);
/* Switching key: for digit j < digits, kb[j] = e_j - a_j*s (all rows) and row j gets
 * + (P mod q_j) * target[j] (ckks.py:151-176; target = s^2 for relinearisation,
 * sigma_g(s) for rotation). */
int heb_make_switch_key(heb_ctx *ctx, const uint64_t *s_eval, const uint64_t *target, const uint64_t *a,
                        const int64_t *e, uint64_t *kb, int digits, void *stream);

/* --- batched layer evaluator (layers.py:92-294 fused per layer) --------------------- */
/* For output o < n_out: raw_o = sum_{t<taps} A[a_idx[o*taps+t]] (x) B[b_idx[o*taps+t]]
 * (degree-2 tensor, lazy 128-bit accumulation); index arrays are device int32. */
int heb_dot_tensor(heb_ctx *ctx, heb_ct a, heb_ct b, const int32_t *a_idx, const int32_t *b_idx, int taps,
                   heb_ct raw, int64_t n_out, int k, void *stream);
/* Convolution layer tensor (layers.py:92-127 fused): A holds channels*m*n input cells
 * (item = c*m*n + i*n + j), B the broadcast weights (item = ((f*channels + c)*kp + p)*kq
 * + q); raw output item f*om*on + i*on + j = sum over (c,p,q) of A (x) B for a valid,
 * `stride`d cross-correlation.  Weights are staged in shared memory per position tile. */
int heb_conv_tensor(heb_ctx *ctx, heb_ct a, heb_ct b, heb_ct raw, int channels, int m, int n, int filters, int kp,
                    int kq, int stride, int k, void *stream);
/* out_o = sum_{t<terms} A[idx[o*terms+t]] over `comps` components (pool windows). */
int heb_sum_gather(heb_ctx *ctx, heb_ct a, const int32_t *idx, int terms, heb_ct out, int64_t n_out, int comps,
                   int k, void *stream);
/* out_o = A[idx[o]] (gather copy of k rows x comps). */
int heb_gather(heb_ctx *ctx, heb_ct a, const int32_t *idx, heb_ct out, int64_t n_out, int comps, int k,
               void *stream);

/* --- layer entry points (one call per encrypted-CNN layer, layers.py:92-294) ---------
 * Operands are batches at `level` (k = level+1 rows); outputs are written at the level
 * the reference's layer returns.  Intermediates live in the stream's scratch arena.
 * evk = prepared relinearisation key (heb_prepare_switch_key).  The host keeps the
 * level / scale / noise ledger (base.py:354-502). */
/* conv2d_enc (layers.py:92-127) for every output cell at once: raw = sum over the
 * valid, strided window (heb_conv_tensor; index-driven heb_dot_tensor beyond its
 * shared-memory stage), raw_finalize (relinearise + rescale), then bias[f] (bias.data
 * NULL: none; else `filters` ciphertexts at >= the output level) added to filter f's
 * cells.  out: filters*om*on ciphertexts at level-1, item f*om*on + i*on + j. */
int heb_conv(heb_ctx *ctx, heb_ct x, heb_ct w, heb_ct bias, heb_ct out, int channels, int m, int n, int filters,
             int kp, int kq, int stride, int level, const uint64_t *evk, void *stream);
/* Standalone x^2 activation: mul_ct_ct(y, y) = tensor + raw_finalize (ckks.py:333-387). */
int heb_square(heb_ctx *ctx, heb_ct y, heb_ct out, int64_t count, int level, const uint64_t *evk, void *stream);
/* approx_relu_cell (layers.py:164-186) with the folded-coefficient plaintexts of
 * _act_plaintexts (:139-161): out = (y^2 (*) pt_quad) + (y (*) pt_lin) + pt_const.
 * pt_quad: level rows (k-1), pt_lin: k rows, pt_const: k-2 rows, each broadcast.
 * out at level-2; level >= 2. */
int heb_poly_act(heb_ctx *ctx, heb_ct y, const uint64_t *pt_quad, const uint64_t *pt_lin, const uint64_t *pt_const,
                 heb_ct out, int64_t count, int level, const uint64_t *evk, void *stream);
/* 2x2 sum pool of a channel-major map (channels, m, n) -> (channels, m/2, n/2):
 * mean_pool_2x2's four-way add (layers.py:189-204) without the divisor. */
int heb_sumpool(heb_ctx *ctx, heb_ct y, heb_ct out, int channels, int m, int n, int level, void *stream);
/* dense_enc (layers.py:248-294): out_o = raw_finalize(sum_t X[x_idx[o*taps+t]] (x)
 * W[w_idx[o*taps+t]]) + bias_o (bias.data NULL: none).  out at level-1. */
int heb_fc(heb_ctx *ctx, heb_ct x, heb_ct w, const int32_t *x_idx, const int32_t *w_idx, int taps, heb_ct bias,
           heb_ct out, int64_t n_out, int level, const uint64_t *evk, void *stream);

/* --- multi-GPU: logit gather ------------------------------------------
 * Ranks evaluate independent image batches with replicated keys; the only exchange is
 * an all-gather of the output logit ciphertexts over NCCL (NVLink / NVSwitch).  NCCL is
 * bound at run time (libnccl.so.2, preferring the copy already loaded in the process).
 * Replaces the reference's in-process fork-join combine (executor.py:161-279), which
 * has no network transport. */
typedef struct heb_comm heb_comm;
/* 128-byte NCCL unique id, created on one rank and shared with the others by the host. */
int heb_comm_unique_id(uint8_t *id_out);
int heb_comm_init(heb_comm **out, const uint8_t *id, int nranks, int rank, int device);
int heb_comm_destroy(heb_comm *comm);
/* recv[r*words + i] = rank r's send[i] (ncclAllGather of u64 words on `stream`). */
int heb_gather_logits(heb_comm *comm, const uint64_t *send, uint64_t *recv, int64_t words, void *stream);

/* --- transport (host <-> device wire format) --------------------------------------- */
/* Residue rows bit-packed at bitlen(p_r) bits per residue: a block of rows 0..rows-1
 * takes heb_packed_words(rows) words (row r: ceil(N*bitlen(p_r)/64) words, in order);
 * blocks are contiguous.  No reference counterpart (its payloads are u64 words). */
int64_t heb_packed_words(heb_ctx *ctx, int rows);
int heb_pack_rows(heb_ctx *ctx, const uint64_t *in, int64_t count, int rows, int64_t in_stride, uint64_t *out,
                  void *stream);
int heb_unpack_rows(heb_ctx *ctx, const uint64_t *in, int64_t count, int rows, uint64_t *out, int64_t out_stride,
                    void *stream);

/* --- instrumentation ---------------------------------------------------------------- */
/* Enable (1) / disable (0) per-kernel CUDA-event timing; enabling clears old records. */
int heb_prof_enable(int on);
/* Writes "kernel launches total_ms total_algorithmic_bytes" lines into buf; returns the
 * full text length. */
int heb_prof_summary(char *buf, size_t len);
/* Override the algorithmic byte count recorded for the next profiled launch on this
 * thread (callers that know operand reuse, e.g. convolution windows). */
int heb_prof_next_bytes(double bytes);
/* Shoup 64-bit modmul throughput microbenchmark (blocks*threads*iters*8 modmuls). */
int heb_bench_modmul(int blocks, int threads, int iters, uint64_t p, double *ms_out, void *stream);
/* NTT butterfly throughput microbenchmark, registers only (blocks*threads*iters*128 butterflies):
 * kind 1 = FP64 engine (p < 2^42), kind 2 = integer Shoup engine.  The measured ceilings of
 * the transform kernels' compute roofline (bench.py `butterfly_roofline`). */
int heb_bench_butterfly(int kind, int blocks, int threads, int iters, uint64_t p, double *ms_out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* HEB200_H */
