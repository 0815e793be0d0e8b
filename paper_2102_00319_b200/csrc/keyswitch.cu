// keyswitch.cu -- rescale, relinearisation (key switch + ModDown + rescale) and rotation.
#include <type_traits>

#include "common.cuh"

// =============================================================================
// rescale (divide_drop_last, kernels.py:270-294), optionally fused with ct x pt
//   head: v = center(INTT_L(c_L [* pt_L]))                      (1 INTT / component)
//   tail: out_i = c_i [* pt_i] * qL^-1 - NTT_i(v * qL^-1 * R)  (k-1 NTTs / component)
// =============================================================================
template <int LOGN, int ENG>
__global__ void ROW_BOUNDS(LOGN) k_rescale_head(Ctx K, heb_ct in, const u64 *pt,
                                                                        int64_t pstride, i64 *V, int comps, int L,
                                                                        int64_t count) {
    extern __shared__ u64 sm[];
    const int c = lbx<LOGN>();
    const PrimeInfo P = K.pi[L];
    const LastConst lc = K.last[L];
    for (int64_t b = blockIdx.y; b < count; b += gridDim.y) {
        u64 x[16];
        load16<LOGN>(at(in, b, c, L, LOGN) + tpos<LOGN>(), x);
        if (pt) {
            u64 y[16];
            load16<LOGN>(pt + b * pstride + ((int64_t)L << LOGN) + tpos<LOGN>(), y);
#pragma unroll
            for (int m = 0; m < 16; ++m) x[m] = mont_mul(x[m], y[m], P.p, P.pinv);
        }
        i64 *dst = V + (b * comps + c) * (1 << LOGN);
        inv_any<LOGN, 16, ENG>(K, L, P, sm, x, [&](int i, u64 v) { dst[i] = center(v, P.p); }, true);
    }
}

template <int LOGN, int ENG>
__global__ void ROW_BOUNDS(LOGN) k_rescale_tail(Ctx K, heb_ct in, const u64 *pt,
                                                                        int64_t pstride, const i64 *V, heb_ct out,
                                                                        int comps, int L, int64_t count, int r0) {
    extern __shared__ u64 sm[];
    const int i = r0 + lbx<LOGN>(), c = blockIdx.z;
    const PrimeInfo P = K.pi[i];
    const LevelConst C = K.lc[(size_t)L * K.num_rows + i];
    for (int64_t b = blockIdx.y; b < count; b += gridDim.y) {
        const i64 *src = V + (b * comps + c) * (1 << LOGN);
        u64 y[16];
        fwd_any<LOGN, 16, ENG>(K, i, P, sm,
                           [&](int j) { return signed_mul_const(__ldcg(src + j), C.beta_r.x, C.beta_r.y, P.p); }, y);
        u64 x[16];
        load16<LOGN>(at(in, b, c, i, LOGN) + tpos<LOGN>(), x);
        if (pt) {
            u64 z[16];
            load16<LOGN>(pt + b * pstride + ((int64_t)i << LOGN) + tpos<LOGN>(), z);
#pragma unroll
            for (int m = 0; m < 16; ++m) x[m] = mont_mul(x[m], z[m], P.p, P.pinv);
        }
#pragma unroll
        for (int m = 0; m < 16; ++m) x[m] = sub_mod(shoup(x[m], C.beta.x, C.beta.y, P.p), y[m], P.p);
        store16<LOGN>(at(out, b, c, i, LOGN) + tpos<LOGN>(), x);
    }
}

template <int LOGN>
static int launch_rescale(heb_ctx *c, heb_ct in, const u64 *pt, int64_t pstride, heb_ct out, int64_t count, int comps,
                          int level, cudaStream_t st) {
    constexpr int T = KT<LOGN>;
    constexpr size_t sm = smem_bytes<LOGN>();
    PREP_ENGINES(k_rescale_head, sm);
    PREP_ENGINES(k_rescale_tail, sm);
    const int64_t chunk = c->chunk > 0 ? c->chunk * 4 : count;
    Scratch V(c, st);
    CUDA_TRY(V.get(sizeof(i64) * (size_t)std::min<int64_t>(count, chunk) * comps * c->n));
    for (int64_t b0 = 0; b0 < count; b0 += chunk) {
        const int64_t cnt = std::min<int64_t>(chunk, count - b0);
        heb_ct ib = in, ob = out;
        ib.data += b0 * in.ct_stride;
        ob.data += b0 * out.ct_stride;
        const u64 *pb = pt ? pt + b0 * pstride : nullptr;
        { PROF("k_rescale_head", st, 8.0 * c->n * (2.0 * cnt * comps + (pt ? (pstride ? cnt : 1) : 0))); CUDA_TRY(launch_rows<LOGN>(c->row_fp[level] ? k_rescale_head<LOGN, 1> : k_rescale_head<LOGN, 2>, dim3(dim3(comps, gdim(cnt))), KT<LOGN>, sm, st, kctx(c), ib, pb, pstride, (i64 *)V.p, comps,
                                                                     level, cnt)); }
        LAUNCH_CHECK();
        { PROF("k_rescale_tail", st, 8.0 * c->n * (cnt * comps * (1.0 + 2.0 * level) + (pt ? level * (pstride ? cnt : 1) : 0))); CUDA_TRY(launch_by_engine<LOGN>(c, ENGINE_KERNELS(k_rescale_tail), 0, level, gdim(cnt), comps, sm, st, kctx(c), ib, pb, pstride,
                                                                            (const i64 *)V.p, ob, comps, level, cnt)); }
        LAUNCH_CHECK();
    }
    return HEB_OK;
}

extern "C" int heb_rescale(heb_ctx *c, heb_ct in, const uint64_t *pt, int64_t pstride, heb_ct out, int64_t count,
                           int comps, int level, void *stream) {
    if (!c || level < 1 || level > c->num_rows - 2 || comps < 1) return fail(HEB_EINVAL, "heb_rescale: bad level %d", level);
    if (count <= 0) return HEB_OK;
    if (out.data == in.data) return fail(HEB_EINVAL, "heb_rescale: output must not alias input");
    DISPATCH_LOGN(c, launch_rescale, c, in, pt, pstride, out, count, comps, level, (cudaStream_t)stream);
}

// =============================================================================
// key switching (relin_accumulate + moddown_special, kernels.py:297-371) and the
// fused ModDown + rescale of raw_finalize (ckks.py:359-387).
//   head : D_j = center(INTT_j(d2_j))                                     k INTT
//   modup: acc_t = sum_j NTT_t(D_j mod p_t) (*) key[j][t]  (t<k and P)      k^2 NTT
//   ModDown+rescale per component c (q_L = row k-1, P = special):
//     aP = center(INTT_P(acc_P));  bL = INTT_L(acc_L + P d_L)              2 INTT
//     sL = (bL - aP) P^-1 mod q_L ; cL = center(sL)
//     out_i = acc_i P^-1 qL^-1 + d_i qL^-1 - NTT_i(aP P^-1 qL^-1 R + cL qL^-1 R)
//                                                                       k-1 NTT
// which equals moddown -> add d -> divide_drop_last of the reference exactly,
// since every step is an identity mod q_i.
// =============================================================================
// Digit layout.  For rows split over a 2-CTA cluster the digits D_j are stored with the
// even positions first, then the odd ones (MODUP_EO): each CTA of the fused ModUp then
// owns one contiguous half (one parity class, ntt::forward_split_eo), stages it into
// shared memory with cp.async while the previous digit's key products run, and the
// digit is read once per (item, target) instead of twice.
#ifndef MODUP_EO
#define MODUP_EO 1
#endif
template <int LOGN>
constexpr bool DIGITS_EO = Row<LOGN>::SP == 2 && MODUP_EO;
template <int LOGN>
__device__ __forceinline__ int digit_index(int i) {
    if constexpr (DIGITS_EO<LOGN>) return ((i & 1) << (LOGN - 1)) | (i >> 1);
    else return i;
}

template <int LOGN, int ENG>
__global__ void ROW_BOUNDS(LOGN) k_ks_head(Ctx K, heb_ct src, int comp, i64 *D, int k,
                                                                   int64_t count, int r0) {
    extern __shared__ u64 sm[];
    const int j = r0 + lbx<LOGN>();
    const PrimeInfo P = K.pi[j];
    const LastConst lc = K.last[j];
    for (int64_t b = blockIdx.y; b < count; b += gridDim.y) {
        u64 x[16];
        load16<LOGN>(at(src, b, comp, j, LOGN) + tpos<LOGN>(), x);
        i64 *dst = D + (b * k + j) * (1 << LOGN);
        inv_any<LOGN, 16, ENG>(K, j, P, sm, x, [&](int i, u64 v) {
            NTT_ASSERT(i >= 0 && i < (1 << LOGN) && b < count && j < k);
            // digits of FP64-engine primes (< 2^42) are stored as the double of the centred
            // value (exact): the FP64 ModUp targets transform them as they are (DigitLoad)
            dst[digit_index<LOGN>(i)] =
                P.use_fp ? (i64)__double_as_longlong(ntt::u2d(v) - (v > (P.p >> 1) ? P.pd : 0.0)) : center(v, P.p);
        }, true);
    }
}

// acc layout: (count, 2, k+1, N); row k is the special prime.
// key: prepared switching key (heb_prepare_switch_key): for digit j, chain row r the
// ulonglong2 pairs (w, floor(w 2^64 / p)) of the b part (N entries) then the a part,
// with w the key residue in standard form, so dig * key is one Shoup product that
// keeps dig's Montgomery factor (identical to the reference's mont_mul(dig, evk)).
//
// ModUp is split in two launches so that the transform kernel carries no
// accumulators (full register budget, two CTAs per SM, independent phases):
//   k_ks_modup_ntt : one CTA per (item, digit j, target t != j):
//                    V[item][t][j] = NTT_t(D_j mod p_t * R)        (k^2 NTTs/item)
//   k_ks_modup_mac : pointwise, acc_t = sum_j v_j (*) key[j][t] with v_t = d2_t
//                    (the centred digit is congruent to d2_t mod its own prime).
// V layout: (count, k+1, k, N); slot (t, t) is unused.
// ModUp input: digit D_j (centred mod q_j, int64) as a canonical residue mod p_t.  The
// reference converts it to Montgomery form first (to_mont, kernels.py:297-340); here the
// factor R lives in the prepared key instead (k_prep_key), and NTT_t is linear, so the
// key products are the same residues.  When q_j / 2 < p_t the centred digit already lies
// in (-p_t, p_t) and needs only a sign fix -- every digit except a wide base digit
// entering a 40-bit target.
template <int LOGN>
struct DigitLoad {
    const i64 *d;
    u64 p, r1s;
    bool small, dbl;  // dbl: the digit's words are doubles (its prime runs on the FP64 engine, see k_ks_head)
    __device__ __forceinline__ DigitLoad(const i64 *d_, const PrimeInfo &P, const PrimeInfo &Pj)
        : d(d_), p(P.p), r1s(P.r1s), small((Pj.p >> 1) < P.p), dbl(Pj.use_fp != 0) {}
    // stored word -> canonical residue mod p
    __device__ __forceinline__ u64 conv(i64 v) const {
        if (dbl) {  // exact integer |x| < 2^41: x + 1.5 * 2^52 keeps 2^51 + x in the mantissa field
            const long long b = __double_as_longlong(__longlong_as_double(v) + FP_MAGIC);
            v = (b & ((1ll << 52) - 1)) - (1ll << 51);
        }
        if (small) return (u64)v + (v < 0 ? p : 0);
        return signed_mul_const(v, 1, r1s, p);
    }
    // by position (the parity-split layout is walked through digit_index: only the
    // fallback paths load by position there)
    __device__ __forceinline__ u64 operator()(int i) const { return conv(__ldcg(d + digit_index<LOGN>(i))); }
};

template <int LOGN>
__global__ void ROW_BOUNDS(LOGN)
    k_ks_modup_ntt(Ctx K, const i64 *D, int k, u64 *V, int64_t count) {
    extern __shared__ u64 sm[];
    // blockIdx.x enumerates the k^2 (t, j) pairs with j != t: k-1 digits for each
    // ciphertext target t < k, then all k digits for the special prime (t = k).
    // Targets 0 (base prime) and k (special prime) are the wide primes that run on
    // the integer engine; their 2k-1 pairs are spread evenly through the launch order
    // so that co-resident CTAs keep both the IMAD and the DFMA pipes busy.
    const int xi = lbx<LOGN>();
    const int total = k * k, nwide = 2 * k - 1;
    const int wide_before = (int)(((long)xi * nwide) / total);
    const bool is_wide = ((long)(xi + 1) * nwide) / total != wide_before;
    int t, j;
    if (is_wide) {  // wide pair #wide_before: t = 0 (j = 1..k-1) then t = k (j = 0..k-1)
        const int w = wide_before;
        if (w < k - 1) {
            t = 0;
            j = w + 1;
        } else {
            t = k;
            j = w - (k - 1);
        }
    } else {  // narrow pair #(xi - wide_before): t = 1..k-1, j != t
        const int q = xi - wide_before;
        t = 1 + q / (k - 1);
        j = q % (k - 1);
        j += (j >= t);
    }
    const int gt = t < k ? t : K.num_rows - 1;
    const PrimeInfo P = K.pi[gt];
    const int n = 1 << LOGN;
    for (int64_t b = blockIdx.y; b < count; b += gridDim.y) {
        const i64 *dj = D + (b * k + j) * n;
        u64 y[16];
        DigitLoad<LOGN> ld(dj, P, K.pi[j]);
        fwd_any<LOGN>(K, gt, P, sm, ld, y);
        store16<LOGN>(V + ((b * (k + 1) + t) * k + j) * n + tpos<LOGN>(), y);
    }
}

// ---------------------------------------------------------------------------------
// Fused ModUp with the accumulators in tensor memory (TMEM).
// One CTA per (item, target t): for every digit j it forms v_j = NTT_t(D_j mod p_t R)
// (v_t = d2_t needs no transform) and accumulates v_j (*) key_b[j][t] and
// v_j (*) key_a[j][t] for its 16 positions per thread.  The two accumulators (32 words
// per position pair... 64 32-bit columns per thread) live in TMEM: 256 columns per CTA,
// warp w owns lane quadrant w % 4 and column group w / 4, so two CTAs (1024 threads)
// fit one SM's 512 columns and the NTT keeps its full register budget.  No ModUp
// intermediate ever reaches HBM and the separate MAC pass disappears.
// Column map per thread: component c, position m -> columns 32 c + 2 m (+1): the 64-bit
// accumulator (FP64 rows: an exact double sum; integer rows: a u64 in [0, 2p)).
__device__ __forceinline__ void tmem_st8(uint32_t a, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t a, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(a)
                 : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// key rows are streamed once per CTA: keep them out of L1 (the transform's twiddles live there)
__device__ __forceinline__ double2 ld_key(const double2 *p) {
    double2 v;
    asm("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ ulonglong2 ld_key(const ulonglong2 *p) {
    ulonglong2 v;
    asm("ld.global.nc.L1::no_allocate.v2.u64 {%0,%1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p));
    return v;
}

// accumulate y (*) key over this thread's 16 line-pair positions, 4 positions per TMEM access
// (RAW: FP64 rows hand y over as raw double bit patterns, FpArithRaw).  The tcgen05 asm
// statements are compiler barriers for memory operations, so the key values of the next
// (q, c) step are loaded explicitly before the current step's TMEM round trip
// (MODUP_KEY_AHEAD steps ahead): their L2 latency then overlaps the products instead of
// adding up over the 8 steps.
#ifndef MODUP_KEY_AHEAD
#define MODUP_KEY_AHEAD 1
#endif
#ifndef MODUP_KEY_AHEAD_INT
#define MODUP_KEY_AHEAD_INT 0  // 64 bytes of key per step: more spills than the load-ahead saves
#endif
template <bool FP>
struct ModupKey {
    using KV = typename std::conditional<FP, double2, ulonglong2>::type;
    static constexpr int NK = FP ? 2 : 4;  // 16-byte key words per step (two position pairs)
};
// key words of accumulation step `it` (q = it >> 1: position pairs 2q, 2q + 1; c = it & 1)
template <int LOGN, bool FP>
__device__ __forceinline__ void modup_key_step(const ulonglong2 *keyrow, int pos, int it,
                                               typename ModupKey<FP>::KV (&kv)[ModupKey<FP>::NK]) {
    const int n = 1 << LOGN;
    constexpr int T = KT<LOGN>;
    const int q = it >> 1, c = it & 1;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int off = pos + 2 * T * (2 * q + h);
        if constexpr (FP) {
            const double *kd = reinterpret_cast<const double *>(keyrow) + (size_t)c * n;
            kv[h] = ld_key(reinterpret_cast<const double2 *>(kd + off));
        } else {
            const ulonglong2 *kp = keyrow + (size_t)c * n + off;
            kv[2 * h] = ld_key(kp);
            kv[2 * h + 1] = ld_key(kp + 1);
        }
    }
}
// PRE: the key words of step 0 were loaded by the caller (`pre`), e.g. before a barrier wait
template <int LOGN, bool FP, bool RAW = false, bool PRE = false>
__device__ __forceinline__ void modup_acc(uint32_t ta, const u64 (&y)[16], const ulonglong2 *keyrow, int pos,
                                          bool first, const PrimeInfo &P,
                                          const typename ModupKey<FP>::KV (&pre)[ModupKey<FP>::NK]) {
    const int n = 1 << LOGN;
    constexpr int T = KT<LOGN>;
    using KV = typename ModupKey<FP>::KV;
    constexpr int NK = ModupKey<FP>::NK;
    auto load_step = [&](int it, KV (&kv)[NK]) {
        if (PRE && it == 0) {
#pragma unroll
            for (int x = 0; x < NK; ++x) kv[x] = pre[x];
            return;
        }
        const int q = it >> 1, c = it & 1;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int off = pos + 2 * T * (2 * q + h);
            if constexpr (FP) {
                const double *kd = reinterpret_cast<const double *>(keyrow) + (size_t)c * n;
                kv[h] = ld_key(reinterpret_cast<const double2 *>(kd + off));
            } else {
                const ulonglong2 *kp = keyrow + (size_t)c * n + off;
                kv[2 * h] = ld_key(kp);
                kv[2 * h + 1] = ld_key(kp + 1);
            }
        }
    };
    // ring of AH + 1 key buffers; every index below is a compile-time constant after unrolling
    constexpr int AH = FP ? MODUP_KEY_AHEAD : MODUP_KEY_AHEAD_INT;
    KV kb[AH + 1][NK];
#pragma unroll
    for (int a = 0; a < AH; ++a) load_step(a, kb[a]);
#pragma unroll
    for (int it = 0; it < 8; ++it) {  // q = it >> 1: positions m = 4q .. 4q+3 = pairs 2q, 2q+1; c = it & 1
        const int q = it >> 1, c = it & 1;
        if (it + AH < 8) load_step(it + AH, kb[(it + AH) % (AH + 1)]);
        KV(&kv)[NK] = kb[it % (AH + 1)];
        uint32_t w[8];
        if (!first) tmem_ld8(ta + 32 * c + 8 * q, w);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int i = 2 * q + h;  // pair index: positions pos + 2T i (+1)
            if constexpr (FP) {
                const double y0 = RAW ? __longlong_as_double((long long)y[2 * i]) : ntt::u2d(y[2 * i]);
                const double y1 = RAW ? __longlong_as_double((long long)y[2 * i + 1]) : ntt::u2d(y[2 * i + 1]);
                double a0 = ntt::fmul(y0, kv[h].x, P.pd, P.pinvd);
                double a1 = ntt::fmul(y1, kv[h].y, P.pd, P.pinvd);
                if (!first) {
                    a0 += __hiloint2double(w[4 * h + 1], w[4 * h]);
                    a1 += __hiloint2double(w[4 * h + 3], w[4 * h + 2]);
                }
                w[4 * h] = __double2loint(a0);
                w[4 * h + 1] = __double2hiint(a0);
                w[4 * h + 2] = __double2loint(a1);
                w[4 * h + 3] = __double2hiint(a1);
            } else {
                u64 a0 = shoup_lazy(y[2 * i], kv[2 * h].x, kv[2 * h].y, P.p);
                u64 a1 = shoup_lazy(y[2 * i + 1], kv[2 * h + 1].x, kv[2 * h + 1].y, P.p);
                if (!first) {
                    a0 = csub(a0 + ((u64)w[4 * h + 1] << 32 | w[4 * h]), 2 * P.p);
                    a1 = csub(a1 + ((u64)w[4 * h + 3] << 32 | w[4 * h + 2]), 2 * P.p);
                }
                w[4 * h] = (uint32_t)a0;
                w[4 * h + 1] = (uint32_t)(a0 >> 32);
                w[4 * h + 2] = (uint32_t)a1;
                w[4 * h + 3] = (uint32_t)(a1 >> 32);
            }
        }
        tmem_st8(ta + 32 * c + 8 * q, w);
    }
    tmem_wait_st();
}

template <int LOGN, bool FP, bool RAW = false>
__device__ __forceinline__ void modup_acc(uint32_t ta, const u64 (&y)[16], const ulonglong2 *keyrow, int pos,
                                          bool first, const PrimeInfo &P) {
    typename ModupKey<FP>::KV none[ModupKey<FP>::NK] = {};
    modup_acc<LOGN, FP, RAW, false>(ta, y, keyrow, pos, first, P, none);
}

template <int LOGN, bool FP>
__device__ __forceinline__ void modup_store(uint32_t ta, u64 *o0, u64 *o1, int pos, const PrimeInfo &P) {
    constexpr int T = KT<LOGN>;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            uint32_t w[8];
            tmem_ld8(ta + 32 * c + 8 * q, w);
            u64 *o = c ? o1 : o0;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int i = 2 * q + h;
                u64 r0, r1;
                if constexpr (FP) {
                    r0 = ntt::fcanon(__hiloint2double(w[4 * h + 1], w[4 * h]), P.pd, P.pinvd);
                    r1 = ntt::fcanon(__hiloint2double(w[4 * h + 3], w[4 * h + 2]), P.pd, P.pinvd);
                } else {
                    r0 = csub((u64)w[4 * h + 1] << 32 | w[4 * h], P.p);
                    r1 = csub((u64)w[4 * h + 3] << 32 | w[4 * h + 2], P.p);
                }
                __stcg(reinterpret_cast<ulonglong2 *>(o + pos + 2 * T * i), make_ulonglong2(r0, r1));
            }
        }
    }
}

// Digit staging for the FP64-engine ModUp (MODUP_STAGE): while a digit's key products
// run (TMEM and key loads only), the next digit's row is copied into the transform's
// shared-memory buffer with cp.async, at the padded positions the first transform group
// reads; each thread then converts its own read set in place and the transform starts
// from shared memory.  Hides the digit-load latency behind the products.
#ifndef MODUP_STAGE
#define MODUP_STAGE 1
#endif
#ifndef MODUP_STAGE_INT
#define MODUP_STAGE_INT 1
#endif
template <int LL>
__device__ __forceinline__ void stage_row_async(u64 *sm, const i64 *src) {
    constexpr int N = 1 << LL;
    constexpr int T = ntt::Shape<LL, 16>::T;
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
#pragma unroll 4
    for (int i = threadIdx.x; i < N; i += T)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(base + 8u * (uint32_t)ntt::pad(i)), "l"(src + i)
                     : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
}
// the first forward group's read set of this thread (start at stage 0, shared memory)
template <int LL, class F>
__device__ __forceinline__ void first_group_positions(F f) {
    using S = ntt::Shape<LL, 16>;
    constexpr int RB0 = S::REM ? S::REM : S::LOGE;
    constexpr int LB0 = LL - RB0;
    constexpr int UPT0 = (S::N >> RB0) / S::T;
#pragma unroll
    for (int kk = 0; kk < UPT0; ++kk)
#pragma unroll
        for (int m = 0; m < (1 << RB0); ++m) f((int)threadIdx.x + kk * S::T + (m << LB0));
}

// TMEM columns a CTA of T threads addresses: 64 per group of four warps (one warp per
// lane quadrant), at least 32, a power of two as tcgen05.alloc requires.  Sized to the
// block so that as many CTAs as the NTT launch bounds make resident also fit the SM's
// 512 columns (an over-sized request leaves co-resident CTAs blocked in the alloc).
template <int T>
__host__ __device__ constexpr uint32_t modup_tmem_cols() {
    constexpr uint32_t c = 64u * (uint32_t)((T / 32 + 3) / 4);
    return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512;
}

// ENG: 0 = both engines in one launch, 1 = FP64-engine targets only, 2 = integer targets only
// integer-engine targets (60-bit rows) may trade residency for registers: the Shoup
// butterflies need more than the 64 registers two 512-thread CTAs per SM leave
#ifndef MODUP_INT_MINB
#define MODUP_INT_MINB(LOGN) NTT_MINB(LOGN)
#endif
#ifndef MODUP_FP_MINB
#define MODUP_FP_MINB(LOGN) NTT_MINB(LOGN)
#endif
// L2 prefetch of this CTA's part of key row (j, gt) (b and a parts): the key products of a
// digit follow its transform, so the key is in L2 by then (cfg4: 160 MB of key, larger
// than L2, re-read for every item).
template <int LOGN, bool FP>
__device__ __forceinline__ void prefetch_key(const ulonglong2 *keyrow) {
    constexpr int LL = Row<LOGN>::LL;
    constexpr uint32_t bytes = (1u << LL) * (FP ? 8u : 16u);
    const size_t stride = (size_t)(1 << LOGN) * (FP ? 8 : 16);
    const char *base = FP ? reinterpret_cast<const char *>(reinterpret_cast<const double *>(keyrow) + (rpart<LOGN>() << LL))
                          : reinterpret_cast<const char *>(keyrow + (rpart<LOGN>() << LL));
#pragma unroll
    for (int c = 0; c < 2; ++c)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + c * stride), "r"(bytes) : "memory");
}

// Targets of one fused-ModUp launch (each NTT engine gets its own launch and list).
struct TargetList {
    int n;
    signed char t[60];
};

#ifndef MODUP_STAGE_SPLIT
#define MODUP_STAGE_SPLIT 0
#endif
// parity-split rows: the first accumulation step's key words are loaded right after the
// cross-CTA stage, before the closing cluster-barrier wait and the staging of the next
// digit, so their L2 latency is covered by both (1 = FP64 targets, 2 = integer targets too).
// Measured r2h (cfg4, fused ModUp ms per 4 steps): off 1394, FP64 targets 1408, both 1440 --
// the 8 / 16 registers held across the barrier cost more spills than the latency saves: off.
#ifndef MODUP_KEY_HOOK
#define MODUP_KEY_HOOK 0
#endif
// parity-split rows: cross-CTA stage fed by st.async pushes (ntt::forward_split_eo_push)
// instead of remote loads between two cluster barriers
#ifndef MODUP_PUSH
#define MODUP_PUSH 0
#endif
// dynamic shared memory of the fused ModUp: the transform buffer, plus the receive region
// of the push exchange for parity-split rows
template <int LOGN>
static constexpr size_t modup_smem_bytes() {
    return smem_bytes<LOGN>() +
           (Row<LOGN>::SP == 2 && MODUP_EO && MODUP_PUSH ? sizeof(u64) * ntt::xchg::recv_words<Row<LOGN>::LL, 16>() : 0);
}
#ifndef MODUP_KEY_PREFETCH
#define MODUP_KEY_PREFETCH 0
#endif
#ifndef MODUP_TS_DEFAULT
#define MODUP_TS_DEFAULT 4
#endif
// Launch order: x = target within a set of TS targets, y = item, z = target set.  CTAs are
// dispatched x-fastest, so the resident CTAs work on ONE set of targets over consecutive
// items: the set's key rows (TS k rows of 16 N bytes) stay in L2 and are shared by all
// resident CTAs, while the digits stream through (each item's digits are read by the
// set's TS CTAs at about the same time).  With every target in flight at once (TS >= all
// targets, the old order) the cfg4 key (157 MB at k = 18) cycles through the 126 MB L2
// and every key row comes from HBM (ncu r2b: 136 GB of DRAM reads per 1000-item launch).
template <int LOGN, int ENG>
__global__ void __launch_bounds__(KT<LOGN>, ENG == 2 ? MODUP_INT_MINB(LOGN) : MODUP_FP_MINB(LOGN)) k_ks_modup_fused(Ctx K, heb_ct src, int comp, const i64 *D, const ulonglong2 *key,
                                                  int k, u64 *acc, int64_t count, TargetList tl, int TS) {
    extern __shared__ u64 sm[];
    __shared__ uint32_t tbase;
    // one (item, target) per CTA (pair): the host sizes the grid to cover every item
    const int ti = (int)blockIdx.z * TS + lbx<LOGN>();
    const int64_t b = blockIdx.y;
    if (ti >= tl.n) return;  // last (partial) set; both CTAs of a cluster agree
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&tbase)),
                     "n"(modup_tmem_cols<KT<LOGN>>())
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t ta = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(64 * (warp >> 2));

    const int t = tl.t[ti];
    const int gt = t < k ? t : K.num_rows - 1;
    const PrimeInfo P = K.pi[gt];
    const int n = 1 << LOGN, R = K.num_rows;
    const int pos = tpos<LOGN>();
    constexpr int LL = Row<LOGN>::LL;
    const int hoff = rpart<LOGN>() << LL;  // this CTA's first position (split rows: part r)
    {
        bool first = true;
        int staged_for = -1;  // digit whose row (this CTA's part) sits in shared memory
        constexpr bool EO = DIGITS_EO<LOGN> && ENG != 0;  // parity-split rows, staged digits
        constexpr bool PUSH = EO && MODUP_PUSH;
        int seq = 0;  // exchanges done (push protocol)
        if constexpr (EO || (Row<LOGN>::SPLIT && MODUP_STAGE_SPLIT && ENG != 0)) {
            // split rows only ever transform from staged digits: stage the first one now
            const int j0 = t == 0 ? 1 : 0;
            if (j0 < k) {
                stage_row_async<LL>(sm, D + (b * k + j0) * n + hoff);
                staged_for = j0;
            }
        }
        if constexpr (PUSH) ntt::xchg::init();
        for (int j = 0; j < k; ++j) {
            if (MODUP_KEY_PREFETCH && ENG != 0 && threadIdx.x == 0)
                prefetch_key<LOGN, ENG == 1>(key + (((size_t)j * R + gt) * 2) * n);
            u64 y[16];
            const ulonglong2 *keyrow = key + (((size_t)j * R + gt) * 2) * n;
            constexpr bool HOOK = EO && !PUSH && (ENG == 1 ? MODUP_KEY_HOOK >= 1 : MODUP_KEY_HOOK >= 2);
            typename ModupKey<ENG == 1>::KV pre[ModupKey<ENG == 1>::NK];
            if (j == t) {
                load16<LOGN>(at(src, b, comp, t, LOGN) + pos, y);  // d2_t: congruent digit, no transform
                if constexpr (ENG == 1) {  // canonical residues -> the raw doubles FpArithRaw hands out
#pragma unroll
                    for (int i = 0; i < 16; ++i) y[i] = (u64)__double_as_longlong(ntt::u2d(y[i]));
                }
            } else {
                const i64 *dj = D + (b * k + j) * n;
                DigitLoad<LOGN> ld(dj, P, K.pi[j]);
                if constexpr (ENG == 0) {
                    fwd_any<LOGN>(K, gt, P, sm, ld, y);
                } else {
                    const bool staged = staged_for == j;
                    if constexpr (ENG == 1) {
                        const ntt::FpArithRaw ar(P.pd, P.pinvd);
                        double *s2 = reinterpret_cast<double *>(sm);
                        const double *tw = K.twf + ((size_t)gt << (LOGN + ntt::TW_ROW_SHIFT));
                        if constexpr (EO) {
                            // the first group reads exactly the words this thread staged; a
                            // double-format digit is transformed as it lies in shared memory
                            asm volatile("cp.async.wait_all;" ::: "memory");
                            if (!ld.dbl) {
                                first_group_positions<LL>([&](int i) {
                                    const int q = ntt::pad(i);
                                    s2[q] = ntt::u2d(ld.conv(reinterpret_cast<const i64 *>(sm)[q]));
                                });
                            }
                            if constexpr (PUSH && MODUP_PUSH == 2) ntt::forward_split_eo_bulk<LL, 16>(ar, s2, tw, y, rpart<LOGN>(), seq++);
                            else if constexpr (PUSH) ntt::forward_split_eo_push<LL, 16>(ar, s2, tw, y, rpart<LOGN>(), seq++);
                            else if constexpr (HOOK) ntt::forward_split_eo<LL, 16>(ar, s2, tw, y, rpart<LOGN>(), [&] { modup_key_step<LOGN, true>(keyrow, pos, 0, pre); });
                            else ntt::forward_split_eo<LL, 16>(ar, s2, tw, y, rpart<LOGN>());
                        } else if constexpr (Row<LOGN>::SPLIT) {
                            if constexpr (MODUP_STAGE_SPLIT) ntt::forward_split_staged<LL, 16, Row<LOGN>::SP>(ar, s2, tw, ld, y, rpart<LOGN>());
                            else ntt::forward_split<LL, 16, Row<LOGN>::SP>(ar, s2, tw, ld, y, rpart<LOGN>());
                        } else if (MODUP_STAGE && staged) {
                            asm volatile("cp.async.wait_all;" ::: "memory");
                            __syncthreads();
                            if (!ld.dbl) {
                                first_group_positions<LL>([&](int i) {
                                    const int q = ntt::pad(i);
                                    s2[q] = ntt::u2d(ld.conv(reinterpret_cast<const i64 *>(sm)[q]));
                                });
                            }
                            ntt::forward_core<LL, 16, true>(ar, s2, tw, 1, ld, y);
                        } else {
                            ntt::forward<LL, 16>(ar, s2, tw, ld, y);
                        }
                    } else {
                        const ntt::IntArith ar(P.p);
                        const ulonglong2 *tw = K.tw + ((size_t)gt << (LOGN + ntt::TW_ROW_SHIFT));
                        if constexpr (EO) {
                            asm volatile("cp.async.wait_all;" ::: "memory");
                            first_group_positions<LL>([&](int i) {
                                const int q = ntt::pad(i);
                                sm[q] = ld.conv(reinterpret_cast<const i64 *>(sm)[q]);
                            });
                            if constexpr (PUSH && MODUP_PUSH == 2) ntt::forward_split_eo_bulk<LL, 16>(ar, sm, tw, y, rpart<LOGN>(), seq++);
                            else if constexpr (PUSH) ntt::forward_split_eo_push<LL, 16>(ar, sm, tw, y, rpart<LOGN>(), seq++);
                            else if constexpr (HOOK) ntt::forward_split_eo<LL, 16>(ar, sm, tw, y, rpart<LOGN>(), [&] { modup_key_step<LOGN, false>(keyrow, pos, 0, pre); });
                            else ntt::forward_split_eo<LL, 16>(ar, sm, tw, y, rpart<LOGN>());
                        } else if constexpr (Row<LOGN>::SPLIT) {
                            if constexpr (MODUP_STAGE_SPLIT) ntt::forward_split_staged<LL, 16, Row<LOGN>::SP>(ar, sm, tw, ld, y, rpart<LOGN>());
                            else ntt::forward_split<LL, 16, Row<LOGN>::SP>(ar, sm, tw, ld, y, rpart<LOGN>());
                        } else if (MODUP_STAGE_INT && staged) {
                            asm volatile("cp.async.wait_all;" ::: "memory");
                            __syncthreads();
                            first_group_positions<LL>([&](int i) {
                                const int q = ntt::pad(i);
                                sm[q] = ld.conv(reinterpret_cast<const i64 *>(sm)[q]);
                            });
                            ntt::forward_core<LL, 16, true>(ar, sm, tw, 1, ld, y);
                        } else {
                            ntt::forward<LL, 16>(ar, sm, tw, ld, y);
                        }
                    }
                    // stage the next digit's row (this CTA's part) during the key products
                    constexpr bool stage_on = EO || (Row<LOGN>::SPLIT ? MODUP_STAGE_SPLIT : (ENG == 1 ? MODUP_STAGE : MODUP_STAGE_INT));
                    if constexpr (stage_on) {
                        int jn = j + 1;
                        if (jn == t) ++jn;
                        if (jn < k) {
                            // every thread has read the transform's output (parity-split
                            // rows: forward_split_eo ended with a cluster barrier)
                            if constexpr (!EO) __syncthreads();
                            stage_row_async<LL>(sm, D + (b * k + jn) * n + hoff);
                            staged_for = jn;
                        }
                    }
                }
            }
            if constexpr (HOOK) {
                if (j != t) modup_acc<LOGN, ENG == 1, ENG == 1, true>(ta, y, keyrow, pos, first, P, pre);
                else modup_acc<LOGN, ENG == 1, ENG == 1>(ta, y, keyrow, pos, first, P);
            } else if (ENG == 1)
                modup_acc<LOGN, true, true>(ta, y, keyrow, pos, first, P);
            else if (ENG == 0 && HEB_FPSEL(P.use_fp))
                modup_acc<LOGN, true>(ta, y, keyrow, pos, first, P);
            else
                modup_acc<LOGN, false>(ta, y, keyrow, pos, first, P);
            first = false;
        }
        u64 *o0 = acc + ((b * 2 + 0) * (k + 1) + t) * n;
        u64 *o1 = acc + ((b * 2 + 1) * (k + 1) + t) * n;
        if (ENG == 1 || (ENG == 0 && HEB_FPSEL(P.use_fp)))
            modup_store<LOGN, true>(ta, o0, o1, pos, P);
        else
            modup_store<LOGN, false>(ta, o0, o1, pos, P);
        if constexpr (PUSH) ntt::xchg::fini();
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(modup_tmem_cols<KT<LOGN>>())
                     : "memory");
}

// acc[item][c][t][x] = sum_j v_j[x] * key_c[j][gt][x]  (Shoup with the prepared key)
// Each thread owns two adjacent positions (16-byte accesses) and issues the loads of
// MJ digits before using them, so every thread keeps MJ HBM reads in flight -- the
// kernel is a stream over V and needs that memory-level parallelism.
#ifndef MAC_MJ
#define MAC_MJ 2
#endif
#ifndef MAC_MINB
#define MAC_MINB 6
#endif
template <bool FP>
__global__ void __launch_bounds__(256, MAC_MINB) k_ks_modup_mac(Ctx K, heb_ct src, int comp, const u64 *V, const ulonglong2 *key, int k, u64 *acc,
                               int64_t count, int logn) {
    const int n = 1 << logn;
    const int x = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
    const int t = blockIdx.y;
    const int gt = t < k ? t : K.num_rows - 1;
    const PrimeInfo P = K.pi[gt];
    const u64 p2 = 2 * P.p;
    if (x >= n || P.use_fp != FP) return;  // launched once per engine; rows of the other engine exit
    for (int64_t b = blockIdx.z; b < count; b += gridDim.z) {
        const u64 *vrow = V + ((b * (k + 1) + t) * k) * n + x;
        const u64 *own = at(src, b, comp, t < k ? t : 0, logn) + x;
        u64 *o0 = acc + ((b * 2 + 0) * (k + 1) + t) * n + x;
        u64 *o1 = acc + ((b * 2 + 1) * (k + 1) + t) * n + x;
        if constexpr (FP) {
            // FP64 rows: the prepared key holds w as doubles (b part then a part);
            // exact FP64 modular products, sums stay exact below 2^47
            double s0x = 0.0, s0y = 0.0, s1x = 0.0, s1y = 0.0;
            for (int j0 = 0; j0 < k; j0 += MAC_MJ) {
                ulonglong2 v[MAC_MJ];
                double2 kb[MAC_MJ], ka[MAC_MJ];
#pragma unroll
                for (int u = 0; u < MAC_MJ; ++u) {
                    const int j = j0 + u;
                    if (j < k) {
                        const u64 *vp = (j == t) ? own : vrow + (size_t)j * n;
                        v[u] = __ldcg(reinterpret_cast<const ulonglong2 *>(vp));
                        const double *kd = reinterpret_cast<const double *>(key + (((size_t)j * K.num_rows + gt) * 2) * n);
                        kb[u] = __ldg(reinterpret_cast<const double2 *>(kd + x));
                        ka[u] = __ldg(reinterpret_cast<const double2 *>(kd + n + x));
                    }
                }
#pragma unroll
                for (int u = 0; u < MAC_MJ; ++u) {
                    if (j0 + u < k) {
                        const double vx = ntt::u2d(v[u].x), vy = ntt::u2d(v[u].y);
                        s0x += ntt::fmul(vx, kb[u].x, P.pd, P.pinvd);
                        s0y += ntt::fmul(vy, kb[u].y, P.pd, P.pinvd);
                        s1x += ntt::fmul(vx, ka[u].x, P.pd, P.pinvd);
                        s1y += ntt::fmul(vy, ka[u].y, P.pd, P.pinvd);
                    }
                }
            }
            __stcg(reinterpret_cast<ulonglong2 *>(o0),
                   make_ulonglong2(ntt::fcanon(s0x, P.pd, P.pinvd), ntt::fcanon(s0y, P.pd, P.pinvd)));
            __stcg(reinterpret_cast<ulonglong2 *>(o1),
                   make_ulonglong2(ntt::fcanon(s1x, P.pd, P.pinvd), ntt::fcanon(s1y, P.pd, P.pinvd)));
        } else {
        u64 s0x = 0, s0y = 0, s1x = 0, s1y = 0;
        for (int j0 = 0; j0 < k; j0 += MAC_MJ) {
            ulonglong2 v[MAC_MJ];
#pragma unroll
            for (int u = 0; u < MAC_MJ; ++u) {
                const int j = j0 + u;
                if (j < k) v[u] = __ldcg(reinterpret_cast<const ulonglong2 *>((j == t) ? own : vrow + (size_t)j * n));
            }
#pragma unroll
            for (int u = 0; u < MAC_MJ; ++u) {
                const int j = j0 + u;
                if (j < k) {
                    const ulonglong2 *kp = key + (((size_t)j * K.num_rows + gt) * 2) * n + x;
                    const ulonglong2 bx = __ldg(kp), by = __ldg(kp + 1), ax = __ldg(kp + n), ay = __ldg(kp + n + 1);
                    s0x = csub(s0x + shoup_lazy(v[u].x, bx.x, bx.y, P.p), p2);
                    s0y = csub(s0y + shoup_lazy(v[u].y, by.x, by.y, P.p), p2);
                    s1x = csub(s1x + shoup_lazy(v[u].x, ax.x, ax.y, P.p), p2);
                    s1y = csub(s1y + shoup_lazy(v[u].y, ay.x, ay.y, P.p), p2);
                }
            }
        }
        __stcg(reinterpret_cast<ulonglong2 *>(o0), make_ulonglong2(csub(s0x, P.p), csub(s0y, P.p)));
        __stcg(reinterpret_cast<ulonglong2 *>(o1), make_ulonglong2(csub(s1x, P.p), csub(s1y, P.p)));
        }
    }
}

// Prepared switching key: Montgomery residue x of digit j, row r -> (w, floor(w 2^64 / p))
// with w = x R^-1 on the diagonal j == r and w = x elsewhere (see DigitLoad).
// floor(w 2^64/p) = w floor(2^64/p) + floor(w (2^64 mod p) / p), the last term by a
// Shoup quotient with one correction -- exact, no 128-bit division.
__global__ void k_prep_key(Ctx K, const u64 *kb, const u64 *ka, ulonglong2 *out, int digits, int logn) {
    const int n = 1 << logn;
    const int r = blockIdx.y, j = blockIdx.z;
    const PrimeInfo P = K.pi[r];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const size_t src = ((size_t)j * K.num_rows + r) * n + i;
        ulonglong2 *dst = out + (((size_t)j * K.num_rows + r) * 2) * n + i;
        double *dstd = reinterpret_cast<double *>(out + (((size_t)j * K.num_rows + r) * 2) * n) + i;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            // j == r: the digit is d2_r itself (Montgomery form) -> w = x R^-1;
            // j != r: the ModUp digit enters without its Montgomery factor (DigitLoad),
            // so the key keeps it: w = x
            const u64 x = c == 0 ? kb[src] : ka[src];
            const u64 w = j == r ? mont_mul(x, 1, P.p, P.pinv) : x;
            if (P.use_fp) {  // FP64 rows: w as a double, b part then a part
                dstd[(size_t)c * n] = (double)w;
                continue;
            }
            u64 q = __umul64hi(w, P.rmod_s);
            const u64 rem = w * P.rmod - q * P.p;
            q += rem >= P.p;
            dst[(size_t)c * n] = make_ulonglong2(w, w * P.r1s + q);
        }
    }
}

extern "C" int heb_prepare_switch_key(heb_ctx *c, const uint64_t *kb, const uint64_t *ka, int digits, uint64_t *out,
                                      void *stream) {
    if (!c || !kb || !ka || !out || digits < 1 || digits > c->num_rows - 1)
        return fail(HEB_EINVAL, "heb_prepare_switch_key: bad args");
    cudaStream_t st = (cudaStream_t)stream;
    {
        PROF("k_prep_key", st, 8.0 * c->n * digits * c->num_rows * 6.0);
        k_prep_key<<<dim3((c->n + 255) / 256, c->num_rows, digits), 256, 0, st>>>(kctx(c), kb, ka, (ulonglong2 *)out,
                                                                                  digits, c->log_n);
    }
    LAUNCH_CHECK();
    return HEB_OK;
}

// which = 0: aP = center_P(INTT_P(acc_P)) ; which = 1: bL = INTT_L(acc_L + P d_L) (std form)
template <int LOGN, int ENG>
__global__ void ROW_BOUNDS(LOGN) k_ks_down_head(Ctx K, const u64 *acc, heb_ct d, int k,
                                                                        i64 *aP, u64 *bL, int64_t count, int which0) {
    extern __shared__ u64 sm[];
    const int which = which0 + lbx<LOGN>(), c = blockIdx.z;
    const int n = 1 << LOGN;
    const int pos = tpos<LOGN>();
    const int row = which == 0 ? K.num_rows - 1 : k - 1;
    const int arow = which == 0 ? k : k - 1;
    const PrimeInfo P = K.pi[row];
    const LastConst lc = K.last[row];
    const LevelConst C = K.lc[(size_t)(k - 1) * K.num_rows + (k - 1)];
    for (int64_t b = blockIdx.y; b < count; b += gridDim.y) {
        u64 x[16];
        load16<LOGN>(acc + ((b * 2 + c) * (k + 1) + arow) * n + pos, x);
        if (which == 1) {
            u64 y[16];
            load16<LOGN>(at(d, b, c, k - 1, LOGN) + pos, y);
#pragma unroll
            for (int m = 0; m < 16; ++m) x[m] = add_mod(x[m], shoup(y[m], C.pmod.x, C.pmod.y, P.p), P.p);
            u64 *dst = bL + (b * 2 + c) * n;
            inv_any<LOGN, 16, ENG>(K, row, P, sm, x, [&](int i, u64 v) { dst[i] = v; }, true);
        } else {
            i64 *dst = aP + (b * 2 + c) * n;
            inv_any<LOGN, 16, ENG>(K, row, P, sm, x, [&](int i, u64 v) { dst[i] = center(v, P.p); }, true);
        }
    }
}

// exact FP64 helpers for the tail's FP64 rows (p < 2^42)
__device__ __forceinline__ double fp_imul(i64 a, double w, double w32, double pd, double pinvd) {
    // a (any signed 64-bit) * w mod p, as (a >> 32) * (2^32 w) + (a & (2^32-1)) * w
    const double hi = (double)(int)(a >> 32), lo = (double)(u32)(a & 0xffffffffu);
    return ntt::fmul(hi, w32, pd, pinvd) + ntt::fmul(lo, w, pd, pinvd);
}

// ModDown head for the rescale path, after k_ks_down_head has stored
// aP = center(INTT_P(acc_P)); one CTA per (item, component):
//   cL = center((INTT_L(acc_L + P d_L) - aP) P^-1 mod q_L)
// cL depends only on (item, component, position); computing it here once (instead of
// in each of the k-1 tail rows) removes most of the tail's integer prologue.
template <int LOGN, int ENG>
__global__ void ROW_BOUNDS(LOGN) k_ks_down_head_cl(Ctx K, const u64 *acc, heb_ct d, int k, const i64 *aP, i64 *cL,
                                                   int64_t count) {
    extern __shared__ u64 sm[];
    const int c = blockIdx.z;
    const int n = 1 << LOGN;
    const int pos = tpos<LOGN>();
    const int L = k - 1;
    const PrimeInfo PL = K.pi[L];
    const LevelConst C = K.lc[(size_t)L * K.num_rows + L];
    for (int64_t b = blockIdx.y; b < count; b += gridDim.y) {
        const i64 *ap = aP + (b * 2 + c) * n;
        i64 *cl = cL + (b * 2 + c) * n;
        u64 x[16], y[16];
        load16<LOGN>(acc + ((b * 2 + c) * (k + 1) + L) * n + pos, x);
        load16<LOGN>(at(d, b, c, L, LOGN) + pos, y);
#pragma unroll
        for (int m = 0; m < 16; ++m) x[m] = add_mod(x[m], shoup(y[m], C.pmod.x, C.pmod.y, PL.p), PL.p);
        inv_any<LOGN, 16, ENG>(K, L, PL, sm, x,
                      [&](int i, u64 v) {
                          const u64 sl = sub_mod(shoup(v, C.pinv.x, C.pinv.y, PL.p),
                                                 signed_mul_const(__ldcg(ap + i), C.pinv.x, C.pinv.y, PL.p), PL.p);
                          cl[i] = center(sl, PL.p);
                      },
                      true);
    }
}

// cL = center((bL - aP) P^-1 mod q_L) elementwise, from bL = INTT_L(acc_L + P d_L) (std
// form, k_ks_down_head which = 1) and aP: the same values k_ks_down_head_cl produces,
// with the two transforms run concurrently (integer P row / FP64 q_L row) before it.
__global__ void k_cl_combine(Ctx K, const u64 *__restrict__ bL, const i64 *__restrict__ aP, int k, i64 *cL,
                             int64_t total) {
    const int L = k - 1;
    const PrimeInfo PL = K.pi[L];
    const LevelConst C = K.lc[(size_t)L * K.num_rows + L];
    auto one = [&](u64 b, i64 a) {
        return center(sub_mod(shoup(b, C.pinv.x, C.pinv.y, PL.p), signed_mul_const(a, C.pinv.x, C.pinv.y, PL.p), PL.p),
                      PL.p);
    };
    // position pairs, 16-byte accesses (total is even: whole rows of N)
    const ulonglong2 *b2 = reinterpret_cast<const ulonglong2 *>(bL);
    const longlong2 *a2 = reinterpret_cast<const longlong2 *>(aP);
    longlong2 *c2 = reinterpret_cast<longlong2 *>(cL);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total / 2; i += (int64_t)gridDim.x * blockDim.x) {
        const ulonglong2 b = __ldcs(b2 + i);
        const longlong2 a = __ldcs(a2 + i);
        c2[i] = make_longlong2(one(b.x, a.x), one(b.y, a.y));
    }
}

// ModDown tail at N = 2^15: forward transform over the parity split instead of the half split
// (bit-exact; measured r2j, cfg4 tail ms per 4 steps: 173 -> 201: the DSMEM exchange and its
// two cluster barriers cost more than the loader evaluated twice; off)
#ifndef TAIL_EO
#define TAIL_EO 0
#endif
template <int LOGN, int ENG>
__global__ void ROW_BOUNDS(LOGN) k_ks_down_rescale_tail(Ctx K, const u64 *acc, heb_ct d, const i64 *aP, const i64 *cL,
                                                        int k, heb_ct out, int64_t count, int r0) {
    extern __shared__ u64 sm[];
    const int i = r0 + lbx<LOGN>(), c = blockIdx.z;
    const int n = 1 << LOGN;
    const int pos = tpos<LOGN>();
    const int L = k - 1;
    const PrimeInfo Pi = K.pi[i];
    const LevelConst Ci = K.lc[(size_t)L * K.num_rows + i];  // level L: drop q_L
    if (eng_fp<ENG>(Pi)) {
        // FP64 row: every product is an exact FP64 modular product (the integer pipe is
        // this kernel's bottleneck otherwise)
        const double pd = Pi.pd, pinvd = Pi.pinvd;
        const double ar = (double)Ci.alpha_r.x, br = (double)Ci.beta_r.x;
        const double ar32 = (double)ntt::fcanon(ntt::fmul(4294967296.0, ar, pd, pinvd), pd, pinvd);
        const double al = (double)Ci.alpha.x, be = (double)Ci.beta.x;
        // the transform takes and returns raw doubles (|v| < 2^47, FpArithRawIO): no
        // canonicalise / convert round trip on either side of it
        const ntt::FpArithRawIO fa(pd, pinvd);
        double *s2 = reinterpret_cast<double *>(sm);
        const double *twf = K.twf + ((size_t)i << (LOGN + ntt::TW_ROW_SHIFT));
        for (int64_t b = blockIdx.y; b < count; b += gridDim.y) {
            const i64 *ap = aP + (b * 2 + c) * n;
            const i64 *cl = cL + (b * 2 + c) * n;
            u64 y[16];
            auto ld = [&](int j) -> u64 {
                const double v = fp_imul(__ldcg(ap + j), ar, ar32, pd, pinvd) +
                                 ntt::fmul((double)__ldcg(cl + j), br, pd, pinvd);
                return (u64)__double_as_longlong(v);
            };
            constexpr int LL = Row<LOGN>::LL;
            if constexpr (Row<LOGN>::SP == 2 && TAIL_EO) {
                // parity split (see ntt::forward_split_eo): each CTA evaluates the loader for
                // its own parity class only -- the half split evaluates it for both halves
                // in both CTAs -- and the last stage crosses the pair through DSMEM
                const int r = rpart<LOGN>();
#pragma unroll 4
                for (int jl = threadIdx.x; jl < (1 << LL); jl += KT<LOGN>)
                    s2[ntt::pad(jl)] = __longlong_as_double((long long)ld(2 * jl + r));
                __syncthreads();
                ntt::forward_split_eo<LL, 16>(fa, s2, twf, y, r);
            } else if constexpr (Row<LOGN>::SPLIT) ntt::forward_split<LL, 16, Row<LOGN>::SP>(fa, s2, twf, ld, y, rpart<LOGN>());
            else ntt::forward<LL, 16>(fa, s2, twf, ld, y);
            u64 x[16], z[16];
            load16<LOGN>(acc + ((b * 2 + c) * (k + 1) + i) * n + pos, x);
            load16<LOGN>(at(d, b, c, i, LOGN) + pos, z);
#pragma unroll
            for (int m = 0; m < 16; ++m)
                x[m] = ntt::fcanon(ntt::fmul(ntt::u2d(x[m]), al, pd, pinvd) + ntt::fmul(ntt::u2d(z[m]), be, pd, pinvd) -
                                       __longlong_as_double((long long)y[m]),
                                   pd, pinvd);
            store16<LOGN>(at(out, b, c, i, LOGN) + pos, x);
        }
        return;
    }
    for (int64_t b = blockIdx.y; b < count; b += gridDim.y) {
        const i64 *ap = aP + (b * 2 + c) * n;
        const i64 *cl = cL + (b * 2 + c) * n;
        u64 y[16];
        fwd_any<LOGN, 16, ENG>(K, i, Pi, sm,
            [&](int j) {
                return add_mod(signed_mul_const(__ldcg(ap + j), Ci.alpha_r.x, Ci.alpha_r.y, Pi.p),
                               signed_mul_const(__ldcg(cl + j), Ci.beta_r.x, Ci.beta_r.y, Pi.p), Pi.p);
            },
            y);
        u64 x[16], z[16];
        load16<LOGN>(acc + ((b * 2 + c) * (k + 1) + i) * n + pos, x);
        load16<LOGN>(at(d, b, c, i, LOGN) + pos, z);
#pragma unroll
        for (int m = 0; m < 16; ++m)
            x[m] = sub_mod(add_mod(shoup(x[m], Ci.alpha.x, Ci.alpha.y, Pi.p), shoup(z[m], Ci.beta.x, Ci.beta.y, Pi.p),
                                   Pi.p),
                           y[m], Pi.p);
        store16<LOGN>(at(out, b, c, i, LOGN) + pos, x);
    }
}

// ModDown without rescale (rotation): out_i = acc_i P^-1 - NTT_i(aP P^-1 R) [+ add0_i for c = 0]
template <int LOGN, int ENG>
__global__ void ROW_BOUNDS(LOGN) k_ks_down_tail(Ctx K, const u64 *acc, const i64 *aP, int k,
                                                                        heb_ct add0, heb_ct out, int64_t count, int r0) {
    extern __shared__ u64 sm[];
    const int i = r0 + lbx<LOGN>(), c = blockIdx.z;
    const int n = 1 << LOGN;
    const int pos = tpos<LOGN>();
    const PrimeInfo Pi = K.pi[i];
    const LevelConst Ci = K.lc[(size_t)(k - 1) * K.num_rows + i];
    for (int64_t b = blockIdx.y; b < count; b += gridDim.y) {
        const i64 *ap = aP + (b * 2 + c) * n;
        u64 y[16];
        fwd_any<LOGN, 16, ENG>(K, i, Pi, sm,
                           [&](int j) { return signed_mul_const(__ldcg(ap + j), Ci.gamma_r.x, Ci.gamma_r.y, Pi.p); }, y);
        u64 x[16];
        load16<LOGN>(acc + ((b * 2 + c) * (k + 1) + i) * n + pos, x);
#pragma unroll
        for (int m = 0; m < 16; ++m) x[m] = sub_mod(shoup(x[m], Ci.gamma.x, Ci.gamma.y, Pi.p), y[m], Pi.p);
        if (c == 0) {
            u64 z[16];
            load16<LOGN>(at(add0, b, 0, i, LOGN) + pos, z);
#pragma unroll
            for (int m = 0; m < 16; ++m) x[m] = add_mod(x[m], z[m], Pi.p);
        }
        store16<LOGN>(at(out, b, c, i, LOGN) + pos, x);
    }
}

template <int LOGN>
static int launch_keyswitch(heb_ctx *c, heb_ct src, int comp, const ulonglong2 *key, heb_ct d, heb_ct out,
                            int64_t count, int level, bool rescale, cudaStream_t st) {
    constexpr int T = KT<LOGN>;
    constexpr size_t sm = smem_bytes<LOGN>();
    PREP_ENGINES(k_ks_head, sm);
    CUDA_TRY(prep_kernel(k_ks_modup_ntt<LOGN>, sm));
    constexpr size_t smu = modup_smem_bytes<LOGN>();
    CUDA_TRY(prep_kernel(k_ks_modup_fused<LOGN, 0>, sm));
    CUDA_TRY(prep_kernel(k_ks_modup_fused<LOGN, 1>, smu));
    CUDA_TRY(prep_kernel(k_ks_modup_fused<LOGN, 2>, smu));
    PREP_ENGINES(k_ks_down_head, sm);
    PREP_ENGINES(k_ks_down_head_cl, sm);
    PREP_ENGINES(k_ks_down_rescale_tail, sm);
    PREP_ENGINES(k_ks_down_tail, sm);
    const int k = level + 1, n = c->n;
    // the fused ModUp gives every item of a chunk its own grid row (gridDim.y <= 65535)
    const int64_t chunk = std::min<int64_t>(c->chunk > 0 ? c->chunk : count, 65535);
    const int64_t cmax = std::min<int64_t>(chunk, count);
    // ModUp sub-chunk: enough (item, t, j) transforms for ~8 CTA waves, V kept small
    static const int64_t target_ctas = [] {
        const char *e = getenv("HEB_MODUP_CTAS");
        return e ? std::max<int64_t>(64, atoll(e)) : (int64_t)2400;
    }();
    const int64_t sub = std::max<int64_t>(4, std::min<int64_t>(cmax, (target_ctas + k * k - 1) / (k * k)));
    // ModUp: TMEM-accumulating fused kernel by default (HEB_MODUP_SPLIT=1: the two-pass
    // NTT + MAC path with the V intermediate in HBM)
    static const bool fused_env = [] {
        const char *e = getenv("HEB_MODUP_SPLIT");
        return !(e && *e && *e != '0');
    }();
    // TMEM accesses are warp-wide: rows of fewer than 32 x 16 residues per CTA take the split path
    const bool fused = fused_env && KT<LOGN> % 32 == 0;
    Scratch sD(c, st), sA(c, st), sP(c, st), sL(c, st), sB(c, st), sV(c, st);
    CUDA_TRY(sD.get(sizeof(i64) * (size_t)cmax * k * n));
    CUDA_TRY(sA.get(sizeof(u64) * (size_t)cmax * 2 * (k + 1) * n));
    CUDA_TRY(sP.get(sizeof(i64) * (size_t)cmax * 2 * n));
    CUDA_TRY(sL.get(sizeof(u64) * (size_t)cmax * 2 * n));
    CUDA_TRY(sB.get(rescale ? sizeof(u64) * (size_t)cmax * 2 * n : 256));
    CUDA_TRY(sV.get(fused ? 256 : sizeof(u64) * (size_t)sub * (k + 1) * k * n));
    const Ctx K = kctx(c);
    for (int64_t b0 = 0; b0 < count; b0 += chunk) {
        const int64_t cnt = std::min<int64_t>(chunk, count - b0);
        heb_ct s = src, dd = d, o = out;
        s.data += b0 * src.ct_stride;
        dd.data += b0 * d.ct_stride;
        o.data += b0 * out.ct_stride;
        const unsigned gy = gdim(cnt);
        { PROF("k_ks_head", st, 16.0 * n * cnt * k); CUDA_TRY(launch_by_engine<LOGN>(c, ENGINE_KERNELS(k_ks_head), 0, k, gy, 1, sm, st, K, s, comp, (i64 *)sD.p, k, cnt)); }
        LAUNCH_CHECK();
        if (fused) {
            // algorithmic: read D (k rows) and the congruent d2 rows (k), the key once, write acc (2(k+1) rows)
            PROF("k_ks_modup_fused", st, 8.0 * n * cnt * (2.0 * k + 4.0 * k * (k + 1) / cnt + 2.0 * (k + 1)));
#ifndef MODUP_ENGINES_SPLIT
#define MODUP_ENGINES_SPLIT 1
#endif
            // each engine's launch covers exactly its own targets (no early-exit CTAs);
            // G items per group, targets in sequence within a group (see the kernel)
            TargetList tl_fp{0, {}}, tl_int{0, {}}, tl_all{0, {}};
            for (int t = 0; t <= k; ++t) {
                const int gt = t < k ? t : c->num_rows - 1;
                TargetList &l = c->row_fp[gt] ? tl_fp : tl_int;
                l.t[l.n++] = (signed char)t;
                tl_all.t[tl_all.n++] = (signed char)t;
            }
            // targets per set (HEB_MODUP_TS; see the kernel): every item gets its own CTA row
            static const int TS_env = [] {
                const char *e = getenv("HEB_MODUP_TS");
                return e ? std::max(1, atoi(e)) : 0;
            }();
            const int TS = TS_env > 0 ? TS_env : MODUP_TS_DEFAULT;
            auto mgrid = [&](const TargetList &l) {
                const int ts = std::min(TS, l.n);
                return dim3((unsigned)ts, (unsigned)cnt, (unsigned)((l.n + ts - 1) / ts));
            };
            auto mts = [&](const TargetList &l) { return std::min(TS, l.n); };
            if (MODUP_ENGINES_SPLIT) {
                // the integer-target and FP64-target launches are independent (disjoint acc
                // rows): the integer one goes to the stream's side stream so their CTAs share
                // SMs and the IMAD/ALU and DFMA pipes work at the same time
                static const bool concurrent = [] {
                    const char *e = getenv("HEB_MODUP_CONCURRENT");
                    return !(e && *e == '0');
                }();
                cudaStream_t ist = st;
                if (concurrent && tl_int.n) CUDA_TRY(side_fork(c, st, &ist));
                if (tl_int.n)
                    CUDA_TRY(launch_rows<LOGN>(k_ks_modup_fused<LOGN, 2>, mgrid(tl_int), KT<LOGN>, smu, ist, K,
                                               s, comp, (const i64 *)sD.p, key, k, (u64 *)sA.p, cnt, tl_int, mts(tl_int)));
                if (tl_fp.n)
                    CUDA_TRY(launch_rows<LOGN>(k_ks_modup_fused<LOGN, 1>, mgrid(tl_fp), KT<LOGN>, smu, st, K,
                                               s, comp, (const i64 *)sD.p, key, k, (u64 *)sA.p, cnt, tl_fp, mts(tl_fp)));
                if (concurrent && tl_int.n) CUDA_TRY(side_join(c, st));
            } else {
                CUDA_TRY(launch_rows<LOGN>(k_ks_modup_fused<LOGN, 0>, mgrid(tl_all), KT<LOGN>, sm, st, K, s,
                                           comp, (const i64 *)sD.p, key, k, (u64 *)sA.p, cnt, tl_all, mts(tl_all)));
            }
        }
        for (int64_t s0 = 0; s0 < (fused ? 0 : cnt); s0 += sub) {
            const int64_t sc = std::min<int64_t>(sub, cnt - s0);
            heb_ct ss = s;
            ss.data += s0 * s.ct_stride;
            const i64 *Dp = (const i64 *)sD.p + s0 * k * n;
            u64 *Ap = (u64 *)sA.p + s0 * 2 * (k + 1) * n;
            {
                PROF("k_ks_modup_ntt", st, 16.0 * n * sc * k * k);
                CUDA_TRY(launch_rows<LOGN>(k_ks_modup_ntt<LOGN>, dim3(dim3(k * k, gdim(sc))), KT<LOGN>, sm, st, K, Dp, k, (u64 *)sV.p, sc));
            }
            LAUNCH_CHECK();
            {
                PROF("k_ks_modup_mac", st, 8.0 * n * (sc * k * (k + 1) + 4.0 * k * (k + 1) + 2.0 * sc * (k + 1)));
                const dim3 mg((n / 2 + 255) / 256, k + 1, gdim(sc));
                k_ks_modup_mac<true><<<mg, 256, 0, st>>>(K, ss, comp, (const u64 *)sV.p, key, k, Ap, sc, LOGN);
                k_ks_modup_mac<false><<<mg, 256, 0, st>>>(K, ss, comp, (const u64 *)sV.p, key, k, Ap, sc, LOGN);
            }
            LAUNCH_CHECK();
        }
        if (rescale) {
            // aP = center(INTT_P(acc_P)) (special prime) and bL = INTT_L(acc_L + P d_L) are
            // independent: the P transform goes to the side stream, then one elementwise
            // pass forms cL (HEB_MODDOWN_CONCURRENT=0: the sequential k_ks_down_head_cl)
            static const bool conc = [] {
                const char *e = getenv("HEB_MODDOWN_CONCURRENT");
                return !(e && *e == '0');
            }();
            auto head_p = c->row_fp[c->num_rows - 1] ? k_ks_down_head<LOGN, 1> : k_ks_down_head<LOGN, 2>;
            if (conc) {
                PROF("k_ks_down_head", st, 8.0 * n * cnt * 2.0 * 2.0 * 2.0);
                cudaStream_t side;
                CUDA_TRY(side_fork(c, st, &side));
                CUDA_TRY(launch_rows<LOGN>(head_p, dim3(dim3(1, gy, 2)), KT<LOGN>, sm, side, K, (const u64 *)sA.p, dd, k,
                                           (i64 *)sP.p, (u64 *)nullptr, cnt, 0));
                CUDA_TRY(launch_rows<LOGN>(c->row_fp[k - 1] ? k_ks_down_head<LOGN, 1> : k_ks_down_head<LOGN, 2>,
                                           dim3(dim3(1, gy, 2)), KT<LOGN>, sm, st, K, (const u64 *)sA.p, dd, k,
                                           (i64 *)nullptr, (u64 *)sB.p, cnt, 1));
                CUDA_TRY(side_join(c, st));
            } else {
                PROF("k_ks_down_head", st, 8.0 * n * cnt * 4.0);
                CUDA_TRY(launch_rows<LOGN>(head_p, dim3(dim3(1, gy, 2)), KT<LOGN>, sm, st, K, (const u64 *)sA.p, dd, k,
                                           (i64 *)sP.p, (u64 *)nullptr, cnt, 0));
            }
            LAUNCH_CHECK();
            if (conc) {
                PROF("k_cl_combine", st, 8.0 * n * cnt * 2.0 * 3.0);
                const int64_t total = cnt * 2 * n;
                k_cl_combine<<<(unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16), 256, 0, st>>>(
                    K, (const u64 *)sB.p, (const i64 *)sP.p, k, (i64 *)sL.p, total);
            } else {
                PROF("k_ks_down_head_cl", st, 8.0 * n * cnt * 2.0 * 4.0);
                CUDA_TRY(launch_rows<LOGN>(c->row_fp[k - 1] ? k_ks_down_head_cl<LOGN, 1> : k_ks_down_head_cl<LOGN, 2>,
                                           dim3(dim3(1, gy, 2)), KT<LOGN>, sm, st, K, (const u64 *)sA.p, dd, k,
                                           (const i64 *)sP.p, (i64 *)sL.p, cnt));
            }
            LAUNCH_CHECK();
            { PROF("k_ks_down_rescale_tail", st, 8.0 * n * cnt * 2.0 * (2 + 3 * (k - 1))); CUDA_TRY(launch_by_engine<LOGN>(c, ENGINE_KERNELS(k_ks_down_rescale_tail), 0, k - 1, gy, 2, sm, st, K, (const u64 *)sA.p, dd,
                                                                             (const i64 *)sP.p, (const i64 *)sL.p, k,
                                                                             o, cnt)); }
            LAUNCH_CHECK();
        } else {
            { PROF("k_ks_down_head", st, 8.0 * n * cnt * 4.0); CUDA_TRY(launch_rows<LOGN>(c->row_fp[c->num_rows - 1] ? k_ks_down_head<LOGN, 1> : k_ks_down_head<LOGN, 2>, dim3(dim3(1, gy, 2)), KT<LOGN>, sm, st, K, (const u64 *)sA.p, dd, k, (i64 *)sP.p,
                                                                 (u64 *)sL.p, cnt, 0)); }
            LAUNCH_CHECK();
            { PROF("k_ks_down_tail", st, 8.0 * n * cnt * (2.0 + 5.0 * k)); CUDA_TRY(launch_by_engine<LOGN>(c, ENGINE_KERNELS(k_ks_down_tail), 0, k, gy, 2, sm, st, K, (const u64 *)sA.p, (const i64 *)sP.p, k, dd, o,
                                                                 cnt)); }
            LAUNCH_CHECK();
        }
    }
    return HEB_OK;
}

extern "C" int heb_relin_rescale(heb_ctx *c, heb_ct raw, const uint64_t *evk, heb_ct out, int64_t count, int level,
                                 void *stream) {
    if (!c || !evk || level < 1 || level > c->num_rows - 2)
        return fail(HEB_EINVAL, "heb_relin_rescale: bad level %d", level);
    if (count <= 0) return HEB_OK;
    // d2 = component 2 of raw; d0/d1 = components 0/1
    DISPATCH_LOGN(c, launch_keyswitch, c, raw, 2, (const ulonglong2 *)evk, raw, out, count, level, true,
                  (cudaStream_t)stream);
}

extern "C" int heb_rotate(heb_ctx *c, heb_ct ct, const uint64_t *gk, heb_ct out, int64_t count, int level,
                          uint64_t galois, void *stream) {
    if (!c || !gk || level < 0 || level > c->num_rows - 2 || !(galois & 1))
        return fail(HEB_EINVAL, "heb_rotate: bad args");
    if (count <= 0) return HEB_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int k = level + 1;
    // sigma_g of both components into a compact scratch batch
    Scratch rot(c, st);
    CUDA_TRY(rot.get(sizeof(u64) * (size_t)count * 2 * k * c->n));
    heb_ct r{(u64 *)rot.p, (int64_t)2 * k * c->n, (int64_t)k * c->n};
    const int64_t lines = count * 2 * k;
    { PROF("k_galois_ct", st, 16.0 * c->n * lines); k_galois_ct<<<pw_grid(c->n, lines), 256, 0, st>>>(ct, r, lines, k, c->log_n, galois % (2ull * c->n)); }
    LAUNCH_CHECK();
    DISPATCH_LOGN(c, launch_keyswitch, c, r, 1, (const ulonglong2 *)gk, r, out, count, level, false, st);
}

