// ntt.cuh -- CTA-cooperative negacyclic NTT engine for sm_100a.
//
// Transform (reference kernels.py:68-114):
//   forward: natural-order input, output position i holds a(psi^(2*brv(i)+1));
//            Cooley-Tukey stages s = 0..n-1, stage s pairs (j, j + N/2^(s+1)) inside
//            block b = j >> (n-s) with twiddle tw[2^s + b] = psi^brv(2^s + b);
//   inverse: the exact inverse map (Gentleman-Sande with tw^-1, stages n-1..0, times
//            n^-1 folded into the last stage), so results are bit-identical to the
//            reference's backwards table walk.
//
// Work split: one CTA of T = N/E threads owns one row of N residues (E = 8 or 16
// elements per thread).  The n stages are processed in register-blocked groups: a
// radix-2^r group gives each thread a "unit" of 2^r elements that stay in registers
// for r stages; units exchange through shared memory between groups (padded index
// i + i/16 keeps 64-bit accesses (nearly) free of bank conflicts).  n = e*G + REM
// (E = 2^e) gives G radix-E groups plus one radix-2^REM group (first in forward
// order, last in inverse order).
//
// Interfaces chosen so that callers can fuse prologues/epilogues:
//   forward: input through a functor load(idx) (coalesced across threads), output
//            left in registers: thread t holds positions [E t, E t + E) of the result;
//   inverse: input given in registers in that same layout, output through a functor
//            store(idx, value) (coalesced).
// Lazy reduction: forward values live in [0, 4p), inverse values in [0, 2p); all
// values handed to the caller are canonical.
#pragma once
#include "modarith.cuh"

namespace ntt {

HD int pad(int i) { return i + (i >> 4); }

template <int LOGN, int E = 16>
struct Shape {
    static_assert(E == 8 || E == 16, "8 or 16 elements per thread");
    static constexpr int LOGE = E == 8 ? 3 : 4;
    static constexpr int N = 1 << LOGN;
    static constexpr int T = N / E;
    static constexpr int REM = LOGN % LOGE;
    static constexpr int G = LOGN / LOGE;
    static constexpr int SMEM_WORDS = N + N / 16;
};

// ---------------------------------------------------------------- forward ----
// One forward group: radix 2^RB covering stages S0 .. S0+RB-1.
// SRC: 0 = functor load, 1 = shared memory.  DST: 0 = shared memory, 1 = registers.
template <int LOGN, int E, int RB, int S0, int SRC, int DST, class Load>
HD void fwd_group(u64 *sm, const ulonglong2 *__restrict__ tw, u64 p, Load &load, u64 (&out)[E]) {
    using S = Shape<LOGN, E>;
    constexpr int R = 1 << RB;
    constexpr int LB = LOGN - S0 - RB;
    constexpr int UPT = (S::N / R) / S::T;
    const u64 p2 = 2 * p;
    const int tid = threadIdx.x;
#pragma unroll
    for (int k = 0; k < UPT; ++k) {
        const int u = tid + k * S::T;
        const int ulow = u & ((1 << LB) - 1);
        const int uhigh = u >> LB;
        const int base = (uhigh << (LOGN - S0)) | ulow;
        u64 x[R];
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const int idx = base + (m << LB);
            if constexpr (SRC == 0) x[m] = load(idx);
            else x[m] = sm[pad(idx)];
        }
#pragma unroll
        for (int q = 0; q < RB; ++q) {
            const int half = R >> (q + 1);
#pragma unroll
            for (int m = 0; m < R; ++m) {
                if (m & half) continue;
                const ulonglong2 w = __ldg(tw + (1 << (S0 + q)) + (uhigh << q) + (m >> (RB - q)));
                u64 a = csub(x[m], p2);
                u64 t = shoup_lazy(x[m + half], w.x, w.y, p);
                x[m] = a + t;
                x[m + half] = a - t + p2;
            }
        }
        if constexpr (DST == 1) {
            static_assert(UPT == 1 && R == E, "register output needs one radix-E unit per thread");
#pragma unroll
            for (int m = 0; m < R; ++m) out[m] = csub(csub(x[m], p2), p);
        } else {
#pragma unroll
            for (int m = 0; m < R; ++m) sm[pad(base + (m << LB))] = x[m];
        }
    }
}

template <int LOGN, int E, int GI, class Load>
HD void fwd_main_groups(u64 *sm, const ulonglong2 *__restrict__ tw, u64 p, Load &load, u64 (&out)[E]) {
    using S = Shape<LOGN, E>;
    constexpr int S0 = S::REM + S::LOGE * GI;
    constexpr bool first = (S0 == 0);
    constexpr bool last = (GI == S::G - 1);
    fwd_group<LOGN, E, S::LOGE, S0, first ? 0 : 1, last ? 1 : 0>(sm, tw, p, load, out);
    if constexpr (!last) {
        __syncthreads();
        fwd_main_groups<LOGN, E, GI + 1>(sm, tw, p, load, out);
    }
}

// Forward NTT of one row.  `load(idx)` returns the input residue at natural position
// idx (in [0, 2p)); on return thread t holds output positions E t .. E t + E - 1.
template <int LOGN, int E = 16, class Load>
__device__ void forward(u64 *sm, const ulonglong2 *__restrict__ tw, u64 p, Load load, u64 (&out)[E]) {
    using S = Shape<LOGN, E>;
    static_assert(LOGN >= 6 && LOGN <= 14, "single-CTA engine covers N = 64 .. 16384");
    __syncthreads();  // shared memory may still be read by a previous transform
    if constexpr (S::REM) {
        fwd_group<LOGN, E, S::REM, 0, 0, 0>(sm, tw, p, load, out);
        __syncthreads();
    }
    fwd_main_groups<LOGN, E, 0>(sm, tw, p, load, out);
}

// ---------------------------------------------------------------- inverse ----
// SRC: 1 = registers, 0 = shared memory.  DST: 0 = shared memory, 1 = functor store.
template <int LOGN, int E, int RB, int S0, int SRC, int DST, class Store>
HD void inv_group(u64 *sm, const ulonglong2 *__restrict__ itw, u64 p, const u64 (&in)[E], Store &store,
                  ulonglong2 last_u, ulonglong2 last_v) {
    using S = Shape<LOGN, E>;
    constexpr int R = 1 << RB;
    constexpr int LB = LOGN - S0 - RB;
    constexpr int UPT = (S::N / R) / S::T;
    const u64 p2 = 2 * p;
    const int tid = threadIdx.x;
#pragma unroll
    for (int k = 0; k < UPT; ++k) {
        const int u = tid + k * S::T;
        const int ulow = u & ((1 << LB) - 1);
        const int uhigh = u >> LB;
        const int base = (uhigh << (LOGN - S0)) | ulow;
        u64 x[R];
        if constexpr (SRC == 1) {
            static_assert(UPT == 1 && R == E, "register input needs one radix-E unit per thread");
#pragma unroll
            for (int m = 0; m < R; ++m) x[m] = in[m];
        } else {
#pragma unroll
            for (int m = 0; m < R; ++m) x[m] = sm[pad(base + (m << LB))];
        }
#pragma unroll
        for (int q = RB - 1; q >= 0; --q) {
            const int half = R >> (q + 1);
#pragma unroll
            for (int m = 0; m < R; ++m) {
                if (m & half) continue;
                const u64 a = x[m], b = x[m + half];
                if (S0 + q == 0) {
                    // final stage: fold n^-1 (and optionally R^-1) and canonicalise
                    x[m] = shoup(a + b, last_u.x, last_u.y, p);
                    x[m + half] = shoup(a - b + p2, last_v.x, last_v.y, p);
                } else {
                    const ulonglong2 w = __ldg(itw + (1 << (S0 + q)) + (uhigh << q) + (m >> (RB - q)));
                    x[m] = csub(a + b, p2);
                    x[m + half] = shoup_lazy(a - b + p2, w.x, w.y, p);
                }
            }
        }
        if constexpr (DST == 1) {
#pragma unroll
            for (int m = 0; m < R; ++m) store(base + (m << LB), x[m]);
        } else {
#pragma unroll
            for (int m = 0; m < R; ++m) sm[pad(base + (m << LB))] = x[m];
        }
    }
}

template <int LOGN, int E, int GI, class Store>
HD void inv_main_groups(u64 *sm, const ulonglong2 *__restrict__ itw, u64 p, const u64 (&in)[E], Store &store,
                        ulonglong2 last_u, ulonglong2 last_v) {
    // GI counts down from G-1 (first inverse group, register input) to 0.
    using S = Shape<LOGN, E>;
    constexpr int S0 = S::REM + S::LOGE * GI;
    constexpr bool first = (GI == S::G - 1);
    constexpr bool last = (S0 == 0);
    inv_group<LOGN, E, S::LOGE, S0, first ? 1 : 0, last ? 1 : 0>(sm, itw, p, in, store, last_u, last_v);
    if constexpr (GI > 0) {
        __syncthreads();
        inv_main_groups<LOGN, E, GI - 1>(sm, itw, p, in, store, last_u, last_v);
    }
}

// Inverse NTT of one row.  Thread t supplies positions E t .. E t + E - 1 (values in
// [0, 2p)); results leave through store(idx, canonical value).  last_u = n^-1 * c and
// last_v = itw[1] * n^-1 * c (Shoup pairs) for a caller-chosen output factor c.
template <int LOGN, int E = 16, class Store>
__device__ void inverse(u64 *sm, const ulonglong2 *__restrict__ itw, u64 p, const u64 (&in)[E], Store store,
                        ulonglong2 last_u, ulonglong2 last_v) {
    using S = Shape<LOGN, E>;
    static_assert(LOGN >= 6 && LOGN <= 14, "single-CTA engine covers N = 64 .. 16384");
    __syncthreads();
    inv_main_groups<LOGN, E, S::G - 1>(sm, itw, p, in, store, last_u, last_v);
    if constexpr (S::REM) {
        __syncthreads();
        inv_group<LOGN, E, S::REM, 0, 0, 1>(sm, itw, p, in, store, last_u, last_v);
    }
}

// =============================================================================
// FP64 engine for primes p < 2^42 (the 40-bit level primes).
//
// On sm_100a the DFMA pipe sustains the same 64 op/clk/SM as 32-bit IMAD, while a
// 64-bit Shoup product costs ~8 IMAD-pipe issue slots (tools/pipes_bench.cu).  With
// p < 2^42 residues are exact doubles and a product modulo p needs 6 FP64 ops:
//     h = y*w;  l = fma(y, w, -h)            (y*w = h + l exactly)
//     q = rint(y * (w/p))                    (fma with the 1.5*2^52 magic constant)
//     r = fma(-q, p, h) + l                  (exact; r in (-p, 2p))
// Values are kept *unreduced and signed* between stages: a forward stage adds at most
// 2p in magnitude, the inverse's sum path doubles and is re-centred at every group
// boundary, so everything stays below 2^47 and every step above stays exact.  Inputs
// and outputs are canonical u64 residues, bit-identical to the integer engine.
// =============================================================================
#define FP_MAGIC 6755399441055744.0  // 1.5 * 2^52

HD double u2d(u64 v) { return __longlong_as_double((long long)(0x4330000000000000ull | v)) - 4503599627370496.0; }
HD double rint_fp(double x) { return (x + FP_MAGIC) - FP_MAGIC; }
// y * w mod p, result in (-p, 2p); the quotient estimate uses the rounded product
// h (relative error 2^-52), so it is off by at most one -- absorbed by the lazy range
HD double fmul(double y, double w, double p, double pinv) {
    const double h = __dmul_rn(y, w);
    const double l = fma(y, w, -h);
    const double q = __dsub_rn(fma(h, pinv, FP_MAGIC), FP_MAGIC);
    return __dadd_rn(fma(-q, p, h), l);
}
// any |x| < 2^50 -> centred representative in about (-p/2, p/2]
HD double fred(double x, double p, double pinv) {
    const double q = __dsub_rn(fma(x, pinv, FP_MAGIC), FP_MAGIC);
    return fma(-q, p, x);
}
// exact canonical residue in [0, p) as u64
HD u64 fcanon(double x, double p, double pinv) {
    double r = fred(x, p, pinv);
    r = r < 0.0 ? r + p : r;
    r = r >= p ? r - p : r;
    return (u64)__double_as_longlong(r + 4503599627370496.0) & 0x000FFFFFFFFFFFFFull;
}

template <int LOGN, int E, int RB, int S0, int SRC, int DST, class Load>
HD void fwd_group_fp(double *sm, const double *__restrict__ tw, double p, double pinv, Load &load,
                     u64 (&out)[E]) {
    using S = Shape<LOGN, E>;
    constexpr int R = 1 << RB;
    constexpr int LB = LOGN - S0 - RB;
    constexpr int UPT = (S::N / R) / S::T;
    const int tid = threadIdx.x;
#pragma unroll
    for (int k = 0; k < UPT; ++k) {
        const int u = tid + k * S::T;
        const int ulow = u & ((1 << LB) - 1);
        const int uhigh = u >> LB;
        const int base = (uhigh << (LOGN - S0)) | ulow;
        double x[R];
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const int idx = base + (m << LB);
            if constexpr (SRC == 0) x[m] = u2d(load(idx));
            else x[m] = sm[pad(idx)];
        }
#pragma unroll
        for (int q = 0; q < RB; ++q) {
            const int half = R >> (q + 1);
#pragma unroll
            for (int m = 0; m < R; ++m) {
                if (m & half) continue;
                const double w = __ldg(tw + (1 << (S0 + q)) + (uhigh << q) + (m >> (RB - q)));
                const double r = fmul(x[m + half], w, p, pinv);
                x[m + half] = x[m] - r;
                x[m] = x[m] + r;
            }
        }
        if constexpr (DST == 1) {
            static_assert(UPT == 1 && R == E, "register output needs one radix-E unit per thread");
#pragma unroll
            for (int m = 0; m < R; ++m) out[m] = fcanon(x[m], p, pinv);
        } else {
#pragma unroll
            for (int m = 0; m < R; ++m) sm[pad(base + (m << LB))] = x[m];
        }
    }
}

template <int LOGN, int E, int GI, class Load>
HD void fwd_main_groups_fp(double *sm, const double *__restrict__ tw, double p, double pinv, Load &load,
                           u64 (&out)[E]) {
    using S = Shape<LOGN, E>;
    constexpr int S0 = S::REM + S::LOGE * GI;
    constexpr bool first = (S0 == 0);
    constexpr bool last = (GI == S::G - 1);
    fwd_group_fp<LOGN, E, S::LOGE, S0, first ? 0 : 1, last ? 1 : 0>(sm, tw, p, pinv, load, out);
    if constexpr (!last) {
        __syncthreads();
        fwd_main_groups_fp<LOGN, E, GI + 1>(sm, tw, p, pinv, load, out);
    }
}

template <int LOGN, int E = 16, class Load>
__device__ void forward_fp(double *sm, const double *__restrict__ tw, double p, double pinv, Load load,
                           u64 (&out)[E]) {
    using S = Shape<LOGN, E>;
    static_assert(LOGN >= 6 && LOGN <= 14, "single-CTA engine covers N = 64 .. 16384");
    __syncthreads();
    if constexpr (S::REM) {
        fwd_group_fp<LOGN, E, S::REM, 0, 0, 0>(sm, tw, p, pinv, load, out);
        __syncthreads();
    }
    fwd_main_groups_fp<LOGN, E, 0>(sm, tw, p, pinv, load, out);
}

template <int LOGN, int E, int RB, int S0, int SRC, int DST, class Store>
HD void inv_group_fp(double *sm, const double *__restrict__ itw, double p, double pinv, const u64 (&in)[E],
                     Store &store, double last_u, double last_v) {
    using S = Shape<LOGN, E>;
    constexpr int R = 1 << RB;
    constexpr int LB = LOGN - S0 - RB;
    constexpr int UPT = (S::N / R) / S::T;
    const int tid = threadIdx.x;
#pragma unroll
    for (int k = 0; k < UPT; ++k) {
        const int u = tid + k * S::T;
        const int ulow = u & ((1 << LB) - 1);
        const int uhigh = u >> LB;
        const int base = (uhigh << (LOGN - S0)) | ulow;
        double x[R];
        if constexpr (SRC == 1) {
            static_assert(UPT == 1 && R == E, "register input needs one radix-E unit per thread");
#pragma unroll
            for (int m = 0; m < R; ++m) x[m] = u2d(in[m]);
        } else {
#pragma unroll
            for (int m = 0; m < R; ++m) x[m] = sm[pad(base + (m << LB))];
        }
#pragma unroll
        for (int q = RB - 1; q >= 0; --q) {
            const int half = R >> (q + 1);
#pragma unroll
            for (int m = 0; m < R; ++m) {
                if (m & half) continue;
                const double a = x[m], b = x[m + half];
                if (S0 + q == 0) {
                    x[m] = fmul(a + b, last_u, p, pinv);
                    x[m + half] = fmul(a - b, last_v, p, pinv);
                } else {
                    const double w = __ldg(itw + (1 << (S0 + q)) + (uhigh << q) + (m >> (RB - q)));
                    x[m] = a + b;
                    x[m + half] = fmul(a - b, w, p, pinv);
                }
            }
        }
        if constexpr (DST == 1) {
#pragma unroll
            for (int m = 0; m < R; ++m) store(base + (m << LB), fcanon(x[m], p, pinv));
        } else {
            // the additive path grew by up to 2^RB: re-centre before the next group
#pragma unroll
            for (int m = 0; m < R; ++m) sm[pad(base + (m << LB))] = fred(x[m], p, pinv);
        }
    }
}

template <int LOGN, int E, int GI, class Store>
HD void inv_main_groups_fp(double *sm, const double *__restrict__ itw, double p, double pinv, const u64 (&in)[E],
                           Store &store, double last_u, double last_v) {
    using S = Shape<LOGN, E>;
    constexpr int S0 = S::REM + S::LOGE * GI;
    constexpr bool first = (GI == S::G - 1);
    constexpr bool last = (S0 == 0);
    inv_group_fp<LOGN, E, S::LOGE, S0, first ? 1 : 0, last ? 1 : 0>(sm, itw, p, pinv, in, store, last_u, last_v);
    if constexpr (GI > 0) {
        __syncthreads();
        inv_main_groups_fp<LOGN, E, GI - 1>(sm, itw, p, pinv, in, store, last_u, last_v);
    }
}

template <int LOGN, int E = 16, class Store>
__device__ void inverse_fp(double *sm, const double *__restrict__ itw, double p, double pinv, const u64 (&in)[E],
                           Store store, double last_u, double last_v) {
    using S = Shape<LOGN, E>;
    static_assert(LOGN >= 6 && LOGN <= 14, "single-CTA engine covers N = 64 .. 16384");
    __syncthreads();
    inv_main_groups_fp<LOGN, E, S::G - 1>(sm, itw, p, pinv, in, store, last_u, last_v);
    if constexpr (S::REM) {
        __syncthreads();
        inv_group_fp<LOGN, E, S::REM, 0, 0, 1>(sm, itw, p, pinv, in, store, last_u, last_v);
    }
}

}  // namespace ntt
