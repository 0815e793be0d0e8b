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
// Two arithmetic policies share the schedule:
//   IntArith  64-bit Shoup products (any prime < 2^62), values in [0,4p) / [0,2p);
//   FpArith   exact FP64 products for primes < 2^42 (the 40-bit level primes): the
//             DFMA pipe sustains 64 op/clk/SM on sm_100a while a 64-bit Shoup product
//             costs ~8 IMAD-pipe slots (tools/pipes_bench.cu).  A product mod p is 6
//             exact FP64 ops; values stay unreduced and signed between stages (< 2^47).
//
// N = 2^15 rows do not fit one CTA's shared memory; they run on a 2-CTA cluster
// (forward_split / inverse_split): the only cross-half stage (s = 0) is folded into
// the forward's loads (each CTA reads both halves) and into the inverse's epilogue
// (each CTA reads the peer's half through distributed shared memory).  Within a half,
// stage s' of the local transform uses global twiddle (2 + h) * 2^s' + block, so the
// same engine runs with a twiddle base multiplier c0 = 2 + h (c0 = 1 otherwise).
//
// Interfaces chosen so that callers can fuse prologues/epilogues:
//   forward: input through a functor load(idx) (coalesced across threads), output
//            left in registers in line-pair order (lpos below) of its row (of its half
//            for split rows);
//   inverse: input given in registers in that same layout, output through a functor
//            store(idx, value) (coalesced).
// All values handed to the caller are canonical residues.
#pragma once
#include <cooperative_groups.h>

#include "modarith.cuh"

namespace ntt {

HD int pad(int i) { return i + (i >> 4); }
// Register layout at the engine boundary ("line pairs"): thread t of T holds positions
// 2t + (m & 1) + 2T (m >> 1), m < E -- every warp-wide 16-byte access covers 512
// contiguous bytes.  The radix-E groups themselves work on E contiguous positions per
// thread, so the forward's last group and the inverse's first group transpose through
// shared memory (conflict-free with the padded index).
HD int lpos(int t, int m, int T) { return 2 * t + (m & 1) + 2 * T * (m >> 1); }

template <int LOGN, int E = 16>
struct Shape {
    static_assert(E == 8 || E == 16 || E == 32, "8, 16 or 32 elements per thread");
    static constexpr int LOGE = E == 8 ? 3 : (E == 16 ? 4 : 5);
    static constexpr int N = 1 << LOGN;
    static constexpr int T = N / E;
    static constexpr int REM = LOGN % LOGE;
    static constexpr int G = LOGN / LOGE;
    static constexpr int SMEM_WORDS = N + N / 16;
};

// ---------------------------------------------------------------- arithmetic ----
struct IntArith {
    using V = u64;
    using W = ulonglong2;
#ifndef INT_THROTTLE
#define INT_THROTTLE 0
#endif
    // >0: compiler barrier every THROTTLE butterflies (bounds twiddle-load hoisting)
    static constexpr int THROTTLE = INT_THROTTLE;
    u64 p, p2;
    HD explicit IntArith(u64 p_) : p(p_), p2(2 * p_) {}
    HD V in(u64 x) const { return x; }
    HD void fwd(V &a, V &b, W w) const {  // a, b in [0,4p) -> [0,4p)
        const u64 x = csub(a, p2);
        const u64 t = shoup_lazy(b, w.x, w.y, p);
        a = x + t;
        b = x - t + p2;
    }
    HD void inv(V &a, V &b, W w) const {  // [0,2p) -> [0,2p)
        const u64 x = a, y = b;
        a = csub(x + y, p2);
        b = shoup_lazy(x - y + p2, w.x, w.y, p);
    }
    HD void inv_last(V &a, V &b, W u, W v) const {  // final stage, canonical outputs
        const u64 x = a, y = b;
        a = shoup(x + y, u.x, u.y, p);
        b = shoup(x - y + p2, v.x, v.y, p);
    }
    HD u64 out_fwd(V x) const { return csub(csub(x, p2), p); }
    HD u64 out_inv(V x) const { return x; }
    HD V to_smem_inv(V x) const { return x; }
    HD V split_fwd(V a, V b, W w1, int h) const {  // stage 0 for half h, a,b in [0,2p)
        const u64 t = shoup_lazy(b, w1.x, w1.y, p);
        return h ? a - t + p2 : a + t;
    }
};

#define FP_MAGIC 6755399441055744.0  // 1.5 * 2^52

HD double u2d(u64 v) { return __longlong_as_double((long long)(0x4330000000000000ull | v)) - 4503599627370496.0; }
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

struct FpArith {
    using V = double;
    using W = double;
    static constexpr int THROTTLE = 0;
    double p, pinv;
    HD FpArith(double p_, double pinv_) : p(p_), pinv(pinv_) {}
    HD V in(u64 x) const { return u2d(x); }
    HD void fwd(V &a, V &b, W w) const {
        const double r = fmul(b, w, p, pinv);
        b = a - r;
        a = a + r;
    }
    HD void inv(V &a, V &b, W w) const {
        const double x = a, y = b;
        a = x + y;
        b = fmul(x - y, w, p, pinv);
    }
    HD void inv_last(V &a, V &b, W u, W v) const {
        const double x = a, y = b;
        a = fmul(x + y, u, p, pinv);
        b = fmul(x - y, v, p, pinv);
    }
    HD u64 out_fwd(V x) const { return fcanon(x, p, pinv); }
    HD u64 out_inv(V x) const { return fcanon(x, p, pinv); }
    // the inverse's additive path grows by up to 2^RB per group: re-centre at exchanges
    HD V to_smem_inv(V x) const { return fred(x, p, pinv); }
    HD V split_fwd(V a, V b, W w1, int h) const {
        const double r = fmul(b, w1, p, pinv);
        return h ? a - r : a + r;
    }
};

// FP64 engine whose forward hands out raw (unreduced, signed, |v| < 2^47) doubles as bit
// patterns instead of canonical residues: for consumers that multiply the transform by
// fmul right away (fmul accepts such operands), e.g. the fused ModUp key products.
struct FpArithRaw : FpArith {
    HD FpArithRaw(double p_, double pinv_) : FpArith(p_, pinv_) {}
    HD u64 out_fwd(V x) const { return (u64)__double_as_longlong(x); }
};
// ... and whose forward also takes raw doubles (bit patterns, |v| < 2^47) as input
struct FpArithRawIO : FpArithRaw {
    HD FpArithRawIO(double p_, double pinv_) : FpArithRaw(p_, pinv_) {}
    HD V in(u64 x) const { return __longlong_as_double((long long)x); }
};

// ---------------------------------------------------------------- forward ----
// One forward group: radix 2^RB covering stages S0 .. S0+RB-1.
// SRC: 0 = functor load, 1 = shared memory.  DST: 0 = shared memory, 1 = registers.
template <int LOGN, int E, int RB, int S0, int SRC, int DST, class A, class Load>
HD void fwd_group(const A &ar, typename A::V *sm, const typename A::W *__restrict__ tw, int c0, Load &load,
                  u64 (&out)[E]) {
    using S = Shape<LOGN, E>;
    using V = typename A::V;
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
        V x[R];
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const int idx = base + (m << LB);
            if constexpr (SRC == 0) x[m] = ar.in(load(idx));
            else x[m] = sm[pad(idx)];
        }
#pragma unroll
        for (int q = 0; q < RB; ++q) {
            const int half = R >> (q + 1);
#pragma unroll
            for (int m = 0; m < R; ++m) {
                if (m & half) continue;
                const auto w = __ldg(tw + (c0 << (S0 + q)) + (uhigh << q) + (m >> (RB - q)));
                ar.fwd(x[m], x[m + half], w);
                if constexpr (A::THROTTLE > 0) {
                    if ((m % A::THROTTLE) == A::THROTTLE - 1) asm volatile("" ::: "memory");
                }
            }
        }
        if constexpr (DST == 1) {
            static_assert(UPT == 1 && R == E && LB == 0, "register output needs one radix-E unit per thread");
            // in place (this unit's own positions), then read back in line-pair order
#pragma unroll
            for (int m = 0; m < R; ++m) sm[pad(base + m)] = x[m];
            __syncthreads();
#pragma unroll
            for (int m = 0; m < R; ++m) out[m] = ar.out_fwd(sm[pad(lpos(tid, m, S::T))]);
        } else {
#pragma unroll
            for (int m = 0; m < R; ++m) sm[pad(base + (m << LB))] = x[m];
        }
    }
}

template <int LOGN, int E, int GI, bool FS, class A, class Load>
HD void fwd_main_groups(const A &ar, typename A::V *sm, const typename A::W *__restrict__ tw, int c0, Load &load,
                        u64 (&out)[E]) {
    using S = Shape<LOGN, E>;
    constexpr int S0 = S::REM + S::LOGE * GI;
    constexpr bool first = (S0 == 0) && !FS;
    constexpr bool last = (GI == S::G - 1);
    fwd_group<LOGN, E, S::LOGE, S0, first ? 0 : 1, last ? 1 : 0>(ar, sm, tw, c0, load, out);
    if constexpr (!last) {
        __syncthreads();
        fwd_main_groups<LOGN, E, GI + 1, FS>(ar, sm, tw, c0, load, out);
    }
}

// FS: the input is already in shared memory (split rows) instead of behind `load`.
template <int LOGN, int E, bool FS, class A, class Load>
__device__ void forward_core(const A &ar, typename A::V *sm, const typename A::W *__restrict__ tw, int c0, Load load,
                             u64 (&out)[E]) {
    using S = Shape<LOGN, E>;
    static_assert(LOGN >= 6 && LOGN <= 14, "one CTA covers N = 64 .. 16384");
    if constexpr (S::REM) {
        fwd_group<LOGN, E, S::REM, 0, FS ? 1 : 0, 0>(ar, sm, tw, c0, load, out);
        __syncthreads();
    }
    fwd_main_groups<LOGN, E, 0, FS>(ar, sm, tw, c0, load, out);
}

// Forward NTT of one row held by one CTA.
template <int LOGN, int E = 16, class A, class Load>
__device__ void forward(const A &ar, typename A::V *sm, const typename A::W *__restrict__ tw, Load load,
                        u64 (&out)[E]) {
    __syncthreads();  // shared memory may still be read by a previous transform
    forward_core<LOGN, E, false>(ar, sm, tw, 1, load, out);
}

// Forward NTT of a 2^(LL+1) row split over a 2-CTA cluster; this CTA (half h) ends
// with positions h*2^LL + E t .. + E-1 in registers.  load(idx) takes global indices.
template <int LL, int E = 16, class A, class Load>
__device__ void forward_split(const A &ar, typename A::V *sm, const typename A::W *__restrict__ tw, Load load,
                              u64 (&out)[E], int h) {
    using S = Shape<LL, E>;
    __syncthreads();
    const auto w1 = __ldg(tw + 1);
    constexpr int half = 1 << LL;
    for (int j = threadIdx.x; j < half; j += S::T)
        sm[pad(j)] = ar.split_fwd(ar.in(load(j)), ar.in(load(j + half)), w1, h);
    __syncthreads();
    forward_core<LL, E, true>(ar, sm, tw, 2 + h, load, out);
}

// ---------------------------------------------------------------- inverse ----
// SRC: 1 = registers, 0 = shared memory.  DST: 0 = shared memory, 1 = functor store.
// LASTS: this group contains global stage 0 (fold n^-1 and canonicalise).
template <int LOGN, int E, int RB, int S0, int SRC, int DST, bool LASTS, class A, class Store>
HD void inv_group(const A &ar, typename A::V *sm, const typename A::W *__restrict__ itw, int c0, const u64 (&in)[E],
                  Store &store, typename A::W last_u, typename A::W last_v) {
    using S = Shape<LOGN, E>;
    using V = typename A::V;
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
        V x[R];
        if constexpr (SRC == 1) {
            static_assert(UPT == 1 && R == E && LB == 0, "register input needs one radix-E unit per thread");
            // line-pair order in registers -> this unit's contiguous positions
#pragma unroll
            for (int m = 0; m < R; ++m) sm[pad(lpos(tid, m, S::T))] = ar.in(in[m]);
            __syncthreads();
#pragma unroll
            for (int m = 0; m < R; ++m) x[m] = sm[pad(base + m)];
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
                if (LASTS && S0 + q == 0) {
                    ar.inv_last(x[m], x[m + half], last_u, last_v);
                } else {
                    const auto w = __ldg(itw + (c0 << (S0 + q)) + (uhigh << q) + (m >> (RB - q)));
                    ar.inv(x[m], x[m + half], w);
                    if constexpr (A::THROTTLE > 0) {
                        if ((m % A::THROTTLE) == A::THROTTLE - 1) asm volatile("" ::: "memory");
                    }
                }
            }
        }
        if constexpr (DST == 1) {
#pragma unroll
            for (int m = 0; m < R; ++m) store(base + (m << LB), ar.out_inv(x[m]));
        } else {
#pragma unroll
            for (int m = 0; m < R; ++m) sm[pad(base + (m << LB))] = ar.to_smem_inv(x[m]);
        }
    }
}

template <int LOGN, int E, int GI, bool NF, class A, class Store>
HD void inv_main_groups(const A &ar, typename A::V *sm, const typename A::W *__restrict__ itw, int c0,
                        const u64 (&in)[E], Store &store, typename A::W last_u, typename A::W last_v) {
    // GI counts down from G-1 (first inverse group, register input) to 0.
    using S = Shape<LOGN, E>;
    constexpr int S0 = S::REM + S::LOGE * GI;
    constexpr bool first = (GI == S::G - 1);
    constexpr bool last = (S0 == 0);
    inv_group<LOGN, E, S::LOGE, S0, first ? 1 : 0, (last && !NF) ? 1 : 0, !NF>(ar, sm, itw, c0, in, store, last_u,
                                                                            last_v);
    if constexpr (GI > 0) {
        __syncthreads();
        inv_main_groups<LOGN, E, GI - 1, NF>(ar, sm, itw, c0, in, store, last_u, last_v);
    }
}

// NF: "no final stage" -- the local transform of a split row; results stay in shared
// memory (re-centred) for the cross-half stage.
template <int LOGN, int E, bool NF, class A, class Store>
__device__ void inverse_core(const A &ar, typename A::V *sm, const typename A::W *__restrict__ itw, int c0,
                             const u64 (&in)[E], Store store, typename A::W last_u, typename A::W last_v) {
    using S = Shape<LOGN, E>;
    static_assert(LOGN >= 6 && LOGN <= 14, "one CTA covers N = 64 .. 16384");
    inv_main_groups<LOGN, E, S::G - 1, NF>(ar, sm, itw, c0, in, store, last_u, last_v);
    if constexpr (S::REM) {
        __syncthreads();
        inv_group<LOGN, E, S::REM, 0, 0, NF ? 0 : 1, !NF>(ar, sm, itw, c0, in, store, last_u, last_v);
    }
}

// Inverse NTT of one row.  Thread t supplies positions E t .. E t + E - 1 (values in
// [0, 2p)); results leave through store(idx, canonical value).  last_u = n^-1 * c and
// last_v = itw[1] * n^-1 * c for a caller-chosen output factor c.
template <int LOGN, int E = 16, class A, class Store>
__device__ void inverse(const A &ar, typename A::V *sm, const typename A::W *__restrict__ itw, const u64 (&in)[E],
                        Store store, typename A::W last_u, typename A::W last_v) {
    __syncthreads();
    inverse_core<LOGN, E, false>(ar, sm, itw, 1, in, store, last_u, last_v);
}

// Inverse NTT of a 2^(LL+1) row over a 2-CTA cluster (half h supplies positions
// h*2^LL + E t ..); store() receives global indices.  Stage 0 pairs (j, j + 2^LL)
// across the halves: CTA h finishes j in [h 2^(LL-1), (h+1) 2^(LL-1)) reading the
// peer half from distributed shared memory.
template <int LL, int E = 16, class A, class Store>
__device__ void inverse_split(const A &ar, typename A::V *sm, const typename A::W *__restrict__ itw,
                              const u64 (&in)[E], Store store, typename A::W last_u, typename A::W last_v, int h) {
    using S = Shape<LL, E>;
    using V = typename A::V;
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    __syncthreads();
    inverse_core<LL, E, true>(ar, sm, itw, 2 + h, in, store, last_u, last_v);
    cluster.sync();
    V *peer = cluster.map_shared_rank(sm, h ^ 1);
    const V *s0 = h ? peer : sm;
    const V *s1 = h ? sm : peer;
    constexpr int half = 1 << LL, quarter = half >> 1;
    for (int j = h * quarter + threadIdx.x; j < (h + 1) * quarter; j += S::T) {
        V a = s0[pad(j)], b = s1[pad(j)];
        ar.inv_last(a, b, last_u, last_v);
        store(j, ar.out_inv(a));
        store(j + half, ar.out_inv(b));
    }
    cluster.sync();  // the peer must not reuse its shared memory while it is being read
}

}  // namespace ntt
