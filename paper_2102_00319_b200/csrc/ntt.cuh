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
// Rows longer than one CTA's part (2^LL, see Row in common.cuh) run on an SP-CTA cluster
// (SP = 2 or 4; forward_split / inverse_split): the log2(SP) cross-part stages work
// column-wise over the parts' shared memories (distributed shared memory), the rest is
// local.  Within part r, stage s' of the local transform uses global twiddle
// (SP + r) * 2^s' + block, so the same engine runs with a twiddle base multiplier
// c0 = SP + r (c0 = 1 otherwise).
//
// Interfaces chosen so that callers can fuse prologues/epilogues:
//   forward: input through a functor load(idx) (coalesced across threads), output
//            left in registers in line-pair order (lpos below) of its row (of its part
//            for split rows);
//   inverse: input given in registers in that same layout, output through a functor
//            store(idx, value) (coalesced).
// All values handed to the caller are canonical residues.
#pragma once
#include <cooperative_groups.h>

#include "modarith.cuh"

// -DHEB_DEVICE_ASSERT=1: bounds asserts on every shared-memory and twiddle index of the
// engine and on the callers' global stores (compute-sanitizer is closed on the GPU pool,
// so this build is the memory checker; see tools/assert_check.sh)
#if defined(HEB_DEVICE_ASSERT) && HEB_DEVICE_ASSERT
#include <cassert>
#define NTT_ASSERT(c) assert(c)
#else
#define NTT_ASSERT(c) ((void)0)
#endif

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

// Twiddle tables hold 4N entries per row (TW_ROW_SHIFT): [0, N) psi^brv(i) in the reference's
// order; [N, 2N) the entries of the last radix-16 group of the full transform (first stage
// S = n - 4) regrouped lane-major, P_S[(2^q - 1 + i) 2^S + g] = tw[((2^S + g) << q) + i]
// for stage S + q, unit g: in that group every thread owns one unit and needs 15
// twiddles of its own; in the reference order a warp's loads of one (q, i) are strided by
// 8 * 2^q bytes (up to 16 lines per request), regrouped they are one contiguous 256-byte
// run (the group was bound by L1 wavefronts, not by the DFMA pipe);  [2N, 3N) the same
// for S = n - 5, the last local group of a parity-split row (forward_split_eo).
constexpr int TW_ROW_SHIFT = 2;
#ifndef NTT_TW_LANE_MAJOR
#define NTT_TW_LANE_MAJOR 1
#endif
// Address of the lane-major twiddles of unit u of this CTA in a last group (LOGN = this
// CTA's part, first stage S0 = LOGN - 4, c0 = its twiddle base multiplier); the entry of
// stage S0 + q, butterfly i is at [((1 << q) - 1 + i) * stride].  PERM 1: full-transform
// group of a row of SP parts (c0 = SP + part); PERM 2: parity-split local group.
template <int LOGN, int S0, int PERM, class W>
HD const W *lane_major_tw(const W *__restrict__ tw, int c0, int u, int &stride) {
    if constexpr (PERM == 2) {
        stride = 1 << S0;
        return tw + (size_t)(4 << LOGN) + u;  // row length 2 * 2^LOGN, region [2N, 3N)
    } else {
        const int sp = c0 >= 4 ? 4 : (c0 >= 2 ? 2 : 1);
        stride = sp << S0;
        return tw + (size_t)(sp << LOGN) + ((c0 - sp) << S0) + u;
    }
}

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

// Barrier over the NT consecutive threads around this thread (NT a power of two).  After
// the group that starts at stage S0 every later forward stage stays inside blocks of
// N / 2^S0 positions, and the thread -> unit map keeps a block with the same T / 2^S0
// consecutive threads in every group, so the exchange between two groups only needs
// those threads: the whole CTA, one named barrier per NT-thread slice, or just the warp.
// A CTA that is alone on its SM (N >= 2^14 parts) then stalls as a whole only around the
// first group and the boundary transposition instead of at every exchange.
#ifndef NTT_FINE_SYNC
#define NTT_FINE_SYNC 1
#endif
template <int T, int NT>
HD void sync_slice() {
    if constexpr (!NTT_FINE_SYNC || NT >= T) {
        __syncthreads();
    } else if constexpr (NT <= 32) {
        __syncwarp();
    } else if constexpr (T / NT > 4) {  // at most four named barriers (1..4) per CTA
        sync_slice<T, NT * 2>();
    } else {
        // immediate barrier numbers: a register operand makes ptxas reserve all 16 barriers
        const int s = (int)threadIdx.x / NT;
        if (s == 0) asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
        else if (s == 1) asm volatile("bar.sync 2, %0;" ::"n"(NT) : "memory");
        else if (s == 2) asm volatile("bar.sync 3, %0;" ::"n"(NT) : "memory");
        else asm volatile("bar.sync 4, %0;" ::"n"(NT) : "memory");
    }
}

// Cluster barrier halves for exchanges through (distributed) shared memory.
// cg::cluster_group::sync() compiles to MEMBAR.ALL.GPU + ERRBAR + CGAERRBAR before the
// arrive (release at cluster scope: every outstanding global access of the thread is
// waited for, 4% of the fused ModUp's stall samples at cfg4, ncu r2g) -- not needed when
// the only data handed over sits in this CTA's shared memory: a CTA barrier has performed
// the CTA's shared-memory writes, and the peer's loads reach this SM after the cluster
// barrier completes.  PUBLISH: this CTA wrote shared memory its peers will read.
#ifndef NTT_RELAXED_CLUSTER_SYNC
#define NTT_RELAXED_CLUSTER_SYNC 1
#endif
template <bool PUBLISH>
__device__ __forceinline__ void cluster_arrive_smem() {
#if NTT_RELAXED_CLUSTER_SYNC
    if constexpr (PUBLISH) __syncthreads();
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
#else
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
#endif
}
__device__ __forceinline__ void cluster_wait() {
#if NTT_RELAXED_CLUSTER_SYNC
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
#else
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
#endif
}
__device__ __forceinline__ unsigned long long word_bits(double v) { return (unsigned long long)__double_as_longlong(v); }
__device__ __forceinline__ unsigned long long word_bits(u64 v) { return v; }
// "This thread is done reading its peers' shared memory": the arrive must not be issued
// while a (remote) load is still in flight -- the peer may overwrite the location as soon
// as the barrier completes -- so it follows a shared-memory store whose data depends on
// every loaded word (the store cannot issue before the loads have returned); it goes to
// a scratch word per lane that nothing reads.
__device__ __forceinline__ unsigned ntt_scratch_addr() {
    __shared__ unsigned scratch[32];
    return (unsigned)__cvta_generic_to_shared(&scratch[threadIdx.x & 31]);
}
template <class V, int NA, int NB>
__device__ __forceinline__ void cluster_arrive_after_loads(V *sm, const V (&a)[NA], const V (&b)[NB]) {
#if NTT_RELAXED_CLUSTER_SYNC
    unsigned long long acc = 0;
#pragma unroll
    for (int i = 0; i < NA; ++i) acc |= word_bits(a[i]);
#pragma unroll
    for (int i = 0; i < NB; ++i) acc |= word_bits(b[i]);
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(ntt_scratch_addr()), "r"((unsigned)(acc >> 32) | (unsigned)acc) : "memory");
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
#else
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
#endif
}

// ---------------------------------------------------------------- forward ----
// One forward group: radix 2^RB covering stages S0 .. S0+RB-1.
// SRC: 0 = functor load, 1 = shared memory.  DST: 0 = shared memory, 1 = registers (line
// pairs), 2 = shared memory in place, natural order, for the last group (LB = 0), 3 = raw
// values of the unit's own positions in registers (last group).
template <int LOGN, int E, int RB, int S0, int SRC, int DST, int PERM, class A, class Load>
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
        constexpr bool LANE_MAJOR = NTT_TW_LANE_MAJOR && PERM != 0 && LB == 0 && RB == 4 && UPT == 1;
        int lm_stride = 0;
        const typename A::W *lm = nullptr;
        if constexpr (LANE_MAJOR) lm = lane_major_tw<LOGN, S0, PERM>(tw, c0, u, lm_stride);
        V x[R];
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const int idx = base + (m << LB);
            NTT_ASSERT(idx >= 0 && idx < S::N);
            if constexpr (SRC == 0) x[m] = ar.in(load(idx));
            else x[m] = sm[pad(idx)];
        }
#pragma unroll
        for (int q = 0; q < RB; ++q) {
            const int half = R >> (q + 1);
#pragma unroll
            for (int m = 0; m < R; ++m) {
                if (m & half) continue;
                NTT_ASSERT((c0 << (S0 + q)) + (uhigh << q) + (m >> (RB - q)) < 4 * S::N && uhigh < (1 << S0));
                typename A::W w;
                if constexpr (LANE_MAJOR) w = __ldg(lm + ((1 << q) - 1 + (m >> (RB - q))) * lm_stride);
                else w = __ldg(tw + (c0 << (S0 + q)) + (uhigh << q) + (m >> (RB - q)));
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
            for (int m = 0; m < R; ++m) {
                NTT_ASSERT(lpos(tid, m, S::T) < S::N && tid < S::T);
                out[m] = ar.out_fwd(sm[pad(lpos(tid, m, S::T))]);
            }
        } else if constexpr (DST == 3) {
            static_assert(UPT == 1 && R == E && LB == 0, "register output needs one radix-E unit per thread");
            // raw results of this unit's own positions base + m (natural order), no exchange
#pragma unroll
            for (int m = 0; m < R; ++m) out[m] = word_bits(x[m]);
        } else if constexpr (DST == 2) {
            static_assert(LB == 0, "in-place output is for the last group");
#pragma unroll
            for (int m = 0; m < R; ++m) sm[pad(base + m)] = x[m];
        } else {
#pragma unroll
            for (int m = 0; m < R; ++m) sm[pad(base + (m << LB))] = x[m];
        }
    }
}

template <int LOGN, int E, int GI, bool FS, int LASTDST, int PERM, class A, class Load>
HD void fwd_main_groups(const A &ar, typename A::V *sm, const typename A::W *__restrict__ tw, int c0, Load &load,
                        u64 (&out)[E]) {
    using S = Shape<LOGN, E>;
    constexpr int S0 = S::REM + S::LOGE * GI;
    constexpr bool first = (S0 == 0) && !FS;
    constexpr bool last = (GI == S::G - 1);
    fwd_group<LOGN, E, S::LOGE, S0, first ? 0 : 1, last ? LASTDST : 0, PERM>(ar, sm, tw, c0, load, out);
    if constexpr (!last) {
        sync_slice<S::T, (S::T >> (S0 < 16 ? S0 : 16))>();  // blocks of stage S0 (0: the whole row)
        fwd_main_groups<LOGN, E, GI + 1, FS, LASTDST, PERM>(ar, sm, tw, c0, load, out);
    }
}

// FS: the input is already in shared memory (split rows) instead of behind `load`.
// LASTDST: 1 = results in registers (line pairs), 2 = left in shared memory (natural order).
// PERM: which lane-major twiddle region the last group reads (see lane_major_tw).
template <int LOGN, int E, bool FS, int LASTDST = 1, int PERM = 1, class A, class Load>
__device__ void forward_core(const A &ar, typename A::V *sm, const typename A::W *__restrict__ tw, int c0, Load load,
                             u64 (&out)[E]) {
    using S = Shape<LOGN, E>;
    static_assert(LOGN >= 6 && LOGN <= 14, "one CTA covers N = 64 .. 16384");
    if constexpr (S::REM) {
        fwd_group<LOGN, E, S::REM, 0, FS ? 1 : 0, 0, 0>(ar, sm, tw, c0, load, out);
        __syncthreads();
    }
    fwd_main_groups<LOGN, E, 0, FS, LASTDST, PERM>(ar, sm, tw, c0, load, out);
}

// Forward NTT of one row held by one CTA.
template <int LOGN, int E = 16, class A, class Load>
__device__ void forward(const A &ar, typename A::V *sm, const typename A::W *__restrict__ tw, Load load,
                        u64 (&out)[E]) {
    __syncthreads();  // shared memory may still be read by a previous transform
    forward_core<LOGN, E, false>(ar, sm, tw, 1, load, out);
}

// Cross-CTA stages of a row split over SP = 2 or 4 CTAs (x[q] = the element of part q at
// one local index j): the first log2(SP) forward stages (CT), in place.
template <int SP, class A>
HD void cross_fwd(const A &ar, typename A::V (&x)[SP], const typename A::W *__restrict__ tw) {
    static_assert(SP == 2 || SP == 4, "2- or 4-CTA rows");
    const auto w1 = __ldg(tw + 1);
    if constexpr (SP == 2) {
        ar.fwd(x[0], x[1], w1);
    } else {
        ar.fwd(x[0], x[2], w1);
        ar.fwd(x[1], x[3], w1);
        ar.fwd(x[0], x[1], __ldg(tw + 2));
        ar.fwd(x[2], x[3], __ldg(tw + 3));
    }
}

// Forward NTT of a 2^LL * SP row split over an SP-CTA cluster (this CTA: part r).  Each
// CTA brings its own part into shared memory (load(idx) with global indices), then the
// cross-part stages run column-wise through distributed shared memory -- CTA r owns local
// columns [r C, (r+1) C), C = 2^LL / SP, reading the column's SP elements (one local) and
// writing them back, so every location has one reader/writer -- and the rest of the
// transform is local (global stage s = log2(SP) + s' uses twiddle (SP + r) 2^s' + block).
// Ends with positions r 2^LL + lpos(t, m) in registers.
template <int LL, int E, int SP, class A>
__device__ void split_cross_and_local(const A &ar, typename A::V *sm, const typename A::W *__restrict__ tw,
                                      u64 (&out)[E], int r) {
    using S = Shape<LL, E>;
    using V = typename A::V;
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();  // every part is in its CTA's shared memory
    V *parts[SP];
#pragma unroll
    for (int q = 0; q < SP; ++q) parts[q] = cluster.map_shared_rank(sm, q);
    constexpr int C = (1 << LL) / SP;
#pragma unroll 2
    for (int j = r * C + (int)threadIdx.x; j < (r + 1) * C; j += S::T) {
        const int i = pad(j);
        V x[SP];
#pragma unroll
        for (int q = 0; q < SP; ++q) x[q] = parts[q][i];
        cross_fwd<SP>(ar, x, tw);
#pragma unroll
        for (int q = 0; q < SP; ++q) parts[q][i] = x[q];
    }
    cluster.sync();  // every column written
    int dummy = 0;
    auto noload = [&](int) { return (u64)dummy; };
    forward_core<LL, E, true>(ar, sm, tw, SP + r, noload, out);
}

// Cross-part stages for one CTA's own output only (part r of SP): 1 (SP = 2) or 3
// (SP = 4) products per element instead of a full column.
template <int SP, class A>
HD typename A::V cross_fwd_part(const A &ar, typename A::V (&x)[SP], const typename A::W *__restrict__ tw, int r) {
    const auto w1 = __ldg(tw + 1);
    if constexpr (SP == 2) {
        ar.fwd(x[0], x[1], w1);
        return r ? x[1] : x[0];
    } else {
        const int h = r >> 1;
        ar.fwd(x[0], x[2], w1);
        ar.fwd(x[1], x[3], w1);
        typename A::V y0 = h ? x[2] : x[0], y1 = h ? x[3] : x[1];
        ar.fwd(y0, y1, __ldg(tw + 2 + h));
        return (r & 1) ? y1 : y0;
    }
}

// Forward NTT of a 2^LL * SP row split over SP CTAs (this CTA: part r), without any
// cross-CTA synchronisation: each CTA reads the SP elements of every one of its columns
// from global memory (load(idx) takes global indices), forms its own part of the
// cross-part stages, then runs the local stages.
template <int LL, int E = 16, int SP = 2, class A, class Load>
__device__ void forward_split(const A &ar, typename A::V *sm, const typename A::W *__restrict__ tw, Load load,
                              u64 (&out)[E], int r) {
    using S = Shape<LL, E>;
    using V = typename A::V;
    __syncthreads();  // shared memory may still be read by a previous transform
    constexpr int PER = (1 << LL) / S::T;
#pragma unroll 4
    for (int k = 0; k < PER; ++k) {
        const int j = (int)threadIdx.x + k * S::T;
        V x[SP];
#pragma unroll
        for (int q = 0; q < SP; ++q) x[q] = ar.in(load((q << LL) + j));
        sm[pad(j)] = cross_fwd_part<SP>(ar, x, tw, r);
    }
    __syncthreads();
    forward_core<LL, E, true>(ar, sm, tw, SP + r, load, out);
}

// The same transform when this CTA's part was staged into shared memory as raw 64-bit
// words by cp.async (thread t copied positions t, t + T, ...): each thread converts its
// own copies in place (conv.conv(raw) -> residue) once they have landed.
template <int LL, int E = 16, int SP = 2, class A, class Conv>
__device__ void forward_split_staged(const A &ar, typename A::V *sm, const typename A::W *__restrict__ tw,
                                     const Conv &conv, u64 (&out)[E], int r) {
    using S = Shape<LL, E>;
    asm volatile("cp.async.wait_all;" ::: "memory");
    const long long *raw = reinterpret_cast<const long long *>(sm);
#pragma unroll 4
    for (int j = threadIdx.x; j < (1 << LL); j += S::T) {
        const int i = pad(j);
        sm[i] = ar.in(conv.conv(raw[i]));
    }
    split_cross_and_local<LL, E, SP>(ar, sm, tw, out, r);
}

// Forward NTT of a 2^(LL+1) row split over a 2-CTA cluster by the PARITY of the position:
// CTA r holds positions 2j' + r at local index j' of its shared memory (already converted
// to A::V).  Stage s < LL pairs positions that differ in bit LL - s >= 1, so it stays
// inside a parity class and is stage s of a 2^LL transform over the local indices with
// the row's own twiddles (block j >> (LL + 1 - s) = j' >> (LL - s)): the local engine
// runs unchanged with c0 = 1.  Only the last stage crosses the CTAs: it pairs (2b, 2b + 1)
// = (CTA 0's b, CTA 1's b) with twiddle tw[2^LL + b].  CTA r finishes the pairs
// b in [r 2^(LL-1), (r+1) 2^(LL-1)) -- one value local, one read through distributed
// shared memory -- which are exactly positions r 2^LL + lpos(t, m) of the row.  Every
// input element is read by one CTA only (forward_split reads each column twice) and no
// butterfly is computed twice.  The closing cluster barrier keeps each CTA's shared
// memory alive until its peer has read it.
template <int LL, int E = 16, class A, class Hook>
__device__ void forward_split_eo(const A &ar, typename A::V *sm, const typename A::W *__restrict__ tw, u64 (&out)[E],
                                 int r, Hook after_last_stage) {
    using S = Shape<LL, E>;
    using V = typename A::V;
    using W = typename A::W;
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    int dummy = 0;
    auto noload = [&](int) { return (u64)dummy; };
    forward_core<LL, E, true, 2, 2>(ar, sm, tw, 1, noload, out);
    cluster_arrive_smem<true>();  // this CTA's parity class is complete
    const V *peer = cluster.map_shared_rank(sm, r ^ 1);
    constexpr int H = (1 << LL) / 2;
    static_assert(H == (E / 2) * S::T, "E/2 pairs per thread");
    V mine[E / 2], other[E / 2];
    W w[E / 2];
    // the local halves of the pairs and the last stage's twiddles do not need the peer
#pragma unroll
    for (int i = 0; i < E / 2; ++i) mine[i] = sm[pad(r * H + (int)threadIdx.x + S::T * i)];
#pragma unroll
    for (int i = 0; i < E / 2; ++i) w[i] = __ldg(tw + (1 << LL) + r * H + (int)threadIdx.x + S::T * i);
    cluster_wait();  // ... and so is the peer's
#pragma unroll
    for (int i = 0; i < E / 2; ++i) other[i] = peer[pad(r * H + (int)threadIdx.x + S::T * i)];
    // both operands have arrived before the peer is told it may reuse its shared memory
    cluster_arrive_after_loads(sm, other, mine);
#pragma unroll
    for (int i = 0; i < E / 2; ++i) {
        V u = r ? other[i] : mine[i], v = r ? mine[i] : other[i];
        ar.fwd(u, v, w[i]);
        out[2 * i] = ar.out_fwd(u);
        out[2 * i + 1] = ar.out_fwd(v);
    }
    after_last_stage();  // the caller's loads for what follows: in flight during the barrier wait
    cluster_wait();      // the peer has read this CTA's results: shared memory may be reused
}
template <int LL, int E = 16, class A>
__device__ void forward_split_eo(const A &ar, typename A::V *sm, const typename A::W *__restrict__ tw, u64 (&out)[E],
                                 int r) {
    forward_split_eo<LL, E>(ar, sm, tw, out, r, [] {});
}

// The same transform with the cross-CTA stage fed by PUSHES instead of remote loads
// (NTT_PUSH_XCHG).  After the last local group every thread holds the 16 results of its
// own unit (local indices 16 t .. 16 t + 15) in registers.  The CTA that finishes a pair
// range needs both parity classes of it: results of this CTA's own range stay in place,
// results of the peer's range are sent to the peer's receive region (behind the
// transform buffer) with st.async, which counts the bytes on the receiver's mbarrier as
// they land.  Against forward_split_eo (remote loads between two cluster barriers: 16%
// of the FP64 launch in the exchange plus 6% in MEMBAR / ERRBAR / UCGABAR, ncu r2g): no
// cluster barrier and no fence in the loop, no load latency over the SM-to-SM network
// (the stores are fire-and-forget and start as each warp finishes its group), no L1
// invalidation (barrier.cluster.wait carries a CCTL.IVALL, which drops the twiddles).
// Protocol per exchange #seq (both CTAs run the same sequence):
//   full  (receiver's): 1 arrival (its thread 0, arrive.expect_tx of 2^LL / 2 words)
//                       + the bytes pushed by the peer; waited with parity seq & 1;
//   free  (sender's):   1 arrival per exchange, made remotely by the receiver once all
//                       its threads have read the receive region; a sender waits for
//                       exchange seq - 1's before it pushes again.
namespace xchg {
__device__ __forceinline__ uint32_t bar_addr(int which) {
    __shared__ __align__(8) unsigned long long bars[2];
    return (uint32_t)__cvta_generic_to_shared(&bars[which]);
}
__device__ __forceinline__ uint32_t peer_addr(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void wait_parity(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n XW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @p bra XD;\n bra XW;\n XD:\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
// Once per CTA before the first exchange: the barriers exist cluster-wide before anything
// is sent to them.
__device__ __forceinline__ void init() {
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_addr(0)) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_addr(1)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Before the CTA exits: the peer's last (remote) arrival on this CTA's barrier has landed.
__device__ __forceinline__ void fini() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
template <int LL, int E>
constexpr size_t recv_words() {
    return (size_t)((1 << LL) / 2 + (1 << LL) / 32);
}
}  // namespace xchg

template <int LL, int E = 16, class A>
__device__ void forward_split_eo_push(const A &ar, typename A::V *sm, const typename A::W *__restrict__ tw,
                                      u64 (&out)[E], int r, int seq) {
    using S = Shape<LL, E>;
    using V = typename A::V;
    using W = typename A::W;
    static_assert(E == 16 && sizeof(V) == 8, "16 eight-byte results per thread");
    constexpr int H = (1 << LL) / 2;
    static_assert(H == (E / 2) * S::T, "E/2 pairs per thread");
    V *recv = sm + S::SMEM_WORDS;
    int dummy = 0;
    auto noload = [&](int) { return (u64)dummy; };
    forward_core<LL, E, true, 3, 2>(ar, sm, tw, 1, noload, out);
    const int base = E * (int)threadIdx.x;  // this thread's unit: local indices base .. base + 15
    const uint32_t full = xchg::bar_addr(0), fre = xchg::bar_addr(1);
    if (threadIdx.x == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full), "r"((uint32_t)(H * 8)) : "memory");
    if ((base >= H) == (r != 0)) {  // warp-uniform: this CTA finishes these pairs itself
#pragma unroll
        for (int m = 0; m < E; ++m) reinterpret_cast<u64 *>(sm)[pad(base + m)] = out[m];
    } else {
        if (seq > 0) xchg::wait_parity(fre, (uint32_t)((seq - 1) & 1));  // the peer has read the previous push
        const uint32_t pfull = xchg::peer_addr(full, (uint32_t)(r ^ 1));
        const uint32_t precv = xchg::peer_addr((uint32_t)__cvta_generic_to_shared(recv), (uint32_t)(r ^ 1));
        const int idx = base - (r ? 0 : H);  // index inside the peer's pair range
        const uint32_t dst = precv + 8u * (uint32_t)pad(idx);  // pad(idx + m) = pad(idx) + m for m < 16
#pragma unroll
        for (int m = 0; m < E; ++m)
            asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(dst + 8u * m),
                         "l"(out[m]), "r"(pfull)
                         : "memory");
    }
    __syncthreads();  // the in-place results are visible to the whole CTA
    V mine[E / 2], other[E / 2];
    W w[E / 2];
#pragma unroll
    for (int i = 0; i < E / 2; ++i) mine[i] = sm[pad(r * H + (int)threadIdx.x + S::T * i)];
#pragma unroll
    for (int i = 0; i < E / 2; ++i) w[i] = __ldg(tw + (1 << LL) + r * H + (int)threadIdx.x + S::T * i);
    xchg::wait_parity(full, (uint32_t)(seq & 1));  // the peer's half of every pair has landed
#pragma unroll
    for (int i = 0; i < E / 2; ++i) other[i] = recv[pad((int)threadIdx.x + S::T * i)];
#pragma unroll
    for (int i = 0; i < E / 2; ++i) {
        V u = r ? other[i] : mine[i], v = r ? mine[i] : other[i];
        ar.fwd(u, v, w[i]);
        out[2 * i] = ar.out_fwd(u);
        out[2 * i + 1] = ar.out_fwd(v);
    }
    __syncthreads();  // every thread has read the buffer and the receive region: both may be reused
    if (threadIdx.x == 0)
        asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(xchg::peer_addr(fre, (uint32_t)(r ^ 1)))
                     : "memory");
}

// Push exchange with ONE bulk copy per exchange (cp.async.bulk shared::cta ->
// shared::cluster, completed on the receiver's mbarrier) instead of per-thread stores:
// the last local group leaves every result in place, and the padded half of the buffer
// that the peer finishes is copied into the peer's receive region as it lies (the
// receive region has the same padded layout).  8-byte st.async pushes from a thread's own
// unit are uncoalesced (one packet per word) and measured 26% slower than remote loads.
// The sender's buffer is being read by the copy engine until the receiver has seen all
// bytes, so the exchange ends by waiting for the peer's "consumed" arrival.
template <int LL, int E = 16, class A>
__device__ void forward_split_eo_bulk(const A &ar, typename A::V *sm, const typename A::W *__restrict__ tw,
                                      u64 (&out)[E], int r, int seq) {
    using S = Shape<LL, E>;
    using V = typename A::V;
    using W = typename A::W;
    constexpr int H = (1 << LL) / 2;
    static_assert(H == (E / 2) * S::T, "E/2 pairs per thread");
    constexpr uint32_t HALF_BYTES = 8u * (uint32_t)(H + H / 16);  // padded half of the buffer
    constexpr int CH = 4;                                          // copies per exchange
    static_assert(HALF_BYTES % (16 * CH) == 0, "16-byte granules");
    V *recv = sm + S::SMEM_WORDS;
    int dummy = 0;
    auto noload = [&](int) { return (u64)dummy; };
    forward_core<LL, E, true, 2, 2>(ar, sm, tw, 1, noload, out);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> visible to the copy engine
    __syncthreads();
    const uint32_t full = xchg::bar_addr(0), fre = xchg::bar_addr(1);
    if (threadIdx.x < CH) {
        if (threadIdx.x == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full), "r"(HALF_BYTES) : "memory");
        const uint32_t off = (uint32_t)threadIdx.x * (HALF_BYTES / CH);
        const uint32_t src = (uint32_t)__cvta_generic_to_shared(sm) + (uint32_t)(r ^ 1) * HALF_BYTES + off;
        const uint32_t dst = xchg::peer_addr((uint32_t)__cvta_generic_to_shared(recv) + off, (uint32_t)(r ^ 1));
        const uint32_t pfull = xchg::peer_addr(full, (uint32_t)(r ^ 1));
        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                     "r"(src), "r"(HALF_BYTES / CH), "r"(pfull)
                     : "memory");
    }
    V mine[E / 2], other[E / 2];
    W w[E / 2];
#pragma unroll
    for (int i = 0; i < E / 2; ++i) mine[i] = sm[pad(r * H + (int)threadIdx.x + S::T * i)];
#pragma unroll
    for (int i = 0; i < E / 2; ++i) w[i] = __ldg(tw + (1 << LL) + r * H + (int)threadIdx.x + S::T * i);
    xchg::wait_parity(full, (uint32_t)(seq & 1));  // the peer's half of every pair has landed
#pragma unroll
    for (int i = 0; i < E / 2; ++i) other[i] = recv[pad((int)threadIdx.x + S::T * i)];
#pragma unroll
    for (int i = 0; i < E / 2; ++i) {
        V u = r ? other[i] : mine[i], v = r ? mine[i] : other[i];
        ar.fwd(u, v, w[i]);
        out[2 * i] = ar.out_fwd(u);
        out[2 * i + 1] = ar.out_fwd(v);
    }
    __syncthreads();  // every thread has read the buffer and the receive region
    if (threadIdx.x == 0)
        asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(xchg::peer_addr(fre, (uint32_t)(r ^ 1)))
                     : "memory");
    xchg::wait_parity(fre, (uint32_t)(seq & 1));  // the peer has everything: this CTA's buffer may be reused
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
        // the first inverse group (register input) is the forward's last group mirrored
        constexpr bool LANE_MAJOR = NTT_TW_LANE_MAJOR && SRC == 1 && LB == 0 && RB == 4 && UPT == 1 && !(LASTS && S0 == 0);
        int lm_stride = 0;
        const typename A::W *lm = nullptr;
        if constexpr (LANE_MAJOR) lm = lane_major_tw<LOGN, S0, 1>(itw, c0, u, lm_stride);
        V x[R];
        if constexpr (SRC == 1) {
            static_assert(UPT == 1 && R == E && LB == 0, "register input needs one radix-E unit per thread");
            // line-pair order in registers -> this unit's contiguous positions
#pragma unroll
            for (int m = 0; m < R; ++m) {
                NTT_ASSERT(lpos(tid, m, S::T) < S::N && tid < S::T);
                sm[pad(lpos(tid, m, S::T))] = ar.in(in[m]);
            }
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
                    NTT_ASSERT((c0 << (S0 + q)) + (uhigh << q) + (m >> (RB - q)) < 4 * S::N && uhigh < (1 << S0));
                    typename A::W w;
                    if constexpr (LANE_MAJOR) w = __ldg(lm + ((1 << q) - 1 + (m >> (RB - q))) * lm_stride);
                    else w = __ldg(itw + (c0 << (S0 + q)) + (uhigh << q) + (m >> (RB - q)));
                    ar.inv(x[m], x[m + half], w);
                    if constexpr (A::THROTTLE > 0) {
                        if ((m % A::THROTTLE) == A::THROTTLE - 1) asm volatile("" ::: "memory");
                    }
                }
            }
        }
        if constexpr (DST == 1) {
#pragma unroll
            for (int m = 0; m < R; ++m) {
                NTT_ASSERT(base + (m << LB) >= 0 && base + (m << LB) < S::N);
                store(base + (m << LB), ar.out_inv(x[m]));
            }
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
        // the next group (first stage S0 - LOGE) reads inside blocks of that stage
        sync_slice<S::T, (S::T >> (S0 - S::LOGE < 16 ? S0 - S::LOGE : 16))>();
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

// Last log2(SP) inverse stages of a split row (GS, global stages log2(SP)-1 .. 0; the
// final one folds n^-1 and the caller's output factor: inv_last with last_u / last_v).
template <int SP, class A>
HD void cross_inv(const A &ar, typename A::V (&x)[SP], const typename A::W *__restrict__ itw, typename A::W last_u,
                  typename A::W last_v) {
    static_assert(SP == 2 || SP == 4, "2- or 4-CTA rows");
    if constexpr (SP == 2) {
        ar.inv_last(x[0], x[1], last_u, last_v);
    } else {
        ar.inv(x[0], x[1], __ldg(itw + 2));
        ar.inv(x[2], x[3], __ldg(itw + 3));
        ar.inv_last(x[0], x[2], last_u, last_v);
        ar.inv_last(x[1], x[3], last_u, last_v);
    }
}

// Inverse NTT of a 2^LL * SP row over an SP-CTA cluster (part r supplies positions
// r 2^LL + lpos(t, m)).  The local stages run first (results left in shared memory), then
// CTA r finishes local columns [r C, (r+1) C) across all parts through distributed shared
// memory and stores all SP outputs of each column: store(idx, v) gets global indices.
template <int LL, int E = 16, int SP = 2, class A, class Store>
__device__ void inverse_split(const A &ar, typename A::V *sm, const typename A::W *__restrict__ itw,
                              const u64 (&in)[E], Store store, typename A::W last_u, typename A::W last_v, int r) {
    using S = Shape<LL, E>;
    using V = typename A::V;
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    __syncthreads();
    inverse_core<LL, E, true>(ar, sm, itw, SP + r, in, store, last_u, last_v);
    cluster_arrive_smem<true>();  // this part's local stages are in shared memory
    cluster_wait();
    const V *parts[SP];
#pragma unroll
    for (int q = 0; q < SP; ++q) parts[q] = cluster.map_shared_rank(sm, q);
    constexpr int C = (1 << LL) / SP;
#pragma unroll 2
    for (int j = r * C + (int)threadIdx.x; j < (r + 1) * C; j += S::T) {
        const int i = pad(j);
        V x[SP];
#pragma unroll
        for (int q = 0; q < SP; ++q) x[q] = parts[q][i];
        cross_inv<SP>(ar, x, itw, last_u, last_v);
#pragma unroll
        for (int q = 0; q < SP; ++q) store((q << LL) + j, ar.out_inv(x[q]));
    }
    // The peers must not reuse their shared memory while it is being read.  Every loaded
    // word has been consumed by a store issued above (memory operations do not move across
    // the arrive), so no load of this thread is still in flight here.
    cluster_arrive_smem<false>();
    cluster_wait();
}

}  // namespace ntt
