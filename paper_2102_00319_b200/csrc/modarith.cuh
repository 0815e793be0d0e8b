// modarith.cuh -- 64-bit modular arithmetic for sm_100a.
//
// Representation contract (reference kernels.py:1-13):
// every stored residue is x*2^64 mod p in [0, p) ("Montgomery form"), p < 2^62.
// Inside kernels we use whichever reduction is cheapest and only promise the
// *canonical* value at the boundary, so results are bit-identical to the
// reference's Montgomery-only arithmetic:
//   * Shoup multiplication by a constant w (precomputed w' = floor(w*2^64/p)):
//     one mulhi + two low products, result in [0, 2p) for ANY 64-bit input,
//     which also performs the true reduction of out-of-range digits;
//   * Montgomery REDC (R = 2^64) for products of two variables;
//   * lazy 128-bit accumulation of products, reduced once.
#pragma once
#include <cstdint>

typedef uint64_t u64;
typedef int64_t i64;
typedef uint32_t u32;

#define HD __device__ __forceinline__

HD u64 csub(u64 x, u64 m) { return x >= m ? x - m : x; }
HD u64 add_mod(u64 x, u64 y, u64 p) { return csub(x + y, p); }
HD u64 sub_mod(u64 x, u64 y, u64 p) { return csub(x + p - y, p); }

// x*w mod p in [0, 2p), any x < 2^64 (Shoup / Harvey).
HD u64 shoup_lazy(u64 x, u64 w, u64 ws, u64 p) {
    u64 q = __umul64hi(x, ws);
    return x * w - q * p;
}
HD u64 shoup(u64 x, u64 w, u64 ws, u64 p) { return csub(shoup_lazy(x, w, ws, p), p); }

// Montgomery product x*y*2^-64 mod p, canonical; needs x*y < p*2^64.
HD u64 mont_mul(u64 x, u64 y, u64 p, u64 pinv) {
    u64 lo = x * y, hi = __umul64hi(x, y);
    u64 m = lo * pinv;
    u64 t = hi + __umul64hi(m, p) + (lo != 0);
    return csub(t, p);
}

// 128-bit accumulator of products.
struct acc128 {
    u64 lo, hi;
};
HD void mac(acc128 &a, u64 x, u64 y) {
    u64 lo = x * y, hi = __umul64hi(x, y);
    u64 s = a.lo + lo;
    a.hi += hi + (s < lo);
    a.lo = s;
}
// Same accumulation with four 32-bit limbs and carry-chained mad.lo/mad.hi: the
// 64x64 -> 128 product is formed once (no separate low/high recomputation), ~1.5x
// the throughput of mac() on sm_100a (measured, tools/pipes_bench.cu).
struct acc4 {
    u32 w0, w1, w2, w3;
};
HD void mac4(acc4 &a, u64 x, u64 y) {
    const u32 x0 = (u32)x, x1 = (u32)(x >> 32), y0 = (u32)y, y1 = (u32)(y >> 32);
    asm("mad.lo.cc.u32  %0, %4, %6, %0;\n\t"
        "madc.hi.cc.u32 %1, %4, %6, %1;\n\t"
        "madc.lo.cc.u32 %2, %5, %7, %2;\n\t"
        "madc.hi.u32    %3, %5, %7, %3;\n\t"
        "mad.lo.cc.u32  %1, %4, %7, %1;\n\t"
        "madc.hi.cc.u32 %2, %4, %7, %2;\n\t"
        "addc.u32       %3, %3, 0;\n\t"
        "mad.lo.cc.u32  %1, %5, %6, %1;\n\t"
        "madc.hi.cc.u32 %2, %5, %6, %2;\n\t"
        "addc.u32       %3, %3, 0;\n\t"
        : "+r"(a.w0), "+r"(a.w1), "+r"(a.w2), "+r"(a.w3)
        : "r"(x0), "r"(x1), "r"(y0), "r"(y1));
}
HD acc128 to128(acc4 a) {
    return acc128{((u64)a.w1 << 32) | a.w0, ((u64)a.w3 << 32) | a.w2};
}

// REDC of a 128-bit value T = hi*2^64 + lo: returns T * 2^-64 mod p, canonical.
// hi is first reduced with a Shoup step (w = 1), so any T < 2^128 is accepted.
HD u64 redc128(acc128 a, u64 p, u64 pinv, u64 r1s /* floor(2^64/p) */) {
    u64 hi = csub(a.hi - __umul64hi(a.hi, r1s) * p, p);  // hi mod p
    u64 m = a.lo * pinv;
    u64 t = hi + __umul64hi(m, p) + (a.lo != 0);
    return csub(t, p);
}

// Signed (centered) integer v -> (v mod p) * w mod p, canonical, Python mod semantics.
HD u64 signed_mul_const(i64 v, u64 w, u64 ws, u64 p) {
    u64 mag = v < 0 ? (u64)(-v) : (u64)v;
    u64 r = shoup(mag, w, ws, p);
    return (v < 0 && r) ? p - r : r;
}

// Standard-form residue in [0, p) -> centered signed representative (kernels.py:200-212).
HD i64 center(u64 x, u64 p) { return x > (p >> 1) ? (i64)x - (i64)p : (i64)x; }

// Per-prime constants resident in device memory.
struct PrimeInfo {
    u64 p;
    u64 pinv;      // -p^-1 mod 2^64
    u64 r1s;       // floor(2^64 / p)   (Shoup of w = 1)
    u64 rmod, rmod_s;        // R mod p and its Shoup companion (std -> Montgomery)
    u64 rinv, rinv_s;        // R^-1 mod p  (Montgomery -> std)
    u64 ninv, ninv_s;        // n^-1 mod p
    u64 ninv_rinv, ninv_rinv_s;  // n^-1 * R^-1 mod p  (INTT + from-Montgomery)
    double pd, pinvd;            // p and 1/p as doubles (FP64 engine)
    u64 use_fp;                  // 1 if p < 2^42: NTTs of this row run on the FP64 pipe
    u64 pad[2];
};

