// conv.cu -- fused tensor-and-accumulate for an encrypted convolution layer.
//
// For every output cell (f, i, j) of a valid, strided, multi-channel convolution the
// layer needs the degree-2 raw product
//     raw = sum_{c,p,q} x[c][i*s+p][j*s+q] (x) w[f][c][p][q]
// (reference conv2d_enc, layers.py:92-127: one mul_ct_ct_raw + raw_add per tap).
// The tensor is pointwise in (row, position), so each (row r, position x) is an
// independent small convolution.  A CTA owns one row and XC consecutive positions:
//   * the weights of FG filters (all taps, both components) for those positions are
//     staged once in shared memory and reused by every output cell;
//   * SW warps-worth of workers stride over the output cells; each thread keeps FG
//     filters' three 128-bit accumulators in registers, so every input tap is loaded
//     once per cell and reused across the FG filters;
//   * products are summed lazily in 128 bits (Karatsuba: a0b0, a1b1,
//     (a0+a1)(b0+b1)) and reduced once per cell with Montgomery REDC, giving the
//     reference's canonical Montgomery residues exactly.
#include "common.cuh"

#include <cstdlib>

static bool getenv_flag(const char *name) {
    const char *v = getenv(name);
    return v && *v && *v != '0';
}

namespace {
// Positions per CTA (256 threads = positions x workers, a worker strides over the output
// cells).  Two widths are compiled: the wide one (512-byte warp accesses) while two CTAs'
// weight stages fit an SM's shared memory, the narrow one beyond that -- cfg4's second
// convolution (45 taps) stages 173 KB at the wide width, which leaves ONE 8-warp CTA per
// SM; at half the width two CTAs are resident (r2h: 78 -> ~52 ms per launch, while the
// 25-tap convolutions are 25% slower narrow).
#ifndef CONV_XC
#define CONV_XC 32  // wide width of the integer-row body (narrow: half)
#endif
#ifndef CONV_FGF
#define CONV_FGF 5
#endif
constexpr int FG = CONV_FGF;  // filters per CTA group
}  // namespace
#ifndef CONV_MINB
#define CONV_MINB 2
#endif
// taps whose inputs are in flight ahead of the one being multiplied (FP64 split-limb body)
#ifndef CONV_AHEAD
#define CONV_AHEAD 1
#endif

// One CTA = (row r, XC positions from bx * XC, filter group): integer rows (and, without
// the split-limb path, FP64 rows with one exact FP64 modular product per term).
// Output cells [cell_lo, cell_hi) of row r (the integer rows split their cells over
// several CTAs, see k_conv_tensor).
template <bool FLUSH, bool ALLOW_FP, int XC>
__device__ __forceinline__ void conv_body(u64 *wsm, const Ctx &K, const heb_ct &A, const heb_ct &B, const heb_ct &D,
                                          int C, int m, int n, int F, int P, int Q, int s, int om, int on, int logn,
                                          int flush, int bx, int r, int cell_lo, int cell_hi) {
    // wsm: [tap][fl][comp][XC]
    constexpr int SW = 256 / XC;  // workers per position
    const int xl = threadIdx.x % XC, w = threadIdx.x / XC;
    const int x = bx * XC + xl;
    const int f0 = blockIdx.z * FG;
    const int nf = min(FG, F - f0);
    const int taps = C * P * Q;
    const PrimeInfo Pr = K.pi[r];
    const u64 p = Pr.p;
    const int64_t roff = ((int64_t)r << logn) + x;

    // stage weights of filters f0 .. f0+nf-1 for positions [x0, x0+XC)
    for (int e = w; e < taps * nf; e += SW) {
        const int tap = e / nf, fl = e % nf;
        const int64_t widx = (int64_t)(f0 + fl) * taps + tap;
        const u64 *src = B.data + widx * B.ct_stride + roff;
        u64 *dst = wsm + ((size_t)(tap * FG + fl) * 2) * XC + xl;
        if (ALLOW_FP && Pr.use_fp) {  // FP64 rows: stage the weights as doubles
            dst[0] = (u64)__double_as_longlong(ntt::u2d(src[0]));
            dst[XC] = (u64)__double_as_longlong(ntt::u2d(src[B.comp_stride]));
        } else {
            dst[0] = src[0];
            dst[XC] = src[B.comp_stride];
        }
    }
    __syncthreads();

    const int cells = om * on;
    if (ALLOW_FP && Pr.use_fp) {
        // Rows with p < 2^42: every product reduced exactly on the FP64 pipe (6 ops),
        // sums exact below 2^47; one R^-1 product per output restores the Montgomery
        // factor of the reference's mont_mul accumulation.
        const double pd = Pr.pd, pinvd = Pr.pinvd, rinv = (double)Pr.rinv;
        const double *wd = reinterpret_cast<const double *>(wsm);
        for (int cell = cell_lo + w; cell < cell_hi; cell += SW) {
            const int i = cell / on, j = cell % on;
            double s0[FG], s1[FG], s2[FG];
#pragma unroll
            for (int fl = 0; fl < FG; ++fl) s0[fl] = s1[fl] = s2[fl] = 0.0;
            for (int c = 0; c < C; ++c) {
                for (int pp = 0; pp < P; ++pp) {
                    const int64_t rowcell = (int64_t)c * m * n + (int64_t)(i * s + pp) * n + j * s;
                    for (int qq = 0; qq < Q; ++qq) {
                        const int tap = (c * P + pp) * Q + qq;
                        const u64 *ap = A.data + (rowcell + qq) * A.ct_stride + roff;
                        const double a0 = ntt::u2d(__ldg(ap)), a1 = ntt::u2d(__ldg(ap + A.comp_stride));
                        const double sa = a0 + a1;
                        const double *wt = wd + (size_t)(tap * FG) * 2 * XC + xl;
#pragma unroll
                        for (int fl = 0; fl < FG; ++fl) {
                            if (fl < nf) {
                                const double b0 = wt[(2 * fl) * XC], b1 = wt[(2 * fl + 1) * XC];
                                s0[fl] += ntt::fmul(a0, b0, pd, pinvd);
                                s2[fl] += ntt::fmul(a1, b1, pd, pinvd);
                                s1[fl] += ntt::fmul(sa, b0 + b1, pd, pinvd);
                            }
                        }
                    }
                }
            }
#pragma unroll
            for (int fl = 0; fl < FG; ++fl) {
                if (fl < nf) {
                    const double e0 = ntt::fmul(s0[fl], rinv, pd, pinvd);
                    const double e2 = ntt::fmul(s2[fl], rinv, pd, pinvd);
                    const double e1 = ntt::fmul(s1[fl], rinv, pd, pinvd) - e0 - e2;
                    u64 *dp = D.data + ((int64_t)(f0 + fl) * cells + cell) * D.ct_stride + roff;
                    dp[0] = ntt::fcanon(e0, pd, pinvd);
                    dp[D.comp_stride] = ntt::fcanon(e1, pd, pinvd);
                    dp[2 * D.comp_stride] = ntt::fcanon(e2, pd, pinvd);
                }
            }
        }
        return;
    }
    for (int cell = cell_lo + w; cell < cell_hi; cell += SW) {
        const int i = cell / on, j = cell % on;
        acc4 s0[FG], s1[FG], s2[FG];
        u64 t0[FG], t1[FG], t2[FG];
#pragma unroll
        for (int fl = 0; fl < FG; ++fl) {
            s0[fl] = s1[fl] = s2[fl] = acc4{0, 0, 0, 0};
            t0[fl] = t1[fl] = t2[fl] = 0;
        }
        int since = 0;
        for (int c = 0; c < C; ++c) {
            for (int pp = 0; pp < P; ++pp) {
                const int64_t rowcell = (int64_t)c * m * n + (int64_t)(i * s + pp) * n + j * s;
                for (int qq = 0; qq < Q; ++qq) {
                    const int tap = (c * P + pp) * Q + qq;
                    const u64 *ap = A.data + (rowcell + qq) * A.ct_stride + roff;
                    const u64 a0 = __ldg(ap), a1 = __ldg(ap + A.comp_stride);
                    const u64 sa = add_mod(a0, a1, p);
                    const u64 *wt = wsm + (size_t)(tap * FG) * 2 * XC + xl;
#pragma unroll
                    for (int fl = 0; fl < FG; ++fl) {
                        if (fl < nf) {
                            const u64 b0 = wt[(2 * fl) * XC], b1 = wt[(2 * fl + 1) * XC];
                            mac4(s0[fl], a0, b0);
                            mac4(s2[fl], a1, b1);
                            mac4(s1[fl], sa, add_mod(b0, b1, p));
                        }
                    }
                    if (FLUSH && ++since == flush) {
#pragma unroll
                        for (int fl = 0; fl < FG; ++fl) {
                            t0[fl] = add_mod(t0[fl], redc128(to128(s0[fl]), p, Pr.pinv, Pr.r1s), p);
                            t1[fl] = add_mod(t1[fl], redc128(to128(s1[fl]), p, Pr.pinv, Pr.r1s), p);
                            t2[fl] = add_mod(t2[fl], redc128(to128(s2[fl]), p, Pr.pinv, Pr.r1s), p);
                            s0[fl] = s1[fl] = s2[fl] = acc4{0, 0, 0, 0};
                        }
                        since = 0;
                    }
                }
            }
        }
#pragma unroll
        for (int fl = 0; fl < FG; ++fl) {
            if (fl < nf) {
                const u64 d0 = add_mod(t0[fl], redc128(to128(s0[fl]), p, Pr.pinv, Pr.r1s), p);
                const u64 d2 = add_mod(t2[fl], redc128(to128(s2[fl]), p, Pr.pinv, Pr.r1s), p);
                const u64 e1 = add_mod(t1[fl], redc128(to128(s1[fl]), p, Pr.pinv, Pr.r1s), p);
                u64 *dp = D.data + ((int64_t)(f0 + fl) * cells + cell) * D.ct_stride + roff;
                dp[0] = d0;
                dp[D.comp_stride] = sub_mod(sub_mod(e1, d0, p), d2, p);
                dp[2 * D.comp_stride] = d2;
            }
        }
    }
}

// ---------------------------------------------------------------------------------
// FP64 rows (p < 2^42): split-limb products.  Every residue is split into 20-bit limbs
// (a = a_h 2^20 + a_l), so each limb product is < 2^42 and is accumulated EXACTLY by
// one DFMA -- no per-product modular reduction.  A Karatsuba component costs 4 DFMA
// (hh, the two cross terms into one accumulator, ll) instead of a 6-op exact FP64
// modular product plus an add; the three partial sums of each component are reduced
// once per output cell.  Bounds: limbs of the component sums < 2^21, so every term is
// < 2^42 and a sum of `taps` terms stays below 2^53 for taps <= 256 (schoolbook middle,
// CONV_SCHOOL: up to four terms < 2^40 per tap into one accumulator, < 2^50).  The weight limbs
// and their Karatsuba sums are staged in shared memory as double pairs
// ([tap][filter][(b0h, b0l), (b1h, b1l) [, (b0h + b1h, b0l + b1l)]][XF]).  Forming the
// Karatsuba sums in registers instead of staging them (CONV_WPAIRS=2 with the Karatsuba
// middle: 2 more DADD per tap and filter) measured 23% SLOWER (more spills at the
// 128-register bound), as did two taps of input loads in flight (CONV_AHEAD=2, +4%).
namespace {
#ifndef CONV_XF
#define CONV_XF 16  // wide width of the split-limb body (narrow: half)
#endif
constexpr int FGF = CONV_FGF;  // filters per CTA group
constexpr int FP_MAX_TAPS = 256;
constexpr u64 M20 = (1ull << 20) - 1;
// CONV_SCHOOL: the middle component as a0 b1 + a1 b0 (8 DFMA per tap and filter) instead of
// the Karatsuba product of the sums (4 DFMA + a third staged pair).  The kernel is bound by
// the shared-memory data pipe, not the DFMA pipe (ncu r2h: a warp-wide 16-byte load costs
// ~3.6 wavefronts whatever the lanes share, 79% of the LSU data pipe at 39% FP64): two
// staged pairs per (tap, filter) instead of three trade a third of that traffic for a
// third more DFMA, with fewer live registers.  Measured r2h (cfg4, ms per conv launch):
// Karatsuba middle 37.55, this 36.32; cfg2 unchanged (1.86 / 1.87).
#ifndef CONV_SCHOOL
#define CONV_SCHOOL 1
#endif
#ifndef CONV_WPAIRS
#define CONV_WPAIRS (CONV_SCHOOL ? 2 : 3)
#endif
// CONV_LDS64: the staged limbs as separate 8-byte arrays ([tap][filter][limb][XF] doubles)
// read with 8-byte loads instead of double2 pairs read with 16-byte loads (measured r2j,
// cfg4 ms per conv launch: 36.40 -> 36.17, cfg2 unchanged: within noise, off)
#ifndef CONV_LDS64
#define CONV_LDS64 0
#endif
constexpr int WPAIRS = CONV_WPAIRS;  // staged weight double2 per (tap, filter): 3 = with the Karatsuba sums
}  // namespace

template <int XF>
__device__ __forceinline__ void conv_body_limbs(double *wl, const Ctx &K, const heb_ct &A, const heb_ct &B,
                                                const heb_ct &D, int C, int m, int n, int F, int P, int Q, int s,
                                                int om, int on, int logn, int bx, int r) {
    constexpr int SF = 256 / XF;  // workers per position
    const int xl = threadIdx.x % XF, w = threadIdx.x / XF;
    const int x = bx * XF + xl;
    const PrimeInfo Pr = K.pi[r];
    const int f0 = blockIdx.z * FGF;
    const int nf = min(FGF, F - f0);
    const int taps = C * P * Q;
    const int64_t roff = ((int64_t)r << logn) + x;
    // weight limbs of the FGF filter slots (zero for slots past the last filter, so the
    // hot loop needs no per-filter guard), and every tap's input offset
    __shared__ int64_t toff[FP_MAX_TAPS];
    for (int e = w; e < taps * FGF; e += SF) {
        const int tap = e / FGF, fl = e % FGF;
        // [tap][filter][pair][XF] double2: (b0h, b0l), (b1h, b1l) [, (b0h + b1h, b0l + b1l)]
        double2 *dst = reinterpret_cast<double2 *>(wl) + (size_t)(tap * FGF + fl) * WPAIRS * XF + xl;
        if (fl < nf) {
            const u64 *src = B.data + ((int64_t)(f0 + fl) * taps + tap) * B.ct_stride + roff;
            const u64 b0 = src[0], b1 = src[B.comp_stride];
            const double b0h = ntt::u2d(b0 >> 20), b0l = ntt::u2d(b0 & M20);
            const double b1h = ntt::u2d(b1 >> 20), b1l = ntt::u2d(b1 & M20);
#if CONV_LDS64
            double *d1 = wl + (size_t)(tap * FGF + fl) * 2 * WPAIRS * XF + xl;
            d1[0] = b0h, d1[XF] = b0l, d1[2 * XF] = b1h, d1[3 * XF] = b1l;
            if constexpr (WPAIRS == 3) d1[4 * XF] = b0h + b1h, d1[5 * XF] = b0l + b1l;
            (void)dst;
#else
            dst[0] = make_double2(b0h, b0l);
            dst[XF] = make_double2(b1h, b1l);
            if constexpr (WPAIRS == 3) dst[2 * XF] = make_double2(b0h + b1h, b0l + b1l);
#endif
        } else {
            dst[0] = dst[XF] = make_double2(0.0, 0.0);
            if constexpr (WPAIRS == 3) dst[2 * XF] = make_double2(0.0, 0.0);
        }
    }
    for (int tap = threadIdx.x; tap < taps; tap += blockDim.x) {
        const int c = tap / (P * Q), pp = (tap / Q) % P, qq = tap % Q;
        toff[tap] = ((int64_t)c * m * n + (int64_t)pp * n + qq) * A.ct_stride;
    }
    __syncthreads();
    const double pd = Pr.pd, pinvd = Pr.pinvd;
    // limb weights with the Montgomery correction folded in: R^-1 * (2^40, 2^20, 1)
    const double c0 = (double)Pr.rinv;
    const double c20 = (double)ntt::fcanon(ntt::fmul(1048576.0, c0, pd, pinvd), pd, pinvd);
    const double c40 = (double)ntt::fcanon(ntt::fmul(1048576.0, c20, pd, pinvd), pd, pinvd);
    const int cells = om * on;
    for (int cell = w; cell < cells; cell += SF) {
        const int i = cell / on, j = cell % on;
        double h0[FGF], q0[FGF], l0[FGF], h1[FGF], q1[FGF], l1[FGF], h2[FGF], q2[FGF], l2[FGF];
#pragma unroll
        for (int fl = 0; fl < FGF; ++fl) h0[fl] = q0[fl] = l0[fl] = h1[fl] = q1[fl] = l1[fl] = h2[fl] = q2[fl] = l2[fl] = 0.0;
        // taps in (c, p, q) order; the next tap's inputs are loaded before this tap's math
        const u64 *base = A.data + ((int64_t)(i * s) * n + j * s) * A.ct_stride + roff;
        u64 na0 = __ldg(base), na1 = __ldg(base + A.comp_stride);
#if CONV_AHEAD == 2
        u64 nb0 = 0, nb1 = 0;
        if (taps > 1) {
            nb0 = __ldg(base + toff[1]);
            nb1 = __ldg(base + toff[1] + A.comp_stride);
        }
#endif
        for (int tap = 0; tap < taps; ++tap) {
            {
                const u64 a0 = na0, a1 = na1;
#if CONV_AHEAD == 2
                na0 = nb0;
                na1 = nb1;
                if (tap + 2 < taps) {
                    const u64 *ap = base + toff[tap + 2];
                    nb0 = __ldg(ap);
                    nb1 = __ldg(ap + A.comp_stride);
                }
#else
                if (tap + 1 < taps) {
                    const u64 *ap = base + toff[tap + 1];
                    na0 = __ldg(ap);
                    na1 = __ldg(ap + A.comp_stride);
                }
#endif
                {
                    const double a0h = ntt::u2d(a0 >> 20), a0l = ntt::u2d(a0 & M20);
                    const double a1h = ntt::u2d(a1 >> 20), a1l = ntt::u2d(a1 & M20);
                    const double ash = a0h + a1h, asl = a0l + a1l;
                    const double2 *wt = reinterpret_cast<const double2 *>(wl) + (size_t)(tap * FGF) * WPAIRS * XF + xl;
#pragma unroll
                    for (int fl = 0; fl < FGF; ++fl) {
                        {  // every slot: zero weights past the last filter
#if CONV_LDS64
                            const double *w8 = wl + (size_t)((tap * FGF + fl) * 2 * WPAIRS) * XF + xl;
                            const double b0h = w8[0], b0l = w8[XF], b1h = w8[2 * XF], b1l = w8[3 * XF];
#else
                            const double2 w0 = wt[(WPAIRS * fl) * XF], w1 = wt[(WPAIRS * fl + 1) * XF];
                            const double b0h = w0.x, b0l = w0.y, b1h = w1.x, b1l = w1.y;
#endif
                            double bsh, bsl;
                            if constexpr (WPAIRS == 3) {
                                const double2 ws = wt[(WPAIRS * fl + 2) * XF];
                                bsh = ws.x;
                                bsl = ws.y;
                            } else {
                                bsh = b0h + b1h;
                                bsl = b0l + b1l;
                            }
                            h0[fl] = fma(a0h, b0h, h0[fl]);
                            q0[fl] = fma(a0h, b0l, fma(a0l, b0h, q0[fl]));
                            l0[fl] = fma(a0l, b0l, l0[fl]);
                            h2[fl] = fma(a1h, b1h, h2[fl]);
                            q2[fl] = fma(a1h, b1l, fma(a1l, b1h, q2[fl]));
                            l2[fl] = fma(a1l, b1l, l2[fl]);
#if CONV_SCHOOL
                            (void)bsh;
                            (void)bsl;
                            h1[fl] = fma(a0h, b1h, fma(a1h, b0h, h1[fl]));
                            q1[fl] = fma(a0h, b1l, fma(a0l, b1h, fma(a1h, b0l, fma(a1l, b0h, q1[fl]))));
                            l1[fl] = fma(a0l, b1l, fma(a1l, b0l, l1[fl]));
#else
                            h1[fl] = fma(ash, bsh, h1[fl]);
                            q1[fl] = fma(ash, bsl, fma(asl, bsh, q1[fl]));
                            l1[fl] = fma(asl, bsl, l1[fl]);
#endif
                        }
                    }
                }
            }
        }
        auto comb = [&](double h, double q, double l) {
            return ntt::fmul(ntt::fred(h, pd, pinvd), c40, pd, pinvd) + ntt::fmul(ntt::fred(q, pd, pinvd), c20, pd, pinvd) +
                   ntt::fmul(ntt::fred(l, pd, pinvd), c0, pd, pinvd);
        };
#pragma unroll
        for (int fl = 0; fl < FGF; ++fl) {
            if (fl < nf) {
                const double e0 = comb(h0[fl], q0[fl], l0[fl]);
                const double e2 = comb(h2[fl], q2[fl], l2[fl]);
                const double e1 = CONV_SCHOOL ? comb(h1[fl], q1[fl], l1[fl]) : comb(h1[fl], q1[fl], l1[fl]) - e0 - e2;
                u64 *dp = D.data + ((int64_t)(f0 + fl) * cells + cell) * D.ct_stride + roff;
                dp[0] = ntt::fcanon(e0, pd, pinvd);
                dp[D.comp_stride] = ntt::fcanon(e1, pd, pinvd);
                dp[2 * D.comp_stride] = ntt::fcanon(e2, pd, pinvd);
            }
        }
    }
}

// Which CTA does what.  FP64 rows take the split-limb body (XF positions per CTA);
// integer rows the 128-bit body (XC positions per CTA, cells split over `cs` CTAs so an
// integer CTA lasts about as long as an FP64 one).  The integer CTAs are spread evenly
// through the launch order, so they run on the IMAD pipe alongside FP64-row CTAs on the
// DFMA pipe instead of occupying most SM slots in the first wave.
struct ConvMap {
    int nfp, nint;           // CTAs of each kind (per filter group)
    int xf_blocks, xc_blocks, cs;
    int8_t fp_rows[32], int_rows[32];
};

template <bool FLUSH, bool LIMBS, bool NARROW>
__global__ void __launch_bounds__(256, CONV_MINB) k_conv_tensor(Ctx K, heb_ct A, heb_ct B, heb_ct D, int C, int m, int n,
                                                         int F, int P, int Q, int s, int om, int on, int logn,
                                                         int flush, ConvMap map) {
    extern __shared__ u64 conv_smem[];
    constexpr int XC = NARROW ? CONV_XC / 2 : CONV_XC, XF = NARROW ? CONV_XF / 2 : CONV_XF;
    const int cells = om * on;
    if (!LIMBS) {
        conv_body<FLUSH, true, XC>(conv_smem, K, A, B, D, C, m, n, F, P, Q, s, om, on, logn, flush, blockIdx.x,
                               blockIdx.y, 0, cells);
        return;
    }
    const int b = blockIdx.x, total = map.nfp + map.nint;
    const int ib = (int)(((long)b * map.nint) / total);
    const bool is_int = ((long)(b + 1) * map.nint) / total != ib;
    if (is_int) {
        const int per_row = map.xc_blocks * map.cs;
        const int rem = ib % per_row, split = rem % map.cs;
        conv_body<FLUSH, false, XC>(conv_smem, K, A, B, D, C, m, n, F, P, Q, s, om, on, logn, flush, rem / map.cs,
                                map.int_rows[ib / per_row], (int)((long)split * cells / map.cs),
                                (int)((long)(split + 1) * cells / map.cs));
    } else {
        const int fb = b - ib;
        conv_body_limbs<XF>(reinterpret_cast<double *>(conv_smem), K, A, B, D, C, m, n, F, P, Q, s, om, on, logn,
                        fb % map.xf_blocks, map.fp_rows[fb / map.xf_blocks]);
    }
}

extern "C" int heb_conv_tensor(heb_ctx *c, heb_ct a, heb_ct b, heb_ct d, int channels, int m, int n, int filters,
                               int kp, int kq, int stride, int k, void *stream) {
    if (!c || channels < 1 || filters < 1 || kp < 1 || kq < 1 || stride < 1 || kp > m || kq > n || k < 1 ||
        k > c->num_rows || c->n % CONV_XC)
        return fail(HEB_EINVAL, "heb_conv_tensor: bad args");
    const int om = (m - kp) / stride + 1, on = (n - kq) / stride + 1;
    const int taps = channels * kp * kq;
    cudaStream_t st = (cudaStream_t)stream;
    const bool need_flush = taps > c->flush;
    // shared-memory stage of one CTA at positions-per-CTA (xc, xf): integer body / split-limb body
    auto stage = [&](int xc, int xf, bool &limbs) {
        const size_t sm = sizeof(u64) * (size_t)taps * FG * 2 * xc;
        const size_t smf = sizeof(double2) * (size_t)taps * FGF * WPAIRS * xf;
        limbs = taps <= FP_MAX_TAPS && smf <= 200 * 1024 && !getenv_flag("HEB_CONV_NO_LIMBS");
        return limbs ? std::max(sm, smf) : sm;
    };
    // wide CTAs while two of them fit an SM (227 KB, 1 KB reserved per CTA plus the static arrays)
    static const int narrow_env = [] {
        const char *e = getenv("HEB_CONV_NARROW");  // 0 / 1 force the width (experiments)
        return e && *e ? atoi(e) : -1;
    }();
    bool limbs = false;
    size_t smem = stage(CONV_XC, CONV_XF, limbs);
    const bool narrow = narrow_env >= 0 ? narrow_env != 0 : smem > 110 * 1024;
    const int XC = narrow ? CONV_XC / 2 : CONV_XC, XF = narrow ? CONV_XF / 2 : CONV_XF;
    if (narrow) smem = stage(XC, XF, limbs);
    if (sizeof(u64) * (size_t)taps * FG * 2 * XC > 220 * 1024)
        return fail(HEB_EUNSUP, "heb_conv_tensor: %d taps exceed the shared-memory stage", taps);
    static_assert(FG == FGF, "both bodies use the same filter groups");
    ConvMap map{};
    map.xf_blocks = c->n / XF;
    map.xc_blocks = c->n / XC;
    static const int cs_env = [] {
        const char *e = getenv("HEB_CONV_CS");
        return e ? std::max(1, atoi(e)) : 4;
    }();
    map.cs = cs_env;
    if (k > 32) return fail(HEB_EUNSUP, "heb_conv_tensor: more than 32 rows");
    int nfr = 0, nir = 0;
    for (int r = 0; r < k; ++r) {
        if (c->row_fp[r]) map.fp_rows[nfr++] = (int8_t)r;
        else map.int_rows[nir++] = (int8_t)r;
    }
    map.nfp = nfr * map.xf_blocks;
    map.nint = nir * map.xc_blocks * map.cs;
    const dim3 grid = limbs ? dim3(map.nfp + map.nint, 1, (filters + FG - 1) / FG)
                            : dim3(c->n / XC, k, (filters + FG - 1) / FG);
    const double nout = (double)filters * om * on;
    PROF("k_conv_tensor", st, 8.0 * c->n * k * (2.0 * channels * m * n + 2.0 * filters * taps + 3.0 * nout));
#define CONV_LAUNCH(FL, LI, NA)                                                                                   \
    {                                                                                                             \
        CUDA_TRY(prep_kernel(k_conv_tensor<FL, LI, NA>, smem));                                                   \
        k_conv_tensor<FL, LI, NA><<<grid, 256, smem, st>>>(kctx(c), a, b, d, channels, m, n, filters, kp, kq, stride, \
                                                           om, on, c->log_n, c->flush, map);                     \
    }
#define CONV_LAUNCH_W(FL, LI) \
    if (narrow) CONV_LAUNCH(FL, LI, true) else CONV_LAUNCH(FL, LI, false)
    if (limbs) {
        if (need_flush) { CONV_LAUNCH_W(true, true) } else { CONV_LAUNCH_W(false, true) }
    } else {
        if (need_flush) { CONV_LAUNCH_W(true, false) } else { CONV_LAUNCH_W(false, false) }
    }
#undef CONV_LAUNCH_W
#undef CONV_LAUNCH
    LAUNCH_CHECK();
    return HEB_OK;
}

// Largest tap count heb_conv sends to the fused kernel: what its shared-memory stage
// holds, capped at 64 (beyond that the index-driven heb_dot_tensor measured faster).
int conv_tensor_max_taps() { return std::min(64, (int)(220 * 1024 / (sizeof(u64) * FG * 2 * (CONV_XC / 2)))); }
