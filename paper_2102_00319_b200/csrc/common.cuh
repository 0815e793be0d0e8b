// common.cuh -- shared declarations of the libheb200 translation units.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/heb200.h"
#include "modarith.cuh"
#include "ntt.cuh"

typedef unsigned __int128 u128;

int fail(int code, const char *fmt, ...);

#define CUDA_TRY(expr)                                                                     \
    do {                                                                                   \
        cudaError_t _e = (expr);                                                           \
        if (_e != cudaSuccess)                                                             \
            return fail(HEB_ECUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), \
                        __FILE__, __LINE__);                                               \
    } while (0)

#define LAUNCH_CHECK() CUDA_TRY(cudaGetLastError())

// Optional per-kernel timing (heb_prof_enable): CUDA events recorded on the launch
// stream around every kernel, resolved in heb_prof_summary.  Off by default.
bool prof_enabled();
int prof_begin(cudaStream_t st);
void prof_end(int slot, const char *name, double bytes, cudaStream_t st);
// Each launch declares its algorithmic bytes (every input read once, every output
// written once); a caller-provided override (heb_prof_next_bytes) takes precedence.
struct ProfScope {
    int slot;
    const char *name;
    double bytes;
    cudaStream_t st;
    ProfScope(const char *n, cudaStream_t s, double b) : slot(-1), name(n), bytes(b), st(s) {
        if (prof_enabled()) slot = prof_begin(s);
    }
    ~ProfScope() {
        if (slot >= 0) prof_end(slot, name, bytes, st);
    }
};
#define PROF(name, st, bytes) ProfScope _prof_scope(name, st, (double)(bytes))

// =============================================================================
// context
// =============================================================================
struct LevelConst {
    // rescale at this level drops q_L (row `level`); valid for rows i < level
    ulonglong2 beta, beta_r;     // q_L^-1, q_L^-1 * R            (mod q_i)
    ulonglong2 alpha, alpha_r;   // P^-1 q_L^-1, P^-1 q_L^-1 R    (mod q_i)
    // key switch at this level (rows i <= level) and the q_L row's own constants
    ulonglong2 gamma, gamma_r;   // P^-1, P^-1 R                  (mod q_i)
    ulonglong2 pmod, pinv;       // P mod q_i, P^-1 mod q_i       (std)
};

struct LastConst {  // final inverse-stage factors (Shoup pairs; FP64 engine: (w, w/p))
    ulonglong2 u_plain, v_plain;  // n^-1,       itw[1] n^-1
    ulonglong2 u_std, v_std;      // n^-1 R^-1,  itw[1] n^-1 R^-1  (fold from-Montgomery)
    double fu_plain, fv_plain, fu_std, fv_std;
};

struct StreamArena {
    struct Block {
        char *base;
        size_t cap;
    };
    std::recursive_mutex mu;
    std::vector<Block> blocks;
    // side stream of this stream (created on first use, outside any capture) and the
    // fork / join events that order it: independent launches of one call overlap on it
    cudaStream_t side = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    size_t blk = 0, off = 0;  // bump position
    // set when scratch was handed out during a CUDA-graph capture on this stream: the
    // graph holds raw block addresses, so the blocks must outlive it
    bool captured = false;
};

struct heb_ctx {
    int device = 0, log_n = 0, n = 0, num_rows = 0, chunk = 1024;
    std::vector<u64> primes;
    std::vector<char> row_fp;  // host copy of PrimeInfo::use_fp per chain row
    PrimeInfo *d_pi = nullptr;
    ulonglong2 *d_tw = nullptr, *d_itw = nullptr;
    double *d_twf = nullptr, *d_itwf = nullptr;  // FP64 engine twiddles (w as double)
    LevelConst *d_lc = nullptr;
    LastConst *d_last = nullptr;
    int flush = 64;  // lazy 128-bit accumulation: products summed before a reduction
    std::mutex arena_mu;
    std::unordered_map<cudaStream_t, std::unique_ptr<StreamArena>> arenas;
    StreamArena *arena(cudaStream_t st) {
        std::lock_guard<std::mutex> g(arena_mu);
        auto &a = arenas[st];
        if (!a) a.reset(new StreamArena());
        return a.get();
    }
};

// Per-stream scratch arena.  Kernel intermediates (key-switch digits, ModUp outputs,
// ...) come from a chain of device blocks owned by the context and keyed by stream;
// Scratch objects take and return space in LIFO order, so a call's scratch is reused by
// the next call on the same stream (stream order makes that safe).  Blocks are only
// ever added (cudaMalloc, during the first calls of a shape) -- steady-state calls and
// CUDA-graph replays touch no allocator, and concurrent streams never share memory.
// One host thread at a time may issue calls on a stream (a recursive lock per stream
// arena covers the lifetime of a call's Scratch objects).
struct Scratch {
    void *p = nullptr;
    StreamArena *a;
    cudaStream_t st;
    size_t blk0, off0;
    std::unique_lock<std::recursive_mutex> lock;
    Scratch(heb_ctx *c, cudaStream_t st);
    cudaError_t get(size_t bytes) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) a->captured = true;
        bytes = (bytes + 255) & ~(size_t)255;
        if (!bytes) bytes = 256;
        while (a->blk < a->blocks.size()) {
            auto &b = a->blocks[a->blk];
            if (a->off + bytes <= b.cap) {
                p = b.base + a->off;
                a->off += bytes;
                return cudaSuccess;
            }
            ++a->blk;
            a->off = 0;
        }
        // a new block holds this request (at least 64 MB, 2 MB granules): no geometric
        // growth, so a multi-GB layer intermediate does not double the arena's footprint
        size_t cap = std::max(bytes, (size_t)64 << 20);
        cap = (cap + ((size_t)2 << 20) - 1) & ~(((size_t)2 << 20) - 1);
        void *q = nullptr;
        cudaError_t e = cudaMalloc(&q, cap);
        if (e != cudaSuccess) return e;
        a->blocks.push_back({(char *)q, cap});
        a->blk = a->blocks.size() - 1;
        p = q;
        a->off = bytes;
        return cudaSuccess;
    }
    ~Scratch() {
        a->blk = blk0;
        a->off = off0;
    }
};
inline Scratch::Scratch(heb_ctx *c, cudaStream_t st_) : a(c->arena(st_)), st(st_), lock(a->mu) {
    blk0 = a->blk;
    off0 = a->off;
}

// =============================================================================
// device helpers
// =============================================================================
struct Ctx {  // kernel-side view of the context
    const PrimeInfo *pi;
    const ulonglong2 *tw, *itw;
    const double *twf, *itwf;
    const LevelConst *lc;
    const LastConst *last;
    int num_rows;
};
static inline Ctx kctx(const heb_ctx *c) {
    return Ctx{c->d_pi, c->d_tw, c->d_itw, c->d_twf, c->d_itwf, c->d_lc, c->d_last, c->num_rows};
}

// ---------------------------------------------------------------------------------
// Row geometry.  A CTA owns 2^LL residues of a row, LL = min(log N, ROW_MAX_LL); longer
// rows are split over an SP-CTA cluster (SP = N / 2^LL = 2 or 4, blockIdx.x = SP *
// logical index + part): parts of 2^13 residues (68 KB of shared memory, 512 threads)
// let two CTAs share an SM, where a 2^14 part (136 KB) leaves one barrier-synchronised
// CTA per SM.  Kernels use lbx() for their logical x index, rpart() for their part,
// tpos() for the first of the positions a thread holds after a forward transform (line
// pairs: tpos + (m & 1) + 2 T (m >> 1), see ntt::lpos; load16/store16 walk that
// pattern), KT for their block size.
#ifndef ROW_MAX_LL
#define ROW_MAX_LL 14
#endif
template <int LOGN>
struct Row {
    static constexpr int LL = LOGN < ROW_MAX_LL ? LOGN : ROW_MAX_LL;  // residues per CTA = 2^LL
    static constexpr int SP = 1 << (LOGN - LL);                      // CTAs per row
    static constexpr bool SPLIT = SP > 1;
    static constexpr int N = 1 << LOGN;
    static_assert(SP <= 4, "rows are split over at most 4 CTAs");
};
template <int LOGN, int E = 16>
constexpr int KT = ntt::Shape<Row<LOGN>::LL, E>::T;
template <int LOGN>
__device__ __forceinline__ int lbx() {
    return (int)blockIdx.x / Row<LOGN>::SP;
}
template <int LOGN>
__device__ __forceinline__ int rpart() {
    return (int)blockIdx.x % Row<LOGN>::SP;
}
template <int LOGN, int E = 16>
__device__ __forceinline__ int tpos() {
    return (rpart<LOGN>() << Row<LOGN>::LL) + 2 * (int)threadIdx.x;
}
// HEB_PATH_PROBE (build experiments only): 1 = FP64 engine only, 2 = integer engine only
#if defined(HEB_PATH_PROBE) && HEB_PATH_PROBE == 1
#define HEB_FPSEL(x) true
#elif defined(HEB_PATH_PROBE) && HEB_PATH_PROBE == 2
#define HEB_FPSEL(x) false
#else
#define HEB_FPSEL(x) (x)
#endif
// Row-dispatched transforms: rows whose prime is < 2^42 run on the FP64 engine, the
// others (50/60-bit base and special primes) on the 64-bit integer engine.  Both read
// u64 residues and return canonical u64 residues, so callers are engine-agnostic.
// ENG (kernels instantiated per engine): 0 = dispatch on the row at run time, 1 = FP64
// engine only, 2 = integer engine only.  One instantiation per engine is register-
// allocated on its own (no spills carried over from the other engine's code).
template <int ENG>
__device__ __forceinline__ bool eng_fp(const PrimeInfo &P) {
    if constexpr (ENG == 1) return true;
    else if constexpr (ENG == 2) return false;
    else return HEB_FPSEL(P.use_fp);
}
template <int ENG>
__device__ __forceinline__ bool eng_skip(const PrimeInfo &P) {  // row belongs to the other instantiation
    return ENG != 0 && (bool)P.use_fp != (ENG == 1);
}
template <int LOGN, int E = 16, int ENG = 0, class Load>
__device__ __forceinline__ void fwd_any(const Ctx &K, int row, const PrimeInfo &P, u64 *sm, Load load,
                                        u64 (&out)[E]) {
    constexpr int LL = Row<LOGN>::LL;
    if constexpr (ENG == 2) {
        const ntt::IntArith ar(P.p);
        const ulonglong2 *tw = K.tw + ((size_t)row << (LOGN + ntt::TW_ROW_SHIFT));
        if constexpr (Row<LOGN>::SPLIT) ntt::forward_split<LL, E, Row<LOGN>::SP>(ar, sm, tw, load, out, rpart<LOGN>());
        else ntt::forward<LL, E>(ar, sm, tw, load, out);
        return;
    }
    if (ENG == 1 || HEB_FPSEL(P.use_fp)) {
        const ntt::FpArith ar(P.pd, P.pinvd);
        double *s = reinterpret_cast<double *>(sm);
        const double *tw = K.twf + ((size_t)row << (LOGN + ntt::TW_ROW_SHIFT));
        if constexpr (Row<LOGN>::SPLIT) ntt::forward_split<LL, E, Row<LOGN>::SP>(ar, s, tw, load, out, rpart<LOGN>());
        else ntt::forward<LL, E>(ar, s, tw, load, out);
    } else if constexpr (ENG == 0) {
        const ntt::IntArith ar(P.p);
        const ulonglong2 *tw = K.tw + ((size_t)row << (LOGN + ntt::TW_ROW_SHIFT));
        if constexpr (Row<LOGN>::SPLIT) ntt::forward_split<LL, E, Row<LOGN>::SP>(ar, sm, tw, load, out, rpart<LOGN>());
        else ntt::forward<LL, E>(ar, sm, tw, load, out);
    }
}
// std_out: fold the from-Montgomery factor R^-1 into the final stage
template <int LOGN, int E = 16, int ENG = 0, class Store>
__device__ __forceinline__ void inv_any(const Ctx &K, int row, const PrimeInfo &P, u64 *sm, const u64 (&in)[E],
                                        Store store, bool std_out) {
    constexpr int LL = Row<LOGN>::LL;
    const LastConst &lc = K.last[row];
    if constexpr (ENG == 2) {
        const ntt::IntArith ar(P.p);
        const ulonglong2 *itw = K.itw + ((size_t)row << (LOGN + ntt::TW_ROW_SHIFT));
        const ulonglong2 u = std_out ? lc.u_std : lc.u_plain, v = std_out ? lc.v_std : lc.v_plain;
        if constexpr (Row<LOGN>::SPLIT) ntt::inverse_split<LL, E, Row<LOGN>::SP>(ar, sm, itw, in, store, u, v, rpart<LOGN>());
        else ntt::inverse<LL, E>(ar, sm, itw, in, store, u, v);
        return;
    }
    if (ENG == 1 || HEB_FPSEL(P.use_fp)) {
        const ntt::FpArith ar(P.pd, P.pinvd);
        double *s = reinterpret_cast<double *>(sm);
        const double *itw = K.itwf + ((size_t)row << (LOGN + ntt::TW_ROW_SHIFT));
        const double u = std_out ? lc.fu_std : lc.fu_plain, v = std_out ? lc.fv_std : lc.fv_plain;
        if constexpr (Row<LOGN>::SPLIT) ntt::inverse_split<LL, E, Row<LOGN>::SP>(ar, s, itw, in, store, u, v, rpart<LOGN>());
        else ntt::inverse<LL, E>(ar, s, itw, in, store, u, v);
    } else if constexpr (ENG == 0) {
        const ntt::IntArith ar(P.p);
        const ulonglong2 *itw = K.itw + ((size_t)row << (LOGN + ntt::TW_ROW_SHIFT));
        const ulonglong2 u = std_out ? lc.u_std : lc.u_plain, v = std_out ? lc.v_std : lc.v_plain;
        if constexpr (Row<LOGN>::SPLIT) ntt::inverse_split<LL, E, Row<LOGN>::SP>(ar, sm, itw, in, store, u, v, rpart<LOGN>());
        else ntt::inverse<LL, E>(ar, sm, itw, in, store, u, v);
    }
}

// Launch a row kernel: split rows get SP times the CTAs along x, clustered SP at a time.
template <int LOGN, class Kern, class... Args>
static cudaError_t launch_rows(Kern kernel, dim3 grid, int block, size_t smem, cudaStream_t st, Args... args) {
    if constexpr (Row<LOGN>::SPLIT) {
        grid.x *= Row<LOGN>::SP;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(block);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = Row<LOGN>::SP;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kernel, args...);
    } else {
        kernel<<<grid, block, smem, st>>>(args...);
        return cudaGetLastError();
    }
}

// Launch a row kernel over chain rows [a, b) (its blockIdx.x row = r0 + lbx, r0 passed
// as the kernel's last argument).  When the integer-engine rows form a prefix of the
// range (the usual chain layout: wide base prime first, 40-bit level primes after) the
// rows are split over the integer-only and FP64-only instantiations, each register-
// allocated on its own; otherwise the run-time dispatching instantiation covers all.
// Fork `st`'s side stream off st (the side stream and its events are created on first
// use, outside any graph capture) / join it back.  Work on the side stream between the
// two overlaps the work on st.
static inline cudaError_t side_fork(heb_ctx *c, cudaStream_t st, cudaStream_t *side) {
    StreamArena *ar = c->arena(st);
    std::lock_guard<std::recursive_mutex> g(ar->mu);
    if (!ar->side) {
        cudaError_t e = cudaStreamCreateWithFlags(&ar->side, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ar->fork, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ar->join, cudaEventDisableTiming);
        if (e != cudaSuccess) return e;
    }
    cudaError_t e = cudaEventRecord(ar->fork, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(ar->side, ar->fork, 0);
    *side = ar->side;
    return e;
}
static inline cudaError_t side_join(heb_ctx *c, cudaStream_t st) {
    StreamArena *ar = c->arena(st);
    cudaError_t e = cudaEventRecord(ar->join, ar->side);
    return e == cudaSuccess ? cudaStreamWaitEvent(st, ar->join, 0) : e;
}

template <int LOGN, class K0, class K1, class K2, class... Args>
static cudaError_t launch_by_engine(const heb_ctx *cc, K0 k0, K1 k1, K2 k2, int a, int b, unsigned gy, unsigned gz,
                                    size_t smem, cudaStream_t st, Args... args) {
    heb_ctx *c = const_cast<heb_ctx *>(cc);
    if (b <= a) return cudaSuccess;
#ifndef ENGINE_SPLIT_ROWS
#define ENGINE_SPLIT_ROWS 1  // with the integer rows on the side stream: cfg1 relin +8%, cfg2 neutral
#endif
    if (!ENGINE_SPLIT_ROWS) return launch_rows<LOGN>(k0, dim3(b - a, gy, gz), KT<LOGN>, smem, st, args..., a);
    int nint = 0;
    while (a + nint < b && !c->row_fp[a + nint]) ++nint;
    bool rest_fp = true;
    for (int r = a + nint; r < b; ++r) rest_fp = rest_fp && c->row_fp[r];
    if (!rest_fp) return launch_rows<LOGN>(k0, dim3(b - a, gy, gz), KT<LOGN>, smem, st, args..., a);
    // integer rows on the side stream, concurrent with the FP64 rows (IMAD/ALU vs DFMA)
#ifndef ENGINE_SIDE_STREAM
#define ENGINE_SIDE_STREAM 1
#endif
    const bool both = ENGINE_SIDE_STREAM && nint && b - a - nint;
    cudaStream_t ist = st;
    cudaError_t e = both ? side_fork(c, st, &ist) : cudaSuccess;
    // The integer rows take the run-time-dispatching instantiation: the integer-only
    // instantiation of k_ks_head faults at N = 512 (found by smoke(); all other sizes
    // pass), and k0 measured the same speed for these short launches.
#ifndef ENGINE_INT_ONLY_INST
#define ENGINE_INT_ONLY_INST 0
#endif
    if (e == cudaSuccess && nint)
        e = launch_rows<LOGN>(ENGINE_INT_ONLY_INST ? k2 : k0, dim3(nint, gy, gz), KT<LOGN>, smem, ist, args..., a);
    if (e == cudaSuccess && b - a - nint)
        e = launch_rows<LOGN>(k1, dim3(b - a - nint, gy, gz), KT<LOGN>, smem, st, args..., a + nint);
    if (e == cudaSuccess && both) e = side_join(c, st);
    return e;
}
#define ENGINE_KERNELS(KERN) KERN<LOGN, 0>, KERN<LOGN, 1>, KERN<LOGN, 2>
#define PREP_ENGINES(KERN, SM)                       \
    CUDA_TRY(prep_kernel(KERN<LOGN, 0>, SM));        \
    CUDA_TRY(prep_kernel(KERN<LOGN, 1>, SM));        \
    CUDA_TRY(prep_kernel(KERN<LOGN, 2>, SM))

template <int LOGN>
__device__ __forceinline__ const ulonglong2 *tw_row(const Ctx &k, int row) {
    return k.tw + ((size_t)row << (LOGN + ntt::TW_ROW_SHIFT));
}
template <int LOGN>
__device__ __forceinline__ const ulonglong2 *itw_row(const Ctx &k, int row) {
    return k.itw + ((size_t)row << (LOGN + ntt::TW_ROW_SHIFT));
}

// a thread's 16 line-pair positions starting at src = row + tpos(): 16-byte accesses,
// each warp-wide access covers 512 contiguous bytes
template <int LOGN>
__device__ __forceinline__ void load16(const u64 *__restrict__ src, u64 (&v)[16]) {
    const ulonglong2 *s = reinterpret_cast<const ulonglong2 *>(src);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        ulonglong2 t = __ldcg(s + i * KT<LOGN>);
        v[2 * i] = t.x;
        v[2 * i + 1] = t.y;
    }
}
template <int LOGN>
__device__ __forceinline__ void store16(u64 *__restrict__ dst, const u64 (&v)[16]) {
    ulonglong2 *d = reinterpret_cast<ulonglong2 *>(dst);
#pragma unroll
    for (int i = 0; i < 8; ++i) __stcg(d + i * KT<LOGN>, make_ulonglong2(v[2 * i], v[2 * i + 1]));
}

// minimum resident CTAs per SM for the NTT kernels: caps registers at 64/thread
#ifndef NTT_REGS_PER_THREAD
#define NTT_REGS_PER_THREAD 64
#endif
#define NTT_MINB_LL(LL) \
    (((65536 / NTT_REGS_PER_THREAD) >> ((LL) - 4)) > 32 ? 32 : (((65536 / NTT_REGS_PER_THREAD) >> ((LL) - 4)) < 1 ? 1 : ((65536 / NTT_REGS_PER_THREAD) >> ((LL) - 4))))
#define NTT_MINB(LOGN) NTT_MINB_LL(Row<LOGN>::LL)
// min CTAs/SM for a block of T threads at NTT_REGS_PER_THREAD registers
#define NTT_MINB_T(T) \
    ((65536 / NTT_REGS_PER_THREAD / (T)) > 32 ? 32 : ((65536 / NTT_REGS_PER_THREAD / (T)) < 1 ? 1 : (65536 / NTT_REGS_PER_THREAD / (T))))

// E line-pair positions (engine with E elements per thread) through L2
template <int LOGN, int E>
__device__ __forceinline__ void loadv(const u64 *__restrict__ src, u64 (&v)[E]) {
    const ulonglong2 *s = reinterpret_cast<const ulonglong2 *>(src);
#pragma unroll
    for (int i = 0; i < E / 2; ++i) {
        ulonglong2 t = __ldcg(s + i * KT<LOGN, E>);
        v[2 * i] = t.x;
        v[2 * i + 1] = t.y;
    }
}
template <int LOGN, int E>
__device__ __forceinline__ void storev(u64 *__restrict__ dst, const u64 (&v)[E]) {
    ulonglong2 *d = reinterpret_cast<ulonglong2 *>(dst);
#pragma unroll
    for (int i = 0; i < E / 2; ++i) __stcg(d + i * KT<LOGN, E>, make_ulonglong2(v[2 * i], v[2 * i + 1]));
}
// launch bounds of a row kernel (E = 16 engine)
#define ROW_BOUNDS(LOGN) __launch_bounds__(KT<LOGN>, NTT_MINB(LOGN))

template <int LOGN>
static constexpr size_t smem_bytes() {
    return sizeof(u64) * ntt::Shape<Row<LOGN>::LL>::SMEM_WORDS;
}

template <class K>
static cudaError_t prep_kernel(K kernel, size_t smem) {
    // the 48 KB default limit covers static + dynamic shared memory: opt in early enough
    // that a kernel's static arrays (a few KB) never push a launch over it
    if (smem > 32 * 1024)
        return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return cudaSuccess;
}

#define DISPATCH_LOGN(ctx, FN, ...)                                          \
    switch ((ctx)->log_n) {                                                  \
        case 6: return FN<6>(__VA_ARGS__);                                   \
        case 7: return FN<7>(__VA_ARGS__);                                   \
        case 8: return FN<8>(__VA_ARGS__);                                   \
        case 9: return FN<9>(__VA_ARGS__);                                   \
        case 10: return FN<10>(__VA_ARGS__);                                 \
        case 11: return FN<11>(__VA_ARGS__);                                 \
        case 12: return FN<12>(__VA_ARGS__);                                 \
        case 13: return FN<13>(__VA_ARGS__);                                 \
        case 14: return FN<14>(__VA_ARGS__);                                 \
        case 15: return FN<15>(__VA_ARGS__);                                 \
        default: return fail(HEB_EUNSUP, "unsupported log_n %d", (ctx)->log_n); \
    }

static inline unsigned gdim(int64_t v) { return (unsigned)(v < 65535 ? (v < 1 ? 1 : v) : 65535); }

// =============================================================================
// pointwise kernels (HBM-bound)
// =============================================================================
// grid.y enumerates (item, comp, row) "lines"; grid.x * block covers N.
struct LineIdx {
    int64_t b;
    int c, r;
};
__device__ __forceinline__ LineIdx line_of(int64_t line, int comps, int k) {
    LineIdx L;
    L.r = (int)(line % k);
    int64_t t = line / k;
    L.c = (int)(t % comps);
    L.b = t / comps;
    return L;
}
__device__ __forceinline__ u64 *at(const heb_ct &x, int64_t b, int c, int r, int logn) {
    return x.data + b * x.ct_stride + c * x.comp_stride + ((int64_t)r << logn);
}


static inline dim3 pw_grid(int n, int64_t lines) {
    int bx = (n + 255) / 256;
    return dim3(bx, gdim(lines));
}

__global__ void k_galois_ct(heb_ct in, heb_ct out, int64_t lines, int k, int logn, u64 g);
