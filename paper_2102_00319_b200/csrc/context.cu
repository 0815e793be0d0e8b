// context.cu -- error state, host-side number theory, context tables, memory API.
#include "common.cuh"

static thread_local std::string g_err;

int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

// =============================================================================
// host-side number theory (cold path, exact 128-bit arithmetic)
// =============================================================================
static u64 mulmod_h(u64 a, u64 b, u64 p) { return (u64)((u128)a * b % p); }
static u64 powmod_h(u64 a, u64 e, u64 p) {
    u64 r = 1 % p;
    a %= p;
    while (e) {
        if (e & 1) r = mulmod_h(r, a, p);
        a = mulmod_h(a, a, p);
        e >>= 1;
    }
    return r;
}
static u64 invmod_h(u64 a, u64 p) { return powmod_h(a, p - 2, p); }  // p prime
static u64 shoup_companion(u64 w, u64 p) { return (u64)(((u128)w << 64) / p); }
static ulonglong2 shoup_pair(u64 w, u64 p) {
    ulonglong2 r;
    r.x = w % p;
    r.y = shoup_companion(r.x, p);
    return r;
}
static u64 r_mod(u64 p) { return (u64)(((u128)1 << 64) % p); }
static u64 neg_inv64(u64 p) {
    u64 x = p;  // Newton iteration for p^-1 mod 2^64
    for (int i = 0; i < 6; ++i) x *= 2 - p * x;
    return (u64)0 - x;
}
// first element of exact order 2n (reference kernels.py:439-446)
static u64 find_2n_root_h(u64 n, u64 p) {
    u64 e = (p - 1) / (2 * n);
    for (u64 x = 2; x < (1u << 20); ++x) {
        u64 y = powmod_h(x, e, p);
        if (powmod_h(y, n, p) == p - 1) return y;
    }
    return 0;
}
static u32 brv_h(u32 x, int bits) {
    u32 y = 0;
    for (int i = 0; i < bits; ++i) y |= ((x >> i) & 1u) << (bits - 1 - i);
    return y;
}

extern "C" int heb_version(void) { return 1; }
extern "C" const char *heb_last_error(void) { return g_err.c_str(); }
extern "C" int heb_device_count(int *count) {
    CUDA_TRY(cudaGetDeviceCount(count));
    return HEB_OK;
}

extern "C" int heb_ctx_create(heb_ctx **out, int device, int log_n, int num_rows, const uint64_t *primes,
                              const uint64_t *psi) {
    if (!out || !primes || num_rows < 2) return fail(HEB_EINVAL, "heb_ctx_create: bad arguments");
    if (log_n < 6 || log_n > 15) return fail(HEB_EUNSUP, "ring degree 2^%d not supported (2^6 .. 2^15)", log_n);
    const int n = 1 << log_n;
    auto *c = new heb_ctx();
    if (const char *e = getenv("HEB_CHUNK")) c->chunk = std::max(1, atoi(e));  // key-switch chunk override
    c->device = device;
    c->log_n = log_n;
    c->n = n;
    c->num_rows = num_rows;
    c->primes.assign(primes, primes + num_rows);
    u64 pmax = 0;
    for (u64 p : c->primes) {
        if (p >= (1ull << 62) || p % (2ull * n) != 1) {
            delete c;
            return fail(HEB_EINVAL, "prime %llu is not an NTT prime < 2^62 for n=%d", (unsigned long long)p, n);
        }
        pmax = p > pmax ? p : pmax;
    }
    // products of canonical residues are < p^2; allow as many in a 128-bit accumulator
    {
        u128 lim = (~(u128)0) / ((u128)pmax * pmax);
        c->flush = lim > 64 ? 64 : (int)lim;
    }
    std::vector<PrimeInfo> pi(num_rows);
    // 4n entries per row: reference order, then the lane-major regions (ntt.cuh, TW_ROW_SHIFT)
    const size_t rs = (size_t)n << ntt::TW_ROW_SHIFT;
    std::vector<ulonglong2> tw((size_t)num_rows * rs, make_ulonglong2(0, 0)), itw((size_t)num_rows * rs, make_ulonglong2(0, 0));
    std::vector<double> twf((size_t)num_rows * rs, 0.0), itwf((size_t)num_rows * rs, 0.0);
    std::vector<LastConst> last(num_rows);
    const char *fp_env = getenv("HEB_DISABLE_FP64_NTT");
    const bool fp_disabled = fp_env && fp_env[0] == '1';
    for (int r = 0; r < num_rows; ++r) {
        const u64 p = c->primes[r];
        const u64 g = psi ? psi[r] : find_2n_root_h(n, p);
        if (!g || powmod_h(g, n, p) != p - 1) {
            delete c;
            return fail(HEB_EINVAL, "psi for prime %llu has wrong order", (unsigned long long)p);
        }
        PrimeInfo &q = pi[r];
        memset(&q, 0, sizeof q);
        q.p = p;
        q.pinv = neg_inv64(p);
        q.r1s = shoup_companion(1, p);
        q.rmod = r_mod(p);
        q.rmod_s = shoup_companion(q.rmod, p);
        q.rinv = invmod_h(q.rmod, p);
        q.rinv_s = shoup_companion(q.rinv, p);
        q.ninv = invmod_h((u64)n % p, p);
        q.ninv_s = shoup_companion(q.ninv, p);
        q.ninv_rinv = mulmod_h(q.ninv, q.rinv, p);
        q.ninv_rinv_s = shoup_companion(q.ninv_rinv, p);
        // powers of psi in bit-reversed order: tw[i] = psi^brv(i)   (kernels.py:464-475, std form)
        std::vector<u64> pw(n);
        pw[0] = 1;
        for (int i = 1; i < n; ++i) pw[i] = mulmod_h(pw[i - 1], g, p);
        for (int i = 0; i < n; ++i) {
            u64 w = pw[brv_h((u32)i, log_n)];
            tw[(size_t)r * rs + i] = shoup_pair(w, p);
            itw[(size_t)r * rs + i] = shoup_pair(invmod_h(w, p), p);
        }
        // lane-major copies of the last radix-16 group's twiddles: first stage S = log_n - 4
        // at [n, 2n), S = log_n - 5 at [2n, 3n)
        for (int region = 1; region <= 2; ++region) {
            const int S = log_n - 3 - region;
            if (S < 0) continue;
            const size_t base = (size_t)r * rs + (size_t)region * n;
            for (int q = 0; q < 4; ++q)
                for (int i = 0; i < (1 << q); ++i)
                    for (int g = 0; g < (1 << S); ++g) {
                        const size_t src = (size_t)r * rs + ((((size_t)1 << S) + g) << q) + i;
                        const size_t dst = base + ((size_t)((1 << q) - 1 + i) << S) + g;
                        tw[dst] = tw[src];
                        itw[dst] = itw[src];
                    }
        }
        const u64 it1 = itw[(size_t)r * rs + 1].x;
        last[r].u_plain = shoup_pair(q.ninv, p);
        last[r].v_plain = shoup_pair(mulmod_h(it1, q.ninv, p), p);
        last[r].u_std = shoup_pair(q.ninv_rinv, p);
        last[r].v_std = shoup_pair(mulmod_h(it1, q.ninv_rinv, p), p);
        // FP64 engine (p < 2^42): doubles (w, w/p) for every twiddle / final-stage factor
        q.pd = (double)p;
        q.pinvd = 1.0 / (double)p;
        q.use_fp = (p < (1ull << 42)) && !fp_disabled;
        c->row_fp.push_back(q.use_fp ? 1 : 0);
        auto fpair = [&](u64 w) { return (double)w; };
        for (size_t i = 0; i < rs; ++i) {
            twf[(size_t)r * rs + i] = fpair(tw[(size_t)r * rs + i].x);
            itwf[(size_t)r * rs + i] = fpair(itw[(size_t)r * rs + i].x);
        }
        last[r].fu_plain = fpair(last[r].u_plain.x);
        last[r].fv_plain = fpair(last[r].v_plain.x);
        last[r].fu_std = fpair(last[r].u_std.x);
        last[r].fv_std = fpair(last[r].v_std.x);
    }
    // per-level constants; P = special prime (last row)
    const int levels = num_rows - 1;  // level 0 .. num_rows-2
    const u64 P = c->primes[num_rows - 1];
    std::vector<LevelConst> lc((size_t)levels * num_rows);
    memset(lc.data(), 0, lc.size() * sizeof(LevelConst));
    for (int lvl = 0; lvl < levels; ++lvl) {
        const u64 qL = c->primes[lvl];
        for (int i = 0; i <= lvl; ++i) {
            const u64 q = c->primes[i];
            const u64 R = r_mod(q);
            LevelConst &L = lc[(size_t)lvl * num_rows + i];
            const u64 pinv = invmod_h(P % q, q);
            L.gamma = shoup_pair(pinv, q);
            L.gamma_r = shoup_pair(mulmod_h(pinv, R, q), q);
            L.pmod = shoup_pair(P % q, q);
            L.pinv = shoup_pair(pinv, q);
            if (i < lvl) {
                const u64 qinv = invmod_h(qL % q, q);
                L.beta = shoup_pair(qinv, q);
                L.beta_r = shoup_pair(mulmod_h(qinv, R, q), q);
                const u64 a = mulmod_h(pinv, qinv, q);
                L.alpha = shoup_pair(a, q);
                L.alpha_r = shoup_pair(mulmod_h(a, R, q), q);
            }
        }
    }
    cudaError_t e;
    if ((e = cudaSetDevice(device)) != cudaSuccess ||
        (e = cudaMalloc(&c->d_pi, sizeof(PrimeInfo) * num_rows)) != cudaSuccess ||
        (e = cudaMalloc(&c->d_tw, sizeof(ulonglong2) * tw.size())) != cudaSuccess ||
        (e = cudaMalloc(&c->d_itw, sizeof(ulonglong2) * itw.size())) != cudaSuccess ||
        (e = cudaMalloc(&c->d_twf, sizeof(double) * twf.size())) != cudaSuccess ||
        (e = cudaMalloc(&c->d_itwf, sizeof(double) * itwf.size())) != cudaSuccess ||
        (e = cudaMemcpy(c->d_twf, twf.data(), sizeof(double) * twf.size(), cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(c->d_itwf, itwf.data(), sizeof(double) * itwf.size(), cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMalloc(&c->d_lc, sizeof(LevelConst) * lc.size())) != cudaSuccess ||
        (e = cudaMalloc(&c->d_last, sizeof(LastConst) * num_rows)) != cudaSuccess ||
        (e = cudaMemcpy(c->d_pi, pi.data(), sizeof(PrimeInfo) * num_rows, cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(c->d_tw, tw.data(), sizeof(ulonglong2) * tw.size(), cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(c->d_itw, itw.data(), sizeof(ulonglong2) * itw.size(), cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(c->d_lc, lc.data(), sizeof(LevelConst) * lc.size(), cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(c->d_last, last.data(), sizeof(LastConst) * num_rows, cudaMemcpyHostToDevice)) != cudaSuccess) {
        heb_ctx_destroy(c);
        return fail(HEB_ECUDA, "context upload failed: %s", cudaGetErrorString(e));
    }
    // heb_alloc memory is stream-ordered: keep freed blocks in the pool (no unmapping
    // around every synchronisation).  Never let the pool satisfy an allocation on one
    // stream with memory freed on another by inserting a wait on that stream: with
    // concurrent inference pipelines such hidden dependencies serialise the pipelines.
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t keep = ~0ull;
        int no = 0;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &no);
    }
    *out = c;
    return HEB_OK;
}

extern "C" int heb_ctx_destroy(heb_ctx *c) {
    if (!c) return HEB_OK;
    cudaFree(c->d_pi);
    cudaFree(c->d_tw);
    cudaFree(c->d_itw);
    cudaFree(c->d_twf);
    cudaFree(c->d_itwf);
    cudaFree(c->d_lc);
    cudaFree(c->d_last);
    if (!c->arenas.empty()) {
        cudaDeviceSynchronize();  // scratch may still be in use by queued work
        for (auto &kv : c->arenas) {
            for (auto &b : kv.second->blocks) cudaFree(b.base);
            if (kv.second->side) {
                cudaStreamDestroy(kv.second->side);
                cudaEventDestroy(kv.second->fork);
                cudaEventDestroy(kv.second->join);
            }
        }
    }
    delete c;
    return HEB_OK;
}

extern "C" int heb_ctx_release_scratch(heb_ctx *c, void *stream) {
    if (!c) return fail(HEB_EINVAL, "heb_ctx_release_scratch: null context");
    StreamArena *a;
    {
        std::lock_guard<std::mutex> g(c->arena_mu);
        auto it = c->arenas.find((cudaStream_t)stream);
        if (it == c->arenas.end()) return HEB_OK;
        a = it->second.get();
    }
    std::lock_guard<std::recursive_mutex> g(a->mu);
    if (a->blk != 0 || a->off != 0) return fail(HEB_EINVAL, "heb_ctx_release_scratch: scratch in use");
    if (a->captured)
        return fail(HEB_EINVAL,
                    "heb_ctx_release_scratch: CUDA graphs captured on this stream use its scratch "
                    "(destroy them, then heb_ctx_clear_captured)");
    CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));  // queued work may still read it
    for (auto &b : a->blocks) cudaFree(b.base);
    a->blocks.clear();
    return HEB_OK;
}

extern "C" int heb_ctx_clear_captured(heb_ctx *c, void *stream) {
    if (!c) return fail(HEB_EINVAL, "heb_ctx_clear_captured: null context");
    std::lock_guard<std::mutex> g(c->arena_mu);
    auto it = c->arenas.find((cudaStream_t)stream);
    if (it != c->arenas.end()) {
        std::lock_guard<std::recursive_mutex> ga(it->second->mu);
        it->second->captured = false;
    }
    return HEB_OK;
}

extern "C" int heb_ctx_ring_degree(const heb_ctx *c) { return c ? c->n : 0; }
extern "C" int heb_ctx_set_chunk(heb_ctx *c, int items) {
    if (!c || items < 1) return fail(HEB_EINVAL, "bad chunk");
    c->chunk = items;
    return HEB_OK;
}

// =============================================================================
// memory
// =============================================================================
extern "C" int heb_alloc(size_t bytes, void **out, void *stream) {
    if (cudaMallocAsync(out, bytes ? bytes : 8, (cudaStream_t)stream) != cudaSuccess)
        return fail(HEB_ENOMEM, "cudaMallocAsync(%zu) failed", bytes);
    return HEB_OK;
}
extern "C" int heb_free(void *ptr, void *stream) {
    CUDA_TRY(cudaFreeAsync(ptr, (cudaStream_t)stream));
    return HEB_OK;
}
extern "C" int heb_h2d(void *dst, const void *src, size_t bytes, void *stream) {
    CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, (cudaStream_t)stream));
    return HEB_OK;
}
extern "C" int heb_d2h(void *dst, const void *src, size_t bytes, void *stream) {
    CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    return HEB_OK;
}
extern "C" int heb_sync(void *stream) {
    CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
    return HEB_OK;
}


// =============================================================================
// per-kernel event profiler (used by bench.py for the roofline's launch durations)
// =============================================================================
#include <map>
#include <mutex>

namespace {
struct ProfRec {
    cudaEvent_t a, b;
    const char *name;
    double bytes;
};
thread_local double t_next_bytes = -1.0;
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof_recs;
std::vector<cudaEvent_t> g_prof_pool;

cudaEvent_t take_event() {
    if (!g_prof_pool.empty()) {
        cudaEvent_t e = g_prof_pool.back();
        g_prof_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}
}  // namespace

bool prof_enabled() { return g_prof_on; }

int prof_begin(cudaStream_t st) {
    std::lock_guard<std::mutex> g(g_prof_mu);
    ProfRec r{take_event(), take_event(), nullptr, 0.0};
    cudaEventRecord(r.a, st);
    g_prof_recs.push_back(r);
    return (int)g_prof_recs.size() - 1;
}

void prof_end(int slot, const char *name, double bytes, cudaStream_t st) {
    std::lock_guard<std::mutex> g(g_prof_mu);
    if (slot < 0 || slot >= (int)g_prof_recs.size()) return;
    g_prof_recs[slot].name = name;
    g_prof_recs[slot].bytes = t_next_bytes >= 0 ? t_next_bytes : bytes;
    t_next_bytes = -1.0;
    cudaEventRecord(g_prof_recs[slot].b, st);
}

extern "C" int heb_prof_enable(int on) {
    std::lock_guard<std::mutex> g(g_prof_mu);
    for (auto &r : g_prof_recs) {
        g_prof_pool.push_back(r.a);
        g_prof_pool.push_back(r.b);
    }
    g_prof_recs.clear();
    g_prof_on = on != 0;
    return HEB_OK;
}

extern "C" int heb_prof_next_bytes(double bytes) {
    t_next_bytes = bytes;
    return HEB_OK;
}

// "name launches total_ms total_bytes" lines, one per kernel, after synchronising the events.
extern "C" int heb_prof_summary(char *buf, size_t len) {
    std::lock_guard<std::mutex> g(g_prof_mu);
    struct Agg {
        long n = 0;
        double ms = 0, bytes = 0;
    };
    std::map<std::string, Agg> agg;
    for (auto &r : g_prof_recs) {
        if (!r.name) continue;
        cudaEventSynchronize(r.b);
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) return fail(HEB_ECUDA, "event timing failed");
        auto &e = agg[r.name];
        e.n += 1;
        e.ms += ms;
        e.bytes += r.bytes;
    }
    std::string out;
    char line[256];
    for (auto &kv : agg) {
        snprintf(line, sizeof line, "%s %ld %.6f %.0f\n", kv.first.c_str(), kv.second.n, kv.second.ms,
                 kv.second.bytes);
        out += line;
    }
    if (buf && len) {
        strncpy(buf, out.c_str(), len - 1);
        buf[len - 1] = 0;
    }
    return (int)out.size();
}

// =============================================================================
// integer modmul microbenchmark: the INT64 roofline denominator
// =============================================================================
__global__ void k_bench_modmul(u64 *sink, u64 p, u64 w, u64 ws, int iters) {
    u64 x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = (threadIdx.x + blockIdx.x * blockDim.x) * 8 + i + 1;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = shoup_lazy(x[i], w, ws, p);
    }
    u64 s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s ^= x[i];
    if (s == 0x9e3779b97f4a7c15ull) sink[0] = s;
}

// Launch blocks x threads threads each doing iters x 8 Shoup modmuls; elapsed ms out.
extern "C" int heb_bench_modmul(int blocks, int threads, int iters, uint64_t p, double *ms_out, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    u64 *sink;
    CUDA_TRY(cudaMallocAsync(&sink, 8, st));
    const u64 w = (p >> 1) + 12345, ws = (u64)(((u128)w << 64) / p);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_bench_modmul<<<blocks, threads, 0, st>>>(sink, p, w, ws, 16);  // warm-up
    cudaEventRecord(a, st);
    k_bench_modmul<<<blocks, threads, 0, st>>>(sink, p, w, ws, iters);
    cudaEventRecord(b, st);
    CUDA_TRY(cudaEventSynchronize(b));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    *ms_out = ms;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    CUDA_TRY(cudaFreeAsync(sink, st));
    return HEB_OK;
}

// =============================================================================
// NTT butterfly microbenchmark: the compute-roofline denominators of the transform
// kernels.  Each thread keeps one radix-16 unit (16 residues) in registers and runs
// `iters` transform-equivalents of 4 register groups (4 levels x 8 butterflies each, the
// engines' own ar.fwd) with twiddles in registers and no memory traffic; the FP64 engine
// re-centres once per transform-equivalent like a real transform's output does.
//   kind 1: FP64 engine (p < 2^42, DFMA pipe)   kind 2: integer Shoup engine (IMAD / ALU)
// =============================================================================
template <class A>
__device__ __forceinline__ void bench_unit(const A &ar, typename A::V (&x)[16], const typename A::W (&w)[4]) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int half = 8 >> q;
#pragma unroll
        for (int m = 0; m < 16; ++m) {
            if (m & half) continue;
            ar.fwd(x[m], x[m + half], w[q]);
        }
    }
}
__global__ void __launch_bounds__(256) k_bench_bfly_fp(double *sink, double p, double pinv, int iters) {
    const ntt::FpArith ar(p, pinv);
    double x[16], w[4];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = (double)((threadIdx.x * 16 + i) * 2654435761u % 1000003u);
#pragma unroll
    for (int q = 0; q < 4; ++q) w[q] = floor(p * (0.31 + 0.17 * q));
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int g = 0; g < 4; ++g) bench_unit(ar, x, w);
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = ntt::fred(x[i], p, pinv);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += x[i];
    if (s == 0.123456789) sink[0] = s;
}
__global__ void __launch_bounds__(256) k_bench_bfly_int(u64 *sink, u64 p, int iters) {
    const ntt::IntArith ar(p);
    u64 x[16];
    ulonglong2 w[4];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = ((u64)(threadIdx.x * 16 + i) * 0x9e3779b97f4a7c15ull) % p;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const u64 v = (p >> 1) + 12345 + 77 * q;
        w[q] = make_ulonglong2(v, (u64)(((u128)v << 64) / p));
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int g = 0; g < 4; ++g) bench_unit(ar, x, w);
    }
    u64 s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s ^= x[i];
    if (s == 0x9e3779b97f4a7c15ull) sink[0] = s;
}

// blocks x threads threads, each iters x 128 butterflies; elapsed ms out.
extern "C" int heb_bench_butterfly(int kind, int blocks, int threads, int iters, uint64_t p, double *ms_out,
                                   void *stream) {
    if ((kind != 1 && kind != 2) || blocks < 1 || threads < 32 || threads > 256 || iters < 1 || !ms_out)
        return fail(HEB_EINVAL, "heb_bench_butterfly: bad args");
    if (kind == 1 && p >= (1ull << 42)) return fail(HEB_EINVAL, "heb_bench_butterfly: FP64 engine needs p < 2^42");
    cudaStream_t st = (cudaStream_t)stream;
    void *sink;
    CUDA_TRY(cudaMallocAsync(&sink, 8, st));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int pass = 0; pass < 2; ++pass) {  // warm-up, then the timed launch
        const int n = pass ? iters : 4;
        if (pass) cudaEventRecord(a, st);
        if (kind == 1) k_bench_bfly_fp<<<blocks, threads, 0, st>>>((double *)sink, (double)p, 1.0 / (double)p, n);
        else k_bench_bfly_int<<<blocks, threads, 0, st>>>((u64 *)sink, p, n);
    }
    cudaEventRecord(b, st);
    CUDA_TRY(cudaEventSynchronize(b));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    *ms_out = ms;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    CUDA_TRY(cudaFreeAsync(sink, st));
    return HEB_OK;
}
