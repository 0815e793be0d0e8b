// packing.cu -- dense wire format for residue rows (host <-> device transport).
//
// A residue of row r is < p_r < 2^b_r (b_r = bit length of the prime: 40 for the
// level primes, 60 for the base / special primes of configs 2-4), yet it occupies a
// 64-bit word in HBM.  For the host -> device leg of serving (the encrypted input grid
// is the dominant transfer, ~617 MB per cfg2 batch) the rows are bit-packed at b_r bits
// per residue: row r of a block takes ceil(N b_r / 64) words, rows follow each other,
// blocks (one ciphertext component: rows 0..rows-1) follow each other.  Lossless; the
// unpack is one coalesced pass on the device.  No reference counterpart (the
// reference's payloads are coefficient-form u64 words, ckks.py:389-436).
#include "common.cuh"

namespace {
constexpr int MAXR = 64;
struct PackGeom {
    int bits[MAXR];
    int64_t off[MAXR + 1];  // word offset of row r inside a block; off[rows] = block words
};

PackGeom geometry(const heb_ctx *c, int rows) {
    PackGeom g{};
    g.off[0] = 0;
    for (int r = 0; r < rows; ++r) {
        int b = 0;
        while (b < 64 && (c->primes[r] >> b)) ++b;
        g.bits[r] = b;
        g.off[r + 1] = g.off[r] + (((int64_t)c->n * b + 63) >> 6);
    }
    return g;
}
}  // namespace

// one thread per output word: gathers the <= 64/b + 1 residues overlapping it
__global__ void k_pack_rows(const u64 *__restrict__ in, int64_t in_stride, u64 *__restrict__ out, PackGeom g,
                            int rows, int logn, int64_t count) {
    const int r = blockIdx.y;
    const int b = g.bits[r];
    const int64_t words = g.off[r + 1] - g.off[r];
    const int n = 1 << logn;
    const u64 mask = b == 64 ? ~0ull : ((1ull << b) - 1);
    for (int64_t blk = blockIdx.z; blk < count; blk += gridDim.z) {
        const u64 *src = in + blk * in_stride + ((int64_t)r << logn);
        u64 *dst = out + blk * g.off[rows] + g.off[r];
        for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x) {
            const int64_t lo = w << 6, hi = lo + 64;  // bit range of this word
            int64_t i = lo / b;
            u64 acc = 0;
            for (; i < n && i * b < hi; ++i) {
                const u64 v = __ldg(src + i) & mask;
                const int64_t o = i * b - lo;  // bit offset of value i relative to the word
                acc |= o >= 0 ? (v << o) : (v >> -o);
            }
            dst[w] = acc;
        }
    }
}

// one thread per residue pair: reads the (at most three) words holding them, one
// 16-byte streaming store
__device__ __forceinline__ u64 unpack_one(const u64 *__restrict__ src, int64_t i, int b, u64 mask) {
    const int64_t o = i * b;
    const int64_t w = o >> 6;
    const int s = (int)(o & 63);
    u64 v = __ldg(src + w) >> s;
    if (s + b > 64) v |= __ldg(src + w + 1) << (64 - s);
    return v & mask;
}
__global__ void k_unpack_rows(const u64 *__restrict__ in, u64 *__restrict__ out, int64_t out_stride, PackGeom g,
                              int rows, int logn, int64_t count) {
    const int r = blockIdx.y;
    const int b = g.bits[r];
    const int n = 1 << logn;
    const u64 mask = b == 64 ? ~0ull : ((1ull << b) - 1);
    for (int64_t blk = blockIdx.z; blk < count; blk += gridDim.z) {
        const u64 *src = in + blk * g.off[rows] + g.off[r];
        ulonglong2 *dst = reinterpret_cast<ulonglong2 *>(out + blk * out_stride + ((int64_t)r << logn));
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n / 2; i += gridDim.x * blockDim.x)
            __stcs(dst + i, make_ulonglong2(unpack_one(src, 2 * i, b, mask), unpack_one(src, 2 * i + 1, b, mask)));
    }
}

extern "C" int64_t heb_packed_words(heb_ctx *c, int rows) {
    if (!c || rows < 1 || rows > c->num_rows || rows > MAXR) return fail(HEB_EINVAL, "heb_packed_words: bad rows");
    return geometry(c, rows).off[rows];
}

extern "C" int heb_pack_rows(heb_ctx *c, const uint64_t *in, int64_t count, int rows, int64_t in_stride,
                             uint64_t *out, void *stream) {
    if (!c || !in || !out || rows < 1 || rows > c->num_rows || rows > MAXR)
        return fail(HEB_EINVAL, "heb_pack_rows: bad args");
    if (count <= 0) return HEB_OK;
    const PackGeom g = geometry(c, rows);
    const int64_t maxw = ((int64_t)c->n * 64 + 63) >> 6;
    const dim3 grid((unsigned)((maxw + 255) / 256), rows, gdim(count));
    {
        PROF("k_pack_rows", (cudaStream_t)stream, 8.0 * (double)count * ((double)rows * c->n + g.off[rows]));
        k_pack_rows<<<grid, 256, 0, (cudaStream_t)stream>>>(in, in_stride, out, g, rows, c->log_n, count);
    }
    LAUNCH_CHECK();
    return HEB_OK;
}

extern "C" int heb_unpack_rows(heb_ctx *c, const uint64_t *in, int64_t count, int rows, uint64_t *out,
                               int64_t out_stride, void *stream) {
    if (!c || !in || !out || rows < 1 || rows > c->num_rows || rows > MAXR)
        return fail(HEB_EINVAL, "heb_unpack_rows: bad args");
    if (count <= 0) return HEB_OK;
    const PackGeom g = geometry(c, rows);
    if (out_stride & 1) return fail(HEB_EINVAL, "heb_unpack_rows: odd output stride");
    const dim3 grid((unsigned)((c->n / 2 + 255) / 256), rows, gdim(count));
    {
        PROF("k_unpack_rows", (cudaStream_t)stream, 8.0 * (double)count * ((double)rows * c->n + g.off[rows]));
        k_unpack_rows<<<grid, 256, 0, (cudaStream_t)stream>>>(in, out, out_stride, g, rows, c->log_n, count);
    }
    LAUNCH_CHECK();
    return HEB_OK;
}
