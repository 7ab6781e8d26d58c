// Graph ingest on the device:
//
//   fw_build_csr_device   reswalk build_csr (graph.py:138-169): CSR from an
//                         edge list, neighbour lists sorted by target with
//                         duplicates in input order -- np.lexsort((dst, src))
//                         semantics -- via a stable LSD radix sort of the
//                         packed (src, dst) keys carrying the input index.
//   fw_fwg1_info / fw_fwg1_read
//                         reswalk load_binary (graph.py:225-254): the FWG1 file
//                         streamed through pinned double buffers straight into
//                         device arrays, its CRC-32 (zlib's) computed on the
//                         device.
//
// The sort is reduce-then-scan per 8-bit digit over a persistent grid: each
// CTA owns one contiguous segment of the keys, (1) histograms it, (2) one
// scan turns the [digit][CTA] table into global output offsets, (3) the CTA
// re-reads its segment tile by tile, in order, ranks each key within its
// digit by warp match + per-warp counters (row order, then warp order), and
// stages the tile in shared memory in digit order so each digit's run is
// stored with coalesced writes.  Equal digits keep their input order: every
// pass is stable, hence the whole sort is (the lexsort tie rule).  Only keys
// move unless weights or labels come along (then a 32-bit value: the weight
// itself when there are no labels, else the input index for a gather).  Passes whose digit is constant over
// all keys are skipped.  HBM-bound integer work: no tensor cores.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/flowwalk.h"

namespace fwi {

int set_err_ingest(int code, const char *fmt, ...);
int staged_h2d(int n, const void *const *src, void *const *dst, const uint64_t *bytes);

#define CUI(expr)                                                                          \
    do {                                                                                   \
        cudaError_t e_ = (expr);                                                           \
        if (e_ != cudaSuccess)                                                             \
            return set_err_ingest(e_ == cudaErrorMemoryAllocation ? FW_ENOMEM : FW_ECUDA,  \
                                  "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_),         \
                                  __FILE__, __LINE__);                                     \
    } while (0)

constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr int kThreads = 256, kWarps = kThreads / 32, kRows = 8;
constexpr int kTile = kWarps * kRows * 32;  // keys per scatter tile
constexpr int kRadix = 256;
static_assert(kThreads == kRadix, "k_scatter: one thread per digit");

__global__ void k_max_id(const uint32_t *__restrict__ a, const uint32_t *__restrict__ b,
                         uint64_t m, unsigned *out) {
    unsigned mx = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x)
        mx = max(mx, max(a[i], b[i]));
    mx = __reduce_max_sync(FULL, mx);
    if ((threadIdx.x & 31) == 0) atomicMax(out, mx);
}

// vals: the input index (labels to gather), or -- weights without labels --
// the weight's bits themselves, so the sorted weights need no random gather
__global__ void k_make_keys(const uint32_t *__restrict__ src, const uint32_t *__restrict__ dst,
                            uint64_t m, int bv, const float *__restrict__ w_carry,
                            uint64_t *__restrict__ keys, uint32_t *__restrict__ vals) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        keys[i] = ((uint64_t)src[i] << bv) | dst[i];
        if (vals) vals[i] = w_carry ? __float_as_uint(w_carry[i]) : (uint32_t)i;
    }
}

// (1) per-CTA digit histogram of its segment -> hist[d * G + cta]
__global__ void __launch_bounds__(kThreads) k_hist(const uint64_t *__restrict__ keys, uint64_t m,
                                                   uint64_t seg, int shift, uint32_t *hist) {
    __shared__ uint32_t h[kWarps][kRadix];
    const int w = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kWarps * kRadix; i += kThreads) (&h[0][0])[i] = 0;
    __syncthreads();
    const uint64_t lo = blockIdx.x * seg, hi = min(m, lo + seg);
    for (uint64_t i = lo + threadIdx.x; i < hi; i += kThreads)
        atomicAdd(&h[w][(keys[i] >> shift) & 0xFF], 1u);
    __syncthreads();
    for (int d = threadIdx.x; d < kRadix; d += kThreads) {
        uint32_t s = 0;
        for (int x = 0; x < kWarps; x++) s += h[x][d];
        hist[(uint64_t)d * gridDim.x + blockIdx.x] = s;
    }
}

// (2) exclusive scan of the [digit][CTA] table (one CTA; n = 256 * G).
// Also reports the largest single-digit count (== m: the pass is a no-op).
__global__ void __launch_bounds__(1024) k_scan(uint32_t *t, uint32_t n, uint32_t G,
                                                unsigned *max_digit) {
    __shared__ uint32_t part[1024];
    const uint32_t per = (n + 1023) / 1024;
    const uint32_t lo = threadIdx.x * per, hi = min(n, lo + per);
    uint32_t s = 0;
    for (uint32_t i = lo; i < hi; i++) s += t[i];
    part[threadIdx.x] = s;
    __syncthreads();
    for (int d = 1; d < 1024; d <<= 1) {
        const uint32_t v = threadIdx.x >= (unsigned)d ? part[threadIdx.x - d] : 0;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    uint32_t run = part[threadIdx.x] - s;
    for (uint32_t i = lo; i < hi; i++) {
        const uint32_t x = t[i];
        t[i] = run;
        run += x;
    }
    __syncthreads();
    // per-digit totals: start of digit d+1 minus start of digit d
    for (uint32_t d = threadIdx.x; d < kRadix; d += 1024) {
        const uint32_t a = t[d * G];
        const uint32_t b = d + 1 < kRadix ? t[(d + 1) * G] : part[1023];
        atomicMax(max_digit, b - a);
    }
}

// (3) stable scatter of the CTA's segment, staged through shared memory.
// Per tile: keys are ranked within their digit (warp match, then warp order),
// written to shared memory in digit-sorted order, and only then stored to
// global memory by consecutive threads -- each digit's run of the tile goes
// out as contiguous, coalesced stores instead of 32 scattered sectors per warp
// store.  Order within a digit is row-major input order, so the pass is
// stable.  VALS: carry the 32-bit input index (weights/labels to gather).
template <bool VALS>
__global__ void __launch_bounds__(kThreads) k_scatter(const uint64_t *__restrict__ kin,
                                                      const uint32_t *__restrict__ vin, uint64_t m,
                                                      uint64_t seg, int shift,
                                                      const uint32_t *__restrict__ offs,
                                                      uint64_t *__restrict__ kout,
                                                      uint32_t *__restrict__ vout) {
    __shared__ uint32_t run[kRadix];     // this CTA's global cursor per digit
    __shared__ uint32_t tstart[kRadix];  // tile-local start of each digit
    __shared__ uint32_t wsum[kWarps];
    __shared__ uint32_t wc[kWarps][kRadix];
    __shared__ uint64_t sk[kTile];
    __shared__ uint32_t sv[VALS ? kTile : 1];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1;
    for (int d = threadIdx.x; d < kRadix; d += kThreads)
        run[d] = offs[(uint64_t)d * gridDim.x + blockIdx.x];
    const uint64_t lo = blockIdx.x * seg, hi = min(m, lo + seg);
    for (uint64_t t0 = lo; t0 < hi; t0 += kTile) {
        const uint32_t tn = (uint32_t)(hi - t0 < (uint64_t)kTile ? hi - t0 : (uint64_t)kTile);
        for (int d = lane; d < kRadix; d += 32) wc[w][d] = 0;
        __syncwarp();
        uint64_t key[kRows];
        uint32_t val[kRows], rank[kRows], dig[kRows];
#pragma unroll
        for (int r = 0; r < kRows; r++) {
            const uint64_t i = t0 + (uint64_t)(w * kRows + r) * 32 + lane;
            const bool ok = i < hi;
            key[r] = ok ? kin[i] : 0;
            val[r] = (VALS && ok) ? vin[i] : 0;
            dig[r] = ok ? (uint32_t)((key[r] >> shift) & 0xFF) : kRadix;  // 256: past the end
        }
#pragma unroll
        for (int r = 0; r < kRows; r++) {
            const unsigned peers = __match_any_sync(FULL, dig[r]);
            const uint32_t base = dig[r] < kRadix ? wc[w][dig[r]] : 0;
            __syncwarp();
            if (dig[r] < kRadix && lane == __ffs(peers) - 1) wc[w][dig[r]] = base + __popc(peers);
            __syncwarp();
            rank[r] = base + __popc(peers & lt);
        }
        __syncthreads();
        // per digit (thread d): warp-order prefixes within the digit and the
        // tile total; then an exclusive scan of the totals over the digits
        uint32_t tot = 0;
        {
            const int d = threadIdx.x;  // kThreads == kRadix
#pragma unroll
            for (int x = 0; x < kWarps; x++) {
                const uint32_t c = wc[x][d];
                wc[x][d] = tot;
                tot += c;
            }
            uint32_t incl = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) wsum[w] = incl;
            __syncthreads();
            uint32_t wofs = 0;
            for (int x = 0; x < w; x++) wofs += wsum[x];
            tstart[d] = wofs + incl - tot;
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < kRows; r++) {
            if (dig[r] < kRadix) {
                const uint32_t lp = tstart[dig[r]] + wc[w][dig[r]] + rank[r];
                sk[lp] = key[r];
                if (VALS) sv[lp] = val[r];
            }
        }
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < tn; i += kThreads) {
            const uint64_t k = sk[i];
            const uint32_t d = (uint32_t)((k >> shift) & 0xFF);
            const uint32_t pos = run[d] + (i - tstart[d]);
            kout[pos] = k;
            if (VALS) vout[pos] = sv[i];
        }
        __syncthreads();
        run[threadIdx.x] += tot;  // kThreads == kRadix: thread d owns digit d
        __syncthreads();
    }
}

// CSR arrays from the sorted keys: targets, and weights/labels gathered by
// the carried input index (a thread per key) ...
// (carried: idx holds the sorted weights' bits, see k_make_keys)
__global__ void k_csr_edges(const uint64_t *__restrict__ keys, const uint32_t *__restrict__ idx,
                            bool carried, uint64_t m, int bv, const float *__restrict__ w_in,
                            const uint8_t *__restrict__ l_in, uint32_t *__restrict__ tgt,
                            float *__restrict__ w_out, uint8_t *__restrict__ l_out) {
    const uint64_t mask = (1ull << bv) - 1;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m;
         e += (uint64_t)gridDim.x * blockDim.x) {
        tgt[e] = (uint32_t)(keys[e] & mask);
        const uint32_t j = idx ? idx[e] : 0;
        if (w_out) w_out[e] = carried ? __uint_as_float(j) : (w_in ? w_in[j] : 1.0f);
        if (l_out) l_out[e] = (l_in && !carried) ? l_in[j] : 0;
    }
}

// ... and offsets[v] = #keys with source < v = lower_bound(keys, v << bv)
// (a branchless binary search per vertex; any id distribution, including
// long runs of isolated vertices, costs the same).
__global__ void k_csr_offsets(const uint64_t *__restrict__ keys, uint64_t m, uint64_t V, int bv,
                              int64_t *__restrict__ off) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v <= V;
         v += (uint64_t)gridDim.x * blockDim.x) {
        if (v == V) {
            off[v] = (int64_t)m;
            continue;
        }
        const uint64_t want = v << bv;
        uint64_t lo = 0, n = m;  // first index with keys[i] >= want, in [0, m]
        while (n > 0) {
            const uint64_t half = n >> 1;
            if (__ldg(keys + lo + half) < want) {
                lo += half + 1;
                n -= half + 1;
            } else {
                n = half;
            }
        }
        off[v] = (int64_t)lo;
    }
}

__global__ void k_fill_i64(int64_t *p, uint64_t n, int64_t v) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

static int sm_count() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

// ---------------------------------------------------------------------------
// CRC-32 (zlib: reflected polynomial 0xEDB88320, init and final xor ~0).
// raw(D) = the CRC register after D from a zero register.  With shift(c, n)
// = c * x^(8n) mod P: raw(A || B) = shift(raw(A), |B|) ^ raw(B), and
// zlib.crc32(D) = raw(D) ^ shift(~0, |D|) ^ ~0.  Segments of the device
// arrays are reduced by threads, then combined pairwise up a tree.
// ---------------------------------------------------------------------------
constexpr uint32_t kPoly = 0xEDB88320u;
constexpr uint32_t kSeg = 4096;  // bytes per thread segment

__host__ __device__ inline uint32_t gf2_mul(uint32_t a, uint32_t b) {  // a * b mod P (reflected)
    uint32_t p = 0;
    for (int i = 0; i < 32; i++) {
        if (a & 0x80000000u) p ^= b;
        a <<= 1;
        b = (b & 1) ? (b >> 1) ^ kPoly : b >> 1;
    }
    return p;
}

// x^(2^k) mod P for k = 0..63 (host table, reflected: x^0 = 0x80000000)
static uint32_t xpow2(int k) {
    static uint32_t t[64];
    static bool init = false;
    if (!init) {
        t[0] = 0x40000000u;  // x^1
        for (int i = 1; i < 64; i++) t[i] = gf2_mul(t[i - 1], t[i - 1]);
        init = true;
    }
    return t[k];
}
static uint32_t x8n(uint64_t nbytes) {  // x^(8n) mod P
    uint32_t r = 0x80000000u;
    const uint64_t e = nbytes * 8;
    for (int k = 0; k < 64; k++)
        if ((e >> k) & 1) r = gf2_mul(r, xpow2(k));
    return r;
}

__constant__ uint32_t c_crc_tab[4][256];

static void crc_tables(uint32_t t[4][256]) {
    for (uint32_t i = 0; i < 256; i++) {
        uint32_t c = i;
        for (int k = 0; k < 8; k++) c = (c & 1) ? (c >> 1) ^ kPoly : c >> 1;
        t[0][i] = c;
    }
    for (uint32_t i = 0; i < 256; i++)
        for (int s = 1; s < 4; s++) t[s][i] = (t[s - 1][i] >> 8) ^ t[0][t[s - 1][i] & 0xFF];
}

__device__ __forceinline__ uint32_t crc_word(const uint32_t (*T)[256], uint32_t c, uint32_t x) {
    c ^= x;
    return T[3][c & 0xFF] ^ T[2][(c >> 8) & 0xFF] ^ T[1][(c >> 16) & 0xFF] ^ T[0][c >> 24];
}

// raw CRC of nseg full kSeg-byte segments (16-byte aligned base): thread per
// segment, each iteration consuming one 128-byte line it loads whole.
__global__ void __launch_bounds__(256) k_crc_seg(const uint8_t *__restrict__ data, uint64_t nseg,
                                                 uint32_t *__restrict__ out) {
    __shared__ uint32_t T[4][256];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) (&T[0][0])[i] = (&c_crc_tab[0][0])[i];
    __syncthreads();
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < nseg;
         s += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 *p = reinterpret_cast<const uint4 *>(data + s * kSeg);
        uint32_t c = 0;
        for (int line = 0; line < (int)(kSeg / 128); line++) {
            uint4 q[8];
#pragma unroll
            for (int j = 0; j < 8; j++) q[j] = __ldg(p + line * 8 + j);
#pragma unroll
            for (int j = 0; j < 8; j++) {
                c = crc_word(T, c, q[j].x);
                c = crc_word(T, c, q[j].y);
                c = crc_word(T, c, q[j].z);
                c = crc_word(T, c, q[j].w);
            }
        }
        out[s] = c;
    }
}

// raw CRC of a short unaligned byte range (the tail; one thread)
__global__ void k_crc_tail(const uint8_t *__restrict__ data, uint64_t n, uint32_t *out) {
    uint32_t c = 0;
    for (uint64_t i = 0; i < n; i++) c = (c >> 8) ^ c_crc_tab[0][(c ^ data[i]) & 0xFF];
    *out = c;
}

// one tree level: out[i] = shift(in[2i], seg_bytes) ^ in[2i+1]
__global__ void k_crc_combine(const uint32_t *__restrict__ in, uint64_t npairs, uint32_t xs,
                              uint32_t *__restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < npairs;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = gf2_mul(in[2 * i], xs) ^ in[2 * i + 1];
}

// raw CRC of a device byte range
static int device_raw_crc(const uint8_t *d, uint64_t n, cudaStream_t st, uint32_t *out) {
    static bool tab = false;
    if (!tab) {
        uint32_t t[4][256];
        crc_tables(t);
        CUI(cudaMemcpyToSymbol(c_crc_tab, t, sizeof(t)));
        tab = true;
    }
    const uint64_t nseg = ((uintptr_t)d % 16 == 0) ? n / kSeg : 0;
    uint64_t p2 = 1;
    while (p2 < nseg) p2 <<= 1;
    uint32_t *buf = nullptr;
    CUI(cudaMallocAsync(&buf, (2 * p2 + 2) * sizeof(uint32_t), st));
    uint32_t *a = buf, *b = buf + p2, *tail = buf + 2 * p2;
    // zero segments in front of the real ones do not change a raw CRC
    CUI(cudaMemsetAsync(a, 0, (p2 - nseg) * sizeof(uint32_t), st));
    const int sms = sm_count();
    if (nseg) k_crc_seg<<<sms * 8, 256, 0, st>>>(d, nseg, a + (p2 - nseg));
    uint64_t len = kSeg;
    for (uint64_t cnt = p2; cnt > 1; cnt >>= 1, len <<= 1) {
        k_crc_combine<<<std::max<uint64_t>(1, std::min<uint64_t>(sms * 8, cnt / 512 + 1)), 256, 0,
                        st>>>(a, cnt / 2, x8n(len), b);
        std::swap(a, b);
    }
    const uint64_t body = nseg * kSeg;
    k_crc_tail<<<1, 1, 0, st>>>(d + body, n - body, tail);
    CUI(cudaGetLastError());
    uint32_t h[2] = {0, 0};
    CUI(cudaMemcpyAsync(&h[0], a, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    CUI(cudaMemcpyAsync(&h[1], tail, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    CUI(cudaFreeAsync(buf, st));
    CUI(cudaStreamSynchronize(st));
    const uint32_t body_crc = nseg ? h[0] : 0;
    *out = gf2_mul(body_crc, x8n(n - body)) ^ h[1];
    return FW_OK;
}

}  // namespace fwi

using namespace fwi;

// ---------------------------------------------------------------------------
extern "C" int fw_edges_max_id(const uint32_t *d_src, const uint32_t *d_dst, uint64_t m,
                               uint64_t *out_max, void *stream) {
    if (!out_max) return set_err_ingest(FW_EVALIDATION, "null output");
    cudaStream_t st = (cudaStream_t)stream;
    unsigned *d = nullptr;
    CUI(cudaMallocAsync(&d, sizeof(unsigned), st));
    CUI(cudaMemsetAsync(d, 0, sizeof(unsigned), st));
    if (m) k_max_id<<<sm_count() * 8, 256, 0, st>>>(d_src, d_dst, m, d);
    unsigned h = 0;
    CUI(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
    CUI(cudaFreeAsync(d, st));
    CUI(cudaStreamSynchronize(st));
    *out_max = h;
    return FW_OK;
}

extern "C" int fw_build_csr_device(const uint32_t *d_src, const uint32_t *d_dst,
                                   const float *d_w, const uint8_t *d_lab, uint64_t m, uint64_t V,
                                   int64_t *d_off, uint32_t *d_tgt, float *d_w_out,
                                   uint8_t *d_lab_out, void *stream) {
    if (!d_off || (m && (!d_src || !d_dst || !d_tgt)))
        return set_err_ingest(FW_EVALIDATION, "fw_build_csr_device: null array");
    if (m >= (1ull << 32)) return set_err_ingest(FW_ECONFIG, "edge count must be < 2^32");
    if (V > (1ull << 32)) return set_err_ingest(FW_ECONFIG, "vertex count must be <= 2^32");
    cudaStream_t st = (cudaStream_t)stream;
    const int sms = sm_count();
    if (m == 0) {
        k_fill_i64<<<sms, 256, 0, st>>>(d_off, V + 1, 0);
        CUI(cudaGetLastError());
        return FW_OK;
    }
    uint64_t mx = 0;
    int rc = fw_edges_max_id(d_src, d_dst, m, &mx, stream);
    if (rc) return rc;
    if (mx >= V)
        return set_err_ingest(FW_EVALIDATION, "vertex id %llu out of range for vertex_count=%llu",
                              (unsigned long long)mx, (unsigned long long)V);
    int bv = 1;
    while (bv < 32 && (1ull << bv) < V) bv++;  // bits of a vertex id
    const int nbits = 2 * bv;
    uint64_t *k0, *k1;
    uint32_t *v0, *v1, *hist;
    unsigned *dmax;
    {   // the sort's scratch (24 B per edge) comes from the device's default
        // pool; keep up to 8 GB of it mapped between builds (remapping the
        // pages dominated repeated builds: 0.2-1.7 s vs 73 ms of kernels at
        // 2^28 edges), larger builds give theirs back
        int dev = 0;
        cudaMemPool_t pool;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = 8ull << 30;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    }
    const uint32_t G = (uint32_t)std::min<uint64_t>((uint64_t)sms * 4, (m + kTile - 1) / kTile);
    const uint64_t seg = ((m + G - 1) / G + kTile - 1) / kTile * kTile;  // whole tiles per CTA
    // the input index rides along only when weights or labels must be gathered
    const bool vals = d_w || d_lab;
    v0 = v1 = nullptr;
    CUI(cudaMallocAsync(&k0, m * sizeof(uint64_t), st));
    CUI(cudaMallocAsync(&k1, m * sizeof(uint64_t), st));
    if (vals) {
        CUI(cudaMallocAsync(&v0, m * sizeof(uint32_t), st));
        CUI(cudaMallocAsync(&v1, m * sizeof(uint32_t), st));
    }
    CUI(cudaMallocAsync(&hist, (size_t)kRadix * G * sizeof(uint32_t), st));
    CUI(cudaMallocAsync(&dmax, sizeof(unsigned), st));
    const bool carried = d_w && !d_lab;
    k_make_keys<<<sms * 8, 256, 0, st>>>(d_src, d_dst, m, bv, carried ? d_w : nullptr, k0, v0);
    for (int shift = 0; shift < nbits; shift += 8) {
        CUI(cudaMemsetAsync(dmax, 0, sizeof(unsigned), st));
        k_hist<<<G, kThreads, 0, st>>>(k0, m, seg, shift, hist);
        k_scan<<<1, 1024, 0, st>>>(hist, kRadix * G, G, dmax);
        unsigned h = 0;
        CUI(cudaMemcpyAsync(&h, dmax, sizeof(h), cudaMemcpyDeviceToHost, st));
        CUI(cudaStreamSynchronize(st));
        if (h == m) continue;  // every key has the same digit: the pass is the identity
        if (vals)
            k_scatter<true><<<G, kThreads, 0, st>>>(k0, v0, m, seg, shift, hist, k1, v1);
        else
            k_scatter<false><<<G, kThreads, 0, st>>>(k0, nullptr, m, seg, shift, hist, k1, nullptr);
        std::swap(k0, k1);
        std::swap(v0, v1);
    }
    k_csr_edges<<<sms * 8, 256, 0, st>>>(k0, v0, carried, m, bv, d_w, d_lab, d_tgt, d_w_out,
                                         d_lab_out);
    k_csr_offsets<<<sms * 16, 256, 0, st>>>(k0, m, V, bv, d_off);
    CUI(cudaGetLastError());
    cudaFreeAsync(k0, st);
    cudaFreeAsync(k1, st);
    if (v0) cudaFreeAsync(v0, st);
    if (v1) cudaFreeAsync(v1, st);
    cudaFreeAsync(hist, st);
    cudaFreeAsync(dmax, st);
    CUI(cudaStreamSynchronize(st));
    return FW_OK;
}

// ---------------------------------------------------------------------------
// FWG1 (graph.py:204-254): "FWG1", <QQB (V, E, flags), offsets u64[V+1],
// targets u32[E], weights f32[E], [labels u8[E] if flags & 2], crc32 u32.
// ---------------------------------------------------------------------------
static const uint64_t kHeader = 21;
// FWG1 streaming: reader threads x 2 pinned chunks, kept for the process
static const uint64_t kFwg1Chunk = 16ull << 20;
static const int kFwg1Threads = 8;
static std::mutex g_pin_mu;
static std::vector<void *> g_pin;

extern "C" int fw_fwg1_info(const char *path, uint64_t *V, uint64_t *E, int32_t *flags) {
    if (!path || !V || !E || !flags) return set_err_ingest(FW_EVALIDATION, "null argument");
    const int fd = open(path, O_RDONLY);
    if (fd < 0) return set_err_ingest(FW_EFORMAT, "%s: cannot open (%s)", path, strerror(errno));
    struct stat sb;
    fstat(fd, &sb);
    unsigned char h[kHeader];
    const ssize_t got = pread(fd, h, kHeader, 0);
    close(fd);
    if (got < (ssize_t)kHeader || memcmp(h, "FWG1", 4) != 0)
        return set_err_ingest(FW_EFORMAT, "%s: bad magic (not a graph file)", path);
    uint64_t v, e;
    memcpy(&v, h + 4, 8);
    memcpy(&e, h + 12, 8);
    const int f = h[20];
    const unsigned __int128 need = (unsigned __int128)kHeader + 8 * ((unsigned __int128)v + 1) +
                                   8 * (unsigned __int128)e + ((f & 2) ? e : 0) + 4;
    if ((unsigned __int128)sb.st_size != need)
        return set_err_ingest(FW_EFORMAT, "%s: truncated or oversized file (%lld bytes, want %llu)",
                              path, (long long)sb.st_size, (unsigned long long)need);
    *V = v;
    *E = e;
    *flags = f;
    return FW_OK;
}

// Host arrays -> device arrays through the process's pinned pool: kFwg1Threads
// threads, each memcpy-ing 16 MB chunks of the concatenated arrays into its two
// pinned buffers while the previous chunk's H2D runs on its own stream
// (fw_graph_create's upload: one thread and per-call pinned buffers moved
// ~6 GB/s).
int fwi::staged_h2d(int n, const void *const *src, void *const *dst, const uint64_t *bytes) {
    uint64_t total = 0;
    for (int i = 0; i < n; i++) total += bytes[i];
    if (!total) return FW_OK;
    const uint64_t chunk = kFwg1Chunk;
    const int nthreads = kFwg1Threads;
    int dev = 0;
    cudaGetDevice(&dev);
    std::unique_lock<std::mutex> pin_lk(g_pin_mu);
    if (g_pin.empty()) {
        g_pin.assign(2 * nthreads, nullptr);
        for (auto &p : g_pin) {
            if (cudaMallocHost(&p, chunk) != cudaSuccess) {
                for (auto &q : g_pin)
                    if (q) cudaFreeHost(q);
                g_pin.clear();
                return set_err_ingest(FW_ENOMEM, "pinned staging allocation failed");
            }
        }
    }
    std::vector<int> trc(nthreads, FW_OK);
    auto worker = [&](int tid) {
        cudaSetDevice(dev);
        void *pin[2] = {g_pin[2 * tid], g_pin[2 * tid + 1]};
        cudaEvent_t ev[2];
        cudaStream_t ts;
        cudaStreamCreateWithFlags(&ts, cudaStreamNonBlocking);
        cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming);
        cudaEventRecord(ev[0], ts);
        cudaEventRecord(ev[1], ts);
        int slot = 0;
        for (uint64_t c0 = (uint64_t)tid * chunk; c0 < total; c0 += (uint64_t)nthreads * chunk, slot ^= 1) {
            const uint64_t cn = std::min(chunk, total - c0);
            cudaEventSynchronize(ev[slot]);
            uint64_t base = 0;
            for (int i = 0; i < n; i++) {  // the chunk's intersection with each array
                const uint64_t lo = std::max(c0, base), hi = std::min(c0 + cn, base + bytes[i]);
                if (lo < hi) {
                    memcpy((char *)pin[slot] + (lo - c0), (const char *)src[i] + (lo - base), hi - lo);
                    cudaMemcpyAsync((char *)dst[i] + (lo - base), (char *)pin[slot] + (lo - c0),
                                    hi - lo, cudaMemcpyHostToDevice, ts);
                }
                base += bytes[i];
            }
            cudaEventRecord(ev[slot], ts);
        }
        if (cudaStreamSynchronize(ts) != cudaSuccess) trc[tid] = FW_ECUDA;
        cudaEventDestroy(ev[0]);
        cudaEventDestroy(ev[1]);
        cudaStreamDestroy(ts);
    };
    std::vector<std::thread> th;
    for (int t = 0; t < nthreads; t++) th.emplace_back(worker, t);
    for (auto &t : th) t.join();
    for (int t = 0; t < nthreads; t++)
        if (trc[t]) return set_err_ingest(trc[t], "host-to-device upload failed");
    return FW_OK;
}

extern "C" int fw_fwg1_read(const char *path, uint64_t V, uint64_t E, int32_t flags,
                            int64_t *d_off, uint32_t *d_tgt, float *d_w, uint8_t *d_lab,
                            uint32_t *crc_out, void *stream) {
    uint64_t v2, e2;
    int32_t f2;
    int rc = fw_fwg1_info(path, &v2, &e2, &f2);
    if (rc) return rc;
    if (v2 != V || e2 != E || f2 != flags)
        return set_err_ingest(FW_EVALIDATION, "%s: header does not match the arguments", path);
    const bool has_lab = (flags & 2) != 0;
    if (!d_off || (E && (!d_tgt || !d_w)) || (E && has_lab && !d_lab))
        return set_err_ingest(FW_EVALIDATION, "fw_fwg1_read: null device array");
    // payload pieces in file order
    struct Piece {
        uint64_t off, bytes;
        uint8_t *dst;
    };
    std::vector<Piece> pieces;
    uint64_t pos = kHeader;
    pieces.push_back({pos, 8 * (V + 1), (uint8_t *)d_off});
    pos += 8 * (V + 1);
    pieces.push_back({pos, 4 * E, (uint8_t *)d_tgt});
    pos += 4 * E;
    pieces.push_back({pos, 4 * E, (uint8_t *)d_w});
    pos += 4 * E;
    if (has_lab) {
        pieces.push_back({pos, E, d_lab});
        pos += E;
    }
    const uint64_t payload_end = pos;
    const int fd = open(path, O_RDONLY);
    if (fd < 0) return set_err_ingest(FW_EFORMAT, "%s: cannot open", path);
    // Reader threads, each with its own stream and two pinned buffers: a
    // thread reads chunk c (pread) while its previous chunk's H2D runs.  The
    // pinned buffers are allocated once per process and reused (pinning 256
    // MB per call cost more than the copies of a 2 GB file).
    const uint64_t chunk = kFwg1Chunk;
    const int nthreads = kFwg1Threads;
    int dev = 0;
    cudaGetDevice(&dev);
    std::unique_lock<std::mutex> pin_lk(g_pin_mu);  // one FWG1 read at a time owns the pool
    if (g_pin.empty()) {
        g_pin.assign(2 * nthreads, nullptr);
        for (auto &p : g_pin) {
            if (cudaMallocHost(&p, chunk) != cudaSuccess) {
                for (auto &q : g_pin)
                    if (q) cudaFreeHost(q);
                g_pin.clear();
                return set_err_ingest(FW_ENOMEM, "pinned staging allocation failed");
            }
        }
    }
    std::vector<int> trc(nthreads, FW_OK);
    std::vector<std::string> terr(nthreads);
    auto worker = [&](int tid) {
        cudaSetDevice(dev);
        void *pin[2] = {g_pin[2 * tid], g_pin[2 * tid + 1]};
        cudaEvent_t ev[2];
        cudaStream_t ts;
        cudaStreamCreateWithFlags(&ts, cudaStreamNonBlocking);
        cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming);
        cudaEventRecord(ev[0], ts);
        cudaEventRecord(ev[1], ts);
        int slot = 0;
        for (uint64_t c0 = kHeader + (uint64_t)tid * chunk; c0 < payload_end;
             c0 += (uint64_t)nthreads * chunk, slot ^= 1) {
            const uint64_t n = std::min(chunk, payload_end - c0);
            cudaEventSynchronize(ev[slot]);
            uint64_t got = 0;
            while (got < n) {
                const ssize_t r = pread(fd, (char *)pin[slot] + got, n - got, (off_t)(c0 + got));
                if (r <= 0) break;
                got += (uint64_t)r;
            }
            if (got != n) {
                trc[tid] = FW_EFORMAT;
                terr[tid] = std::string(path) + ": short read";
                break;
            }
            for (const Piece &p : pieces) {  // the chunk's intersection with each array
                const uint64_t lo = std::max(c0, p.off), hi = std::min(c0 + n, p.off + p.bytes);
                if (lo < hi)
                    cudaMemcpyAsync(p.dst + (lo - p.off), (char *)pin[slot] + (lo - c0), hi - lo,
                                    cudaMemcpyHostToDevice, ts);
            }
            cudaEventRecord(ev[slot], ts);
        }
        if (cudaStreamSynchronize(ts) != cudaSuccess && trc[tid] == FW_OK) {
            trc[tid] = FW_ECUDA;
            terr[tid] = "H2D copy failed";
        }
        cudaEventDestroy(ev[0]);
        cudaEventDestroy(ev[1]);
        cudaStreamDestroy(ts);
    };
    std::vector<std::thread> th;
    for (int t = 0; t < nthreads; t++) th.emplace_back(worker, t);
    for (auto &t : th) t.join();
    uint32_t stored = 0;
    const bool crc_ok = pread(fd, &stored, 4, (off_t)payload_end) == 4;
    close(fd);
    for (int t = 0; t < nthreads; t++)
        if (trc[t]) return set_err_ingest(trc[t], "%s", terr[t].c_str());
    if (!crc_ok) return set_err_ingest(FW_EFORMAT, "%s: short read", path);
    // CRC-32 of the payload on the device, array by array, then combined
    cudaStream_t st = (cudaStream_t)stream;
    uint32_t raw = 0;
    uint64_t total = 0;
    for (const Piece &p : pieces) {
        uint32_t r = 0;
        rc = device_raw_crc(p.dst, p.bytes, st, &r);
        if (rc) return rc;
        raw = gf2_mul(raw, x8n(p.bytes)) ^ r;
        total += p.bytes;
    }
    const uint32_t crc = raw ^ gf2_mul(0xFFFFFFFFu, x8n(total)) ^ 0xFFFFFFFFu;
    if (crc_out) *crc_out = crc;
    if (crc != stored) return set_err_ingest(FW_EFORMAT, "%s: checksum mismatch", path);
    return FW_OK;
}

// raw-free CRC-32 of a device range (zlib value), for tests and writers
extern "C" int fw_crc32_device(const uint8_t *d, uint64_t n, uint32_t *out, void *stream) {
    if (!out || (n && !d)) return set_err_ingest(FW_EVALIDATION, "null argument");
    uint32_t raw = 0;
    const int rc = device_raw_crc(d, n, (cudaStream_t)stream, &raw);
    if (rc) return rc;
    *out = raw ^ gf2_mul(0xFFFFFFFFu, x8n(n)) ^ 0xFFFFFFFFu;
    return FW_OK;
}
