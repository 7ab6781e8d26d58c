// C ABI of libflowwalk.so (declared in include/flowwalk.h): device-resident
// CSR handle, walk launch (device and host buffers), GPU validator and the
// synthetic-input generators.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/flowwalk.h"
#include "fw_common.cuh"
#include "fw_walk.cuh"

using namespace fw;

static thread_local std::string g_err;

static int set_err(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CU(expr)                                                                         \
    do {                                                                                 \
        cudaError_t e_ = (expr);                                                         \
        if (e_ != cudaSuccess)                                                           \
            return set_err(e_ == cudaErrorMemoryAllocation ? FW_ENOMEM : FW_ECUDA,       \
                           "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__,    \
                           __LINE__);                                                    \
    } while (0)

struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
    cudaError_t reserve(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e == cudaSuccess) cap = bytes;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

constexpr int kQueueRing = 64;

struct fw_graph {
    int device = 0;
    uint64_t V = 0, E = 0;
    int64_t *off = nullptr;
    uint32_t *tgt = nullptr;
    float *w = nullptr;
    uint8_t *lab = nullptr;
    bool owned = false;
    fw_graph_info info{};
    unsigned long long *queues = nullptr;  // ring of per-launch cursors
    unsigned call_counter = 0;
    // a cursor slot (and its schema copy) is reused only after the kernel
    // that last used it has finished, whatever stream either runs on
    cudaEvent_t slot_ev[kQueueRing] = {};
    bool slot_used[kQueueRing] = {};
    std::mutex mu;
    std::mutex host_mu;  // serialises fw_walk's host-buffer scratch
    // host-buffer walk scratch (grow-only); [1] only for sub-launched walks
    DevBuf starts[2], seq[2], len[2], stats, done;
    std::vector<DevBuf> schema_ring;
    uint64_t scratch_limit = 0;  // bytes, 0 = auto
    int sm_count = 0;
    // fw_walk's streams and events, created on first use and kept (creating
    // them per call cost tens of microseconds against millisecond walks)
    cudaStream_t walk_st = nullptr, copy_st = nullptr;
    cudaEvent_t ev[6] = {};
    cudaEvent_t buf_free[2] = {};  // sub-launch ping-pong: buffer's D2H done

    int64_t aux_bytes() const {  // the engine's own scratch (AllocationMeter analogue)
        int64_t b = kQueueRing * sizeof(unsigned long long) + stats.cap + done.cap;
        for (const DevBuf &x : schema_ring) b += x.cap;
        return b;
    }
    int64_t aux_allocations() const {
        int64_t n = 1 + (stats.cap ? 1 : 0) + (done.cap ? 1 : 0);
        for (const DevBuf &x : schema_ring) n += x.cap ? 1 : 0;
        return n;
    }
};

extern "C" const char *fw_last_error(void) { return g_err.c_str(); }

namespace fwi {  // csrc/fw_ingest.cu reports through the same thread-local message
int set_err_ingest(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}
}  // namespace fwi

extern "C" int fw_device_count(int *out) {
    CU(cudaGetDeviceCount(out));
    return FW_OK;
}

// ---------------------------------------------------------------------------
// Graph profile kernels (run once at upload).
// ---------------------------------------------------------------------------
__global__ void k_degree_max(const int64_t *__restrict__ off, uint64_t V,
                             unsigned long long *out) {
    unsigned long long best = 0;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < V;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long d = (unsigned long long)(off[v + 1] - off[v]);
        const unsigned long long key = (d << 32) | (0xFFFFFFFFull - (v & 0xFFFFFFFFull));
        best = key > best ? key : best;
    }
    for (int o = 16; o; o >>= 1) {
        unsigned long long x = __shfl_xor_sync(FULL, best, o);
        best = x > best ? x : best;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(out, best);
}

__global__ void k_weight_profile(const float *__restrict__ w, uint64_t E, int *minlow,
                                 unsigned *maxbits, int *bad) {
    int lo = INT_MAX;
    unsigned mx = 0;
    int b = 0;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < E;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const float x = w[e];
        const unsigned bits = __float_as_uint(x);
        if (!(x >= 0.0f) || isinf(x)) { b = 1; continue; }
        if (x > 0.0f) {
            const int ex = (bits >> 23) & 0xFF;
            const unsigned man = bits & 0x7FFFFFu;
            int low;
            if (ex == 0) low = -149 + __ffs(man) - 1;
            else low = ex - 150 + __ffs(man | 0x800000u) - 1;
            lo = min(lo, low);
            mx = max(mx, bits);
        }
    }
    for (int o = 16; o; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(FULL, lo, o));
        mx = max(mx, __shfl_xor_sync(FULL, mx, o));
        b |= __shfl_xor_sync(FULL, b, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(minlow, lo);
        atomicMax(maxbits, mx);
        if (b) atomicOr(bad, 1);
    }
}

// CSR checks (reference Graph.validate, graph.py:70-81): offsets
// non-decreasing, targets < V; per-vertex sortedness is recorded (the
// reference accepts unsorted lists, but its Node2Vec membership test is a
// binary search over N(prev), _kernels.py:293-306, which our window tables
// reproduce only for sorted lists).  Flags: 1 = offsets decrease, 2 = target
// out of range, 4 = some list unsorted.
__global__ void k_check_offsets(const int64_t *__restrict__ off, uint64_t V, uint64_t E,
                                uint32_t *bounds, int *flags) {
    int f = 0;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < V;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const int64_t a = off[v], b = off[v + 1];
        if (b < a || a < 0 || b > (int64_t)E) { f |= 1; continue; }
        if (b > a) atomicOr(bounds + (a >> 5), 1u << (a & 31));  // a list starts at a
    }
    if (f) atomicOr(flags, f);
}

__global__ void k_check_targets(const uint32_t *__restrict__ tgt, uint64_t E, uint64_t V,
                                const uint32_t *__restrict__ bounds, int *flags) {
    int f = 0;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < E;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t t = tgt[e];
        if ((uint64_t)t >= V) f |= 2;
        if (e + 1 < E && t > tgt[e + 1] && !((bounds[(e + 1) >> 5] >> ((e + 1) & 31)) & 1)) f |= 4;
    }
    f |= __shfl_xor_sync(FULL, f, 16);
    f |= __shfl_xor_sync(FULL, f, 8);
    f |= __shfl_xor_sync(FULL, f, 4);
    f |= __shfl_xor_sync(FULL, f, 2);
    f |= __shfl_xor_sync(FULL, f, 1);
    if ((threadIdx.x & 31) == 0 && f) atomicOr(flags, f);
}

static int check_csr(fw_graph *g) {
    int64_t ends[2] = {0, 0};
    CU(cudaMemcpy(&ends[0], g->off, sizeof(int64_t), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(&ends[1], g->off + g->V, sizeof(int64_t), cudaMemcpyDeviceToHost));
    if (ends[0] != 0 || (uint64_t)ends[1] != g->E)
        return set_err(FW_EVALIDATION, "offsets must start at 0 and end at edge_count");
    if (g->E && (!g->tgt || !g->w))
        return set_err(FW_EVALIDATION, "null targets or weights for a non-empty graph");
    uint32_t *bounds = nullptr;
    int *flags = nullptr;
    const size_t nw = (g->E + 1 + 31) / 32;
    CU(cudaMalloc(&bounds, nw * sizeof(uint32_t)));
    CU(cudaMalloc(&flags, sizeof(int)));
    cudaMemset(bounds, 0, nw * sizeof(uint32_t));
    cudaMemset(flags, 0, sizeof(int));
    const int grid = g->sm_count * 8;
    if (g->V) k_check_offsets<<<grid, 256>>>(g->off, g->V, g->E, bounds, flags);
    int f = 0;
    cudaError_t e = cudaMemcpy(&f, flags, sizeof(int), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && !(f & 1) && g->E) {
        k_check_targets<<<grid, 256>>>(g->tgt, g->E, g->V, bounds, flags);
        e = cudaMemcpy(&f, flags, sizeof(int), cudaMemcpyDeviceToHost);
    }
    cudaFree(bounds);
    cudaFree(flags);
    CU(e);
    if (f & 1) return set_err(FW_EVALIDATION, "offsets must be non-decreasing");
    if (f & 2) return set_err(FW_EVALIDATION, "target id out of range");
    g->info.sorted_lists = (f & 4) ? 0 : 1;
    return FW_OK;
}

static int profile_graph(fw_graph *g) {
    int rc = check_csr(g);
    if (rc) return rc;
    unsigned long long *d_deg;
    int *d_i;
    CU(cudaMalloc(&d_deg, sizeof(unsigned long long)));
    CU(cudaMalloc(&d_i, 3 * sizeof(int)));
    CU(cudaMemset(d_deg, 0, sizeof(unsigned long long)));
    int init[3] = {INT_MAX, 0, 0};
    CU(cudaMemcpy(d_i, init, sizeof(init), cudaMemcpyHostToDevice));
    const int grid = g->sm_count * 8;
    if (g->V) k_degree_max<<<grid, 256>>>(g->off, g->V, d_deg);
    if (g->E) k_weight_profile<<<grid, 256>>>(g->w, g->E, d_i, (unsigned *)(d_i + 1), d_i + 2);
    CU(cudaGetLastError());
    unsigned long long key = 0;
    int res[3];
    CU(cudaMemcpy(&key, d_deg, sizeof(key), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(res, d_i, sizeof(res), cudaMemcpyDeviceToHost));
    cudaFree(d_deg);
    cudaFree(d_i);
    g->info.max_degree = g->V ? (int64_t)(key >> 32) : 0;
    g->info.max_degree_vertex = g->V ? (int64_t)(0xFFFFFFFFull - (key & 0xFFFFFFFFull)) : -1;
    g->info.min_weight_lowbit_exp = res[0];
    unsigned mb = (unsigned)res[1];
    float mw;
    memcpy(&mw, &mb, sizeof(mw));
    g->info.max_weight = mw;
    g->info.has_labels = g->lab != nullptr;
    g->info.bad_weights = res[2];  // non-finite / negative weight flag
    return FW_OK;
}

static int graph_common_init(fw_graph *g, int device) {
    g->device = device;
    CU(cudaSetDevice(device));
    CU(cudaDeviceGetAttribute(&g->sm_count, cudaDevAttrMultiProcessorCount, device));
    CU(cudaMalloc(&g->queues, kQueueRing * sizeof(unsigned long long)));
    return FW_OK;
}

namespace fwi {
int staged_h2d(int n, const void *const *src, void *const *dst, const uint64_t *bytes);
}

extern "C" int fw_graph_create(const int64_t *offsets, const uint32_t *targets,
                               const float *weights, const uint8_t *labels, uint64_t V,
                               uint64_t E, int device, fw_graph **out) {
    if (!out || !offsets || (E && (!targets || !weights)))
        return set_err(FW_EVALIDATION, "fw_graph_create: null array");
    if (offsets[0] != 0 || (uint64_t)offsets[V] != E)
        return set_err(FW_EVALIDATION, "offsets must start at 0 and end at edge_count");
    fw_graph *g = new fw_graph();
    int rc = graph_common_init(g, device);
    if (rc) { delete g; return rc; }
    g->V = V;
    g->E = E;
    g->owned = true;
    auto fail = [&](int code) {
        fw_graph_destroy(g);
        return code;
    };
    cudaError_t e;
    if ((e = cudaMalloc(&g->off, (V + 1) * sizeof(int64_t))) != cudaSuccess ||
        (e = cudaMalloc(&g->tgt, (E + 4) * sizeof(uint32_t))) != cudaSuccess ||  // +4: tail of
        (e = cudaMalloc(&g->w, (E + 4) * sizeof(float))) != cudaSuccess ||        // 16-byte tiles
        (labels && (e = cudaMalloc(&g->lab, std::max<uint64_t>(E, 1))) != cudaSuccess))
        return fail(set_err(FW_ENOMEM, "graph allocation: %s", cudaGetErrorString(e)));
    {   // one pass through the process's pinned pool, 8 copy threads
        const void *src[4] = {offsets, targets, weights, labels};
        void *dst[4] = {g->off, g->tgt, g->w, g->lab};
        const uint64_t bytes[4] = {(V + 1) * sizeof(int64_t), E * sizeof(uint32_t),
                                   E * sizeof(float), labels ? E : 0};
        rc = fwi::staged_h2d(4, src, dst, bytes);  // sets fw_last_error on failure
    }
    if (rc) return fail(rc);
    if ((rc = profile_graph(g))) return fail(rc);
    *out = g;
    return FW_OK;
}

extern "C" int fw_graph_create_device(const int64_t *d_off, const uint32_t *d_tgt,
                                      const float *d_w, const uint8_t *d_lab, uint64_t V,
                                      uint64_t E, int device, fw_graph **out) {
    if (!out || !d_off) return set_err(FW_EVALIDATION, "fw_graph_create_device: null array");
    fw_graph *g = new fw_graph();
    int rc = graph_common_init(g, device);
    if (rc) { delete g; return rc; }
    g->V = V;
    g->E = E;
    g->off = const_cast<int64_t *>(d_off);
    g->tgt = const_cast<uint32_t *>(d_tgt);
    g->w = const_cast<float *>(d_w);
    g->lab = const_cast<uint8_t *>(d_lab);
    g->owned = false;
    if ((rc = profile_graph(g))) {
        fw_graph_destroy(g);
        return rc;
    }
    *out = g;
    return FW_OK;
}

// Replica of a resident CSR on another device: device-to-device peer copies
// (NVLink on NVSwitch systems; staged by the driver when peers are not
// enabled), no host round trip and no re-validation.
extern "C" int fw_graph_replicate(fw_graph *src, int device, fw_graph **out) {
    if (!src || !out) return set_err(FW_EVALIDATION, "null handle");
    fw_graph *g = new fw_graph();
    int rc = graph_common_init(g, device);
    if (rc) { delete g; return rc; }
    g->V = src->V;
    g->E = src->E;
    g->owned = true;
    g->info = src->info;
    const uint64_t V = g->V, E = g->E;
    auto fail = [&](int code) {
        fw_graph_destroy(g);
        return code;
    };
    cudaError_t e;
    if ((e = cudaMalloc(&g->off, (V + 1) * sizeof(int64_t))) != cudaSuccess ||
        (e = cudaMalloc(&g->tgt, (E + 4) * sizeof(uint32_t))) != cudaSuccess ||
        (e = cudaMalloc(&g->w, (E + 4) * sizeof(float))) != cudaSuccess ||
        (src->lab && (e = cudaMalloc(&g->lab, std::max<uint64_t>(E, 1))) != cudaSuccess))
        return fail(set_err(FW_ENOMEM, "replica allocation: %s", cudaGetErrorString(e)));
    int can = 0;
    if (device != src->device && cudaDeviceCanAccessPeer(&can, device, src->device) == cudaSuccess &&
        can) {
        e = cudaDeviceEnablePeerAccess(src->device, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
    }
    cudaStream_t st;
    if ((e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)) != cudaSuccess)
        return fail(set_err(FW_ECUDA, "stream: %s", cudaGetErrorString(e)));
    e = cudaMemcpyPeerAsync(g->off, device, src->off, src->device, (V + 1) * sizeof(int64_t), st);
    if (e == cudaSuccess && E)
        e = cudaMemcpyPeerAsync(g->tgt, device, src->tgt, src->device, E * sizeof(uint32_t), st);
    if (e == cudaSuccess && E)
        e = cudaMemcpyPeerAsync(g->w, device, src->w, src->device, E * sizeof(float), st);
    if (e == cudaSuccess && E && src->lab)
        e = cudaMemcpyPeerAsync(g->lab, device, src->lab, src->device, E, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
    if (e != cudaSuccess) return fail(set_err(FW_ECUDA, "peer copy: %s", cudaGetErrorString(e)));
    *out = g;
    return FW_OK;
}

extern "C" int fw_graph_destroy(fw_graph *g) {
    if (!g) return FW_OK;
    cudaSetDevice(g->device);
    if (g->owned) {
        cudaFree(g->off);
        cudaFree(g->tgt);
        cudaFree(g->w);
        if (g->lab) cudaFree(g->lab);
    }
    if (g->queues) cudaFree(g->queues);
    for (int i = 0; i < 2; i++) {
        g->starts[i].release();
        g->seq[i].release();
        g->len[i].release();
        if (g->buf_free[i]) cudaEventDestroy(g->buf_free[i]);
    }
    g->stats.release();
    g->done.release();
    for (int i = 0; i < kQueueRing; i++)
        if (g->slot_ev[i]) cudaEventDestroy(g->slot_ev[i]);
    if (g->walk_st) {
        for (cudaEvent_t e : g->ev) cudaEventDestroy(e);
        cudaStreamDestroy(g->walk_st);
        cudaStreamDestroy(g->copy_st);
    }
    for (auto &b : g->schema_ring) b.release();
    delete g;
    return FW_OK;
}

extern "C" int fw_graph_set_scratch_limit(fw_graph *g, uint64_t bytes) {
    if (!g) return set_err(FW_EVALIDATION, "null handle");
    std::lock_guard<std::mutex> lk(g->host_mu);
    g->scratch_limit = bytes;
    return FW_OK;
}

extern "C" int fw_graph_info_get(fw_graph *g, fw_graph_info *out) {
    if (!g || !out) return set_err(FW_EVALIDATION, "null handle");
    *out = g->info;
    return FW_OK;
}

// ---------------------------------------------------------------------------
// Exact-order predicate: every app weight is an integer multiple
// of 2^G and every per-step partial sum is <= d_max * x_max <= 2^(52+G), so
// all fp64 partial sums are exact and any summation order reproduces the
// reference's sequential `run += w` bit-for-bit.
// ---------------------------------------------------------------------------
static bool exact_order_ok(const fw_graph_info &gi, const fw_app &app, long *g_out = nullptr,
                           double *xmax_out = nullptr) {
    if (gi.bad_weights) return false;  // non-finite or negative weights: be literal
    std::vector<double> F{1.0};
    if (app.app_id == FW_APP_NODE2VEC) {
        F.push_back(app.inv_a);
        F.push_back(app.inv_b);
    }
    const bool weighted = app.weighted != 0;
    if (weighted && !(gi.max_weight > 0.0f)) return true;  // every weight is zero
    long G = LONG_MAX;
    double xmax = 0.0;
    for (double f : F) {
        if (!(f > 0.0) || !std::isfinite(f)) return false;
        int ex;
        const double m = std::frexp(f, &ex);  // f = m * 2^ex, m in [0.5, 1)
        uint64_t M = (uint64_t)std::ldexp(m, 53);
        const int tz = __builtin_ctzll(M);
        M >>= tz;
        const int bits = 64 - __builtin_clzll(M);
        const long low = (long)ex - 53 + tz;  // f = M * 2^low, M odd
        if (weighted) {
            if (bits + 24 > 53) return false;  // f * w would round
            G = std::min(G, low + (long)gi.min_weight_lowbit_exp);
            xmax = std::max(xmax, f * (double)gi.max_weight);
        } else {
            G = std::min(G, low);
            xmax = std::max(xmax, f);
        }
    }
    if (G < -1000) return false;
    if (g_out) *g_out = G;
    if (xmax_out) *xmax_out = xmax;
    const double lim = std::ldexp(1.0, (int)(52 + G));
    return (double)gi.max_degree * xmax <= lim;
}

static int check_cfg(fw_graph *g, const fw_app *app, const fw_engine *eng) {
    if (!g || !app || !eng) return set_err(FW_EVALIDATION, "null argument");
    if (app->app_id < 0 || app->app_id > 3) return set_err(FW_EVALIDATION, "unknown app id");
    if (app->length < 1) return set_err(FW_EVALIDATION, "walk length must be >= 1");
    if (app->length >= (1u << 20))
        return set_err(FW_ECONFIG, "walk length exceeds the replay stream-id field");
    if (app->app_id == FW_APP_METAPATH && app->schema_len == 0)
        return set_err(FW_EVALIDATION, "metapath needs a non-empty schema");
    if (!(1 <= eng->k_small && eng->k_small <= eng->k_big))
        return set_err(FW_ECONFIG, "lane widths must satisfy 1 <= k_small <= k_big");
    if (eng->k_big > 1000) return set_err(FW_ECONFIG, "k_big larger than the stream-id lane field");
    if (eng->d_t < 1) return set_err(FW_ECONFIG, "degree threshold must be >= 1");
    if (eng->sampler_id != FW_SAMPLER_ZPRS && eng->sampler_id != FW_SAMPLER_DPRS)
        return set_err(FW_ECONFIG, "unknown sampler id");
    if (app->app_id == FW_APP_NODE2VEC && !g->info.sorted_lists)
        return set_err(FW_EVALIDATION,
                       "node2vec needs every neighbour list sorted (build_csr order)");
    return FW_OK;
}

static int launch(fw_graph *g, const int64_t *d_starts, uint64_t n, uint64_t base_qid,
                  const fw_app *app, const fw_engine *eng, uint64_t seed, uint32_t *d_seq,
                  uint32_t *d_len, int64_t *d_stats, cudaStream_t stream, int *mode_out,
                  int *grid_out, unsigned *d_done = nullptr, uint64_t piece_q = 0) {
    if (base_qid + n > (1ull << 33))
        return set_err(FW_ECONFIG, "query ids exceed the replay stream-id field (2^33)");
    long G = 0;
    double xmax = 0.0;
    // FW_FORCE_CERT=1 (tests): certified mode even where every sum is exact
    const char *force_cert = getenv("FW_FORCE_CERT");
    const bool fc = force_cert && force_cert[0] == '1';
    const bool exact = eng->order_mode == FW_ORDER_AUTO && !fc &&
                       exact_order_ok(g->info, *app, &G, &xmax);
    // certified mode (weights whose sums round, e.g. log-normal):
    // tree-order scans with certified accept tests; needs nonnegative finite
    // weights and sums far from overflow (cert_accept's bound)
    int mode = exact ? 1 : 0;
    if (!exact && eng->order_mode == FW_ORDER_AUTO && !(app->weighted && g->info.bad_weights)) {
        double fmax = 1.0;
        if (app->app_id == FW_APP_NODE2VEC) fmax = std::max({1.0, app->inv_a, app->inv_b});
        const double wmax = app->weighted ? (double)g->info.max_weight : 1.0;
        const double tot = (double)g->info.max_degree * fmax * wmax;
        const char *env = getenv("FW_CERT");  // A/B override: 0 keeps the ordered kernels
        if (std::isfinite(fmax) && tot < 1e290 && !(env && env[0] == '0')) mode = 2;
    }
    if (mode_out) *mode_out = mode;
    if (n == 0) return FW_OK;
    WalkArgs a{};
    a.off = g->off;
    a.tgt = g->tgt;
    a.w = g->w;
    a.lab = g->lab;
    a.starts = d_starts;
    a.n = n;
    a.base_qid = base_qid;
    a.out_seq = d_seq;
    a.out_len = d_len;
    a.L = app->length;
    a.weighted = app->weighted;
    a.stop_prob = app->stop_prob;
    a.inv_a = app->inv_a;
    a.inv_b = app->inv_b;
    a.fac[0] = app->inv_b;
    a.fac[1] = 1.0;
    a.fac[2] = app->inv_a;
    a.fac[3] = app->inv_a;
    {   // largest app weight, rounded up to fp32 (node2vec accept prefilter)
        double fmax = 1.0;
        if (app->app_id == FW_APP_NODE2VEC) fmax = std::max({1.0, app->inv_a, app->inv_b});
        const double wm = fmax * (app->weighted ? (double)g->info.max_weight : 1.0);
        float f = (float)wm;
        if ((double)f < wm) f = std::nextafter(f, INFINITY);
        // inf: prefilter off.  Negative or non-finite weights (reserved) let
        // the running prefix shrink, which the prefilter's bound assumes away.
        const bool lit = app->weighted && g->info.bad_weights;
        a.accept_wmax = (std::isfinite(f) && f <= 1e37f && !lit) ? f : INFINITY;
    }
    {   // fp32 factor path: 1/a, 1/b = 2^k and every w * 2^k exact in fp32
        auto pow2_exp = [](double f, int *k) {
            int e;
            const double m = std::frexp(f, &e);
            *k = e - 1;
            return f > 0.0 && m == 0.5;
        };
        int ka = 0, kb = 0;
        bool ok = app->app_id == FW_APP_NODE2VEC && pow2_exp(app->inv_a, &ka) &&
                  pow2_exp(app->inv_b, &kb) && std::abs(ka) <= 16 && std::abs(kb) <= 16;
        if (ok && app->weighted) {
            const int kmin = std::min({0, ka, kb}), kmax = std::max({0, ka, kb});
            ok = !g->info.bad_weights &&
                 (!(g->info.max_weight > 0.0f) ||
                  ((long)g->info.min_weight_lowbit_exp + kmin >= -149 &&
                   std::ldexp((double)g->info.max_weight, kmax) <= (double)FLT_MAX));
        }
        const char *env = getenv("FW_FAC32");  // A/B override: 0 forces the fp64 factor path
        a.fac32 = ok && !(env && env[0] == '0') ? 1 : 0;
        a.inv_a32 = (float)app->inv_a;
        a.inv_b32 = (float)app->inv_b;
    }
    {   // integer tile sums (node2vec fp32 factor path): every app weight is
        // an integer multiple of 2^G, so w * 2^-G is an exact integer; a
        // lane's 4 of them must fit a u32 and the scaled prefilter bound
        // must stay finite
        double sc = std::ldexp(1.0, (int)-G);
        const char *env = getenv("FW_ISCAN");  // A/B override: 0 forces the fp64 tile scan
        const bool iscan_ok = !(env && env[0] == '0');
        bool qscan = false;
        a.qscale = 1.0;
        if (mode == 2 && !a.fac32 && app->weighted && app->app_id == FW_APP_NODE2VEC &&
            g->info.max_weight > 0.0f && iscan_ok) {
            // fp64 factors (1/a, 1/b not powers of two): scale the fp64
            // products f * w by 2^s < 2^29 / max; exact in fp64, then rounded
            const double xm = std::max({1.0, app->inv_a, app->inv_b}) * (double)g->info.max_weight;
            int e2 = 0;
            std::frexp(xm, &e2);
            const int sh = 29 - e2;
            if (sh >= -900 && sh <= 900 && std::isfinite(xm)) {
                a.qscale = std::ldexp(1.0, sh);
                a.iscan = 1;  // selects the quantized tile sums for fp64 factors
            }
        }
        if (mode == 2 && a.fac32 && app->weighted && app->app_id == FW_APP_NODE2VEC &&
            g->info.max_weight > 0.0f && iscan_ok) {
            // certified mode: quantized integer tile sums.  Scale 2^s so every
            // scaled app weight is < 2^29 (a lane's 4 fit a u32); the scaled
            // products stay exact in fp32 (power-of-two factors, no underflow)
            const double xm = std::max({1.0, app->inv_a, app->inv_b}) * (double)g->info.max_weight;
            int e2 = 0;
            std::frexp(xm, &e2);  // xm < 2^e2
            const int sh = 29 - e2;
            int ka = 0, kb = 0;
            std::frexp(app->inv_a, &ka);
            std::frexp(app->inv_b, &kb);
            const int kmin = std::min({0, ka - 1, kb - 1});
            if (sh >= -100 && sh <= 100 &&
                (long)g->info.min_weight_lowbit_exp + kmin + sh >= -149) {
                sc = std::ldexp(1.0, sh);
                xmax = xm;
                qscan = true;
            }
        }
        const double ws = (double)a.accept_wmax * sc;  // the kernel's prefilter has no disable
        const bool q64 = a.iscan == 1;  // set just above: fp64-factor quantized sums
        a.iscan = q64 || (((exact && G >= -126 && G <= 126) || qscan) && a.fac32 &&
                  4.0 * xmax * sc < 2147483648.0 &&
                  std::max({1.0, app->inv_a, app->inv_b}) * sc <= 1e37 && std::isfinite(ws) &&
                  ws <= 1e37 && iscan_ok) ? 1 : 0;
        a.iscale = a.iscan ? (float)sc : 1.0f;
        a.accept_wmax_s = a.iscan ? (float)ws : INFINITY;
        a.fa32 = a.inv_a32 * a.iscale;  // powers of two: exact
        a.f132 = a.iscale;
        a.fb32 = a.inv_b32 * a.iscale;
    }
    a.k_small = eng->k_small;
    a.k_big = eng->k_big;
    a.d_t = eng->d_t;
    a.h = mix64(seed + GOLDEN);
    a.cert_slack = 0x1p-50;
    if (const char *cs = getenv("FW_CERT_SLACK"))  // tests: widen the ambiguity band
        a.cert_slack = std::ldexp(1.0, -50 + atoi(cs));
    {
        const char *mr = getenv("FW_MERGE_RATIO");
        a.merge_ratio = mr ? (uint32_t)atoi(mr) : 4u;  // measured: 4 > 8 > 16 > 32 (s22 +7.8%, s27 +1.7%)
    }
    a.stats = (long long *)d_stats;
    a.done = d_done;
    a.piece_q = piece_q ? piece_q : 1;
    std::unique_lock<std::mutex> lk(g->mu);  // held until the slot's event is recorded
    const unsigned slot = g->call_counter++ % kQueueRing;
    if (g->schema_ring.empty()) g->schema_ring.resize(kQueueRing);
    if (!g->slot_ev[slot]) CU(cudaEventCreateWithFlags(&g->slot_ev[slot], cudaEventDisableTiming));
    // the slot's previous kernel (possibly on another stream) must be done
    // before its cursor is re-zeroed or its schema copy overwritten
    if (g->slot_used[slot]) CU(cudaStreamWaitEvent(stream, g->slot_ev[slot], 0));
    a.queue = g->queues + slot;
    CU(cudaMemsetAsync(a.queue, 0, sizeof(unsigned long long), stream));
    if (app->app_id == FW_APP_METAPATH) {
        a.schema_len = app->schema_len;
        if (app->schema_len <= kSchemaInline) {  // in the kernel arguments: no device copy
            for (uint32_t i = 0; i < app->schema_len; i++) a.schema_inline[i] = app->schema[i];
            a.schema = nullptr;
        } else {
            DevBuf &sb = g->schema_ring[slot];
            if (sb.cap < app->schema_len * sizeof(int64_t)) CU(cudaStreamSynchronize(stream));
            CU(sb.reserve(app->schema_len * sizeof(int64_t)));
            CU(cudaMemcpyAsync(sb.p, app->schema, app->schema_len * sizeof(int64_t),
                               cudaMemcpyHostToDevice, stream));
            a.schema = (const int64_t *)sb.p;
        }
    }
    const int occ = std::max(1, walk_occupancy(app->app_id, eng->sampler_id, mode));
    const uint64_t warps_needed = n;
    uint64_t grid = (uint64_t)g->sm_count * occ;
    const uint64_t max_useful = (warps_needed + (kWalkThreads / 32) - 1) / (kWalkThreads / 32);
    if (grid > max_useful) grid = max_useful;
    if (grid_out) *grid_out = (int)grid;
    CU(launch_walk(a, app->app_id, eng->sampler_id, mode, (int)grid, stream));
    CU(cudaEventRecord(g->slot_ev[slot], stream));
    g->slot_used[slot] = true;
    return FW_OK;
}

extern "C" int fw_walk_device(fw_graph *g, const int64_t *d_starts, uint64_t n,
                              uint64_t base_qid, const fw_app *app, const fw_engine *eng,
                              uint64_t seed, uint32_t *d_seq, uint32_t *d_len,
                              int64_t *d_stats, void *stream) {
    int rc = check_cfg(g, app, eng);
    if (rc) return rc;
    CU(cudaSetDevice(g->device));
    return launch(g, d_starts, n, base_qid, app, eng, seed, d_seq, d_len, d_stats,
                  (cudaStream_t)stream, nullptr, nullptr);
}

// cuStreamWaitValue32 through the runtime's driver entry point (no link-time
// dependency on libcuda); null when the driver does not provide it or
// FW_D2H_OVERLAP=0.
typedef CUresult (*WaitValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static WaitValue32Fn wait_value32() {
    static WaitValue32Fn fn = [] {
        const char *env = getenv("FW_D2H_OVERLAP");
        if (env && env[0] == '0') return (WaitValue32Fn) nullptr;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &p, 12000, cudaEnableDefault,
                                             &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (WaitValue32Fn) nullptr;
        return (WaitValue32Fn)p;
    }();
    return fn;
}

constexpr uint64_t kD2hPieces = 16;         // result pieces for the overlapped D2H
constexpr uint64_t kD2hMinQueries = 65536;  // below this, copy after the walk

extern "C" int fw_walk(fw_graph *g, const int64_t *starts, uint64_t n, uint64_t base_qid,
                       const fw_app *app, const fw_engine *eng, uint64_t seed,
                       uint32_t *out_seq, uint32_t *out_len, fw_stats *stats) {
    static const bool trace = [] {
        const char *e = getenv("FW_HOST_TRACE");
        return e && e[0] == '1';
    }();
    const auto t_in = std::chrono::steady_clock::now();
    auto us = [&]() {
        return (long)std::chrono::duration_cast<std::chrono::microseconds>(
                   std::chrono::steady_clock::now() - t_in).count();
    };
    int rc = check_cfg(g, app, eng);
    if (rc) return rc;
    CU(cudaSetDevice(g->device));
    std::lock_guard<std::mutex> lk(g->host_mu);
    const uint64_t L = app->length;
    // Device staging per query: the path row, its length and its start.
    // Above the scratch limit the walk runs in sub-launches over two
    // alternating buffers (Eq. 3's ping-pong, applied to
    // device memory); each buffer's D2H overlaps the next sub-launch.
    const uint64_t per_q = L * sizeof(uint32_t) + sizeof(uint32_t) + sizeof(int64_t);
    uint64_t limit = g->scratch_limit;
    uint64_t held = 0;
    for (int i = 0; i < 2; i++) held += g->starts[i].cap + g->seq[i].cap + g->len[i].cap;
    const bool fits0 = g->starts[0].cap >= n * sizeof(int64_t) &&
                       g->seq[0].cap >= n * L * sizeof(uint32_t) &&
                       g->len[0].cap >= n * sizeof(uint32_t);
    if (!limit && fits0) {
        limit = std::max(held, n * per_q);  // one launch in the staging already held
    } else if (!limit) {
        // cudaMemGetInfo costs ~0.5 ms: asked only when the staging must grow
        size_t fr = 0, tot = 0;
        CU(cudaMemGetInfo(&fr, &tot));
        limit = (uint64_t)((double)(fr + held) * 0.9);
    }
    const uint64_t rows_cap = std::max<uint64_t>(limit / per_q, 2);
    const bool single = n <= rows_cap;
    const uint64_t chunk = single ? std::max<uint64_t>(n, 1) : rows_cap / 2;
    const uint64_t nsub = single ? 1 : (n + chunk - 1) / chunk;
    for (int i = 0; i < (nsub > 1 ? 2 : 1); i++) {
        CU(g->starts[i].reserve(chunk * sizeof(int64_t)));
        CU(g->seq[i].reserve(chunk * L * sizeof(uint32_t)));
        CU(g->len[i].reserve(chunk * sizeof(uint32_t)));
    }
    CU(g->stats.reserve(ST_WORDS * sizeof(int64_t)));
    // Single launch: pieces of the result are copied back on a second stream
    // as soon as all of a piece's queries are done (the kernel counts them;
    // the copy stream waits on the count), so only the last piece's D2H
    // trails the walk.
    WaitValue32Fn wv = single && n >= kD2hMinQueries ? wait_value32() : nullptr;
    const uint64_t P = wv ? kD2hPieces : 0;
    const uint64_t piece_q = P ? (n + P - 1) / P : 0;
    if (P) CU(g->done.reserve(P * sizeof(unsigned)));
    if (!g->walk_st) {
        CU(cudaStreamCreateWithFlags(&g->walk_st, cudaStreamNonBlocking));
        CU(cudaStreamCreateWithFlags(&g->copy_st, cudaStreamNonBlocking));
        for (int i = 0; i < 4; i++) CU(cudaEventCreate(&g->ev[i]));
        CU(cudaEventCreateWithFlags(&g->ev[4], cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&g->ev[5], cudaEventDisableTiming));
        for (int i = 0; i < 2; i++) CU(cudaEventCreateWithFlags(&g->buf_free[i], cudaEventDisableTiming));
    }
    cudaStream_t st = g->walk_st, cs = g->copy_st;
    cudaEvent_t e0 = g->ev[0], e1 = g->ev[1], e2 = g->ev[2], e3 = g->ev[3], ez = g->ev[4];
    cudaEventRecord(e0, st);
    cudaMemsetAsync(g->stats.p, 0, ST_WORDS * sizeof(int64_t), st);
    int exact = 0;
    int grid = 0, pieces = 0, launches = 0;
    if (single) {
        if (P) cudaMemsetAsync(g->done.p, 0, P * sizeof(unsigned), st);
        if (n) cudaMemcpyAsync(g->starts[0].p, starts, n * sizeof(int64_t), cudaMemcpyHostToDevice, st);
        cudaEventRecord(e1, st);
        cudaEventRecord(ez, st);  // the counters are zero from here on
        rc = launch(g, (const int64_t *)g->starts[0].p, n, base_qid, app, eng, seed,
                    (uint32_t *)g->seq[0].p, (uint32_t *)g->len[0].p, (int64_t *)g->stats.p, st,
                    &exact, &grid, P ? (unsigned *)g->done.p : nullptr, piece_q);
        launches = n ? 1 : 0;
        cudaEventRecord(e2, st);
        if (!rc) {
            if (P) {
                cudaStreamWaitEvent(cs, ez, 0);
                for (uint64_t i = 0; i < P && i * piece_q < n; i++) {
                    const uint64_t q0 = i * piece_q, cnt = std::min(piece_q, n - q0);
                    const CUdeviceptr dc = (CUdeviceptr)((unsigned *)g->done.p + i);
                    if (wv(cs, dc, (cuuint32_t)cnt, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS) {
                        rc = set_err(FW_ECUDA, "cuStreamWaitValue32 failed");
                        break;
                    }
                    cudaMemcpyAsync(out_seq + q0 * L, (uint32_t *)g->seq[0].p + q0 * L,
                                    cnt * L * sizeof(uint32_t), cudaMemcpyDeviceToHost, cs);
                    cudaMemcpyAsync(out_len + q0, (uint32_t *)g->len[0].p + q0,
                                    cnt * sizeof(uint32_t), cudaMemcpyDeviceToHost, cs);
                    pieces++;
                }
                cudaStreamWaitEvent(st, e2, 0);
            } else if (n) {
                cudaMemcpyAsync(out_seq, g->seq[0].p, n * L * sizeof(uint32_t),
                                cudaMemcpyDeviceToHost, st);
                cudaMemcpyAsync(out_len, g->len[0].p, n * sizeof(uint32_t),
                                cudaMemcpyDeviceToHost, st);
            }
        }
    } else {
        cudaEventRecord(e1, st);
        for (uint64_t j = 0; j < nsub && !rc; j++) {
            const int b = (int)(j & 1);
            const uint64_t q0 = j * chunk, cnt = std::min(chunk, n - q0);
            if (j >= 2) cudaStreamWaitEvent(st, g->buf_free[b], 0);  // D2H of sub-launch j-2 done
            cudaMemcpyAsync(g->starts[b].p, starts + q0, cnt * sizeof(int64_t),
                            cudaMemcpyHostToDevice, st);
            rc = launch(g, (const int64_t *)g->starts[b].p, cnt, base_qid + q0, app, eng, seed,
                        (uint32_t *)g->seq[b].p, (uint32_t *)g->len[b].p,
                        (int64_t *)g->stats.p, st, &exact, &grid);
            if (rc) break;
            launches++;
            cudaEventRecord(ez, st);
            cudaStreamWaitEvent(cs, ez, 0);
            cudaMemcpyAsync(out_seq + q0 * L, g->seq[b].p, cnt * L * sizeof(uint32_t),
                            cudaMemcpyDeviceToHost, cs);
            cudaMemcpyAsync(out_len + q0, g->len[b].p, cnt * sizeof(uint32_t),
                            cudaMemcpyDeviceToHost, cs);
            cudaEventRecord(g->buf_free[b], cs);
        }
        cudaEventRecord(e2, st);
    }
    int64_t hst[ST_WORDS] = {0};
    if (!rc) {
        cudaMemcpyAsync(hst, g->stats.p, sizeof(hst), cudaMemcpyDeviceToHost, st);
        if (P || !single) {  // the end event covers both streams
            cudaEventRecord(g->ev[5], cs);
            cudaStreamWaitEvent(st, g->ev[5], 0);
        }
        cudaEventRecord(e3, st);
    }
    const long t_issued = us();
    // always drain both streams: no copy may still target the caller's buffers
    cudaError_t ce = cudaStreamSynchronize(st);
    const cudaError_t ce2 = cudaStreamSynchronize(cs);
    if (ce == cudaSuccess) ce = ce2;
    if (ce != cudaSuccess && !rc) rc = set_err(FW_ECUDA, "walk failed: %s", cudaGetErrorString(ce));
    if (!rc && stats) {
        float kms = 0.f, tms = 0.f;
        cudaEventElapsedTime(&kms, e1, e2);
        cudaEventElapsedTime(&tms, e0, e3);
        stats->steps = hst[ST_STEPS];
        stats->edges_scanned = hst[ST_EDGES];
        stats->collectives = hst[ST_COLLECTIVES];
        stats->draws = hst[ST_DRAWS];
        stats->small_tasks = hst[ST_SMALL];
        stats->large_tasks = hst[ST_LARGE];
        stats->sampled_steps = hst[ST_SAMPLED];
        stats->alg_bytes = hst[ST_BYTES];
        stats->kernel_ms = kms;
        stats->total_ms = tms;
        stats->exact_order = exact;
        stats->grid_ctas = grid;
        stats->kernel_launches = launches;
        stats->d2h_pieces = pieces;
        const uint64_t last = (uint64_t)hst[ST_T_LAST], first = ~(uint64_t)hst[ST_T_FIRST_NEG];
        stats->tail_ms = (n && last >= first) ? (double)(last - first) * 1e-6 : 0.0;
        stats->aux_bytes = g->aux_bytes();
        stats->aux_allocations = g->aux_allocations();
        int64_t sb = 0;
        for (int i = 0; i < 2; i++) sb += g->starts[i].cap + g->seq[i].cap + g->len[i].cap;
        stats->scratch_bytes = sb;
    }
    if (trace)
        fprintf(stderr, "fw_walk host: issued %ld us, returned %ld us (n=%llu)\n", t_issued, us(),
                (unsigned long long)n);
    return rc;
}

// ---------------------------------------------------------------------------
// validate_walks on device (_kernels.py:486-546): one thread per query.
// ---------------------------------------------------------------------------
__global__ void k_validate(const int64_t *__restrict__ off, const uint32_t *__restrict__ tgt,
                           const uint8_t *__restrict__ lab, const int64_t *__restrict__ starts,
                           uint64_t n, const uint32_t *__restrict__ seq,
                           const uint32_t *__restrict__ len, uint32_t L,
                           const int64_t *__restrict__ schema, uint32_t schema_len,
                           unsigned long long *bad) {
    unsigned long long nb = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        int64_t cur = starts[i];
        const int64_t ln = len[i];
        if (ln > (int64_t)L) { nb++; continue; }
        const uint32_t *row = seq + i * (uint64_t)L;
        for (int64_t j = 0; j < ln; j++) {
            const int64_t nxt = row[j];
            int64_t lo = off[cur], hi = off[cur + 1], found = -1;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                const int64_t tv = tgt[mid];
                if (tv < nxt) lo = mid + 1;
                else if (tv > nxt) hi = mid;
                else { found = mid; break; }
            }
            if (found < 0) { nb++; break; }
            if (schema_len > 0) {
                if (j >= (int64_t)schema_len) { nb++; break; }
                const int64_t want = schema[j];
                bool ok = false;
                for (int64_t e = found; e >= off[cur] && (int64_t)tgt[e] == nxt; e--)
                    if ((lab ? (int64_t)lab[e] : 0) == want) { ok = true; break; }
                for (int64_t e = found + 1; !ok && e < off[cur + 1] && (int64_t)tgt[e] == nxt; e++)
                    if ((lab ? (int64_t)lab[e] : 0) == want) { ok = true; break; }
                if (!ok) { nb++; break; }
            }
            cur = nxt;
        }
        for (int64_t j = ln; j < (int64_t)L; j++)
            if (row[j] != 0xFFFFFFFFu) { nb++; break; }
    }
    if (nb) atomicAdd(bad, nb);
}

extern "C" int fw_validate_device(fw_graph *g, const int64_t *d_starts, uint64_t n,
                                  const uint32_t *d_seq, const uint32_t *d_len, uint32_t L,
                                  const int64_t *schema, uint32_t schema_len, int64_t *d_bad,
                                  void *stream) {
    if (!g) return set_err(FW_EVALIDATION, "null handle");
    CU(cudaSetDevice(g->device));
    cudaStream_t st = (cudaStream_t)stream;
    int64_t *d_schema = nullptr;
    if (schema_len) {
        CU(cudaMallocAsync(&d_schema, schema_len * sizeof(int64_t), st));
        CU(cudaMemcpyAsync(d_schema, schema, schema_len * sizeof(int64_t),
                           cudaMemcpyHostToDevice, st));
    }
    if (n)
        k_validate<<<g->sm_count * 8, 128, 0, st>>>(g->off, g->tgt, g->lab, d_starts, n, d_seq,
                                                   d_len, L, d_schema, schema_len,
                                                   (unsigned long long *)d_bad);
    CU(cudaGetLastError());
    if (d_schema) CU(cudaFreeAsync(d_schema, st));
    return FW_OK;
}

// ---------------------------------------------------------------------------
// Sampler trials (csrc/fw_trials.cu).
// ---------------------------------------------------------------------------
namespace fw {
cudaError_t launch_trials(int method, const double *w, uint32_t n, uint32_t k, uint64_t key,
                          uint64_t trials, const double *prob, const int64_t *alias,
                          double w_max, uint32_t max_rounds, uint32_t *picks, int64_t *aux,
                          cudaStream_t stream);
}

extern "C" int fw_sampler_trials_device(int32_t method, const double *d_w, uint32_t n,
                                        uint32_t k, uint64_t key, uint64_t trials,
                                        const double *d_prob, const int64_t *d_alias,
                                        double w_max, uint32_t max_rounds, uint32_t *d_picks,
                                        int64_t *d_aux, void *stream) {
    if (method < 0 || method > 6) return set_err(FW_EVALIDATION, "unknown sampler method");
    if ((method == 1 || method == 2) && (k < 1 || k > 1000))
        return set_err(FW_ECONFIG, "lane width k must be in [1, 1000]");
    if (method == 4 && n && (!d_prob || !d_alias))
        return set_err(FW_EVALIDATION, "alias sampling needs a table");
    if (trials && !d_picks) return set_err(FW_EVALIDATION, "null picks buffer");
    CU(launch_trials(method, d_w, n, k, key, trials, d_prob, d_alias, w_max, max_rounds,
                     d_picks, d_aux, (cudaStream_t)stream));
    return FW_OK;
}

// ---------------------------------------------------------------------------
// Synthetic inputs (counter-hash; paper_2404_08364_b200/rmat.py is the
// bit-identical numpy twin).
// ---------------------------------------------------------------------------
__host__ __device__ static inline uint64_t perm_bits(uint64_t x, int s, uint64_t key) {
    if (s == 0) return 0;
    const uint64_t mask = s >= 64 ? ~0ull : ((1ull << s) - 1);
    const int sh = (s + 1) / 2;
    x = (x ^ key) & mask;
    x = (x * GOLDEN) & mask;
    x ^= x >> sh;
    x = (x * MIX1) & mask;
    x ^= x >> sh;
    x = (x * MIX2) & mask;
    x ^= x >> sh;
    return x;
}

__global__ void k_rmat(uint64_t h, int s, uint32_t ta, uint32_t tab, uint32_t tabc,
                       uint64_t pkey, uint64_t e0, uint64_t m, uint32_t *src, uint32_t *dst) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t base = mix64(h ^ ((e0 + i) * MIX1));
        uint64_t u = 0, v = 0;
        for (int l = 0; l < s; l++) {
            const uint32_t r = (uint32_t)(mix64(base + (uint64_t)l * GOLDEN) >> 32);
            const uint64_t sb = r >= tab;
            const uint64_t db = (r >= ta && r < tab) || r >= tabc;
            u = (u << 1) | sb;
            v = (v << 1) | db;
        }
        src[i] = (uint32_t)perm_bits(u, s, pkey);
        dst[i] = (uint32_t)perm_bits(v, s, pkey);
    }
}

static uint32_t thresh(double p) {
    if (p <= 0) return 0;
    const double t = std::floor(p * 4294967296.0);
    return t >= 4294967295.0 ? 0xFFFFFFFFu : (uint32_t)t;
}

extern "C" int fw_rmat_edges_device(uint64_t seed, int32_t scale, double a, double b, double c,
                                    uint64_t e0, uint64_t m, uint32_t *d_src, uint32_t *d_dst,
                                    void *stream) {
    if (scale < 0 || scale > 32) return set_err(FW_ECONFIG, "scale must be in [0, 32]");
    if (a < 0 || b < 0 || c < 0 || a + b + c > 1.0)
        return set_err(FW_ECONFIG, "R-MAT probabilities must be >= 0 and sum <= 1");
    const uint64_t h = mix64(seed + GOLDEN);
    const uint64_t pkey = mix64(seed ^ 0x5555555555555555ull);
    if (m) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        k_rmat<<<sms * 8, 256, 0, (cudaStream_t)stream>>>(h, scale, thresh(a), thresh(a + b),
                                                         thresh(a + b + c), pkey, e0, m,
                                                         d_src, d_dst);
        CU(cudaGetLastError());
    }
    return FW_OK;
}

__global__ void k_synth_w(uint64_t h, uint64_t e0, uint64_t m, float *w) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t z = mix64(h + (e0 + i) * GOLDEN);
        const double u = __dmul_rn(__ull2double_rn(z >> 11), 0x1.0p-53);
        float x = __double2float_rn(__dadd_rn(1.0, __dmul_rn(4.0, u)));
        if (x >= 5.0f) x = 4.99999952316284180f;  // nextafter(5, 1), graph.py:181-182
        w[i] = x;
    }
}

__global__ void k_synth_l(uint64_t h, uint32_t nl, uint64_t e0, uint64_t m, uint8_t *l) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t z = mix64(h + (e0 + i) * GOLDEN);
        l[i] = (uint8_t)((z >> 32) % nl);
    }
}

extern "C" int fw_synth_weights_device(uint64_t seed, uint64_t e0, uint64_t m, float *d_w,
                                       void *stream) {
    if (m) {
        k_synth_w<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(mix64(seed + GOLDEN), e0, m, d_w);
        CU(cudaGetLastError());
    }
    return FW_OK;
}

extern "C" int fw_synth_labels_device(uint64_t seed, uint32_t label_count, uint64_t e0,
                                      uint64_t m, uint8_t *d_l, void *stream) {
    if (label_count < 1 || label_count > 256)
        return set_err(FW_EVALIDATION, "label_count must be in [1, 256]");
    if (m) {
        k_synth_l<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(mix64(seed + GOLDEN), label_count,
                                                             e0, m, d_l);
        CU(cudaGetLastError());
    }
    return FW_OK;
}
