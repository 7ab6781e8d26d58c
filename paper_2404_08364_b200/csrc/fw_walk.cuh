#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace fw {

#ifndef FW_WALK_THREADS
#define FW_WALK_THREADS 128
#endif
constexpr int kWalkThreads = FW_WALK_THREADS;  // 4 warp walkers per CTA
// Resident CTAs per SM the register budget is sized for.  Node2Vec's tile
// loop runs at 72 registers / 28 warps per SM (measured faster than 64 / 32
// and 80 / 24); the first-order apps at 64 / 32.
#ifndef FW_MIN_BLOCKS
#define FW_MIN_BLOCKS 8
#endif
#ifndef FW_MIN_BLOCKS_N2V
#define FW_MIN_BLOCKS_N2V 7
#endif
#ifndef FW_MIN_BLOCKS_MP
#define FW_MIN_BLOCKS_MP FW_MIN_BLOCKS
#endif
constexpr int walk_min_blocks(int app) {
    return app == 2 ? FW_MIN_BLOCKS_N2V : app == 3 ? FW_MIN_BLOCKS_MP : FW_MIN_BLOCKS;
}
// Per-warp shared memory (32-bit words):
//   [0, slots)            first-order apps: ZPRS weight staging (kHashSlots);
//                         node2vec: the N(prev) window table (kTabSlots)
//   [slots, +512)         256 x u64: ZPRS lane prefixes / node2vec draw words
//   [stats, +16)          8 x u64 RunStats counters
//   [ctl, +8)             node2vec window control words; [4],[5]: N(prev) start
// node2vec's larger table keeps 28 warps (7 CTAs x 4) resident per SM.
constexpr uint32_t kHashSlots = 1024;
constexpr uint32_t kTabSlots = 1472;
constexpr uint32_t kChunk = 256;  // N(prev) entries per table window
#ifndef FW_MP_SLOTS
#define FW_MP_SLOTS 1024
#endif
constexpr uint32_t kMpSlots = FW_MP_SLOTS;  // MetaPath staging (occupancy trade)
static_assert(kMpSlots <= kHashSlots, "MetaPath staging is at most the first-order size");
__host__ __device__ constexpr uint32_t warp_slots(int app) {
    return app == 2 ? kTabSlots : app == 3 ? kMpSlots : kHashSlots;
}
__host__ __device__ constexpr uint32_t stats_word(int app) { return warp_slots(app) + 2 * 256; }
__host__ __device__ constexpr uint32_t ctl_word(int app) { return stats_word(app) + 2 * 8; }
__host__ __device__ constexpr uint32_t warp_words(int app) { return ctl_word(app) + 8; }
__host__ __device__ constexpr int walk_smem_bytes(int app) { return (kWalkThreads / 32) * warp_words(app) * 4; }
constexpr uint32_t kCtlWord = ctl_word(2);  // node2vec control words

// Kernel arguments (passed by value through the constant bank).
struct WalkArgs {
    const int64_t *off;   // offsets int64[V+1]      (graph.py:44)
    const uint32_t *tgt;  // targets uint32[E]       (graph.py:45)
    const float *w;       // weights float32[E]      (graph.py:46)
    const uint8_t *lab;   // labels uint8[E] or null (graph.py:47, 68-76)
    const int64_t *starts;
    uint64_t n;
    uint64_t base_qid;
    uint32_t *out_seq;    // n * L, sentinel padded
    uint32_t *out_len;    // n
    uint32_t L;
    uint32_t schema_len;
    const int64_t *schema;  // device copy, or null: schema_inline holds it
    int64_t schema_inline[16];
    int32_t weighted;
    double stop_prob, inv_a, inv_b;
    double fac[4];  // node2vec factor by 2*is_prev + is_member: {1/b, 1, 1/a, 1/a}
    int64_t k_small, k_big, d_t;
    uint64_t h;  // mix64(seed + GOLDEN), hoisted stream-key hash
    uint32_t merge_ratio;  // node2vec: N(prev) windows when d_prev <= ratio*d_cur + 2*kChunk, else bsearch
    float accept_wmax;     // upper bound on any app weight (exact node2vec accept prefilter)
    // node2vec: 1/a and 1/b are powers of two and w * {1/a, 1/b} is exact in
    // fp32 for every weight, so factor * weight is formed in fp32 and widened
    int32_t fac32;
    float inv_a32, inv_b32;
    // node2vec fp32 factor path in exact order: tile sums as integers in
    // units of 2^G (iscale = 2^-G); accept_wmax_s = accept_wmax * 2^-G
    // fa32/f132/fb32 = {1/a, 1, 1/b} (* 2^-G when iscan): the fp32 factors
    int32_t iscan;
    float iscale, accept_wmax_s;
    float fa32, f132, fb32;
    // per-piece completion counters (null: off).  A warp that finishes
    // query qi bumps done[qi / piece_q] after a device-scope fence, so the
    // host's copy stream can wait on a piece (cuStreamWaitValue32) and copy
    // its paths back while the walk continues.
    unsigned *done;
    uint64_t piece_q;
    // mode 2: certified accept tests; slack = 2^-50 (FW_CERT_SLACK scales it
    // up in tests to force the ordered re-run)
    double cert_slack;
    // mode 2, fp64 factors: the power-of-two scale of the quantized integer
    // tile sums (the fp32-factor path folds it into fa32/f132/fb32)
    double qscale;
    unsigned long long *queue;
    long long *stats;  // ST_COUNT counters (accumulated)
};

constexpr uint32_t kSchemaInline = 16;  // metapath schemas up to this length ride in the args

// mode: 0 ordered (the reference's summation order), 1 exact (tree scans,
// every partial sum exact), 2 certified (tree scans + certified accept
// tests, ambiguous steps re-run in order)
cudaError_t launch_walk(const WalkArgs &a, int app, int sampler, int mode, int grid,
                        cudaStream_t stream);
int walk_occupancy(int app, int sampler, int mode);

}  // namespace fw
