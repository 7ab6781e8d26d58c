/*
 * flowwalk.h -- C ABI of the B200-native walk engine (libflowwalk.so).
 *
 * Plain pointers and sizes only; no torch types.  Every entry point returns
 * an int status (FW_OK or one of the FW_E* codes) and records a message
 * readable through fw_last_error().  The Python host layer
 * (paper_2404_08364_b200/engine.py) maps the codes onto the reference's
 * exception classes (reswalk errors.py:4-45).
 *
 * Reference interfaces replaced (paths relative to /root/reference):
 *   fw_graph_create / fw_graph_create_device / fw_graph_destroy
 *       -- the read-only CSR arrays of reswalk.graph.Graph (pkg/src/reswalk/graph.py:40-87)
 *          that the reference passes by reference into every step_pass call
 *          (engine.py:209-221); here they are uploaded once and stay resident in HBM.
 *   fw_walk / fw_walk_device
 *       -- the worker loop Worker.run_batch / pass_once (engine.py:199-230) driving
 *          the numba operator _kernels.step_pass (_kernels.py:320-483, 33 positional
 *          args), for one batch of queries with global ids base_qid + i, plus the
 *          sentinel pre-fill of the batch buffers (engine.py:299-300) and the
 *          per-worker stats accumulation (engine.py:342-353).
 *   fw_validate_device
 *       -- _kernels.validate_walks (_kernels.py:486-546).
 *   fw_sampler_trials_device
 *       -- the sampler trial kernels seq_rs/dprs/zprs/its/alias/rjs/uniform_control_trials
 *          (_kernels.py:84-277) behind trials.run_trials (trials.py:46-90).
 *   fw_build_csr_device / fw_edges_max_id
 *       -- reswalk build_csr (graph.py:138-169): CSR from an edge list, lists sorted by
 *          target with duplicates in input order (np.lexsort semantics), on the device.
 *   fw_fwg1_info / fw_fwg1_read / fw_crc32_device
 *       -- reswalk load_binary (graph.py:225-254): the FWG1 file streamed into device
 *          arrays, its zlib CRC-32 checked on the device.
 *   fw_rmat_edges_device / fw_synth_weights_device / fw_synth_labels_device
 *       -- synthetic inputs; the reference only ships random/star edge lists and
 *          numpy-seeded synthesis (graph.py:172-201, 257-277), see DESIGN.md.
 */
#ifndef FLOWWALK_H
#define FLOWWALK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    FW_OK = 0,
    FW_EVALIDATION = 1, /* reswalk ValidationError (engine.py:274-275, apps.py:48-59) */
    FW_ECONFIG = 2,     /* reswalk ConfigError (engine.py:64-77, 276-277) */
    FW_ECUDA = 3,       /* CUDA runtime failure */
    FW_ENOMEM = 4,      /* device allocation failure */
    FW_EFORMAT = 5,     /* reswalk FormatError (graph.py:232-244): bad magic, size or CRC */
};

/* app ids: reswalk apps.py:21-24 (APP_IDS) / _kernels.py:41-44 */
enum { FW_APP_DEEPWALK = 0, FW_APP_PPR = 1, FW_APP_NODE2VEC = 2, FW_APP_METAPATH = 3 };
/* sampler ids: _kernels.py:46-47 (resolved by EngineConfig.resolve_sampler, engine.py:79-87) */
enum { FW_SAMPLER_ZPRS = 0, FW_SAMPLER_DPRS = 1 };
/* fp64 summation order: auto picks tree-order scans when every partial sum
 * is provably exact (so any order is bit-identical to the reference's
 * sequential order); otherwise, for nonnegative finite weights, tree-order
 * scans with certified accept tests (a step whose test cannot be decided from
 * the error bound is re-run in the reference's order), else the
 * reference's sequential order.  SEQUENTIAL always replays the reference's
 * order.  fw_stats.exact_order reports 1 (exact), 2 (certified) or 0. */
enum { FW_ORDER_AUTO = 0, FW_ORDER_SEQUENTIAL = 1 };

typedef struct fw_graph fw_graph;

/* AppConfig (apps.py:38-59) as the step kernel consumes it (engine.py:213-215). */
typedef struct {
    int32_t app_id;
    int32_t weighted;
    uint32_t length;       /* l_max, < 2^20 */
    uint32_t schema_len;   /* metapath only, else 0 */
    const int64_t *schema; /* host pointer, schema_len entries */
    double stop_prob;      /* ppr */
    double inv_a;          /* 1.0 / a, computed by the caller in fp64 */
    double inv_b;          /* 1.0 / b */
} fw_app;

/* EngineConfig (engine.py:51-87): only the bit-relevant fields. */
typedef struct {
    int32_t k_small;     /* 1 <= k_small <= k_big <= 1000 */
    int32_t k_big;
    int64_t d_t;         /* degree_threshold */
    int32_t sampler_id;  /* FW_SAMPLER_* (already resolved) */
    int32_t order_mode;  /* FW_ORDER_* */
} fw_engine;

/* RunStats counters (engine.py:245-260; _kernels.py:32-39) plus device metrics. */
typedef struct {
    int64_t steps;          /* ST_STEPS: attempts incl. terminal ones */
    int64_t edges_scanned;  /* ST_EDGES */
    int64_t collectives;    /* ST_COLLECTIVES */
    int64_t draws;          /* ST_DRAWS */
    int64_t small_tasks;    /* ST_SMALL */
    int64_t large_tasks;    /* ST_LARGE */
    int64_t sampled_steps;  /* sum of lengths */
    int64_t alg_bytes;      /* algorithmic HBM bytes */
    double kernel_ms;       /* walk kernel time (CUDA events) */
    double total_ms;        /* incl. H2D/D2H for fw_walk */
    int32_t exact_order;    /* summation order: 0 the reference's sequential order replayed,
                               1 tree-order scans (every partial sum exact), 2 tree-order
                               scans with certified accept tests */
    int32_t grid_ctas;
    int32_t kernel_launches;
    int32_t d2h_pieces;     /* fw_walk: result pieces copied back while the walk ran
                               (0: copied after the kernel) */
    double tail_ms;         /* first to last warp exit: the load-imbalance tail */
    int64_t aux_bytes;      /* device scratch the engine holds besides the graph and the
                               result buffers (cursor slots, counters, piece counters,
                               schema copies): the reference's AllocationMeter total
                               (engine.py:35-48), independent of d_max and |Q| */
    int64_t aux_allocations;
    int64_t scratch_bytes;  /* fw_walk: device result/start staging in use */
} fw_stats;

typedef struct {
    int64_t max_degree;
    int64_t max_degree_vertex;
    float max_weight;
    int32_t min_weight_lowbit_exp; /* min over w>0 of exponent of w's lowest set bit */
    int32_t has_labels;
    int32_t bad_weights;   /* some weight is negative or non-finite */
    int32_t sorted_lists;  /* every neighbour list is non-decreasing (Node2Vec needs it) */
    int32_t pad_;
} fw_graph_info;

const char *fw_last_error(void);
int fw_device_count(int *out);

/* Upload host CSR arrays once (pinned staging); labels may be NULL.
 * Both constructors check the CSR on the device before returning a handle:
 * offsets[0] == 0, offsets[V] == E, offsets non-decreasing and every target
 * < V (FW_EVALIDATION otherwise, the reference's Graph.validate,
 * graph.py:70-81); per-vertex sortedness is recorded in fw_graph_info and
 * required by Node2Vec walks (its membership test binary-searches N(prev),
 * _kernels.py:293-306). */
int fw_graph_create(const int64_t *offsets, const uint32_t *targets, const float *weights,
                    const uint8_t *labels_or_null, uint64_t vertex_count, uint64_t edge_count,
                    int device, fw_graph **out);
/* Wrap device-resident CSR arrays already on `device` (borrowed, not freed).
 * Contract: d_targets and d_weights stay readable 16 bytes past element E-1
 * (the walk kernel loads 16-byte tiles). */
int fw_graph_create_device(const int64_t *d_offsets, const uint32_t *d_targets,
                           const float *d_weights, const uint8_t *d_labels_or_null,
                           uint64_t vertex_count, uint64_t edge_count, int device,
                           fw_graph **out);
/* Replica of a resident graph on another device by device-to-device peer
 * copies (the multi-GPU fan-out of SURVEY §8(e)); the new handle owns its
 * arrays.  Works for device == src's device too (a second private copy). */
int fw_graph_replicate(fw_graph *src, int device, fw_graph **out);
int fw_graph_destroy(fw_graph *g);
/* Device scratch cap for fw_walk's result/start staging (bytes; 0 = auto:
 * 90% of the device's free memory at call time).  Reference analogue: the
 * Eq. 3 memory budget (engine.py:90-105) applied to device memory. */
int fw_graph_set_scratch_limit(fw_graph *g, uint64_t bytes);
int fw_graph_info_get(fw_graph *g, fw_graph_info *out);

/* Host-buffer walk: H2D starts, walk, D2H sequences (n*length u32, sentinel
 * padded) and lengths (n u32).  Stats are written (not accumulated).  When
 * n * (length + 3) * 4 bytes exceed the handle's scratch limit the queries are
 * walked in sub-launches over two alternating device buffers, each one's D2H
 * overlapping the next launch (PAPER.md:394-400 ping-pong). */
int fw_walk(fw_graph *g, const int64_t *starts, uint64_t n, uint64_t base_qid,
            const fw_app *app, const fw_engine *eng, uint64_t seed,
            uint32_t *out_seq, uint32_t *out_len, fw_stats *stats);

/* Device-buffer walk, asynchronous on `stream` (a cudaStream_t, may be NULL).
 * Launches on different streams may overlap: each takes its own work-queue
 * cursor slot, and a slot is reused only after its previous kernel finished.
 * d_stats (int64[10], device) is ACCUMULATED: steps, edges, collectives, draws,
 * small, large, sampled_steps, alg_bytes; words 8/9 take the max of the warps'
 * exit time and of its complement (%globaltimer ns, zero them per launch). */
int fw_walk_device(fw_graph *g, const int64_t *d_starts, uint64_t n, uint64_t base_qid,
                   const fw_app *app, const fw_engine *eng, uint64_t seed,
                   uint32_t *d_out_seq, uint32_t *d_out_len, int64_t *d_stats,
                   void *stream);

/* validate_walks on device; *d_bad (int64, device) accumulates violations. */
int fw_validate_device(fw_graph *g, const int64_t *d_starts, uint64_t n,
                       const uint32_t *d_seq, const uint32_t *d_len, uint32_t l_max,
                       const int64_t *schema_host, uint32_t schema_len,
                       int64_t *d_bad, void *stream);

/* Sampler trials (one pick per trial; trial t draws from streams (t<<10)|lane).
 * method: 0 seq, 1 dprs, 2 zprs, 3 its, 4 alias (d_prob/d_alias = alias table),
 * 5 rjs (w_max, max_rounds), 6 uniform-control.  d_aux (nullable) receives the
 * per-trial collectives (dprs/zprs) or rejection rounds (rjs).  All device pointers. */
int fw_sampler_trials_device(int32_t method, const double *d_w, uint32_t n, uint32_t k,
                             uint64_t key, uint64_t trials, const double *d_prob,
                             const int64_t *d_alias, double w_max, uint32_t max_rounds,
                             uint32_t *d_picks, int64_t *d_aux, void *stream);

/* ---- graph ingest (csrc/fw_ingest.cu); all arrays are device pointers ---- */
/* Largest vertex id over src and dst (m edges). */
int fw_edges_max_id(const uint32_t *d_src, const uint32_t *d_dst, uint64_t m,
                    uint64_t *out_max, void *stream);
/* build_csr: out offsets int64[V+1], targets u32[m], weights f32[m] (w_in NULL:
 * all 1), labels u8[m] (lab_in NULL: all 0; lab_out NULL: not written).  m < 2^32.
 * FW_EVALIDATION if some id >= V. */
int fw_build_csr_device(const uint32_t *d_src, const uint32_t *d_dst, const float *d_w_in,
                        const uint8_t *d_lab_in, uint64_t m, uint64_t vertex_count,
                        int64_t *d_offsets, uint32_t *d_targets, float *d_w_out,
                        uint8_t *d_lab_out, void *stream);
/* FWG1 header: V, E, flags (bit 1: labels present); FW_EFORMAT on bad magic/size. */
int fw_fwg1_info(const char *path, uint64_t *vertex_count, uint64_t *edge_count,
                 int32_t *flags);
/* Stream the FWG1 payload into device arrays (pinned double buffers, reader
 * threads), then check its CRC-32 on the device (FW_EFORMAT on mismatch). */
int fw_fwg1_read(const char *path, uint64_t vertex_count, uint64_t edge_count, int32_t flags,
                 int64_t *d_offsets, uint32_t *d_targets, float *d_weights,
                 uint8_t *d_labels_or_null, uint32_t *crc_out, void *stream);
/* zlib CRC-32 of n device bytes. */
int fw_crc32_device(const uint8_t *d_bytes, uint64_t n, uint32_t *out, void *stream);

/* Synthetic R-MAT (Graph500 a,b,c; d = 1-a-b-c) edges, counter-hash driven so
 * host (numpy) and device generate identical lists.  Writes m (src, dst)
 * pairs for edge ids [e0, e0 + m). */
int fw_rmat_edges_device(uint64_t seed, int32_t scale, double a, double b, double c,
                         uint64_t e0, uint64_t m, uint32_t *d_src, uint32_t *d_dst,
                         void *stream);
/* w[e] = U[1,5) float32 from (seed, e); labels[e] = hash(seed, e) % label_count. */
int fw_synth_weights_device(uint64_t seed, uint64_t e0, uint64_t m, float *d_w, void *stream);
int fw_synth_labels_device(uint64_t seed, uint32_t label_count, uint64_t e0, uint64_t m,
                           uint8_t *d_l, void *stream);

#ifdef __cplusplus
}
#endif
#endif
