/*
 * TEST INFRASTRUCTURE ONLY -- not part of the product path.
 *
 * CPU restatement of the reference's replay-mode walk step
 * (reswalk `_kernels.step_pass`, /root/reference/pkg/src/reswalk/_kernels.py:320-483)
 * used as the parity checker for the sm_100a walk kernel.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 *
 * Pinning: tests/test_oracle.py checks this file bit-for-bit against golden
 * vectors produced by running the reference itself (tests/golden/gen_golden.py).
 *
 * Semantics followed (file:line in the reference):
 *   mix64 / stream_base / u01 ........ _kernels.py:50-66   (spec rng.py:24-41)
 *   _edge_weight ..................... _kernels.py:280-308 (spec apps.py:62-124)
 *   routing, PPR stop draw, checks ... _kernels.py:340-388
 *   DPRS block ....................... _kernels.py:399-430 (spec samplers.py:156-185)
 *   ZPRS block ....................... _kernels.py:431-464 (spec samplers.py:188-220)
 *   commit / stop conditions ......... _kernels.py:466-482
 *   query init (prev=-1, emitted=0) .. engine.py:171-188
 *   validate_walks ................... _kernels.py:486-546
 *
 * Replay mode makes every query a pure function of (graph, seed, global qid,
 * app, k_small, k_big, d_t, sampler), so the oracle walks one query at a time
 * (the reference's worker/pool schedule cannot change the result).  Sums are
 * accumulated in exactly the reference's order (sequential per chunk for DPRS,
 * per lane in chunk order + a sequential lane scan for ZPRS) so that the
 * oracle is bit-exact for arbitrary (non-dyadic) weights too.  Compile with
 * -ffp-contract=off: numba emits no FMAs in step_pass.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define GOLDEN 0x9E3779B97F4A7C15ULL
#define MIX1 0xBF58476D1CE4E5B9ULL
#define MIX2 0x94D049BB133111EBULL
#define TAG_REPLAY (1ULL << 63)
#define STOP_LANE 1023ULL

enum { ST_STEPS = 0, ST_EDGES, ST_COLLECTIVES, ST_DRAWS, ST_SMALL, ST_LARGE, ST_COUNT };
enum { APP_DEEPWALK = 0, APP_PPR = 1, APP_NODE2VEC = 2, APP_METAPATH = 3 };
enum { SAMPLER_ZPRS = 0, SAMPLER_DPRS = 1 };

uint64_t fwo_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * MIX1;
    z = (z ^ (z >> 27)) * MIX2;
    return z ^ (z >> 31);
}

uint64_t fwo_stream_base(uint64_t key, uint64_t sid) {
    uint64_t h = fwo_mix64(key + GOLDEN);
    return fwo_mix64(h ^ (sid * MIX1));
}

double fwo_u01(uint64_t base, uint64_t ctr) {
    uint64_t z = fwo_mix64(base + ctr * GOLDEN);
    return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

typedef struct {
    const int64_t *offsets;
    const uint32_t *targets;
    const float *weights;
    const uint8_t *labels; /* NULL -> zero labels (graph.py:68-76) */
    int app_id, weighted, sampler_id;
    uint32_t length;
    double stop_prob, inv_a, inv_b;
    const int64_t *schema;
    uint32_t schema_len;
    int64_t k_small, k_big, d_t;
    uint64_t key;
} walk_cfg;

static inline double edge_weight(const walk_cfg *c, int64_t e, int64_t prev_v,
                                 int64_t plo, int64_t phi, int64_t want_label) {
    if (c->app_id == APP_METAPATH) {
        int64_t lab = c->labels ? (int64_t)c->labels[e] : 0;
        if (lab != want_label) return 0.0;
        return c->weighted ? (double)c->weights[e] : 1.0;
    }
    if (c->app_id == APP_NODE2VEC && prev_v >= 0) {
        int64_t u = (int64_t)c->targets[e];
        double base;
        if (u == prev_v) {
            base = c->inv_a;
        } else {
            int64_t lo = plo, hi = phi;
            int found = 0;
            while (lo < hi) {
                int64_t mid = (lo + hi) >> 1;
                int64_t tv = (int64_t)c->targets[mid];
                if (tv < u) lo = mid + 1;
                else if (tv > u) hi = mid;
                else { found = 1; break; }
            }
            base = found ? 1.0 : c->inv_b;
        }
        return c->weighted ? base * (double)c->weights[e] : base;
    }
    return c->weighted ? (double)c->weights[e] : 1.0;
}

typedef struct {
    double *lane_w, *lane_prefix;
    int64_t *lane_cand;
    uint64_t *lane_base;
} scratch_t;

/* One query, replay mode.  Returns emitted; writes out[0..emitted). */
static uint32_t walk_one(const walk_cfg *c, scratch_t *s, uint64_t q, int64_t start,
                         uint32_t *out, int64_t *stats) {
    int64_t cur = start, prev = -1;
    uint32_t emitted = 0;
    for (;;) {
        int64_t v = cur;
        int64_t elo = c->offsets[v];
        int64_t deg = c->offsets[v + 1] - elo;
        int small = deg <= c->d_t;
        int64_t k = small ? c->k_small : c->k_big;
        stats[small ? ST_SMALL : ST_LARGE] += 1;
        stats[ST_STEPS] += 1;
        uint64_t step = emitted;
        uint64_t sid_hi = TAG_REPLAY | (q << 30) | (step << 10);
        if (c->app_id == APP_PPR) {
            double r = fwo_u01(fwo_stream_base(c->key, sid_hi | STOP_LANE), 0);
            stats[ST_DRAWS] += 1;
            if (r < c->stop_prob) break;
        }
        if (deg == 0) break;
        if (c->app_id == APP_METAPATH && step >= c->schema_len) break;
        int64_t plo = 0, phi = 0;
        if (c->app_id == APP_NODE2VEC && prev >= 0) {
            plo = c->offsets[prev];
            phi = c->offsets[prev + 1];
        }
        int64_t want_label = c->app_id == APP_METAPATH ? c->schema[step] : 0;
        int64_t chunks = (deg + k - 1) / k;
        int64_t nlanes = k < deg ? k : deg;
        for (int64_t j = 0; j < nlanes; j++)
            s->lane_base[j] = fwo_stream_base(c->key, sid_hi | (uint64_t)j);
        int64_t sel = 0;
        if (c->sampler_id == SAMPLER_DPRS) {
            for (int64_t j = 0; j < k; j++) s->lane_cand[j] = 0;
            double carry = 0.0;
            for (int64_t ch = 0; ch < chunks; ch++) {
                int64_t b0 = ch * k;
                int64_t m = k < deg - b0 ? k : deg - b0;
                double run = 0.0;
                for (int64_t j = 0; j < m; j++) {
                    double wv = edge_weight(c, elo + b0 + j, prev, plo, phi, want_label);
                    run += wv;
                    s->lane_w[j] = wv;
                    s->lane_prefix[j] = run;
                }
                stats[ST_COLLECTIVES] += 1;
                for (int64_t j = 0; j < m; j++) {
                    double r = fwo_u01(s->lane_base[j], (uint64_t)ch);
                    double wv = s->lane_w[j];
                    if (wv > 0.0 && r * (s->lane_prefix[j] + carry) < wv)
                        s->lane_cand[j] = b0 + j + 1;
                }
                int64_t best = 0;
                for (int64_t j = 0; j < k; j++)
                    if (s->lane_cand[j] > best) best = s->lane_cand[j];
                stats[ST_COLLECTIVES] += 1;
                sel = best;
                carry += run;
            }
            stats[ST_EDGES] += deg;
        } else {
            for (int64_t j = 0; j < k; j++) { s->lane_w[j] = 0.0; s->lane_cand[j] = 0; }
            for (int64_t ch = 0; ch < chunks; ch++) {
                int64_t b0 = ch * k;
                int64_t m = k < deg - b0 ? k : deg - b0;
                for (int64_t j = 0; j < m; j++)
                    s->lane_w[j] += edge_weight(c, elo + b0 + j, prev, plo, phi, want_label);
            }
            double run = 0.0;
            for (int64_t j = 0; j < k; j++) {
                s->lane_prefix[j] = run;
                run += s->lane_w[j];
            }
            stats[ST_COLLECTIVES] += 1;
            for (int64_t ch = 0; ch < chunks; ch++) {
                int64_t b0 = ch * k;
                int64_t m = k < deg - b0 ? k : deg - b0;
                for (int64_t j = 0; j < m; j++) {
                    double wv = edge_weight(c, elo + b0 + j, prev, plo, phi, want_label);
                    s->lane_prefix[j] += wv;
                    double r = fwo_u01(s->lane_base[j], (uint64_t)ch);
                    if (wv > 0.0 && r * s->lane_prefix[j] < wv) s->lane_cand[j] = b0 + j + 1;
                }
            }
            for (int64_t j = k - 1; j >= 0; j--)
                if (s->lane_cand[j] > 0) { sel = s->lane_cand[j]; break; }
            stats[ST_COLLECTIVES] += 1;
            stats[ST_EDGES] += 2 * deg;
        }
        stats[ST_DRAWS] += chunks * k;
        if (sel == 0) break;
        int64_t u = (int64_t)c->targets[elo + sel - 1];
        out[step] = (uint32_t)u;
        prev = v;
        cur = u;
        emitted = (uint32_t)step + 1;
        if (emitted >= c->length) break;
        if (c->app_id == APP_METAPATH && emitted >= c->schema_len) break;
    }
    return emitted;
}

typedef struct {
    const walk_cfg *cfg;
    const int64_t *starts;
    uint64_t n, base_qid;
    uint32_t *out_seq, *out_len;
    volatile uint64_t *cursor;
    pthread_mutex_t *mu;
    int64_t stats[ST_COUNT];
} worker_arg;

static void *worker_main(void *p) {
    worker_arg *a = (worker_arg *)p;
    const walk_cfg *c = a->cfg;
    int64_t kb = c->k_big > c->k_small ? c->k_big : c->k_small;
    scratch_t s;
    s.lane_w = (double *)malloc(sizeof(double) * kb);
    s.lane_prefix = (double *)malloc(sizeof(double) * kb);
    s.lane_cand = (int64_t *)malloc(sizeof(int64_t) * kb);
    s.lane_base = (uint64_t *)malloc(sizeof(uint64_t) * kb);
    memset(a->stats, 0, sizeof(a->stats));
    const uint64_t grain = 64;
    for (;;) {
        uint64_t lo = __atomic_fetch_add(a->cursor, grain, __ATOMIC_RELAXED);
        if (lo >= a->n) break;
        uint64_t hi = lo + grain < a->n ? lo + grain : a->n;
        for (uint64_t i = lo; i < hi; i++) {
            uint32_t *row = a->out_seq + i * (uint64_t)c->length;
            for (uint32_t t = 0; t < c->length; t++) row[t] = 0xFFFFFFFFu;
            a->out_len[i] = walk_one(c, &s, a->base_qid + i, a->starts[i], row, a->stats);
        }
    }
    free(s.lane_w); free(s.lane_prefix); free(s.lane_cand); free(s.lane_base);
    return NULL;
}

/*
 * Walk queries starts[0..n) with global qids base_qid + i.  out_seq is
 * n*length u32 (sentinel padded), out_len n u32, stats[6] int64 accumulated
 * (ST_STEPS, ST_EDGES, ST_COLLECTIVES, ST_DRAWS, ST_SMALL, ST_LARGE).
 */
int fwo_walk(const int64_t *offsets, const uint32_t *targets, const float *weights,
             const uint8_t *labels, const int64_t *starts, uint64_t n, uint64_t base_qid,
             int app_id, int weighted, uint32_t length, double stop_prob, double inv_a,
             double inv_b, const int64_t *schema, uint32_t schema_len, int sampler_id,
             int64_t k_small, int64_t k_big, int64_t d_t, uint64_t seed,
             uint32_t *out_seq, uint32_t *out_len, int64_t *stats, int threads) {
    walk_cfg c = {offsets, targets, weights, labels, app_id, weighted, sampler_id, length,
                  stop_prob, inv_a, inv_b, schema, schema_len, k_small, k_big, d_t, seed};
    if (threads < 1) threads = 1;
    volatile uint64_t cursor = 0;
    worker_arg *args = (worker_arg *)calloc((size_t)threads, sizeof(worker_arg));
    pthread_t *tids = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    for (int t = 0; t < threads; t++) {
        args[t].cfg = &c; args[t].starts = starts; args[t].n = n; args[t].base_qid = base_qid;
        args[t].out_seq = out_seq; args[t].out_len = out_len; args[t].cursor = &cursor;
        if (t > 0) pthread_create(&tids[t], NULL, worker_main, &args[t]);
    }
    worker_main(&args[0]);
    for (int t = 1; t < threads; t++) pthread_join(tids[t], NULL);
    for (int t = 0; t < threads; t++)
        for (int i = 0; i < ST_COUNT; i++) stats[i] += args[t].stats[i];
    free(args); free(tids);
    return 0;
}

/* validate_walks restatement (_kernels.py:486-546); returns #violations. */
int64_t fwo_validate(const int64_t *offsets, const uint32_t *targets, const uint8_t *labels,
                     const int64_t *starts, uint64_t n, const uint32_t *result,
                     const uint32_t *lengths, uint32_t l_max, const int64_t *schema,
                     uint32_t schema_len) {
    int64_t bad = 0;
    for (uint64_t i = 0; i < n; i++) {
        int64_t cur = starts[i];
        int64_t ln = lengths[i];
        if (ln > (int64_t)l_max) { bad++; continue; }
        const uint32_t *row = result + i * (uint64_t)l_max;
        for (int64_t j = 0; j < ln; j++) {
            int64_t nxt = row[j];
            int64_t lo = offsets[cur], hi = offsets[cur + 1], found = -1;
            while (lo < hi) {
                int64_t mid = (lo + hi) >> 1;
                int64_t tv = targets[mid];
                if (tv < nxt) lo = mid + 1;
                else if (tv > nxt) hi = mid;
                else { found = mid; break; }
            }
            if (found < 0) { bad++; break; }
            if (schema_len > 0) {
                if (j >= (int64_t)schema_len) { bad++; break; }
                int64_t want = schema[j];
                int ok = 0;
                for (int64_t e = found; e >= offsets[cur] && (int64_t)targets[e] == nxt; e--)
                    if ((labels ? (int64_t)labels[e] : 0) == want) { ok = 1; break; }
                for (int64_t e = found + 1; !ok && e < offsets[cur + 1] && (int64_t)targets[e] == nxt; e++)
                    if ((labels ? (int64_t)labels[e] : 0) == want) { ok = 1; break; }
                if (!ok) { bad++; break; }
            }
            cur = nxt;
        }
        for (int64_t j = ln; j < (int64_t)l_max; j++)
            if (row[j] != 0xFFFFFFFFu) { bad++; break; }
    }
    return bad;
}
