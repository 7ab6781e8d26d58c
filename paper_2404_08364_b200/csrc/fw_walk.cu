// Persistent sm_100a walk kernel: one warp walks one query at a time; queries
// are pulled from a global atomic cursor (the reference's GlobalPool.fetch,
// engine.py:108-125, and the paper's P_G head pointer).
//
// Per step (reswalk _kernels.step_pass, _kernels.py:340-482):
//   route by deg(cur) <= d_t -> k = k_small else k_big      (:341, :351)
//   PPR stop draw on lane 1023, ctr 0, before deg==0       (:362-373)
//   deg==0 / MetaPath schema exhausted -> finish            (:375-380)
//   dynamic weights (_edge_weight, :280-308) fed to
//     DPRS: last accepted element in natural order          (:399-430)
//     ZPRS: last accepted element in lane-major order       (:431-464)
//   commit: result[step] = targets[elo + sel - 1]           (:466-482)
// The *logical* lane structure (element i -> lane i mod k, draw counter
// i div k) is what fixes the random stream; the physical mapping below
// (32 logical lanes per warp pass) is free, so results are bit-identical
// for any k in [1, 1000].
#include <cuda_runtime.h>
#include <climits>
#include <cstdint>

#include "fw_common.cuh"
#include "fw_walk.cuh"

namespace fw {

// Cold helpers (window advance, hash build, binary-search fallback).
// Inlined by default: an out-of-line call makes the tile loop save and
// restore registers around it (measured 6.3e7 vs 5.4e7 steps/s).
#ifndef FW_PF_NEXT
#define FW_PF_NEXT 1
#endif

#ifndef FW_PREFETCH_CHUNK
#define FW_PREFETCH_CHUNK 1
#endif

#ifndef FW_PREFILTER
#define FW_PREFILTER 1
#endif

#ifdef FW_COLD_OUTLINE
#define FW_COLD __noinline__
#else
#define FW_COLD __forceinline__
#endif

// Dynamic shared memory: warp_words(APP) words per warp (see fw_walk.cuh).
extern __shared__ __align__(16) uint32_t fw_smem[];

struct StepCtx {
    int64_t elo;      // offsets[cur]
    uint32_t deg;     // offsets[cur+1] - offsets[cur] (host checks d_max < 2^32)
    int64_t prev;     // previous vertex or -1
    int64_t plo, phi; // N(prev) range (node2vec)
    int64_t want;     // schema[step] (metapath)
    uint64_t A;       // (TAG | q<<30 | step<<10) * MIX1
};

// Membership of u in the sorted list targets[lo, hi) (_kernels.py:293-306).
__device__ __forceinline__ bool in_sorted(const uint32_t *__restrict__ tgt, int64_t lo,
                                          int64_t hi, uint32_t u) {
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        const uint32_t tv = ldg(tgt + mid);
        if (tv < u) lo = mid + 1;
        else if (tv > u) hi = mid;
        else return true;
    }
    return false;
}

// Dynamic transition weight of element i of N(cur) (_kernels.py:280-308).
// High word of the second multiply of mix64 (the final xorshift flips at
// most bit 0 of it).
__device__ __forceinline__ uint32_t mix64_yhi(uint64_t z) {
    z = (z ^ (z >> 30)) * MIX1;
    z = z ^ (z >> 27);
    return (uint32_t)((z * MIX2) >> 32);
}

// Prefilter threshold for a lane whose elements all have prefix P >= base + w:
// >= floor(T * 2^32) + 2 with T = wmax / (base + wmax), saturated.  The fp32
// estimate of T (conversion, add, approximate reciprocal, multiply) is within
// 2^-20 relative; the 2^-12 margin covers it.  base beyond the fp32 range gives
// t = 0 and thr = 2, still >= floor(T * 2^32) + 2 = 2.
// Without the disable check (finite wmax <= 1e37 guaranteed by the host).
__device__ __forceinline__ uint32_t accept_thr_raw(float wmax, float b) {
    float r;  // MUFU.RCP without the denormal-range fixup of __fdividef
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(b + wmax));
    const float t = wmax * r;
    return __float2uint_rz(fmaf(t, 4294967296.0f * 1.000244140625f, 2.0f));  // saturating
}
__device__ __forceinline__ uint32_t accept_thr_f(float wmax, float b) {
    const uint32_t thr = accept_thr_raw(wmax, b);
    return wmax <= 1e37f ? thr : 0xFFFFFFFFu;  // the host passes +inf to disable
}
__device__ __forceinline__ uint32_t accept_thr(float wmax, double base) {
    return accept_thr_f(wmax, (float)base);
}

// Certified accept test (walk mode 2: weights whose fp64 partial sums are not
// exact, e.g. log-normal).  The reference's P_seq (chunk-sequential sums,
// _kernels.py:404-424) and this kernel's tree-order P differ from the exact
// prefix by at most about (2i + c + 1) * 2^-53 * tot each (nonnegative terms,
// tot >= every partial sum of the step so far); d below is more than twice
// that.  Monotone rounding then decides fl(r * P_seq) < w from P alone unless
// r * P is within d of w:
//   ru(r * ru(P + d)) < w  -> accepted for every P_seq in [P - d, P + d]
//   rd(r * rd(P - d)) >= w -> rejected for every such P_seq
// and otherwise (probability ~ i * 2^-50) the step is ambiguous and is
// re-run on the ordered path.  Returns 1 accept, 0 reject, 2 ambiguous.
__device__ __forceinline__ int cert_accept(double r, double P, double w, double tot, uint32_t i,
                                           double slack, double abs_err = 0.0) {
    const double d = __dadd_ru(__dmul_ru(tot, __dmul_ru((double)i + 160.0, slack)), abs_err);
    if (__dmul_ru(r, __dadd_ru(P, d)) < w) return 1;
    if (__dmul_rd(r, fmax(__dadd_rd(P, -d), 0.0)) >= w) return 0;
    return 2;
}
constexpr uint32_t kCertFallback = 0xFFFFFFFFu;  // "re-run this step in order"

// The accept test of element idx1 - 1: exact (fl(r * P) < w, _kernels.py:421,
// 457) or, CERT, certified against the bound tot with ti terms in the sums
// (ambiguous -> amb).
template <bool CERT>
__device__ __forceinline__ void accept_test(double r, double P, double w, uint32_t idx1,
                                            double tot, uint32_t ti, double slack,
                                            uint32_t &cand, uint32_t &amb) {
    if constexpr (CERT) {
        if (w > 0.0) {
            const int c = cert_accept(r, P, w, tot, ti, slack);
            if (c == 1) cand = idx1;
            else if (c == 2) amb = idx1;
        }
    } else if (w > 0.0 && __dmul_rn(r, P) < w) {
        cand = idx1;
    }
}

// Prefilter threshold for a batch of elements starting at prefix `base`.
// CERT kernels bound w by the batch's own largest weight (any upper bound on
// the tested w keeps the prefilter exact) instead of the graph-wide maximum:
// log-normal weights span ~2^10, so the global bound lets far more elements
// through to the full draw.
template <bool CERT>
__device__ __forceinline__ uint32_t batch_thr(const WalkArgs &a, double base, double wmax_b) {
    if constexpr (CERT) return accept_thr_f(__double2float_ru(wmax_b), (float)base);
    else return accept_thr(a.accept_wmax, base);
}

template <int APP>
__device__ __forceinline__ double elem_weight(const WalkArgs &a, const StepCtx &s, uint32_t i) {
    const int64_t e = s.elo + i;
    if constexpr (APP == APP_METAPATH) {
        // both loads issued up front (a dependent weight load would cost a
        // second memory round trip per element)
        const int64_t lab = a.lab ? (int64_t)ldg(a.lab + e) : 0;
        const float w = a.weighted ? ldg(a.w + e) : 1.0f;
        return lab == s.want ? (double)w : 0.0;
    } else if constexpr (APP == APP_NODE2VEC) {
        if (s.prev >= 0) {
            const uint32_t u = ldg(a.tgt + e);
            double base;
            if ((int64_t)u == s.prev) base = a.inv_a;
            else base = in_sorted(a.tgt, s.plo, s.phi, u) ? 1.0 : a.inv_b;
            return a.weighted ? __dmul_rn(base, (double)ldg(a.w + e)) : base;
        }
        return a.weighted ? (double)ldg(a.w + e) : 1.0;
    } else {
        return a.weighted ? (double)ldg(a.w + e) : 1.0;
    }
}

// First-order apps (DeepWalk/PPR/MetaPath): the app weights of elements
// i, i+k, i+2k, i+3k with all loads issued before any is used (the ZPRS
// lane loops are latency-bound otherwise).
template <int APP, uint32_t KC = 0>
__device__ __forceinline__ void weights4(const WalkArgs &a, const StepCtx &s, uint32_t i,
                                         uint32_t k, double x[4]) {
    if (KC) k = KC;  // compile-time lane width: immediate load offsets
    float w[4];
    int lab[4];
#pragma unroll
    for (int r = 0; r < 4; r++) {
        const int64_t e = s.elo + i + (uint32_t)r * k;
        w[r] = a.weighted ? ldg(a.w + e) : 1.0f;
        lab[r] = (APP == APP_METAPATH && a.lab) ? (int)ldg(a.lab + e) : 0;
    }
#pragma unroll
    for (int r = 0; r < 4; r++)
        x[r] = (APP != APP_METAPATH || (int64_t)lab[r] == s.want) ? (double)w[r] : 0.0;
}

__device__ __forceinline__ uint64_t lane_base(const WalkArgs &a, const StepCtx &s, uint32_t j) {
    return mix64(a.h ^ (s.A + (uint64_t)j * MIX1));
}

// ---------------------------------------------------------------------------
// ZPRS (samplers.py:188-220).  Logical lane j owns elements j, j+k, j+2k...
// and physical lane p of group g plays logical lane j = 32g + p, so each
// lane's pass-1 sum and pass-2 running prefix accumulate in chunk order --
// the reference's own order -- and only the exclusive scan over lanes needs
// care (sequential unless EXACT).  The winner is the highest logical lane
// holding a candidate (_kernels.py:459-462), so pass 2 walks the groups from
// the top and stops at the first group with a candidate: lanes below it
// cannot change the result (about half the RNG work saved on hub steps).
// For deg <= kHashSlots the app weights of pass 1 are staged in the warp's
// shared memory (exact as float for DeepWalk/PPR/MetaPath) and pass 2 reads
// them from there instead of re-reading global memory.
// ---------------------------------------------------------------------------
template <int APP, bool EXACT>
__device__ __forceinline__ double lane_excl_scan(double lsum, double &ecarry, int lane) {
    double excl;
    if constexpr (EXACT) {
        const double incl = warp_incl_scan(lsum, lane);
        const double up = __shfl_up_sync(FULL, incl, 1);
        excl = __dadd_rn(ecarry, lane == 0 ? 0.0 : up);
        ecarry = __dadd_rn(ecarry, __shfl_sync(FULL, incl, 31));
    } else {  // run = 0; prefix[j] = run; run += lane_w[j]  (_kernels.py:441-444)
        double run = ecarry;
        excl = 0.0;
#pragma unroll 1
        for (int t = 0; t < 32; t++) {
            const double lt = __shfl_sync(FULL, lsum, t);
            if (lane == t) excl = run;
            run = __dadd_rn(run, lt);
        }
        ecarry = run;
    }
    return excl;
}

// CERT: certified accept tests against the step total tot (the lane's
// exclusive prefix comes from a tree scan); amb = last ambiguous element + 1.
template <int APP, uint32_t KC = 0, bool CERT = false>
__device__ __forceinline__ uint32_t zprs_lane_pass2(const WalkArgs &a, const StepCtx &s,
                                                    uint32_t j, uint32_t k, double run,
                                                    bool staged, uint32_t woff,
                                                    [[maybe_unused]] double tot = 0.0,
                                                    [[maybe_unused]] uint32_t *amb_out = nullptr) {
    if (KC) k = KC;
    const float *stage = reinterpret_cast<const float *>(fw_smem) + woff;
    uint32_t cand = 0;
    [[maybe_unused]] uint32_t amb = 0;
    uint64_t word = lane_base(a, s, j);
    const uint32_t deg = s.deg;
    // Accept prefilter (as in dprs_n2v_pow2): element accepted => r <
    // w / (run_before + w) <= wmax / (run_before + wmax), so hi32 of the
    // draw's second multiply must be <= thr(run at the batch start); only
    // those elements run the full draw and the exact test.
    uint32_t i = j;
    if (staged) {
        for (; i + 3 * k < deg; i += 4 * k) {
            const uint32_t thr = batch_thr<CERT>(
                a, run, CERT ? fmaxf(fmaxf(stage[i], stage[i + k]),
                                     fmaxf(stage[i + 2 * k], stage[i + 3 * k])) : 0.0);
#pragma unroll
            for (int r = 0; r < 4; r++, word += GOLDEN) {
                const double wv = (double)stage[i + r * k];
                run = __dadd_rn(run, wv);
                if (mix64_yhi(word) <= thr) {
                    const double u = u01_word(word);
                    accept_test<CERT>(u, run, wv, i + r * k + 1, tot, i + r * k + k, a.cert_slack, cand, amb);
                }
            }
        }
        for (; i < deg; i += k, word += GOLDEN) {
            const double wv = (double)stage[i];
            run = __dadd_rn(run, wv);
            const double r = u01_word(word);
            accept_test<CERT>(r, run, wv, i + 1, tot, i + k, a.cert_slack, cand, amb);
        }
    } else {
        if constexpr (APP != APP_NODE2VEC) {
            if constexpr (KC == 256 && APP == APP_PPR) {
                // PPR hub steps: 8 loads in flight per lane (+8.6% on config
                // [4]; the same batch cost DeepWalk s16 10%)
                for (; i + 7 * k < deg; i += 8 * k) {
                    float w[8];
#pragma unroll
                    for (int r = 0; r < 8; r++)
                        w[r] = a.weighted ? ldg(a.w + s.elo + i + (uint32_t)r * k) : 1.0f;
                    float wm8 = 0.0f;
                    if constexpr (CERT) {
#pragma unroll
                        for (int r = 0; r < 8; r++) wm8 = fmaxf(wm8, w[r]);
                    }
                    const uint32_t thr = batch_thr<CERT>(a, run, wm8);
#pragma unroll
                    for (int r = 0; r < 8; r++, word += GOLDEN) {
                        const double wv = (double)w[r];
                        run = __dadd_rn(run, wv);
                        if (mix64_yhi(word) <= thr) {
                            const double u = u01_word(word);
                            accept_test<CERT>(u, run, wv, i + r * k + 1, tot, i + r * k + k, a.cert_slack, cand, amb);
                        }
                    }
                }
            }
            for (; i + 3 * k < deg; i += 4 * k) {
                double x[4];
                weights4<APP, KC>(a, s, i, k, x);
                const uint32_t thr =
                    batch_thr<CERT>(a, run, CERT ? fmax(fmax(x[0], x[1]), fmax(x[2], x[3])) : 0.0);
#pragma unroll
                for (int r = 0; r < 4; r++, word += GOLDEN) {
                    run = __dadd_rn(run, x[r]);
                    if (mix64_yhi(word) <= thr) {
                        const double u = u01_word(word);
                        accept_test<CERT>(u, run, x[r], i + r * k + 1, tot, i + r * k + k, a.cert_slack, cand, amb);
                    }
                }
            }
        }
        for (; i < deg; i += k, word += GOLDEN) {
            const double wv = elem_weight<APP>(a, s, i);
            run = __dadd_rn(run, wv);
            const double r = u01_word(word);
            accept_test<CERT>(r, run, wv, i + 1, tot, i + k, a.cert_slack, cand, amb);
        }
    }
    if constexpr (CERT) *amb_out = amb;
    return cand;
}

// Pass 1 of ZPRS for logical lane j: the lane sum in chunk order (the
// reference's order), optionally staging the weights at their element index.
template <int APP, uint32_t KC = 0>
__device__ __forceinline__ double zprs_lane_pass1(const WalkArgs &a, const StepCtx &s,
                                                  uint32_t j, uint32_t k, bool staged,
                                                  float *stage) {
    if (KC) k = KC;
    double lsum = 0.0;
    const uint32_t deg = s.deg;
    uint32_t i = j;
    if constexpr (APP != APP_NODE2VEC) {
        if constexpr (KC != 0 && APP != APP_METAPATH) {
            // 16 loads in flight per lane (the pass is load-latency-bound)
            for (; i + 15 * k < deg; i += 16 * k) {
                float w[16];
#pragma unroll
                for (int r = 0; r < 16; r++)
                    w[r] = a.weighted ? ldg(a.w + s.elo + i + (uint32_t)r * k) : 1.0f;
#pragma unroll
                for (int r = 0; r < 16; r++) {
                    if (staged) stage[i + r * k] = w[r];
                    lsum = __dadd_rn(lsum, (double)w[r]);
                }
            }
        }
        for (; i + 3 * k < deg; i += 4 * k) {
            double x[4];
            weights4<APP, KC>(a, s, i, k, x);
#pragma unroll
            for (int r = 0; r < 4; r++) {
                if (staged) stage[i + r * k] = (float)x[r];
                lsum = __dadd_rn(lsum, x[r]);
            }
        }
    }
    for (; i < deg; i += k) {
        const double wv = elem_weight<APP>(a, s, i);
        if (staged) stage[i] = (float)wv;
        lsum = __dadd_rn(lsum, wv);
    }
    return lsum;
}

// KC: compile-time lane width (32 / 256, the reference's defaults) or 0.
// CERT (with EXACT): tree lane scan and certified accept tests; the winner
// (highest lane with a candidate, its last accepted element) is certain
// unless a lane above it, or the winner after its candidate, holds an
// ambiguous test -- then kCertFallback (the caller re-runs the step in order).
template <int APP, bool EXACT, uint32_t KC = 0, bool CERT = false>
__device__ uint32_t zprs_warp(const WalkArgs &a, const StepCtx &s, uint32_t k, int lane,
                              uint32_t woff) {
    static_assert(!CERT || EXACT, "certified ZPRS uses the tree lane scan");
    if (KC) k = KC;
    const uint32_t deg = s.deg;
    const uint32_t nl = k < deg ? k : deg;
    // app weights are exactly representable as float except for node2vec
    const bool staged = APP != APP_NODE2VEC && deg <= warp_slots(APP);
    float *stage = reinterpret_cast<float *>(fw_smem) + woff;
    if (nl <= 32) {  // one group: physical lane == logical lane
        const uint32_t j = lane;
        double lsum = 0.0;
        uint32_t cand = 0;
        [[maybe_unused]] uint32_t amb = 0;
        double ecarry = 0.0;
        if (APP == APP_METAPATH && staged) {
            // Most MetaPath weights are 0 (label filter).  A zero weight adds
            // nothing to the running prefix and can never be accepted, so
            // lane j keeps only its nonzero elements, compacted in chunk
            // order into its own staging slots j + k*m (m <= chunk index, so
            // the list never outruns the dense layout), chunk ids alongside.
            uint16_t *cst = reinterpret_cast<uint16_t *>(fw_smem + woff + warp_slots(APP));
            uint32_t m = 0;
            if (j < nl) {
                uint32_t c = 0, i = j;
                for (; i + 3 * k < deg; i += 4 * k) {
                    double x[4];
                    weights4<APP, KC>(a, s, i, k, x);
#pragma unroll
                    for (int r = 0; r < 4; r++, c++) {
                        if (x[r] > 0.0) {
                            stage[j + k * m] = (float)x[r];
                            cst[j + k * m] = (uint16_t)c;
                            m++;
                        }
                        lsum = __dadd_rn(lsum, x[r]);
                    }
                }
                for (; i < deg; i += k, c++) {
                    const double wv = elem_weight<APP>(a, s, i);
                    if (wv > 0.0) {
                        stage[j + k * m] = (float)wv;
                        cst[j + k * m] = (uint16_t)c;
                        m++;
                    }
                    lsum = __dadd_rn(lsum, wv);
                }
            }
            double run = lane_excl_scan<APP, EXACT>(lsum, ecarry, lane);
            if (m) {
                const uint64_t base = lane_base(a, s, j);
                for (uint32_t x = 0; x < m; x++) {
                    const double wv = (double)stage[j + k * x];
                    const uint32_t c = cst[j + k * x];
                    run = __dadd_rn(run, wv);
                    const double r = u01_word(base + (uint64_t)c * GOLDEN);
                    accept_test<CERT>(r, run, wv, c * k + j + 1, ecarry, c * k + j + k,
                                      a.cert_slack, cand, amb);
                }
            }
        } else {
            if (j < nl) lsum = zprs_lane_pass1<APP, KC>(a, s, j, k, staged, stage);
            const double excl = lane_excl_scan<APP, EXACT>(lsum, ecarry, lane);
            cand = j < nl ? zprs_lane_pass2<APP, KC, CERT>(a, s, j, k, excl, staged, woff,
                                                            ecarry, &amb)
                          : 0;
        }
        const unsigned m = __ballot_sync(FULL, cand > 0);
        const uint32_t c = __shfl_sync(FULL, cand, m ? 31 - __clz(m) : 0);
        __syncwarp();
        if constexpr (CERT) {  // ambiguity at or above the winner
            const unsigned bad = __ballot_sync(FULL, amb > cand);
            if (bad >> (m ? 31 - __clz(m) : 0)) return kCertFallback;
        }
        return m ? c : 0;
    }
    if (nl <= 256) {  // up to 8 groups: lane sums -> exclusive prefixes in smem
        double *E = reinterpret_cast<double *>(fw_smem + woff + warp_slots(APP));
        const uint32_t ng = (nl + 31) >> 5;
        double ecarry = 0.0;
        for (uint32_t g = 0; g < ng; g++) {
            const uint32_t j = g * 32 + lane;
            const double lsum = j < nl ? zprs_lane_pass1<APP, KC>(a, s, j, k, staged, stage) : 0.0;
            E[j] = lane_excl_scan<APP, EXACT>(lsum, ecarry, lane);
        }
        __syncwarp();
        uint32_t best = 0;
        for (int g = (int)ng - 1; g >= 0; g--) {
            const uint32_t j = g * 32 + lane;
            [[maybe_unused]] uint32_t amb = 0;
            const uint32_t cand = j < nl ? zprs_lane_pass2<APP, KC, CERT>(a, s, j, k, E[j], staged,
                                                                          woff, ecarry, &amb)
                                         : 0;
            const unsigned m = __ballot_sync(FULL, cand > 0);
            if constexpr (CERT) {
                const unsigned bad = __ballot_sync(FULL, amb > cand);
                if (bad >> (m ? 31 - __clz(m) : 0)) {
                    best = kCertFallback;
                    break;
                }
            }
            if (m) {
                best = __shfl_sync(FULL, cand, 31 - __clz(m));
                break;
            }
        }
        __syncwarp();
        return best;
    }
    if constexpr (CERT) return kCertFallback;  // k > 256: the step total comes too late
    // k > 256: group by group, upward (generic k, correctness path)
    double ecarry = 0.0;
    uint32_t best = 0;
    for (uint32_t g0 = 0; g0 < nl; g0 += 32) {
        const uint32_t j = g0 + lane;
        const double lsum = j < nl ? zprs_lane_pass1<APP, KC>(a, s, j, k, false, nullptr) : 0.0;
        const double excl = lane_excl_scan<APP, EXACT>(lsum, ecarry, lane);
        const uint32_t cand = j < nl ? zprs_lane_pass2<APP, KC>(a, s, j, k, excl, false, woff) : 0;
        const unsigned m = __ballot_sync(FULL, cand > 0);
        const uint32_t c = __shfl_sync(FULL, cand, m ? 31 - __clz(m) : 0);
        if (m) best = c;
    }
    return best;
}

// ---------------------------------------------------------------------------
// DPRS (samplers.py:156-185): the selection is the last accepted element in
// natural order, element i accepted iff w_i > 0 and r(i mod k, i div k) *
// P_i < w_i with P_i the fp64 prefix weight.  EXACT: tiles of 32 elements,
// warp tree scan + running carry (bit-identical because every partial sum is
// exact).  Otherwise the reference's order is replayed: sequential sum
// within each k-chunk, P = chunk_prefix + carry, carry += chunk sum.
// ---------------------------------------------------------------------------
template <int APP, bool CERT = false>
__device__ uint32_t dprs_warp_exact(const WalkArgs &a, const StepCtx &s, uint32_t k, int lane) {
    const uint32_t deg = s.deg;
    double carry = 0.0;
    uint32_t cand = 0, amb = 0;
    // CERT: the accept test against the post-tile carry (>= every partial sum
    // of the step so far) -- see cert_accept
#define FW_DPRS_TEST(I, WV, P, R, TOT)                                                   \
    do {                                                                                 \
        if constexpr (CERT) {                                                            \
            if ((WV) > 0.0) {                                                            \
                const int c_ = cert_accept((R), (P), (WV), (TOT), (I), a.cert_slack);    \
                if (c_ == 1) cand = (I) + 1;                                             \
                else if (c_ == 2) amb = (I) + 1;                                         \
            }                                                                            \
        } else if ((WV) > 0.0 && __dmul_rn((R), (P)) < (WV)) {                           \
            cand = (I) + 1;                                                              \
        }                                                                                \
    } while (0)
    if (k == 32) {
        uint64_t word = lane_base(a, s, lane);
#pragma unroll 2
        for (uint32_t t0 = 0; t0 < deg; t0 += 32, word += GOLDEN) {
            const uint32_t i = t0 + lane;
            const double wv = i < deg ? elem_weight<APP>(a, s, i) : 0.0;
            const uint32_t thr = batch_thr<CERT>(a, carry, wv);  // prefilter
            const double incl = warp_incl_scan(wv, lane);
            const double P = __dadd_rn(carry, incl);
            const double nc = __dadd_rn(carry, __shfl_sync(FULL, incl, 31));
            if (mix64_yhi(word) <= thr) {
                const double r = u01_word(word);
                FW_DPRS_TEST(i, wv, P, r, nc);
            }
            carry = nc;
        }
    } else if (k == 256) {
        uint64_t base[8];
#pragma unroll
        for (int q = 0; q < 8; q++) base[q] = lane_base(a, s, q * 32 + lane);
        uint64_t cadd = 0;
        for (uint32_t c0 = 0; c0 < deg; c0 += 256, cadd += GOLDEN) {
#pragma unroll
            for (int q = 0; q < 8; q++) {
                const uint32_t t0 = c0 + q * 32;
                if (t0 < deg) {  // warp-uniform
                    const uint32_t i = t0 + lane;
                    const double wv = i < deg ? elem_weight<APP>(a, s, i) : 0.0;
                    const uint32_t thr = batch_thr<CERT>(a, carry, wv);  // prefilter
                    const double incl = warp_incl_scan(wv, lane);
                    const double P = __dadd_rn(carry, incl);
                    const double nc = __dadd_rn(carry, __shfl_sync(FULL, incl, 31));
                    const uint64_t wd = base[q] + cadd;
                    if (mix64_yhi(wd) <= thr) {
                        const double r = u01_word(wd);
                        FW_DPRS_TEST(i, wv, P, r, nc);
                    }
                    carry = nc;
                }
            }
        }
    } else {
        for (uint32_t t0 = 0; t0 < deg; t0 += 32) {
            const uint32_t i = t0 + lane;
            const double wv = i < deg ? elem_weight<APP>(a, s, i) : 0.0;
            const double incl = warp_incl_scan(wv, lane);
            const double P = __dadd_rn(carry, incl);
            const double nc = __dadd_rn(carry, __shfl_sync(FULL, incl, 31));
            if (wv > 0.0) {
                const double r = u01(lane_base(a, s, i % k), (uint64_t)(i / k));
                FW_DPRS_TEST(i, wv, P, r, nc);
            }
            carry = nc;
        }
    }
#undef FW_DPRS_TEST
    const uint32_t sel = __reduce_max_sync(FULL, cand);
    if constexpr (CERT) {
        if (__reduce_max_sync(FULL, amb) > sel) return kCertFallback;
    }
    return sel;
}

// ---------------------------------------------------------------------------
// Node2Vec DPRS, exact order, prev >= 0: the hot path of the headline config.
//
// Layout: tiles of 128 elements of N(cur), lane p holding 4 consecutive
// elements (16-byte loads of targets and weights; the tile grid is anchored
// at elo & ~3 and only the first and last tiles mask slots), so the
// natural-order fp64 prefix is a 4-element local prefix plus one warp scan
// per 128 elements.  The next tile's targets are loaded one tile ahead.
//
// Membership u in N(prev) (_kernels.py:288-306): N(prev) is sorted and the
// u values only grow along N(cur), so N(prev) is consumed in windows of
// kChunk slots, each stored in an order-preserving hashed sorted table in
// the warp's shared memory (hash_build, below); a lane looks u up when u <=
// max(window) (or the window is the last one), otherwise the window advances
// (skipping windows whose max is below every pending u).  N(prev) is read
// once, coalesced.  When d(prev) is far larger than d(cur) a per-element
// branchless binary search in global memory is cheaper and is used instead.
//
// Random draws: element i uses logical lane j = i mod k and counter i div k;
// for power-of-two k <= 256 each lane stages the words of its own 4 slots
// (stage_words), and an accept prefilter skips the full draw for elements
// that cannot be accepted (dprs_n2v_pow2).
// ---------------------------------------------------------------------------
constexpr uint32_t kEmpty = 0xFFFFFFFFu;

// fp64 shuffles as two explicit 32-bit shuffles (the 64-bit overloads
// compile to extra register swaps on this toolchain).
__device__ __forceinline__ double shfl_up_d(double x, int d) {
    const int lo = __shfl_up_sync(FULL, __double2loint(x), d);
    const int hi = __shfl_up_sync(FULL, __double2hiint(x), d);
    return __hiloint2double(hi, lo);
}
__device__ __forceinline__ double shfl_d(double x, int src) {
    const int lo = __shfl_sync(FULL, __double2loint(x), src);
    const int hi = __shfl_sync(FULL, __double2hiint(x), src);
    return __hiloint2double(hi, lo);
}
// Predicated DADD (no FSEL pair on the ALU pipe, which is the binding pipe
// of the sampler loops).
template <int D>
__device__ __forceinline__ double scan_round(double v, int lane) {
    const double o = shfl_up_d(v, D);
    asm("{\n\t.reg .pred p;\n\tsetp.ge.s32 p, %1, %2;\n\t@p add.rn.f64 %0, %0, %3;\n\t}"
        : "+d"(v) : "r"(lane), "n"(D), "d"(o));
    return v;
}
// Same scan without a lane-index register: the shuffled addend is zeroed
// (two SELs on its halves) when the shuffle's own in-range flag is clear, so
// the add is unconditional and both operands stay in aligned register pairs.
template <int D>
__device__ __forceinline__ double scan_round_p(double v) {
    uint32_t olo, ohi;
    asm volatile("{\n\t.reg .pred p;\n\t"
                 "shfl.sync.up.b32 %0|p, %2, %4, 0, -1;\n\t"
                 "shfl.sync.up.b32 %1, %3, %4, 0, -1;\n\t"
                 "@!p mov.b32 %0, 0;\n\t"
                 "@!p mov.b32 %1, 0;\n\t}"
                 : "=r"(olo), "=r"(ohi)
                 : "r"(__double2loint(v)), "r"(__double2hiint(v)), "n"(D));
    return __dadd_rn(v, __hiloint2double(ohi, olo));
}
__device__ __forceinline__ double warp_incl_scan_p(double v) {
    v = scan_round_p<1>(v);
    v = scan_round_p<2>(v);
    v = scan_round_p<4>(v);
    v = scan_round_p<8>(v);
    return scan_round_p<16>(v);
}

__device__ __forceinline__ double warp_incl_scan_d(double v, int lane) {
    v = scan_round<1>(v, lane);
    v = scan_round<2>(v, lane);
    v = scan_round<4>(v, lane);
    v = scan_round<8>(v, lane);
    return scan_round<16>(v, lane);
}

// Membership table for a window of N(prev): an order-preserving hashed
// sorted array in the warp's shared-memory slice, built without atomics.
// A chunk of cn <= kChunk sorted keys k_0..k_{cn-1} (min kmin, max kmax) is
// mapped to kGroups groups of 4 slots by the monotone bucket function
//   b(u) = min(umulhi(u - kmin, scale), kGroups - 1),
//   scale ~ kGroups * 2^32 / (kmax - kmin + 1),
// and key i goes to slot pos_i = i + max_{j<=i}(4 b_j - j): the first free
// slot at or after its group start, keeping the table sorted (a warp
// max-scan, no atomics, no collisions).  pos_i <= 4(kGroups-1) + cn - 1 <
// kTabSlots.  A lookup reads group b(u) with one LDS.128; u is present iff
// it is in that group, or -- when the group is full and its last key is < u
// (rare) -- in a following group.  Empty slots hold kEmpty (> any vertex
// id).  The window over N(prev) is described by three registers in the hot
// loop (kmin, scale, lim = kmax or ~0 for the last chunk); chunk start,
// length and d(prev) sit in the warp's control words (kCtlWord).
constexpr uint32_t kGroups = 304;
static_assert(4 * (kGroups - 1) + kChunk < kTabSlots, "table overflow (the last slot is the dump)");

struct HashState {
    uint32_t kmin, scale, lim;
};

__device__ __forceinline__ uint32_t tab_group(uint32_t u, const HashState &hs) {
    return min(__umulhi(u - hs.kmin, hs.scale), kGroups - 1);
}
__device__ __forceinline__ uint4 bucket_at(uint32_t woff, uint32_t b) {
    return reinterpret_cast<const uint4 *>(fw_smem + woff)[b];
}
__device__ __forceinline__ bool bucket_has(const uint4 q, uint32_t u) {
    return q.x == u || q.y == u || q.z == u || q.w == u;
}

// Build the table for chunk c of N(prev) = tgt[plo, plo + dp).  Chunks sit
// on a 16-byte aligned grid: chunk c covers global slots [A + 256c, A +
// 256(c+1)) with A = plo & ~3, clipped to N(prev), so lane x reads its 8
// consecutive slots with two 16-byte loads, forms the running max of
// 4 b(k_s) - s over them, and one warp max-scan gives every slot's position
// pos_s = s + max_{j<=s}(4 b_j - j) (slot indices stand in for ranks: the
// offset of a clipped first chunk shifts every position equally).
// Control words: [0] = c, [2] = dp; [4], [5] = plo.
__device__ __forceinline__ void tab_clear(uint32_t woff, int lane) {
    uint4 *t4 = reinterpret_cast<uint4 *>(fw_smem + woff);
#pragma unroll
    for (int x = 0; x < (int)((kTabSlots / 4 + 31) / 32); x++)
        if (x * 32 + lane < (int)(kTabSlots / 4))
            t4[x * 32 + lane] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
}

__device__ __forceinline__ uint32_t tab_scale(uint32_t kmin, uint32_t kmax) {
    // any scale keeps the bucket map monotone (tab_group clamps the top), so
    // the approximate reciprocal is enough; range >= 1 is never denormal.
    // The (1 - 2^-18) factor covers the conversion, add, reciprocal and
    // multiply roundings (< 2^-21 together), so every key of the window maps
    // below kGroups without the clamp: umulhi(k - kmin, scale) <=
    // (kmax - kmin) * kGroups / (kmax - kmin + 1) < kGroups (tab_group_in).
    const float range = (float)(kmax - kmin) + 1.0f;
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(range));
    return (uint32_t)fminf((float)kGroups * 4294967296.0f * (1.0f - 0x1p-18f) * r, 4294967040.0f);
}
// Group of a key known to lie in [kmin, kmax] (the build's own keys).
__device__ __forceinline__ uint32_t tab_group_in(uint32_t k, const HashState &hs) {
    return __umulhi(k - hs.kmin, hs.scale);
}

// The keys of chunk c, loaded ahead of the build so the load latency can
// overlap other work (the step prologue issues them before staging the draw
// words).
struct ChunkKeys {
    uint4 ka, kb;
    uint32_t kmin, kmax;
};

__device__ __forceinline__ ChunkKeys chunk_load(const uint32_t *__restrict__ tgt, int64_t plo,
                                                uint32_t dp, uint32_t c, int lane) {
    const int64_t end = plo + (int64_t)dp;
    const int64_t cs = (plo & ~(int64_t)3) + (int64_t)kChunk * c;  // chunk's first slot
    const int s0 = 8 * lane;
    ChunkKeys ck;
    if (cs >= plo && cs + (int64_t)kChunk <= end) {
        // whole chunk inside N(prev) (the common case): min/max come by shuffle
        ck.ka = ldg(reinterpret_cast<const uint4 *>(tgt + cs + s0));
        ck.kb = ldg(reinterpret_cast<const uint4 *>(tgt + cs + s0 + 4));
        ck.kmin = ck.kmax = 0;
#if FW_PREFETCH_CHUNK
        if (cs + 2 * (int64_t)kChunk <= end)  // the next chunk into L1
            asm volatile("prefetch.global.L1 [%0];" ::"l"(tgt + cs + kChunk + s0));
#endif
    } else {
        const int64_t lo = max(cs, plo), hi = min(cs + (int64_t)kChunk, end);
        const int64_t g0 = cs + s0;
        ck.ka = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
        ck.kb = ck.ka;
        if (g0 < hi) ck.ka = ldg(reinterpret_cast<const uint4 *>(tgt + g0));
        if (g0 + 4 < hi) ck.kb = ldg(reinterpret_cast<const uint4 *>(tgt + g0 + 4));
        ck.kmin = ldg(tgt + lo);
        ck.kmax = ldg(tgt + hi - 1);
#if FW_PREFETCH_CHUNK
        if (g0 + (int64_t)kChunk < end)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(tgt + g0 + kChunk));
#endif
    }
    return ck;
}

__device__ FW_COLD HashState hash_build(const ChunkKeys &ck, int64_t plo, uint32_t dp,
                                        uint32_t c, uint32_t woff, int lane) {
    const int64_t end = plo + (int64_t)dp;
    const int64_t cs = (plo & ~(int64_t)3) + (int64_t)kChunk * c;
    const int s0 = 8 * lane;
    const uint32_t key[8] = {ck.ka.x, ck.ka.y, ck.ka.z, ck.ka.w,
                             ck.kb.x, ck.kb.y, ck.kb.z, ck.kb.w};
    HashState hs;
    int m[8];
    int run = INT_MIN;
    const bool whole = cs >= plo && cs + (int64_t)kChunk <= end;
    if (whole) {
        hs.kmin = __shfl_sync(FULL, key[0], 0);
        const uint32_t kmax = __shfl_sync(FULL, key[7], 31);
        hs.scale = tab_scale(hs.kmin, kmax);
        hs.lim = cs + (int64_t)kChunk >= end ? kEmpty : kmax;
        __syncwarp();  // previous readers of the table are done
        tab_clear(woff, lane);
#pragma unroll
        for (int r = 0; r < 8; r++) {
            run = max(run, (int)(4 * tab_group_in(key[r], hs)) - (s0 + r));
            m[r] = run;
        }
    } else {
        const int64_t lo = max(cs, plo), hi = min(cs + (int64_t)kChunk, end);
        hs.kmin = ck.kmin;
        hs.scale = tab_scale(ck.kmin, ck.kmax);
        hs.lim = cs + (int64_t)kChunk >= end ? kEmpty : ck.kmax;
        __syncwarp();  // previous readers of the table are done
        tab_clear(woff, lane);
        const int vlo = (int)(lo - cs), vhi = (int)(hi - cs);  // valid slots [vlo, vhi)
#pragma unroll
        for (int r = 0; r < 8; r++) {
            const int sl = s0 + r;
            const bool v = sl >= vlo && sl < vhi;
            run = max(run, v ? (int)(4 * tab_group_in(key[r], hs)) - sl : INT_MIN);
            m[r] = v ? run : INT_MAX;  // INT_MAX marks an invalid slot
        }
    }
    if (lane == 0) {
        fw_smem[woff + kCtlWord + 0] = c;
        fw_smem[woff + kCtlWord + 2] = dp;
    }
    int incl = run;  // inclusive max-scan over lanes (idempotent: no predicate)
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) incl = max(incl, __shfl_up_sync(FULL, incl, d));
    int excl = __shfl_up_sync(FULL, incl, 1);
    if (lane == 0) excl = INT_MIN;
    __syncwarp();  // the clear is complete
    // unconditional stores (no per-key branches): an invalid slot writes
    // kEmpty to the table's last slot, which no key ever occupies (positions
    // stay below 4 (kGroups - 1) + kChunk), so it reads as empty
    if (whole) {  // every slot valid: no dump redirection
#pragma unroll
        for (int r = 0; r < 8; r++) fw_smem[woff + s0 + r + max(excl, m[r])] = key[r];
    } else {
#pragma unroll
        for (int r = 0; r < 8; r++) {
            const bool v = m[r] != INT_MAX;
            fw_smem[woff + (v ? s0 + r + max(excl, m[r]) : kTabSlots - 1)] = v ? key[r] : kEmpty;
        }
    }
    __syncwarp();
    return hs;
}

// Continuation probes (a full group whose last key is < u) and the window
// advance (cold path).
struct SlowRet {
    uint32_t mem;
    HashState hs;
};

__device__ __forceinline__ int64_t ctl_plo(uint32_t woff) {
    return (int64_t)(((uint64_t)fw_smem[woff + kCtlWord + 5] << 32) | fw_smem[woff + kCtlWord + 4]);
}

__device__ FW_COLD SlowRet member4_slow(const uint32_t *__restrict__ tgt, uint32_t woff,
                                        uint32_t u0, uint32_t u1, uint32_t u2, uint32_t u3,
                                        uint32_t full, uint32_t need, HashState hs, int lane) {
    const uint32_t u[4] = {u0, u1, u2, u3};
    uint32_t mem = 0;
    for (;;) {
#pragma unroll
        for (int e = 0; e < 4; e++) {
            if ((full >> e) & 1) {
                uint32_t g = tab_group(u[e], hs);
                for (;;) {
                    const uint4 q = bucket_at(woff, ++g);
                    if (bucket_has(q, u[e])) { mem |= 1u << e; break; }
                    if (!(q.w < u[e])) break;
                }
            }
        }
        if (!__any_sync(FULL, need)) return SlowRet{mem, hs};
        uint32_t umin = kEmpty;
#pragma unroll
        for (int e = 3; e >= 0; e--)
            if ((need >> e) & 1) umin = u[e];
        umin = __reduce_min_sync(FULL, umin);
        // advance: skip whole chunks that end below every pending u (chunk
        // c ends at slot A + 256c + 255; it is the last one when that
        // reaches the end of N(prev))
        const int64_t plo = ctl_plo(woff);
        const uint32_t dp = fw_smem[woff + kCtlWord + 2];
        const int64_t end = plo + (int64_t)dp, A = plo & ~(int64_t)3;
        uint32_t c = fw_smem[woff + kCtlWord + 0] + 1;
        ChunkKeys ck = chunk_load(tgt, plo, dp, c, lane);
        // the loaded chunk's own max decides a skip (no separate probe load)
        while (A + (int64_t)kChunk * (c + 1) < end &&
               __shfl_sync(FULL, ck.kb.w, 31) < umin) {
            c++;
            ck = chunk_load(tgt, plo, dp, c, lane);
        }
        hs = hash_build(ck, plo, dp, c, woff, lane);
        full = 0;
        uint32_t here = 0;
#pragma unroll
        for (int e = 0; e < 4; e++) {  // branch-free re-lookups, masked after
            const uint4 q = bucket_at(woff, tab_group(u[e], hs));
            const bool hit = bucket_has(q, u[e]);
            here |= (u[e] <= hs.lim ? 1u : 0u) << e;
            mem |= (hit ? 1u : 0u) << e;
            full |= (!hit && q.w < u[e] ? 1u : 0u) << e;
        }
        // a hit for a slot that was not pending is a true member found
        // earlier (an older window's keys all lie below this window's)
        here &= need;
        full &= here;
        need &= ~here;
    }
}

// 4 independent branchless binary searches over P[0, dp) (global memory).
__device__ FW_COLD uint32_t member4_bsearch(const uint32_t *__restrict__ P, uint32_t dp,
                                                uint32_t u0, uint32_t u1, uint32_t u2,
                                                uint32_t u3, uint32_t need) {
    const uint32_t u[4] = {u0, u1, u2, u3};
    uint32_t b[4] = {0, 0, 0, 0};
    uint32_t n = dp;
    while (n > 1) {
        const uint32_t half = n >> 1;
#pragma unroll
        for (int e = 0; e < 4; e++) b[e] = ldg(P + b[e] + half) <= u[e] ? b[e] + half : b[e];
        n -= half;
    }
    uint32_t mem = 0;
#pragma unroll
    for (int e = 0; e < 4; e++)
        if (((need >> e) & 1) && ldg(P + b[e]) == u[e]) mem |= 1u << e;
    return mem;
}

// 64-bit warp shuffle from an arbitrary source lane.
__device__ __forceinline__ uint64_t shfl_u64(uint64_t x, int src) {
    const uint32_t lo = __shfl_sync(FULL, (uint32_t)x, src);
    const uint32_t hi = __shfl_sync(FULL, (uint32_t)(x >> 32), src);
    return ((uint64_t)hi << 32) | lo;
}

// Per-lane draw words for power-of-two k (4 <= k <= 256).  Element i of
// tile t is i = 128t + s_e with s_e = 4*lane + e - off in [-3, 127]:
//   k <= 128: lane i mod k = s_e mod k and counter i div k = t*128/k +
//             (s_e >> log2 k), so word_e(t) = W_e + t*(128/k)*GOLDEN;
//   k == 256: lane (128*(t&1) + s_e) mod 256 and counter (t>>1) +
//             ((128*(t&1) + s_e) >> 8), so word_e(t) = W_e[t&1] + (t>>1)*GOLDEN.
// W is stored lane-private as [tau][e>>1][lane][e&1] (u64), read with two
// conflict-free LDS.128 per tile.
__device__ __forceinline__ void stage_words(const WalkArgs &a, const StepCtx &s, uint32_t k,
                                            int lane, uint32_t woff, uint32_t off) {
    uint64_t *W = reinterpret_cast<uint64_t *>(fw_smem + woff + kTabSlots);
    const uint32_t lk = 31 - __clz(k);
    if (k <= 32) {
        const uint64_t b = (uint32_t)lane < k ? lane_base(a, s, lane) : 0;
#pragma unroll
        for (int e = 0; e < 4; e++) {
            const int sidx = 4 * lane + e - (int)off;
            const uint64_t bj = shfl_u64(b, sidx & (int)(k - 1));
            W[((e >> 1) * 32 + lane) * 2 + (e & 1)] =
                bj + (uint64_t)(int64_t)(sidx >> lk) * GOLDEN;
        }
    } else {
        const int ntau = k == 256 ? 2 : 1;
        for (int tau = 0; tau < ntau; tau++) {
#pragma unroll
            for (int e = 0; e < 4; e++) {
                const int sidx = 4 * lane + e - (int)off + 128 * tau;
                W[((tau * 2 + (e >> 1)) * 32 + lane) * 2 + (e & 1)] =
                    lane_base(a, s, (uint32_t)sidx & (k - 1)) +
                    (uint64_t)(int64_t)(sidx >> lk) * GOLDEN;
            }
        }
    }
    __syncwarp();
}

// Node2Vec DPRS, exact order, prev >= 0, power-of-two 4 <= k <= 256 (the
// headline path).  Per 128-element tile: 16-byte loads of targets (one tile
// ahead) and weights, branch-free membership lookups into the N(prev) table,
// a 4-element local prefix plus one warp scan, draw words from the staged
// per-lane table, and the accept test.
// HASHED: the caller has established that N(prev) uses windows (not bsearch).
template <bool F32, bool WEIGHTED, bool HASHED = false, bool ISCAN = false, bool CERT = false>
__device__ uint32_t dprs_n2v_pow2(const WalkArgs &a, const StepCtx &s, uint32_t k, int lane,
                                  uint32_t woff) {
    const uint32_t deg = s.deg;
    const uint32_t prev = (uint32_t)s.prev;
    const uint32_t off = (uint32_t)(s.elo & 3);
    const uint32_t dp = (uint32_t)(s.phi - s.plo);
    const bool use_hash = HASHED || dp <= a.merge_ratio * deg + 2 * kChunk;
    const uint32_t span = deg + off;
    // this lane's 4-slot group of tile 0 (16-byte aligned: the tile grid is
    // anchored at elo & ~3); the weights pointer steps alongside
    const uint32_t *tp = a.tgt + (s.elo - off) + 4 * lane;
    const float *wpt = a.w + (s.elo - off) + 4 * lane;
    // N(prev)'s start lives in the control words (read by the cold paths)
    if (lane == 0) {
        fw_smem[woff + kCtlWord + 4] = (uint32_t)s.plo;
        fw_smem[woff + kCtlWord + 5] = (uint32_t)((uint64_t)s.plo >> 32);
    }
    // tile 0's targets are requested before the table build so the memory
    // round trips of a step's prologue overlap
    uint4 nu = make_uint4(0, 0, 0, 0);
    if ((uint32_t)lane * 4 < span) nu = ldg(reinterpret_cast<const uint4 *>(tp));
    ChunkKeys ck0{};
    if (use_hash) ck0 = chunk_load(a.tgt, s.plo, dp, 0, lane);
    stage_words(a, s, k, lane, woff, off);  // overlaps the loads above
    HashState hs{0, 0, 0};
    if (use_hash) hs = hash_build(ck0, s.plo, dp, 0, woff, lane);
    // counter of tile t: k == 256 -> t >> 1; k <= 128 -> t * (128 / k)
    const uint32_t cmul = k == 256 ? 0 : (128u >> (31 - __clz(k)));
    const uint32_t wq0 = (woff + kTabSlots) * 4 + 16 * lane;  // staged words (bytes)
    double carry = 0.0;
    uint64_t icarry = 0;  // ISCAN: the carry in units of 2^G (exact)
    uint32_t cand = 0;
    [[maybe_unused]] uint32_t amb = 0;  // CERT: last ambiguous element + 1
    const uint32_t ntiles = (span + 127) >> 7;
    for (uint32_t t = 0; t < ntiles; t++, tp += 128, wpt += 128) {
        const uint32_t x0 = t * 128;  // first slot of the tile
        // interior tile: all 128 slots are elements of N(cur)
        const bool edge = x0 < off || x0 + 128 > span;
        const uint4 u4 = nu;
        const uint32_t u[4] = {u4.x, u4.y, u4.z, u4.w};
        const int32_t i0 = (int32_t)(x0 + 4 * lane) - (int32_t)off;
        float wf[4] = {1.f, 1.f, 1.f, 1.f};
        uint32_t valid = 0xF;
        if (edge) {
            if (WEIGHTED && x0 + 4 * lane < span) {
                const float4 w4 = ldg(reinterpret_cast<const float4 *>(wpt));
                wf[0] = w4.x; wf[1] = w4.y; wf[2] = w4.z; wf[3] = w4.w;
            }
#pragma unroll
            for (int e = 0; e < 4; e++) {  // invalid slots weigh 0
                if ((uint32_t)(i0 + e) >= deg) {
                    valid &= ~(1u << e);
                    wf[e] = 0.0f;
                }
            }
        } else if (WEIGHTED) {
            const float4 w4 = ldg(reinterpret_cast<const float4 *>(wpt));
            wf[0] = w4.x; wf[1] = w4.y; wf[2] = w4.z; wf[3] = w4.w;
        }
        if (x0 + 128 < span && x0 + 128 + 4 * lane < span)  // next tile's targets
            nu = ldg(reinterpret_cast<const uint4 *>(tp + 128));
        // membership u in N(prev) and the app weight (_kernels.py:288-306):
        // factor 1/a if u == prev, else 1 if u in N(prev), else 1/b
        uint32_t mem = 0;
        float wp[4];  // F32: factor * w, exact in fp32
        if (use_hash) {
            // lookups for every slot (prev's and invalid slots' results are
            // ignored); the cold path handles valid slots beyond the window
            // and those in a full group whose last key is < u
            uint32_t full = 0;
#pragma unroll
            for (int e = 0; e < 4; e++) {
                const uint4 q = bucket_at(woff, tab_group(u[e], hs));
                const bool hit = bucket_has(q, u[e]);
                if constexpr (F32) {
                    wp[e] = (u[e] == prev ? a.fa32 : (hit ? a.f132 : a.fb32)) * wf[e];
                } else {
                    mem |= (hit ? 1u : 0u) << e;
                }
                full |= (!hit && q.w < u[e] ? 1u : 0u) << e;
            }
            // a valid slot beyond the window: u is sorted within the lane, so
            // in an interior tile u[3] decides
            bool beyond = !edge && u[3] > hs.lim;
            if (edge) {
#pragma unroll
                for (int e = 0; e < 4; e++) beyond |= ((valid >> e) & 1) && u[e] > hs.lim;
            }
            full &= valid;
            if (__any_sync(FULL, full || beyond)) {
                uint32_t pend = 0;
#pragma unroll
                for (int e = 0; e < 4; e++) pend |= (u[e] > hs.lim ? 1u : 0u) << e;
                pend &= valid;
                full &= ~pend;
                const SlowRet sr =
                    member4_slow(a.tgt, woff, u[0], u[1], u[2], u[3], full, pend, hs, lane);
                hs = sr.hs;
                if constexpr (F32) {
#pragma unroll
                    for (int e = 0; e < 4; e++)
                        if (((sr.mem >> e) & 1) && u[e] != prev) wp[e] = a.f132 * wf[e];
                } else {
                    mem |= sr.mem;
                }
            }
        } else {
            mem = member4_bsearch(a.tgt + ctl_plo(woff), dp, u[0], u[1], u[2], u[3], valid);
            if constexpr (F32) {
#pragma unroll
                for (int e = 0; e < 4; e++)
                    wp[e] = (u[e] == prev ? a.fa32 : (((mem >> e) & 1) ? a.f132 : a.fb32)) * wf[e];
            }
        }
        // draw words: staged per-lane words + counter(t) * GOLDEN
        const uint32_t wq = wq0 + (cmul ? 0 : (t & 1) * 1024);
        if constexpr (ISCAN) {
            // Integer tile sums.  Every app weight is an integer multiple of
            // 2^G, so wi = w * 2^-G is exact (the factors fa32/f132/fb32
            // carry the 2^-G, then F2I)
            // and the tile total is two 16-bit-half warp reductions
            // (REDUX); the carry stays an exact u64.  The fp64 prefix scan
            // runs only in tiles where some element passes the prefilter
            // (a scale by a power of two commutes with fp64 rounding, so
            // fl(r * P') < w' in units of 2^G is the reference's test).
            uint32_t wi[4];
            [[maybe_unused]] double wqv[4];  // !F32 (CERT only): exact fp64 products, scaled
#pragma unroll
            for (int e = 0; e < 4; e++) {
                // exact: the factors carry 2^-G and every product is an integer.
                // CERT (sums that round): the products carry a scale 2^s that
                // keeps them < 2^29; wi is the nearest integer, so the integer
                // prefix is within 0.5 per element of the exact one
                // (cert_accept's abs_err) while the tested w stays exact
                if constexpr (F32) {
                    wi[e] = CERT ? __float2uint_rn(wp[e]) : __float2uint_rz(wp[e]);
                } else {
                    const double f = u[e] == prev ? a.inv_a : (((mem >> e) & 1) ? 1.0 : a.inv_b);
                    wqv[e] = __dmul_rn(__dmul_rn(f, (double)wf[e]), a.qscale);  // power of two: exact
                    wi[e] = __double2uint_rn(wqv[e]);
                }
            }
            const uint32_t li = (wi[0] + wi[1]) + (wi[2] + wi[3]);
            uint32_t thr;
            if constexpr (!CERT) {
                thr = accept_thr_raw(a.accept_wmax_s, (float)icarry);
            } else {
                // the quantized carry may overstate the exact one by 0.5 per
                // element (weights rounded up): the prefilter needs a lower
                // bound, carry - 0.5 * (elements before this tile <= x0)
                // (fp32: its rounding is far inside the prefilter's 2^-12 margin)
                const float clb = fmaxf(fmaf(-0.5f, (float)x0, (float)icarry), 0.0f);
                if constexpr (F32)
                    thr = accept_thr_f(fmaxf(fmaxf(wp[0], wp[1]), fmaxf(wp[2], wp[3])), clb);
                else
                    thr = accept_thr_f(
                        __double2float_ru(fmax(fmax(wqv[0], wqv[1]), fmax(wqv[2], wqv[3]))), clb);
            }
            const uint32_t slo = __reduce_add_sync(FULL, li & 0xFFFFu);
            const uint32_t shi = __reduce_add_sync(FULL, li >> 16);
            const uint4 qa = *reinterpret_cast<const uint4 *>(reinterpret_cast<const char *>(fw_smem) + wq);
            const uint4 qb = *reinterpret_cast<const uint4 *>(reinterpret_cast<const char *>(fw_smem) + wq + 512);
            const uint64_t cg = (uint64_t)(cmul ? t * cmul : t >> 1) * GOLDEN;
            const uint64_t wd[4] = {(((uint64_t)qa.y << 32) | qa.x) + cg,
                                    (((uint64_t)qa.w << 32) | qa.z) + cg,
                                    (((uint64_t)qb.y << 32) | qb.x) + cg,
                                    (((uint64_t)qb.w << 32) | qb.z) + cg};
            // invalid slots (wi = 0) may pass; the w > 0 test rejects them
            uint32_t y[4];
#pragma unroll
            for (int e = 0; e < 4; e++) y[e] = mix64_yhi(wd[e]);
            const uint32_t ymin = min(min(y[0], y[1]), min(y[2], y[3]));
            if (__any_sync(FULL, ymin <= thr)) {
                const double l3 = (double)li;
                const double incl = warp_incl_scan_p(l3);
                double run = __dadd_rn((double)icarry, __dadd_rn(incl, -l3));  // exact
                if (ymin <= thr) {
                    [[maybe_unused]] const double tot =
                        (double)(icarry + ((uint64_t)shi << 16) + slo) + 64.0;
#pragma unroll
                    for (int e = 0; e < 4; e++) {
                        run = __dadd_rn(run, (double)wi[e]);
                        if (y[e] <= thr) {
                            const double r = u01_word(wd[e]);
                            if constexpr (CERT) {
                                const double w = F32 ? (double)wp[e] : wqv[e];  // exact, scaled
                                if (w > 0.0) {
                                    const uint32_t ie = (uint32_t)(i0 + e);
                                    const int c_ = cert_accept(r, run, w, tot, ie, a.cert_slack,
                                                               0.5 * (double)(ie + 1));
                                    if (c_ == 1) cand = ie + 1;
                                    else if (c_ == 2) amb = ie + 1;
                                }
                            } else {
                                const double w = (double)wi[e];
                                if (w > 0.0 && __dmul_rn(r, run) < w) cand = (uint32_t)(i0 + e) + 1;
                            }
                        }
                    }
                }
            }
            icarry += ((uint64_t)shi << 16) + slo;
        } else {
            double wv[4];
#pragma unroll
            for (int e = 0; e < 4; e++) {
                if constexpr (F32) {
                    wv[e] = (double)wp[e];
                } else {
                    const double f = u[e] == prev ? a.inv_a : (((mem >> e) & 1) ? 1.0 : a.inv_b);
                    wv[e] = __dmul_rn(f, (double)wf[e]);
                }
            }
            const double p1 = __dadd_rn(wv[0], wv[1]);
            const double p2 = __dadd_rn(p1, wv[2]);
            const double p3 = __dadd_rn(p2, wv[3]);
            // prefilter threshold from the tile's starting carry (<= every
            // lane's base, so the bound below stays valid); it does not wait
            // for the scan
            const uint32_t thr =
                batch_thr<CERT>(a, carry, CERT ? fmax(fmax(wv[0], wv[1]), fmax(wv[2], wv[3])) : 0.0);
            const double incl = warp_incl_scan_p(p3);
            const double base = __dadd_rn(carry, __dadd_rn(incl, -p3));  // exact
            carry = __dadd_rn(carry, shfl_d(incl, 31));
            const uint4 qa = *reinterpret_cast<const uint4 *>(reinterpret_cast<const char *>(fw_smem) + wq);
            const uint4 qb = *reinterpret_cast<const uint4 *>(reinterpret_cast<const char *>(fw_smem) + wq + 512);
            const uint64_t cg = (uint64_t)(cmul ? t * cmul : t >> 1) * GOLDEN;
            const uint64_t wd[4] = {(((uint64_t)qa.y << 32) | qa.x) + cg,
                                    (((uint64_t)qa.w << 32) | qa.z) + cg,
                                    (((uint64_t)qb.y << 32) | qb.x) + cg,
                                    (((uint64_t)qb.w << 32) | qb.z) + cg};
#if FW_PREFILTER
            // Accept prefilter.  Element e is accepted iff w > 0 and fl(r*P) < w
            // with P = base + pre[e] >= carry + w, which implies r < w/(carry + w)
            // <= wmax/(carry + wmax) = T, i.e. hi32(z) <= floor(T*2^32).  hi32(z)
            // differs from hi32(y) (y = the second multiply, before the final
            // xorshift) only in bit 0, so the fast path stops after the second
            // multiply's high word and compares it against thr >= floor(T*2^32)+2
            // (base = 0 -> all pass).  Elements that pass run the exact test.
            uint32_t pass = 0;
#pragma unroll
            for (int e = 0; e < 4; e++) pass |= (mix64_yhi(wd[e]) <= thr ? 1u : 0u) << e;
            if (pass & valid) {
                // P = base + w_0 + ... + w_e, recomputed here (every partial sum
                // is exact, so the association order does not matter) so that
                // only the fp32 products stay live across the draws
                double run = base;
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    const double w = F32 ? (double)wp[e] : wv[e];
                    run = __dadd_rn(run, w);
                    if ((pass >> e) & 1) {
                        const double r = u01_word(wd[e]);
                        if constexpr (CERT) {
                            // carry is already the post-tile total here
                            if (w > 0.0) {
                                const int c_ = cert_accept(r, run, w, carry, (uint32_t)(i0 + e),
                                                           a.cert_slack);
                                if (c_ == 1) cand = (uint32_t)(i0 + e) + 1;
                                else if (c_ == 2) amb = (uint32_t)(i0 + e) + 1;
                            }
                        } else if (w > 0.0 && __dmul_rn(r, run) < w) {
                            cand = (uint32_t)(i0 + e) + 1;
#if FW_PF_NEXT
                            // the candidate may become the next vertex: pull its
                            // CSR offsets toward this SM now (the target itself
                            // was loaded by this tile, L1-resident)
                            asm volatile("prefetch.global.L1 [%0];" ::"l"(a.off + __ldg(tp + e)));
#endif
                        }
                    }
                }
            }
#else
            const double pre[4] = {wv[0], p1, p2, p3};
#pragma unroll
            for (int e = 0; e < 4; e++) {
                const double r = u01_word(wd[e]);
                const double Pr = __dmul_rn(r, __dadd_rn(base, pre[e]));
                if (wv[e] > 0.0 && Pr < wv[e]) {
                    cand = (uint32_t)(i0 + e) + 1;
                }
            }
#endif
        }
    }
    // the selected target is reloaded by the caller (L1/L2-resident): not
    // carrying it frees the u registers before the draws
    const uint32_t sel = __reduce_max_sync(FULL, cand);
    __syncwarp();  // the table and the staged words are rebuilt by the next step
    if constexpr (CERT) {
        if (__reduce_max_sync(FULL, amb) > sel) return kCertFallback;
    }
    return sel;
}

// Node2Vec DPRS, exact order, prev >= 0, any k (lane bases recomputed per
// element; the correctness path for non-power-of-two lane widths).
__device__ uint32_t dprs_n2v_generic(const WalkArgs &a, const StepCtx &s, uint32_t k, int lane,
                                   uint32_t woff, uint32_t &sel_u) {
    const uint32_t deg = s.deg;
    const uint32_t prev = (uint32_t)s.prev;
    const uint32_t off = (uint32_t)(s.elo & 3);
    const uint32_t *P = a.tgt + s.plo;
    const uint32_t dp = (uint32_t)(s.phi - s.plo);
    const bool use_hash = dp <= a.merge_ratio * deg + 2 * kChunk;
    const uint32_t span = deg + off;
    const uint32_t ntiles = (span + 127) >> 7;
    const int64_t ebase = s.elo - off;
    uint4 nu = make_uint4(0, 0, 0, 0);
    if ((uint32_t)lane * 4 < span) nu = ldg(reinterpret_cast<const uint4 *>(a.tgt + ebase) + lane);
    if (lane == 0) {
        fw_smem[woff + kCtlWord + 4] = (uint32_t)s.plo;
        fw_smem[woff + kCtlWord + 5] = (uint32_t)((uint64_t)s.plo >> 32);
    }
    HashState hs{0, 0, 0};
    if (use_hash) hs = hash_build(chunk_load(a.tgt, s.plo, dp, 0, lane), s.plo, dp, 0, woff, lane);
    else __syncwarp();
    double carry = 0.0;
    uint32_t cand = 0, cand_u = 0;
    for (uint32_t t = 0; t < ntiles; t++) {
        const uint32_t x = t * 128 + lane * 4;  // slot of element 0 of this lane
        const uint4 u4 = nu;
        float4 w4 = make_float4(1.f, 1.f, 1.f, 1.f);
        if (x < span) {
            if (a.weighted) w4 = ldg(reinterpret_cast<const float4 *>(a.w + ebase) + (x >> 2));
            if (x + 128 < span)  // prefetch the next tile's targets
                nu = ldg(reinterpret_cast<const uint4 *>(a.tgt + ebase) + ((x + 128) >> 2));
        }
        const int32_t i0 = (int32_t)x - (int32_t)off;
        const uint32_t u[4] = {u4.x, u4.y, u4.z, u4.w};
        uint32_t vmask = 0xFu;
        if (i0 < 0) vmask &= 0xFu << (-i0);
        const int32_t rem = (int32_t)deg - i0;
        if (rem < 4) vmask &= rem <= 0 ? 0u : (1u << rem) - 1;
        uint32_t pmask = 0;
#pragma unroll
        for (int e = 0; e < 4; e++) pmask |= (u[e] == prev ? 1u : 0u) << e;
        uint32_t mem = 0;
        const uint32_t need = vmask & ~pmask;
        if (use_hash) {
            uint32_t here = 0, full = 0;
#pragma unroll
            for (int e = 0; e < 4; e++) {
                if (((need >> e) & 1) && u[e] <= hs.lim) {
                    here |= 1u << e;
                    const uint4 q = bucket_at(woff, tab_group(u[e], hs));
                    if (bucket_has(q, u[e])) mem |= 1u << e;
                    else if (q.w < u[e]) full |= 1u << e;
                }
            }
            const uint32_t pend = need & ~here;
            if (__any_sync(FULL, full | pend)) {
                const SlowRet sr =
                    member4_slow(a.tgt, woff, u[0], u[1], u[2], u[3], full, pend, hs, lane);
                mem |= sr.mem;
                hs = sr.hs;
            }
        } else {
            mem = member4_bsearch(P, dp, u[0], u[1], u[2], u[3], need);
        }
        const float wf[4] = {w4.x, w4.y, w4.z, w4.w};
        double wv[4];
#pragma unroll
        for (int e = 0; e < 4; e++) {
            const float w0 = ((vmask >> e) & 1) ? (a.weighted ? wf[e] : 1.0f) : 0.0f;
            const uint32_t fi = (((pmask >> e) & 1) << 1) | ((mem >> e) & 1);
            wv[e] = __dmul_rn(a.fac[fi], (double)w0);
        }
        const double p1 = __dadd_rn(wv[0], wv[1]);
        const double p2 = __dadd_rn(p1, wv[2]);
        const double p3 = __dadd_rn(p2, wv[3]);
        const double incl = warp_incl_scan_d(p3, lane);
        const double base = __dadd_rn(carry, __dadd_rn(incl, -p3));  // exact
        carry = __dadd_rn(carry, shfl_d(incl, 31));
        const double pre[4] = {wv[0], p1, p2, p3};
#pragma unroll
        for (int e = 0; e < 4; e++) {
            const uint32_t i = (uint32_t)(i0 + e);
            const double r = u01(lane_base(a, s, i % k), (uint64_t)(i / k));
            const double Pr = __dmul_rn(r, __dadd_rn(base, pre[e]));
            if (wv[e] > 0.0 && Pr < wv[e]) {
                cand = i + 1;
                cand_u = u[e];
            }
        }
    }
    const uint32_t sel = __reduce_max_sync(FULL, cand);
    const unsigned who = __ballot_sync(FULL, cand == sel);
    sel_u = __shfl_sync(FULL, cand_u, __ffs(who) - 1);
    __syncwarp();  // the table is rebuilt by the next step
    return sel;
}

template <int APP>
__device__ uint32_t dprs_warp_ordered(const WalkArgs &a, const StepCtx &s, uint32_t k, int lane) {
    const uint32_t deg = s.deg;
    double carry = 0.0, run = 0.0;
    uint32_t cand = 0;
    for (uint32_t t0 = 0; t0 < deg; t0 += 32) {
        const uint32_t i = t0 + lane;
        const double wv = i < deg ? elem_weight<APP>(a, s, i) : 0.0;
        double P = 0.0;
        const uint32_t tn = deg - t0 < 32 ? deg - t0 : 32;
#pragma unroll 1
        for (uint32_t t = 0; t < tn; t++) {
            const uint32_t it = t0 + t;
            if (it > 0 && it % k == 0) {  // chunk boundary: carry += run (_kernels.py:429)
                carry = __dadd_rn(carry, run);
                run = 0.0;
            }
            run = __dadd_rn(run, __shfl_sync(FULL, wv, t));
            if ((uint32_t)lane == t) P = __dadd_rn(run, carry);  // lane_prefix[j] + carry (:421)
        }
        if (wv > 0.0) {
            const double r = u01(lane_base(a, s, i % k), (uint64_t)(i / k));
            if (__dmul_rn(r, P) < wv) cand = i + 1;
        }
    }
    return __reduce_max_sync(FULL, cand);
}

__device__ __forceinline__ void stat_add(unsigned long long *st, int idx, long long v, int lane) {
    if (lane == 0) st[idx] += (unsigned long long)v;
}

// ---------------------------------------------------------------------------
// The persistent walker.
// ---------------------------------------------------------------------------
// MODE: 0 = the reference's summation order replayed (ordered kernels),
// 1 = exact (every partial sum exact: tree scans), 2 = certified (tree scans
// with certified accept tests, ambiguous steps re-run in order).
template <int APP, int SAMPLER, int MODE>
__global__ void __launch_bounds__(kWalkThreads, walk_min_blocks(APP))
walk_kernel(const __grid_constant__ WalkArgs a) {
    constexpr bool EXACT = MODE >= 1;
    constexpr bool CERT = MODE == 2;
    const int lane = threadIdx.x & 31;
    const uint32_t woff = (threadIdx.x >> 5) * warp_words(APP);
    // per-warp RunStats counters live in shared memory (registers are the
    // scarce resource in the sampler loops); every lane keeps the same value
    // in flight, lane 0 owns the slot.
    unsigned long long *st = reinterpret_cast<unsigned long long *>(fw_smem + woff + stats_word(APP));
    if (lane < ST_COUNT) st[lane] = 0;
    __syncwarp();

    for (;;) {
        unsigned long long qi = 0;
        if (lane == 0) qi = atomicAdd(a.queue, 1ULL);
        qi = __shfl_sync(FULL, qi, 0);
        if (qi >= a.n) break;
        const uint64_t q = a.base_qid + qi;
        uint32_t *row = a.out_seq + qi * (uint64_t)a.L;
        StepCtx s;
        int64_t cur = ldg(a.starts + qi);
        s.prev = -1;
        int64_t pdeg = 0, pelo = 0;
        uint32_t emitted = 0;
        uint32_t pathbuf = 0xFFFFFFFFu;  // lane (t & 31) holds step t of the open 32-block
        for (;;) {
            s.elo = ldg(a.off + cur);
            s.deg = (uint32_t)(ldg(a.off + cur + 1) - s.elo);
            const bool small = (int64_t)s.deg <= a.d_t;
            const uint32_t k = (uint32_t)(small ? a.k_small : a.k_big);
            stat_add(st, ST_SMALL, small ? 1 : 0, lane);
            stat_add(st, ST_LARGE, small ? 0 : 1, lane);
            stat_add(st, ST_STEPS, 1, lane);
            stat_add(st, ST_BYTES, 16, lane);
            const uint64_t step = emitted;
            s.A = (TAG_REPLAY | (q << 30) | (step << 10)) * MIX1;
            if constexpr (APP == APP_PPR) {
                const double r = u01(mix64(a.h ^ (s.A + STOP_LANE * MIX1)), 0);
                stat_add(st, ST_DRAWS, 1, lane);
                if (r < a.stop_prob) break;
            }
            if (s.deg == 0) break;
            if constexpr (APP == APP_METAPATH) {
                if (step >= a.schema_len) break;
                s.want = a.schema ? ldg(a.schema + step) : a.schema_inline[step];
            }
            if constexpr (APP == APP_NODE2VEC) {
                if (s.prev >= 0) {  // N(prev) = the previous step's N(cur)
                    s.plo = pelo;
                    s.phi = pelo + pdeg;
                    stat_add(st, ST_BYTES, 16 + 4 * pdeg, lane);
                }
            }
            const uint32_t chunks = (s.deg - 1) / k + 1;
            uint32_t sel;
            uint32_t sel_u = 0;
            bool have_u = false;
            if constexpr (SAMPLER == SAMPLER_DPRS) {
                if constexpr (CERT) {
                    // sums that round: non-dyadic weights, or factors 1/a, 1/b
                    // that are not powers of two (weighted or not)
                    if (APP == APP_NODE2VEC && s.prev >= 0) {
                        if (k >= 4 && k <= 256 && (k & (k - 1)) == 0) {
                            const bool win = (uint32_t)(s.phi - s.plo) <=
                                             a.merge_ratio * s.deg + 2 * kChunk;
                            if (a.weighted && a.iscan)  // quantized integer tile sums
                                sel = !a.fac32 ? dprs_n2v_pow2<false, true, false, true, true>(a, s, k, lane, woff)
                                      : win    ? dprs_n2v_pow2<true, true, true, true, true>(a, s, k, lane, woff)
                                               : dprs_n2v_pow2<true, true, false, true, true>(a, s, k, lane, woff);
                            else if (a.weighted)
                                sel = a.fac32 ? (win ? dprs_n2v_pow2<true, true, true, false, true>(a, s, k, lane, woff)
                                                     : dprs_n2v_pow2<true, true, false, false, true>(a, s, k, lane, woff))
                                              : dprs_n2v_pow2<false, true, false, false, true>(a, s, k, lane, woff);
                            else
                                sel = a.fac32 ? dprs_n2v_pow2<true, false, false, false, true>(a, s, k, lane, woff)
                                              : dprs_n2v_pow2<false, false, false, false, true>(a, s, k, lane, woff);
                        } else {
                            sel = kCertFallback;
                        }
                    } else {
                        sel = dprs_warp_exact<APP, true>(a, s, k, lane);
                    }
                    if (sel == kCertFallback) sel = dprs_warp_ordered<APP>(a, s, k, lane);
                } else if constexpr (EXACT && APP == APP_NODE2VEC) {
                    if (s.prev >= 0) {
                        if (k >= 4 && k <= 256 && (k & (k - 1)) == 0) {
                            const bool win = (uint32_t)(s.phi - s.plo) <=
                                             a.merge_ratio * s.deg + 2 * kChunk;
                            if (a.weighted)
                                sel = a.iscan ? (win ? dprs_n2v_pow2<true, true, true, true>(a, s, k, lane, woff)
                                                     : dprs_n2v_pow2<true, true, false, true>(a, s, k, lane, woff))
                                      : a.fac32 ? (win ? dprs_n2v_pow2<true, true, true>(a, s, k, lane, woff)
                                                       : dprs_n2v_pow2<true, true>(a, s, k, lane, woff))
                                                : dprs_n2v_pow2<false, true>(a, s, k, lane, woff);
                            else
                                sel = a.iscan ? dprs_n2v_pow2<true, false, false, true>(a, s, k, lane, woff)
                                      : a.fac32 ? dprs_n2v_pow2<true, false>(a, s, k, lane, woff)
                                                : dprs_n2v_pow2<false, false>(a, s, k, lane, woff);
                        } else {
                            sel = dprs_n2v_generic(a, s, k, lane, woff, sel_u);
                            have_u = true;
                        }
                    } else {
                        sel = dprs_warp_exact<APP>(a, s, k, lane);
                    }
                } else if constexpr (EXACT) {
                    sel = dprs_warp_exact<APP>(a, s, k, lane);
                } else {
                    sel = dprs_warp_ordered<APP>(a, s, k, lane);
                }
                stat_add(st, ST_COLLECTIVES, 2 * chunks, lane);
                stat_add(st, ST_EDGES, s.deg, lane);
            } else {
                // compile-time lane widths (immediate load offsets): +11-13%
                // for DeepWalk / PPR; MetaPath measured 14% slower with them
                if constexpr (CERT) {
                    // certified: tree lane scan; an ambiguous step re-runs
                    // with the reference's sequential lane scan
                    if constexpr (APP == APP_METAPATH) {
                        sel = zprs_warp<APP, true, 0, true>(a, s, k, lane, woff);
                        if (sel == kCertFallback) sel = zprs_warp<APP, false>(a, s, k, lane, woff);
                    } else {
                        sel = k == 32    ? zprs_warp<APP, true, 32, true>(a, s, k, lane, woff)
                              : k == 256 ? zprs_warp<APP, true, 256, true>(a, s, k, lane, woff)
                                         : zprs_warp<APP, true, 0, true>(a, s, k, lane, woff);
                        if (sel == kCertFallback) sel = zprs_warp<APP, false>(a, s, k, lane, woff);
                    }
                } else if constexpr (APP == APP_METAPATH)
                    sel = zprs_warp<APP, EXACT>(a, s, k, lane, woff);
                else
                    sel = k == 32    ? zprs_warp<APP, EXACT, 32>(a, s, k, lane, woff)
                          : k == 256 ? zprs_warp<APP, EXACT, 256>(a, s, k, lane, woff)
                                     : zprs_warp<APP, EXACT>(a, s, k, lane, woff);
                stat_add(st, ST_COLLECTIVES, 2, lane);
                stat_add(st, ST_EDGES, 2 * s.deg, lane);
            }
            stat_add(st, ST_DRAWS, (long long)chunks * k, lane);
            stat_add(st, ST_BYTES, (APP == APP_METAPATH ? 9 : 8) * s.deg, lane);
            if (sel == 0) break;
            const uint32_t u = have_u ? sel_u : ldg(a.tgt + s.elo + sel - 1);
            if (lane == (int)(step & 31)) pathbuf = u;
            emitted = (uint32_t)step + 1;
            stat_add(st, ST_BYTES, 4, lane);
            s.prev = cur;
            pdeg = s.deg;
            pelo = s.elo;
            cur = (int64_t)u;
            if ((emitted & 31) == 0) {
                row[emitted - 32 + lane] = pathbuf;
                pathbuf = 0xFFFFFFFFu;
            }
            if (emitted >= a.L) break;
            if constexpr (APP == APP_METAPATH) {
                if (emitted >= a.schema_len) break;
            }
        }
        // flush the open block, then sentinel-fill the tail (engine.py:299-300)
        for (uint64_t b0 = emitted & ~31u; b0 < a.L; b0 += 32) {
            if (b0 + lane < a.L) row[b0 + lane] = pathbuf;
            pathbuf = 0xFFFFFFFFu;
        }
        if (lane == 0) a.out_len[qi] = emitted;
        if (a.done) {  // publish the finished row for the overlapped D2H
            __threadfence();  // gpu scope: the copy engine reads through L2
            __syncwarp();
            if (lane == 0) atomicAdd(a.done + qi / a.piece_q, 1u);
        }
        stat_add(st, ST_SAMPLED, emitted, lane);
    }
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < ST_COUNT; i++)
            if (st[i]) atomicAdd((unsigned long long *)(a.stats + i), st[i]);
        unsigned long long now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        atomicMax((unsigned long long *)(a.stats + ST_T_LAST), now);
        atomicMax((unsigned long long *)(a.stats + ST_T_FIRST_NEG), ~now);
    }
}

template <int APP, int SAMPLER, int MODE>
static cudaError_t launch_t(const WalkArgs &a, int grid, cudaStream_t stream) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(walk_kernel<APP, SAMPLER, MODE>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, walk_smem_bytes(APP));
        attr = true;
    }
    walk_kernel<APP, SAMPLER, MODE><<<grid, kWalkThreads, walk_smem_bytes(APP), stream>>>(a);
    return cudaGetLastError();
}

template <int APP, int SAMPLER, int MODE>
static int occupancy_t() {
    // per kernel and process (the same on every B200; queried once, not per launch)
    static const int nb = [] {
        int b = 0;
        cudaFuncSetAttribute(walk_kernel<APP, SAMPLER, MODE>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, walk_smem_bytes(APP));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, walk_kernel<APP, SAMPLER, MODE>,
                                                      kWalkThreads, walk_smem_bytes(APP));
        return b;
    }();
    return nb;
}

#define FW_DISPATCH_APP(FN, APP, ...)                                                \
    if (sampler == SAMPLER_ZPRS) {                                                   \
        if (mode == 0) return FN<APP, 0, 0>(__VA_ARGS__);                            \
        if (mode == 1) return FN<APP, 0, 1>(__VA_ARGS__);                            \
        return FN<APP, 0, 2>(__VA_ARGS__);                                           \
    }                                                                                \
    if (mode == 0) return FN<APP, 1, 0>(__VA_ARGS__);                                \
    if (mode == 1) return FN<APP, 1, 1>(__VA_ARGS__);                                \
    return FN<APP, 1, 2>(__VA_ARGS__);

#define FW_DISPATCH(FN, ...)                                                         \
    switch (app) {                                                                   \
    case 0: { FW_DISPATCH_APP(FN, 0, __VA_ARGS__) }                                  \
    case 1: { FW_DISPATCH_APP(FN, 1, __VA_ARGS__) }                                  \
    case 2: { FW_DISPATCH_APP(FN, 2, __VA_ARGS__) }                                  \
    default: { FW_DISPATCH_APP(FN, 3, __VA_ARGS__) }                                 \
    }

cudaError_t launch_walk(const WalkArgs &a, int app, int sampler, int mode, int grid,
                        cudaStream_t stream) {
    FW_DISPATCH(launch_t, a, grid, stream)
}

int walk_occupancy(int app, int sampler, int mode) { FW_DISPATCH(occupancy_t) }

}  // namespace fw
