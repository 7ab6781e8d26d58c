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
#include <cstdint>

#include "fw_common.cuh"
#include "fw_walk.cuh"

namespace fw {

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
template <int APP>
__device__ __forceinline__ double elem_weight(const WalkArgs &a, const StepCtx &s, uint32_t i) {
    const int64_t e = s.elo + i;
    if constexpr (APP == APP_METAPATH) {
        const int64_t lab = a.lab ? (int64_t)ldg(a.lab + e) : 0;
        if (lab != s.want) return 0.0;
        return a.weighted ? (double)ldg(a.w + e) : 1.0;
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

__device__ __forceinline__ uint64_t lane_base(const WalkArgs &a, const StepCtx &s, uint32_t j) {
    return mix64(a.h ^ (s.A + (uint64_t)j * MIX1));
}

// ---------------------------------------------------------------------------
// ZPRS (samplers.py:188-220): logical lanes are processed in groups of 32,
// physical lane p of group g owning logical lane j = 32g + p.  Pass 1 sums
// lane j's strided slice in chunk order (the reference's order), the lane
// sums are exclusive-scanned in lane order (sequentially unless EXACT), and
// pass 2 runs lane j's reservoir.  The winner is the highest logical lane
// holding a candidate (_kernels.py:459-462), so later groups override.
// ---------------------------------------------------------------------------
template <int APP, bool EXACT>
__device__ uint32_t zprs_warp(const WalkArgs &a, const StepCtx &s, uint32_t k, int lane) {
    const uint32_t deg = s.deg;
    const uint32_t nl = k < deg ? k : deg;
    double ecarry = 0.0;
    uint32_t best = 0;
    for (uint32_t g0 = 0; g0 < nl; g0 += 32) {
        const uint32_t j = g0 + lane;
        const bool act = j < nl;
        double lsum = 0.0;
        if (act) {
#pragma unroll 4
            for (uint32_t i = j; i < deg; i += k) lsum = __dadd_rn(lsum, elem_weight<APP>(a, s, i));
        }
        double excl;
        if constexpr (EXACT) {
            const double incl = warp_incl_scan(lsum, lane);
            double up = __shfl_up_sync(FULL, incl, 1);
            excl = __dadd_rn(ecarry, lane == 0 ? 0.0 : up);
            ecarry = __dadd_rn(ecarry, __shfl_sync(FULL, incl, 31));
        } else {
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
        uint32_t cand = 0;
        if (act) {
            double run = excl;
            uint64_t word = lane_base(a, s, j);
#pragma unroll 4
            for (uint32_t i = j; i < deg; i += k, word += GOLDEN) {
                const double wv = elem_weight<APP>(a, s, i);
                run = __dadd_rn(run, wv);
                const double r = u01_word(word);
                if (wv > 0.0 && __dmul_rn(r, run) < wv) cand = i + 1;
            }
        }
        const unsigned m = __ballot_sync(FULL, cand > 0);
        const int src = m ? 31 - __clz(m) : 0;
        const uint32_t c = __shfl_sync(FULL, cand, src);
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
template <int APP>
__device__ uint32_t dprs_warp_exact(const WalkArgs &a, const StepCtx &s, uint32_t k, int lane) {
    const uint32_t deg = s.deg;
    double carry = 0.0;
    uint32_t cand = 0;
    if (k == 32) {
        uint64_t word = lane_base(a, s, lane);
#pragma unroll 2
        for (uint32_t t0 = 0; t0 < deg; t0 += 32, word += GOLDEN) {
            const uint32_t i = t0 + lane;
            const double wv = i < deg ? elem_weight<APP>(a, s, i) : 0.0;
            const double incl = warp_incl_scan(wv, lane);
            const double P = __dadd_rn(carry, incl);
            const double r = u01_word(word);
            if (wv > 0.0 && __dmul_rn(r, P) < wv) cand = i + 1;
            carry = __dadd_rn(carry, __shfl_sync(FULL, incl, 31));
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
                    const double incl = warp_incl_scan(wv, lane);
                    const double P = __dadd_rn(carry, incl);
                    const double r = u01_word(base[q] + cadd);
                    if (wv > 0.0 && __dmul_rn(r, P) < wv) cand = i + 1;
                    carry = __dadd_rn(carry, __shfl_sync(FULL, incl, 31));
                }
            }
        }
    } else {
        for (uint32_t t0 = 0; t0 < deg; t0 += 32) {
            const uint32_t i = t0 + lane;
            const double wv = i < deg ? elem_weight<APP>(a, s, i) : 0.0;
            const double incl = warp_incl_scan(wv, lane);
            const double P = __dadd_rn(carry, incl);
            if (wv > 0.0) {
                const double r = u01(lane_base(a, s, i % k), (uint64_t)(i / k));
                if (__dmul_rn(r, P) < wv) cand = i + 1;
            }
            carry = __dadd_rn(carry, __shfl_sync(FULL, incl, 31));
        }
    }
    return __reduce_max_sync(FULL, cand);
}

// ---------------------------------------------------------------------------
// Node2Vec DPRS, exact order, prev >= 0: the hot path of the headline config.
// Membership of u = targets[elo+i] in N(prev) (_kernels.py:288-306) is
// decided by a warp merge: N(cur) is sorted, so tile after tile the lanes'
// u values only increase; a 32-entry window of N(prev) lives in registers
// (lane j holds P[wpos+j]) and each lane runs a 5-step lower_bound over it
// with shuffles.  The window only moves forward, so a step reads N(prev)
// once, coalesced (4*d_prev bytes, the algorithmic count) instead of
// d_cur*log2(d_prev) dependent probes.  When d_prev >> d_cur the merge would
// stream far more of N(prev) than the probes touch, so the per-lane binary
// search is kept (s.merge == false).  The selected target is carried with
// the candidate, so no dependent reload of targets[elo+sel-1] is needed.
// ---------------------------------------------------------------------------
struct N2VWin {
    const uint32_t *P;  // N(prev)
    uint32_t dp;        // d(prev)
    uint32_t wpos;      // window start
    uint32_t pw;        // this lane's window entry (0xFFFFFFFF past the end)
    bool wend;          // window covers the end of N(prev)
    bool merge;
};

__device__ __forceinline__ bool n2v_member(const WalkArgs &a, const StepCtx &s, N2VWin &W,
                                           uint32_t u, bool need, int lane) {
    if (!W.merge) return need && in_sorted(a.tgt, s.plo, s.phi, u);
    bool res = !need, mem = false;
    for (;;) {
        const uint32_t wmax = __shfl_sync(FULL, W.pw, 31);
        const bool here = !res && (u <= wmax || W.wend);
        int pos = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
            const uint32_t v = __shfl_sync(FULL, W.pw, pos + step - 1);
            if (v < u) pos += step;
        }
        const uint32_t v = __shfl_sync(FULL, W.pw, pos);
        if (here) {
            mem = v == u;
            res = true;
        }
        if (__all_sync(FULL, res)) break;
        W.wpos += 32;
        W.pw = W.wpos + lane < W.dp ? ldg(W.P + W.wpos + lane) : 0xFFFFFFFFu;
        W.wend = W.wpos + 32 >= W.dp;
    }
    return mem;
}

template <int KMODE>  // 1: k == 32, 2: k == 256, 0: any k
__device__ uint32_t dprs_n2v_exact(const WalkArgs &a, const StepCtx &s, uint32_t k, int lane,
                                   uint32_t &sel_u) {
    // Tiles of 32 elements in natural order; the targets/weights of the next
    // kPf tiles are in flight while a tile is processed (the step is
    // latency-bound without it: one DRAM round trip per tile).
    constexpr int kPf = 8;  // == tiles per k=256 chunk, so tile % 8 is static
    const uint32_t deg = s.deg;
    const uint32_t ntiles = (deg + 31) >> 5;
    N2VWin W;
    W.P = a.tgt + s.plo;
    W.dp = (uint32_t)(s.phi - s.plo);
    W.merge = W.dp <= a.merge_ratio * deg + 32;
    W.wpos = 0;
    W.pw = (W.merge && (uint32_t)lane < W.dp) ? ldg(W.P + lane) : 0xFFFFFFFFu;
    W.wend = W.dp <= 32;
    const uint32_t prev = (uint32_t)s.prev;
    const uint32_t *tg = a.tgt + s.elo;
    const float *wt = a.w + s.elo;
    uint32_t pu[kPf];
    float pf[kPf];
#pragma unroll
    for (int d = 0; d < kPf; d++) {
        const uint32_t i = d * 32 + lane;
        pu[d] = i < deg ? ldg(tg + i) : 0xFFFFFFFFu;
        pf[d] = (i < deg && a.weighted) ? ldg(wt + i) : 1.0f;
    }
    double carry = 0.0;
    uint32_t cand = 0, cand_u = 0;
    uint64_t base[KMODE == 2 ? 8 : 1];
    if constexpr (KMODE == 1) base[0] = lane_base(a, s, lane);
    if constexpr (KMODE == 2) {
#pragma unroll
        for (int q = 0; q < 8; q++) base[q] = lane_base(a, s, q * 32 + lane);
    }
    for (uint32_t g = 0; g < ntiles; g += kPf) {
#pragma unroll
        for (int d = 0; d < kPf; d++) {
            const uint32_t t = g + d;
            if (t < ntiles) {  // warp-uniform
                const uint32_t i = t * 32 + lane;
                const bool valid = i < deg;
                const uint32_t u = pu[d];
                const float wf = pf[d];
                {  // refill this slot with tile t + kPf
                    const uint32_t i2 = i + kPf * 32;
                    pu[d] = i2 < deg ? ldg(tg + i2) : 0xFFFFFFFFu;
                    pf[d] = (i2 < deg && a.weighted) ? ldg(wt + i2) : 1.0f;
                }
                const bool isprev = valid && u == prev;
                const bool mem = n2v_member(a, s, W, u, valid && !isprev, lane);
                const double bse = isprev ? a.inv_a : (mem ? 1.0 : a.inv_b);
                const double wv = valid ? (a.weighted ? __dmul_rn(bse, (double)wf) : bse) : 0.0;
                const double incl = warp_incl_scan(wv, lane);
                const double P = __dadd_rn(carry, incl);
                double r;
                if constexpr (KMODE == 1) r = u01_word(base[0] + (uint64_t)t * GOLDEN);
                else if constexpr (KMODE == 2) r = u01_word(base[d] + (uint64_t)(t >> 3) * GOLDEN);
                else r = u01(lane_base(a, s, i % k), (uint64_t)(i / k));
                if (wv > 0.0 && __dmul_rn(r, P) < wv) {
                    cand = i + 1;
                    cand_u = u;
                }
                carry = __dadd_rn(carry, __shfl_sync(FULL, incl, 31));
            }
        }
    }
    const uint32_t sel = __reduce_max_sync(FULL, cand);
    const unsigned who = __ballot_sync(FULL, cand == sel);
    sel_u = __shfl_sync(FULL, cand_u, __ffs(who) - 1);
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

// ---------------------------------------------------------------------------
// The persistent walker.
// ---------------------------------------------------------------------------
template <int APP, int SAMPLER, bool EXACT>
__global__ void __launch_bounds__(kWalkThreads, kWalkMinBlocks)
walk_kernel(const WalkArgs a) {
    const int lane = threadIdx.x & 31;
    long long st[ST_COUNT];
#pragma unroll
    for (int i = 0; i < ST_COUNT; i++) st[i] = 0;

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
        int64_t pdeg = 0;
        uint32_t emitted = 0;
        uint32_t pathbuf = 0xFFFFFFFFu;  // lane (t & 31) holds step t of the open 32-block
        for (;;) {
            s.elo = ldg(a.off + cur);
            s.deg = (uint32_t)(ldg(a.off + cur + 1) - s.elo);
            const bool small = (int64_t)s.deg <= a.d_t;
            const uint32_t k = (uint32_t)(small ? a.k_small : a.k_big);
            st[ST_SMALL] += small ? 1 : 0;
            st[ST_LARGE] += small ? 0 : 1;
            st[ST_STEPS] += 1;
            st[ST_BYTES] += 16;
            const uint64_t step = emitted;
            s.A = (TAG_REPLAY | (q << 30) | (step << 10)) * MIX1;
            if constexpr (APP == APP_PPR) {
                const double r = u01(mix64(a.h ^ (s.A + STOP_LANE * MIX1)), 0);
                st[ST_DRAWS] += 1;
                if (r < a.stop_prob) break;
            }
            if (s.deg == 0) break;
            if constexpr (APP == APP_METAPATH) {
                if (step >= a.schema_len) break;
                s.want = ldg(a.schema + step);
            }
            if constexpr (APP == APP_NODE2VEC) {
                if (s.prev >= 0) {
                    s.plo = ldg(a.off + s.prev);
                    s.phi = ldg(a.off + s.prev + 1);
                    st[ST_BYTES] += 16 + 4 * pdeg;
                }
            }
            const uint32_t chunks = (s.deg - 1) / k + 1;
            uint32_t sel;
            uint32_t sel_u = 0;
            bool have_u = false;
            if constexpr (SAMPLER == SAMPLER_DPRS) {
                if constexpr (EXACT && APP == APP_NODE2VEC) {
                    if (s.prev >= 0) {
                        if (k == 32) sel = dprs_n2v_exact<1>(a, s, k, lane, sel_u);
                        else if (k == 256) sel = dprs_n2v_exact<2>(a, s, k, lane, sel_u);
                        else sel = dprs_n2v_exact<0>(a, s, k, lane, sel_u);
                        have_u = true;
                    } else {
                        sel = dprs_warp_exact<APP>(a, s, k, lane);
                    }
                } else if constexpr (EXACT) {
                    sel = dprs_warp_exact<APP>(a, s, k, lane);
                } else {
                    sel = dprs_warp_ordered<APP>(a, s, k, lane);
                }
                st[ST_COLLECTIVES] += 2 * chunks;
                st[ST_EDGES] += s.deg;
            } else {
                sel = zprs_warp<APP, EXACT>(a, s, k, lane);
                st[ST_COLLECTIVES] += 2;
                st[ST_EDGES] += 2 * s.deg;
            }
            st[ST_DRAWS] += (long long)chunks * k;
            st[ST_BYTES] += (APP == APP_METAPATH ? 9 : 8) * s.deg;
            if (sel == 0) break;
            const uint32_t u = have_u ? sel_u : ldg(a.tgt + s.elo + sel - 1);
            if (lane == (int)(step & 31)) pathbuf = u;
            emitted = (uint32_t)step + 1;
            st[ST_BYTES] += 4;
            s.prev = cur;
            pdeg = s.deg;
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
        st[ST_SAMPLED] += emitted;
    }
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < ST_COUNT; i++)
            if (st[i]) atomicAdd((unsigned long long *)(a.stats + i), (unsigned long long)st[i]);
    }
}

template <int APP, int SAMPLER, bool EXACT>
static cudaError_t launch_t(const WalkArgs &a, int grid, cudaStream_t stream) {
    walk_kernel<APP, SAMPLER, EXACT><<<grid, kWalkThreads, 0, stream>>>(a);
    return cudaGetLastError();
}

template <int APP, int SAMPLER, bool EXACT>
static int occupancy_t() {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, walk_kernel<APP, SAMPLER, EXACT>,
                                                  kWalkThreads, 0);
    return nb;
}

#define FW_DISPATCH(FN, ...)                                                         \
    switch (app * 4 + sampler * 2 + (exact ? 1 : 0)) {                               \
    case 0: return FN<0, 0, false>(__VA_ARGS__);                                     \
    case 1: return FN<0, 0, true>(__VA_ARGS__);                                      \
    case 2: return FN<0, 1, false>(__VA_ARGS__);                                     \
    case 3: return FN<0, 1, true>(__VA_ARGS__);                                      \
    case 4: return FN<1, 0, false>(__VA_ARGS__);                                     \
    case 5: return FN<1, 0, true>(__VA_ARGS__);                                      \
    case 6: return FN<1, 1, false>(__VA_ARGS__);                                     \
    case 7: return FN<1, 1, true>(__VA_ARGS__);                                      \
    case 8: return FN<2, 0, false>(__VA_ARGS__);                                     \
    case 9: return FN<2, 0, true>(__VA_ARGS__);                                      \
    case 10: return FN<2, 1, false>(__VA_ARGS__);                                    \
    case 11: return FN<2, 1, true>(__VA_ARGS__);                                     \
    case 12: return FN<3, 0, false>(__VA_ARGS__);                                    \
    case 13: return FN<3, 0, true>(__VA_ARGS__);                                     \
    case 14: return FN<3, 1, false>(__VA_ARGS__);                                    \
    default: return FN<3, 1, true>(__VA_ARGS__);                                     \
    }

cudaError_t launch_walk(const WalkArgs &a, int app, int sampler, bool exact, int grid,
                        cudaStream_t stream) {
    FW_DISPATCH(launch_t, a, grid, stream)
}

int walk_occupancy(int app, int sampler, bool exact) { FW_DISPATCH(occupancy_t) }

}  // namespace fw
