// ---------------------------------------------------------------------------
// Node2Vec DPRS with membership by reverse search (integer tile sums, fp32
// factors, power-of-two k): used when d(prev) is small against d(cur).
//
// _edge_weight (_kernels.py:288-306) asks, for every u in N(cur), whether
// u == prev or u in N(prev).  Both lists are sorted, so the same answer comes
// from the other side: every key p of N(prev) is located in N(cur) by a
// lower-bound search, and the run of positions [A, E) holding p (duplicates
// are consecutive; E by galloping) is recorded as two toggles in a bitmap
// over N(cur)'s slots in the warp's shared memory (the table region,
// kTabSlots words = 47104 slots per segment; longer N(cur) runs in segments,
// each searching only the N(prev) keys inside its value range).  Runs of
// distinct keys are disjoint, so a slot is a member iff an odd number of
// toggles lie at or before it: per tile, a lane's 4 toggle bits give its
// local prefix parity and one ballot gives the carry from lower lanes.
// prev's own positions [pr_lo, pr_hi) come from the same search (one extra
// key).  The tile loop then needs no targets and no lookups.  Cost: about
// d(prev) * log2(d(cur)) probes per step instead of a lookup per element, so
// it pays when d(prev) << d(cur).
// ---------------------------------------------------------------------------
constexpr uint32_t kSegSlots = kTabSlots * 32;
static_assert(kSegSlots % 128 == 0, "segments hold whole tiles");

// First index in T[0, n) with T[idx] >= p (n >= 1): branchless.
__device__ __forceinline__ uint32_t lower_bound1(const uint32_t *__restrict__ T, uint32_t n,
                                                 uint32_t p) {
    uint32_t b = 0;
    while (n > 1) {
        const uint32_t half = n >> 1;
        b = ldg(T + b + half - 1) < p ? b + half : b;
        n -= half;
    }
    return b + (ldg(T + b) < p ? 1u : 0u);
}

// One search round over G keys per lane: key slot j = j0 + 32 g + lane
// (j < nk); slots below nreal are N(prev) keys P[j], slot nreal is prev.
// Members toggle their run ends in the bitmap; the prev slot returns its
// run [A, E) in pa/pe (segment-relative element indices).
template <int G>
__device__ __forceinline__ void rev_round(const uint32_t *__restrict__ Ts, uint32_t n,
                                          const uint32_t *__restrict__ P, uint32_t j0,
                                          uint32_t nreal, uint32_t nk, uint32_t prev,
                                          uint32_t *bm, uint32_t bit0, int lane, uint32_t &pa,
                                          uint32_t &pe) {
    uint32_t p[G], b[G];
#pragma unroll
    for (int g = 0; g < G; g++) {
        const uint32_t j = j0 + 32 * g + lane;
        p[g] = j < nreal ? ldg(P + j) : prev;
        b[g] = 0;
    }
    uint32_t m = n;
    while (m > 1) {
        const uint32_t half = m >> 1;
#pragma unroll
        for (int g = 0; g < G; g++) b[g] = ldg(Ts + b[g] + half - 1) < p[g] ? b[g] + half : b[g];
        m -= half;
    }
    // A = lower bound; hit iff T[A] == p.  E (first index past the run) by
    // galloping from A then bisection, in warp-uniform loops.
    uint32_t lo[G], hi[G], step[G], go = 0, bis = 0;
#pragma unroll
    for (int g = 0; g < G; g++) {
        const uint32_t j = j0 + 32 * g + lane;
        const uint32_t A = b[g] + (ldg(Ts + b[g]) < p[g] ? 1u : 0u);
        const bool hit = j < nk && A < n && ldg(Ts + min(A, n - 1)) == p[g];
        b[g] = A;
        lo[g] = A;   // T[lo] == p
        hi[g] = A + 1;  // probe
        step[g] = 1;
        go |= (hit ? 1u : 0u) << g;
    }
    const uint32_t found = go;
    while (__any_sync(FULL, go)) {
#pragma unroll
        for (int g = 0; g < G; g++) {
            if ((go >> g) & 1) {
                if (hi[g] >= n) {
                    hi[g] = n;
                    go &= ~(1u << g);
                } else if (ldg(Ts + hi[g]) != p[g]) {
                    go &= ~(1u << g);
                } else {
                    lo[g] = hi[g];
                    step[g] <<= 1;
                    hi[g] = lo[g] + step[g];
                }
            }
        }
    }
#pragma unroll
    for (int g = 0; g < G; g++) bis |= (((found >> g) & 1) && hi[g] - lo[g] > 1 ? 1u : 0u) << g;
    while (__any_sync(FULL, bis)) {  // T[lo] == p, T[hi] != p (or hi == n)
#pragma unroll
        for (int g = 0; g < G; g++) {
            if ((bis >> g) & 1) {
                const uint32_t mid = (lo[g] + hi[g]) >> 1;
                if (ldg(Ts + mid) == p[g]) lo[g] = mid;
                else hi[g] = mid;
                if (hi[g] - lo[g] <= 1) bis &= ~(1u << g);
            }
        }
    }
#pragma unroll
    for (int g = 0; g < G; g++) {
        if ((found >> g) & 1) {
            const uint32_t j = j0 + 32 * g + lane;
            if (j < nreal) {
                const uint32_t ba = bit0 + b[g], be = bit0 + hi[g];
                atomicXor(bm + (ba >> 5), 1u << (ba & 31));
                if (hi[g] < n) atomicXor(bm + (be >> 5), 1u << (be & 31));
            } else {
                pa = b[g];
                pe = hi[g];
            }
        }
    }
}

template <bool WEIGHTED>
__device__ uint32_t dprs_n2v_rev(const WalkArgs &a, const StepCtx &s, uint32_t k, int lane,
                                 uint32_t woff) {
    const uint32_t deg = s.deg;
    const uint32_t off = (uint32_t)(s.elo & 3);
    const uint32_t dp = (uint32_t)(s.phi - s.plo);
    const uint32_t span = deg + off;
    const uint32_t prev = (uint32_t)s.prev;
    const uint32_t *__restrict__ T = a.tgt + s.elo;  // N(cur)
    const uint32_t *__restrict__ P = a.tgt + s.plo;  // N(prev)
    uint32_t *bm = fw_smem + woff;
    stage_words(a, s, k, lane, woff, off);
    const uint32_t cmul = k == 256 ? 0 : (128u >> (31 - __clz(k)));
    const uint32_t wq0 = (woff + kTabSlots) * 4 + 16 * lane;
    const uint32_t lmask = (1u << lane) - 1;
    uint64_t icarry = 0;
    uint32_t cand = 0;
    for (uint32_t xs = 0; xs < span; xs += kSegSlots) {
        const uint32_t xe = min(span, xs + kSegSlots);
        // clear the segment's bitmap words (4 per tile)
        const uint32_t nw = ((xe - xs + 127) >> 7) * 4;
        for (uint32_t w0 = 0; w0 < nw; w0 += 128)
            if (w0 + 4 * lane < nw) *reinterpret_cast<uint4 *>(bm + w0 + 4 * lane) = make_uint4(0, 0, 0, 0);
        // the segment's elements [is, ie) and the N(prev) keys in its value range
        const uint32_t is = xs > off ? xs - off : 0, ie = xe - off;
        const uint32_t *__restrict__ Ts = T + is;
        const uint32_t n = ie - is;
        uint32_t klo = 0, khi = dp;
        if (n < deg) {
            const uint32_t kb = lower_bound1(P, dp, (lane & 1) ? ldg(Ts + n - 1) + 1 : ldg(Ts));
            klo = __shfl_sync(FULL, kb, 0);
            khi = __shfl_sync(FULL, kb, 1);
        }
        __syncwarp();  // the clear is complete before any toggle
        const uint32_t nreal = khi - klo, nk = nreal + 1;  // + prev
        const uint32_t bit0 = is + off - xs;  // bitmap bit of the segment's element 0
        uint32_t pa = 0, pe = 0;
        for (uint32_t j0 = 0; j0 < nk; j0 += 32) {
            if (nk - j0 > 64) {
                rev_round<4>(Ts, n, P + klo, j0, nreal, nk, prev, bm, bit0, lane, pa, pe);
                j0 += 96;
            } else {
                rev_round<1>(Ts, n, P + klo, j0, nreal, nk, prev, bm, bit0, lane, pa, pe);
            }
        }
        // prev's run, as slots (the lane holding the prev key had it)
        const uint32_t pl = (nreal & 31) == (uint32_t)lane ? pa : 0, ph = (nreal & 31) == (uint32_t)lane ? pe : 0;
        const uint32_t pr_lo = __shfl_sync(FULL, pl, nreal & 31) + bit0 + xs;
        const uint32_t pr_hi = __shfl_sync(FULL, ph, nreal & 31) + bit0 + xs;
        __syncwarp();  // the bitmap is complete
        const float *wpt = a.w + (s.elo - off) + xs + 4 * lane;
        uint32_t par = 0;  // membership parity carried across tiles
        for (uint32_t x0 = xs; x0 < xe; x0 += 128, wpt += 128) {
            const uint32_t t = x0 >> 7;
            const bool edge = x0 < off || x0 + 128 > span;
            const int32_t i0 = (int32_t)(x0 + 4 * lane) - (int32_t)off;
            float wf[4] = {1.f, 1.f, 1.f, 1.f};
            if (edge) {
                if (WEIGHTED && x0 + 4 * lane < span) {
                    const float4 w4 = ldg(reinterpret_cast<const float4 *>(wpt));
                    wf[0] = w4.x; wf[1] = w4.y; wf[2] = w4.z; wf[3] = w4.w;
                }
#pragma unroll
                for (int e = 0; e < 4; e++)  // invalid slots weigh 0
                    if ((uint32_t)(i0 + e) >= deg) wf[e] = 0.0f;
            } else if (WEIGHTED) {
                const float4 w4 = ldg(reinterpret_cast<const float4 *>(wpt));
                wf[0] = w4.x; wf[1] = w4.y; wf[2] = w4.z; wf[3] = w4.w;
            }
            // membership: prefix parity of the toggles up to each slot
            const uint32_t tg = (bm[((x0 - xs) >> 5) + (lane >> 3)] >> ((lane & 7) * 4)) & 0xFu;
            uint32_t mx = tg ^ (tg << 1);
            mx ^= mx << 2;  // bit e = xor of toggle bits 0..e
            const uint32_t bal = __ballot_sync(FULL, (mx >> 3) & 1);
            const uint32_t cin = (__popc(bal & lmask) + par) & 1;
            par += __popc(bal);
            const uint32_t mem = mx ^ (0u - cin);
            // factor 1/a if u == prev, else 1 if u in N(prev), else 1/b
            float wp[4];
#pragma unroll
            for (int e = 0; e < 4; e++) wp[e] = (((mem >> e) & 1) ? a.f132 : a.fb32) * wf[e];
            if (pr_lo < x0 + 128 && pr_hi > x0) {  // the tile holds a prev position
#pragma unroll
                for (int e = 0; e < 4; e++)
                    if (x0 + 4 * lane + e - pr_lo < pr_hi - pr_lo) wp[e] = a.fa32 * wf[e];
            }
            // integer tile sums, prefilter, exact test (as in dprs_n2v_pow2)
            const uint32_t wq = wq0 + (cmul ? 0 : (t & 1) * 1024);
            uint32_t wi[4];
#pragma unroll
            for (int e = 0; e < 4; e++) wi[e] = __float2uint_rz(wp[e]);
            const uint32_t li = (wi[0] + wi[1]) + (wi[2] + wi[3]);
            const uint32_t thr = accept_thr_raw(a.accept_wmax_s, (float)icarry);
            const uint32_t slo = __reduce_add_sync(FULL, li & 0xFFFFu);
            const uint32_t shi = __reduce_add_sync(FULL, li >> 16);
            const uint4 qa = *reinterpret_cast<const uint4 *>(reinterpret_cast<const char *>(fw_smem) + wq);
            const uint4 qb = *reinterpret_cast<const uint4 *>(reinterpret_cast<const char *>(fw_smem) + wq + 512);
            const uint64_t cg = (uint64_t)(cmul ? t * cmul : t >> 1) * GOLDEN;
            const uint64_t wd[4] = {(((uint64_t)qa.y << 32) | qa.x) + cg,
                                    (((uint64_t)qa.w << 32) | qa.z) + cg,
                                    (((uint64_t)qb.y << 32) | qb.x) + cg,
                                    (((uint64_t)qb.w << 32) | qb.z) + cg};
            uint32_t y[4];
#pragma unroll
            for (int e = 0; e < 4; e++) y[e] = mix64_yhi(wd[e]);
            const uint32_t ymin = min(min(y[0], y[1]), min(y[2], y[3]));
            if (__any_sync(FULL, ymin <= thr)) {
                const double l3 = (double)li;
                const double incl = warp_incl_scan_p(l3);
                double run = __dadd_rn((double)icarry, __dadd_rn(incl, -l3));  // exact
                if (ymin <= thr) {
#pragma unroll
                    for (int e = 0; e < 4; e++) {
                        const double w = (double)wi[e];
                        run = __dadd_rn(run, w);
                        if (y[e] <= thr) {
                            const double r = u01_word(wd[e]);
                            if (w > 0.0 && __dmul_rn(r, run) < w) cand = (uint32_t)(i0 + e) + 1;
                        }
                    }
                }
            }
            icarry += ((uint64_t)shi << 16) + slo;
        }
        __syncwarp();  // readers of this segment's bitmap are done
    }
    const uint32_t sel = __reduce_max_sync(FULL, cand);
    __syncwarp();  // the staged words are rebuilt by the next step
    return sel;
}

