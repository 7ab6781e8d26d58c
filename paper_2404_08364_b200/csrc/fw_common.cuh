// Shared device helpers for the sm_100a walk engine.
//
// RNG: the reference's SplitMix64-finalizer counter hash, bit-exact
// (reswalk _kernels.py:50-66, spec rng.py:24-41):
//   mix64(z)          = xorshift-multiply finalizer, constants MIX1/MIX2
//   stream_base(k,s)  = mix64(mix64(k + GOLDEN) ^ (s * MIX1))
//   u01(base, c)      = (mix64(base + c * GOLDEN) >> 11) * 2^-53
// Replay stream ids (_kernels.py:8-12, 390-396):
//   sid = 1<<63 | qid<<30 | step<<10 | lane      (lane 1023 = PPR stop draw)
// The fields occupy disjoint bits, so sid*MIX1 = (sid_hi*MIX1) + lane*MIX1
// (mod 2^64): one 64-bit multiply per (query, step), one IMAD per lane.
#pragma once
#include <cstdint>

namespace fw {

constexpr uint64_t GOLDEN = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t MIX1 = 0xBF58476D1CE4E5B9ULL;
constexpr uint64_t MIX2 = 0x94D049BB133111EBULL;
constexpr uint64_t TAG_REPLAY = 1ULL << 63;
constexpr uint64_t STOP_LANE = 1023ULL;
constexpr unsigned FULL = 0xFFFFFFFFu;

enum { APP_DEEPWALK = 0, APP_PPR = 1, APP_NODE2VEC = 2, APP_METAPATH = 3 };
enum { SAMPLER_ZPRS = 0, SAMPLER_DPRS = 1 };
enum { ST_STEPS = 0, ST_EDGES, ST_COLLECTIVES, ST_DRAWS, ST_SMALL, ST_LARGE, ST_SAMPLED,
       ST_BYTES, ST_COUNT };
// extra device words after the counters: max over warps of the exit time and
// of its complement (%globaltimer ns) -> first/last warp exit of a launch
enum { ST_T_LAST = ST_COUNT, ST_T_FIRST_NEG, ST_WORDS };

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * MIX1;
    z = (z ^ (z >> 27)) * MIX2;
    return z ^ (z >> 31);
}

// u01 from a pre-advanced counter word (base + ctr*GOLDEN).  z>>11 < 2^53 so
// the int->double conversion and the 2^-53 scaling are both exact.
__device__ __forceinline__ double u01_word(uint64_t word) {
    const uint64_t z = mix64(word);
    return __dmul_rn(__ull2double_rn(z >> 11), 0x1.0p-53);
}

__device__ __forceinline__ double u01(uint64_t base, uint64_t ctr) {
    return u01_word(base + ctr * GOLDEN);
}

// Read-only graph loads through the non-coherent path.
template <typename T>
__device__ __forceinline__ T ldg(const T *p) { return __ldg(p); }

// fp64 warp inclusive scan (Kogge-Stone).  Only used when every partial sum
// is exact, so association order
// cannot change a bit.
__device__ __forceinline__ double warp_incl_scan(double v, int lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double o = __shfl_up_sync(FULL, v, d);
        if (lane >= d) v = __dadd_rn(v, o);
    }
    return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) v = __dadd_rn(v, __shfl_xor_sync(FULL, v, d));
    return v;
}

}  // namespace fw
