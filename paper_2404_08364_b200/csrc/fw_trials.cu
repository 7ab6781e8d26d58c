// Sampler trial kernels: the reference's sampler micro-benchmark / verify
// path (reswalk _kernels.py:69-277, driven by trials.run_trials,
// trials.py:46-90), SURVEY §8(f) rank 4.  Trial t draws from the streams
// sid = (t << 10) | lane (_kernels.py:79-81), so every pick is a pure
// function of (weights, k, key, t) and is reproduced bit for bit.  One
// thread runs one trial with the reference's exact (sequential) fp64
// summation order; the k logical lanes are emulated without scratch arrays:
//   DPRS  last accepted element in natural order, P = chunk_prefix + carry
//   ZPRS  lanes in order, each lane's reservoir seeded with the exclusive
//         lane prefix, last accepted in lane-major order
#include <cuda_runtime.h>

#include <cstdint>

#include "fw_common.cuh"

namespace fw {

enum { TR_SEQ = 0, TR_DPRS = 1, TR_ZPRS = 2, TR_ITS = 3, TR_ALIAS = 4, TR_RJS = 5,
       TR_UNIFORM = 6 };

__device__ __forceinline__ uint64_t trial_base(uint64_t h, uint64_t t, uint64_t lane) {
    return mix64(h ^ (((t << 10) | lane) * MIX1));
}

__global__ void k_trials(int method, const double *__restrict__ w, uint32_t n, uint32_t k,
                         uint64_t h, uint64_t trials, const double *__restrict__ prob,
                         const int64_t *__restrict__ alias, double w_max, uint32_t max_rounds,
                         uint32_t *__restrict__ picks, int64_t *__restrict__ aux) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < trials;
         t += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t sel = 0;
        int64_t ax = 0;
        if (method == TR_SEQ) {  // _kernels.py:84-99
            const uint64_t b = trial_base(h, t, 0);
            double prefix = 0.0;
            for (uint32_t i = 0; i < n; i++) {
                const double wi = w[i];
                prefix = __dadd_rn(prefix, wi);
                if (wi > 0.0 && __dmul_rn(u01(b, i), prefix) < wi) sel = i + 1;
            }
        } else if (method == TR_DPRS) {  // _kernels.py:102-143
            const uint32_t chunks = n ? (n - 1) / k + 1 : 0;
            double carry = 0.0;
            for (uint32_t c = 0; c < chunks; c++) {
                const uint32_t b0 = c * k, m = min(k, n - b0);
                double run = 0.0;
                for (uint32_t j = 0; j < m; j++) {
                    const double wi = w[b0 + j];
                    run = __dadd_rn(run, wi);
                    const double r = u01(trial_base(h, t, j), c);
                    if (wi > 0.0 && __dmul_rn(r, __dadd_rn(run, carry)) < wi) sel = b0 + j + 1;
                }
                carry = __dadd_rn(carry, run);
            }
            ax = 2 * (int64_t)chunks;
        } else if (method == TR_ZPRS) {  // _kernels.py:146-189
            const uint32_t chunks = n ? (n - 1) / k + 1 : 0;
            double excl = 0.0;  // run = 0; prefix[j] = run; run += lane_sum[j]
            for (uint32_t j = 0; j < k; j++) {
                double lsum = 0.0;
                for (uint32_t c = 0; c < chunks; c++)
                    if (c * k + j < n) lsum = __dadd_rn(lsum, w[c * k + j]);
                if (j < n) {
                    const uint64_t b = trial_base(h, t, j);
                    double running = excl;
                    for (uint32_t c = 0; c < chunks; c++) {
                        const uint32_t i = c * k + j;
                        if (i >= n) break;
                        const double wi = w[i];
                        running = __dadd_rn(running, wi);
                        if (wi > 0.0 && __dmul_rn(u01(b, c), running) < wi) sel = i + 1;
                    }
                }
                excl = __dadd_rn(excl, lsum);
            }
            ax = 2;
        } else if (method == TR_ITS) {  // _kernels.py:192-218
            double total = 0.0;
            for (uint32_t i = 0; i < n; i++) total = __dadd_rn(total, w[i]);
            const double r = u01(trial_base(h, t, 0), 0);
            if (n > 0 && total > 0.0) {
                const double target = __dmul_rn(r, total);
                double prefix = 0.0;
                uint32_t lo = n - 1;
                for (uint32_t i = 0; i < n; i++) {  // first i with prefix[i] >= target
                    prefix = __dadd_rn(prefix, w[i]);
                    if (!(prefix < target)) { lo = i; break; }
                }
                sel = lo + 1;
            }
        } else if (method == TR_ALIAS) {  // _kernels.py:221-234
            const uint64_t b = trial_base(h, t, 0);
            uint32_t bucket = (uint32_t)(int64_t)__dmul_rn(u01(b, 0), (double)n);
            if (bucket >= n) bucket = n - 1;
            sel = u01(b, 1) < prob[bucket] ? bucket + 1 : (uint32_t)alias[bucket];
        } else if (method == TR_RJS) {  // _kernels.py:237-265
            const uint64_t b = trial_base(h, t, 0);
            ax = max_rounds;
            if (n > 0 && w_max > 0.0) {
                uint64_t ctr = 0;
                for (uint32_t rd = 0; rd < max_rounds; rd++) {
                    uint32_t i = (uint32_t)(int64_t)__dmul_rn(u01(b, ctr), (double)n);
                    ctr++;
                    if (i >= n) i = n - 1;
                    const double height = __dmul_rn(u01(b, ctr), w_max);
                    ctr++;
                    if (height < w[i]) {
                        sel = i + 1;
                        ax = rd + 1;
                        break;
                    }
                }
            } else {
                ax = 0;
            }
        } else {  // TR_UNIFORM, _kernels.py:268-277
            uint32_t i = (uint32_t)(int64_t)__dmul_rn(u01(trial_base(h, t, 0), 0), (double)n);
            if (i >= n) i = n - 1;
            sel = i + 1;
        }
        picks[t] = sel;
        if (aux) aux[t] = ax;
    }
}

cudaError_t launch_trials(int method, const double *w, uint32_t n, uint32_t k, uint64_t key,
                          uint64_t trials, const double *prob, const int64_t *alias,
                          double w_max, uint32_t max_rounds, uint32_t *picks, int64_t *aux,
                          cudaStream_t stream) {
    if (!trials) return cudaSuccess;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t want = (trials + 127) / 128;
    const int grid = (int)(want < (uint64_t)sms * 16 ? want : (uint64_t)sms * 16);
    k_trials<<<grid, 128, 0, stream>>>(method, w, n, k, mix64(key + GOLDEN), trials, prob,
                                       alias, w_max, max_rounds, picks, aux);
    return cudaGetLastError();
}

}  // namespace fw
