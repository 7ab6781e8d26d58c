// Checks an FMA-pipe formulation of the 64-bit xorshift used by mix64
// against the plain one (scratch experiment; not part of the library).
#include <cstdint>
#include <cstdio>
__device__ __forceinline__ uint64_t mix64_alu(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
template <int S>
__device__ __forceinline__ uint64_t xorshr_fma(uint64_t z) {
    const uint32_t lo = (uint32_t)z, hi = (uint32_t)(z >> 32);
    const uint32_t m = 1u << (32 - S);
    const uint32_t nlo = __umulhi(lo, m) + hi * m;  // (lo >> S) | (hi << (32-S))
    const uint32_t nhi = __umulhi(hi, m);           // hi >> S
    return z ^ (((uint64_t)nhi << 32) | nlo);
}
__device__ __forceinline__ uint64_t mix64_fma(uint64_t z) {
    z = xorshr_fma<30>(z) * 0xBF58476D1CE4E5B9ULL;
    z = xorshr_fma<27>(z) * 0x94D049BB133111EBULL;
    return xorshr_fma<31>(z);
}
__global__ void check(unsigned long long *bad, unsigned long long *sink) {
    uint64_t x = 0x123456789ABCDEFULL + threadIdx.x + blockIdx.x * 1024ull;
    uint64_t acc = 0;
    for (int i = 0; i < 1000; i++) {
        x = x * 6364136223846793005ULL + 1442695040888963407ULL;
        const uint64_t a = mix64_alu(x), b = mix64_fma(x);
        if (a != b) atomicAdd(bad, 1ull);
        acc ^= b;
    }
    if (acc == 42) atomicAdd(sink, 1ull);
}
__global__ void bench_alu(unsigned long long *sink, int iters) {
    uint64_t x = threadIdx.x + blockIdx.x * 977ull, acc = 0;
    for (int i = 0; i < iters; i++) { acc += mix64_alu(x + i * 0x9E3779B97F4A7C15ULL); }
    if (acc == 42) atomicAdd(sink, 1ull);
}
__global__ void bench_fma(unsigned long long *sink, int iters) {
    uint64_t x = threadIdx.x + blockIdx.x * 977ull, acc = 0;
    for (int i = 0; i < iters; i++) { acc += mix64_fma(x + i * 0x9E3779B97F4A7C15ULL); }
    if (acc == 42) atomicAdd(sink, 1ull);
}
int main() {
    unsigned long long *d; cudaMalloc(&d, 16); cudaMemset(d, 0, 16);
    check<<<1184, 256>>>(d, d + 1);
    unsigned long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("mismatches: %llu\n", h[0]);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; rep++) {
        float ta, tf;
        cudaEventRecord(e0); bench_alu<<<1184, 256>>>(d + 1, 20000); cudaEventRecord(e1);
        cudaEventSynchronize(e1); cudaEventElapsedTime(&ta, e0, e1);
        cudaEventRecord(e0); bench_fma<<<1184, 256>>>(d + 1, 20000); cudaEventRecord(e1);
        cudaEventSynchronize(e1); cudaEventElapsedTime(&tf, e0, e1);
        printf("mix64 alu %.3f ms  fma %.3f ms\n", ta, tf);
    }
    return 0;
}
