// Bit-for-bit check of sqrt_rn_fast (device.cuh) against __dsqrt_rn, and of the EUC_2D
// value (int)(sqrt + 0.5) built on it, over
//   (a) every k^2 - k, k^2 - k + 1, k^2, k^2 + k, k^2 + k + 1 for k < 2^24 (the squared
//       distances next to every EUC_2D rounding boundary of coordinates below 1.2e7),
//   (b) 2^31 random integers below 2^48 (squared distances of coordinates below 1e7),
//   (c) 2^31 random bit patterns whose exponent passes sqrt_fast_ok (any double input).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false -I../../paper_1709_03187_b200/csrc ub_sqrt.cu
#include <cstdio>
#include <cstdint>
#include "device.cuh"
using namespace pacob200;

__device__ unsigned long long g_bad[4], g_count[4];

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ void check(int kind, double x) {
    if (!sqrt_fast_ok(x)) return;
    const double a = sqrt_rn_fast(x), b = __dsqrt_rn(x);
    const bool same = __double_as_longlong(a) == __double_as_longlong(b) &&
                      (int32_t)__dadd_rn(a, 0.5) == (int32_t)__dadd_rn(b, 0.5);
    atomicAdd(&g_count[kind], 1ull);
    if (!same && atomicAdd(&g_bad[kind], 1ull) < 4)
        printf("kind %d x=%.17g fast=%.17g ref=%.17g\n", kind, x, a, b);
}
__global__ void k_boundaries() {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= (1ull << 24)) return;
    const double k2 = (double)(k * k);
    const double kk = (double)k;
    check(0, k2 - kk); check(0, k2 - kk + 1.0); check(0, k2); check(0, k2 + kk); check(0, k2 + kk + 1.0);
}
__global__ void k_random(uint64_t base) {
    const uint64_t i = base + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t r = mix(i);
    check(1, (double)(r >> 16));                       // integer below 2^48
    check(2, __longlong_as_double((long long)(mix(r) & 0x7fffffffffffffffull)));  // any positive double
}

int main() {
    k_boundaries<<<(1u << 24) / 256, 256>>>();
    for (int chunk = 0; chunk < 8; ++chunk) k_random<<<(1u << 28) / 256, 256>>>((uint64_t)chunk << 28);
    cudaDeviceSynchronize();
    unsigned long long bad[4], cnt[4];
    cudaMemcpyFromSymbol(bad, g_bad, sizeof bad);
    cudaMemcpyFromSymbol(cnt, g_count, sizeof cnt);
    const char* names[3] = {"EUC_2D rounding boundaries", "integers < 2^48", "random doubles (fast range)"};
    for (int k = 0; k < 3; ++k) printf("%-30s checked %llu mismatches %llu\n", names[k], cnt[k], bad[k]);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return (bad[0] | bad[1] | bad[2]) ? 1 : 0;
}
