#include <cstdio>
#include <cstdint>
__global__ void warm(const uint32_t* g, int n, uint32_t* o) { uint32_t s=0; for (int i = blockIdx.x*blockDim.x+threadIdx.x; i < n; i += gridDim.x*blockDim.x) s += g[i]; if (s == 12345) o[0] = s; }
__global__ void chase(const uint32_t* g, int mask, uint32_t* out, long long* res, int iters, int mode) {
    uint32_t q = threadIdx.x * 977;
    long long t0 = clock64();
    if (mode == 0) for (int i = 0; i < iters; ++i) q = __ldg(&g[q & mask]);
    else for (int i = 0; i < iters; ++i) q = g[q & mask];
    long long t1 = clock64();
    if (threadIdx.x == 0) res[0] = (t1 - t0) / iters;
    out[threadIdx.x] = q;
}
int main() {
    const int N = 1 << 25; // 128 MB
    uint32_t* h = new uint32_t[N];
    for (int i = 0; i < N; ++i) h[i] = (uint32_t)(((uint64_t)i * 2654435761u + 97) % N) ;
    uint32_t *g, *o; long long* r;
    cudaMalloc(&g, (size_t)N * 4); cudaMalloc(&o, 4096); cudaMalloc(&r, 64);
    cudaMemcpy(g, h, (size_t)N * 4, cudaMemcpyHostToDevice);
    int sizes_mb[] = {1, 4, 16, 32, 64, 128};
    for (int s : sizes_mb) {
        int n = s * (1 << 18);  // entries (4 B)
        for (int mode = 0; mode < 2; ++mode) {
            warm<<<1024, 256>>>(g, n, o); warm<<<1024, 256>>>(g, n, o);
            chase<<<1, 32>>>(g, n - 1, o, r, 4000, mode);
            cudaDeviceSynchronize();
            long long v; cudaMemcpy(&v, r, 8, cudaMemcpyDeviceToHost);
            printf("%4d MB %s: %lld cycles\n", s, mode ? "ld.global" : "ldg.nc", v);
        }
    }
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0); printf("clock %d kHz\n", clk);
}
