#include <cstdio>
#include <cstdint>
__global__ void kb(const uint32_t* g, uint32_t* out, long long* res, int iters) {
    __shared__ uint32_t sm[1024];
    const int lane = threadIdx.x;
    for (int i = lane; i < 1024; i += 32) sm[i] = (i * 7 + 1) & 1023;
    __syncwarp();
    uint32_t x = lane;
    long long t0, t1;
    // 1. SHFL.IDX chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) x = __shfl_sync(0xffffffff, x, (x + 1) & 31);
    t1 = clock64(); if (lane == 0) res[0] = (t1 - t0) / iters;
    // 2. SHFL.UP + FADD chain
    float v = x;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { float y = __shfl_up_sync(0xffffffff, v, 1); if (lane >= 1) v = v + y; }
    t1 = clock64(); if (lane == 0) res[1] = (t1 - t0) / iters; x += (uint32_t)v;
    // 3. LDS chain
    uint32_t p = lane;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) p = sm[p & 1023];
    t1 = clock64(); if (lane == 0) res[2] = (t1 - t0) / iters; x += p;
    // 4. LDG chain (L2/L1): pointer chase over g (1M entries), stride large
    uint32_t q = lane * 4099;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) q = __ldg(&g[q & ((1<<22)-1)]);
    t1 = clock64(); if (lane == 0) res[3] = (t1 - t0) / iters; x += q;
    // 5. ballot + ffs + shfl chain
    uint32_t r = lane;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { unsigned b = __ballot_sync(0xffffffff, ((r + i) & 3) == 0); r = __shfl_sync(0xffffffff, r + 1, __ffs(b) - 1); }
    t1 = clock64(); if (lane == 0) res[4] = (t1 - t0) / iters; x += r;
    // 6. syncwarp
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { __syncwarp(); x ^= i; }
    t1 = clock64(); if (lane == 0) res[5] = (t1 - t0) / iters;
    // 7. LDG chain on small table (L1 resident): 4K entries
    q = lane;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) q = __ldg(&g[q & 4095]);
    t1 = clock64(); if (lane == 0) res[6] = (t1 - t0) / iters; x += q;
    // 8. FADD chain
    float f = x;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) f = f * 1.0000001f + 0.5f;
    t1 = clock64(); if (lane == 0) res[7] = (t1 - t0) / iters; x += (uint32_t)f;
    out[lane] = x;
}
int main() {
    const int N = 1 << 22;
    uint32_t* h = new uint32_t[N];
    for (int i = 0; i < N; ++i) h[i] = (uint32_t)(((uint64_t)i * 2654435761u + 12345) % N);
    uint32_t *g, *o; long long* r;
    cudaMalloc(&g, N * 4); cudaMalloc(&o, 128); cudaMalloc(&r, 64 * 8);
    cudaMemcpy(g, h, N * 4, cudaMemcpyHostToDevice);
    kb<<<1, 32>>>(g, o, r, 100); cudaDeviceSynchronize();
    kb<<<1, 32>>>(g, o, r, 2000); 
    long long hr[8]; cudaMemcpy(hr, r, 64, cudaMemcpyDeviceToHost);
    const char* names[] = {"shfl.idx chain", "shfl.up+fadd", "lds chain", "ldg chain 16MB (L2)", "ballot+ffs+shfl", "syncwarp", "ldg chain 16KB (L1)", "ffma chain"};
    for (int i = 0; i < 8; ++i) printf("%-24s %lld cycles\n", names[i], hr[i]);
}
