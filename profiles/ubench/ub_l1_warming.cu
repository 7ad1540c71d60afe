#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t ld(const uint32_t* p) { uint32_t v; asm volatile("ld.global.u32 %0, [%1];" : "=r"(v) : "l"(p)); return v; }
__device__ __forceinline__ void pfl1(const void* p) { asm volatile("prefetch.global.L1 [%0];" :: "l"(p)); }
// list[i] = node id of step i; g[node*32] holds a value used to make the chain dependent (always 0)
__global__ void run(const uint32_t* g, const uint32_t* list, int steps, int mode, int D, long long* res, uint32_t* out) {
    __shared__ uint32_t sm[64];
    uint32_t acc = 0, x = 0;
    long long t0 = clock64();
    for (int i = 0; i < steps; ++i) {
        if (mode == 1) pfl1(&g[list[i + D] * 32 + threadIdx.x]);
        if (mode == 2) acc += ld(&g[list[i + D] * 32 + threadIdx.x]);
        if (mode == 3) { uint32_t dst = (uint32_t)__cvta_generic_to_shared(&sm[threadIdx.x]);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(dst), "l"(&g[list[i + D] * 32 + threadIdx.x])); asm volatile("cp.async.commit_group;"); }
        x = ld(&g[(list[i] + x) * 32 + threadIdx.x]);   // x == 0 always; dependent chain
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) res[0] = (t1 - t0) / steps;
    out[threadIdx.x] = x + acc;
}
int main() {
    const int nodes = 1 << 18, steps = 4000;
    uint32_t *g, *list, *o; long long* r;
    cudaMalloc(&g, (size_t)nodes * 128); cudaMemset(g, 0, (size_t)nodes * 128);
    uint32_t* hl = new uint32_t[steps + 64];
    for (int i = 0; i < steps + 64; ++i) hl[i] = (uint32_t)(((uint64_t)i * 2654435761u) % nodes);
    cudaMalloc(&list, (steps + 64) * 4); cudaMemcpy(list, hl, (steps + 64) * 4, cudaMemcpyHostToDevice);
    cudaMalloc(&o, 4096); cudaMalloc(&r, 64);
    // warm L2 with the whole table
    run<<<1, 32>>>(g, list, steps, 0, 0, r, o); cudaDeviceSynchronize();
    const char* nm[] = {"none", "prefetch.L1", "dummy ld", "cp.async"};
    for (int mode = 0; mode < 4; ++mode) for (int D : {1, 2, 4, 8}) {
        if (mode == 0 && D > 1) continue;
        run<<<1, 32>>>(g, list, steps, mode, D, r, o); cudaDeviceSynchronize();
        long long v; cudaMemcpy(&v, r, 8, cudaMemcpyDeviceToHost);
        printf("%-12s D=%d: %lld cycles/step\n", nm[mode], D, v);
    }
}
