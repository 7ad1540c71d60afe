// L2 read bandwidth of one B200 (the denominator of the L2-resident roofline).
// A grid of 8 CTAs per SM streams a buffer of S bytes with 16-byte `ld.global.cg` loads
// (L1 bypassed), eight independent loads in flight per thread, `reps` times over. For S
// well inside the 126 MB L2 every pass after the first is served by L2; S = 1 GiB is the
// HBM reference point. Reported: bytes delivered per second over the timed launch (CUDA
// events), best of 5, each launch >= ~2 ms.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o ub_l2_bw ub_l2_bw.cu && ./ub_l2_bw
#include <cstdint>
#include <cstdio>

__global__ void __launch_bounds__(256) k_read(const uint4* __restrict__ buf, size_t n16, int reps,
                                              unsigned long long* sink) {
    uint32_t acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    const size_t t0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int r = 0; r < reps; ++r) {
        for (size_t i = t0; i < n16; i += 8 * stride) {
            uint4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const size_t j = i + u * stride;
                v[u] = make_uint4(0, 0, 0, 0);
                if (j < n16)
                    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                                 : "l"(buf + j));
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
        }
    }
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    const size_t sizes_mb[] = {16, 32, 48, 64, 96, 1024};
    printf("{\"sms\": %d, \"runs\": [", sms);
    bool first = true;
    for (size_t mb : sizes_mb) {
        const size_t bytes = mb << 20, n16 = bytes / 16;
        uint4* buf;
        cudaMalloc(&buf, bytes);
        cudaMemset(buf, 1, bytes);
        const int threads = 256, blocks = sms * 8;
        const int reps = (int)(((size_t)16 << 30) / bytes);  // ~16 GiB per launch
        k_read<<<blocks, threads>>>(buf, n16, 1, sink);     // warm L2
        cudaDeviceSynchronize();
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        float best = 1e30f;
        for (int t = 0; t < 5; ++t) {
            cudaEventRecord(a);
            k_read<<<blocks, threads>>>(buf, n16, reps, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        const double gbs = (double)bytes * reps / (best * 1e-3) / 1e9;
        printf("%s{\"mb\": %zu, \"reps\": %d, \"gb_per_s\": %.1f, \"ms\": %.3f}", first ? "" : ", ", mb, reps, gbs, best);
        first = false;
        cudaFree(buf);
    }
    printf("]}\n");
    return 0;
}
