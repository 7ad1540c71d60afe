// Decision-loop scheduling study (second round): the K2 loop on a synthetic 200k-city,
// 16-candidate table, with scheduling changes that keep the chosen sequence identical:
//   DEFER  - set the visited bit of the current city after this decision's bitmap probe
//            (a city is never its own candidate), so the probe does not queue behind the
//            shared-memory atomic of the previous decision;
//   RPHIL  - every lane computes the same Philox block once per 4 decisions (no shuffle
//            to hand out the draw);
//   BATCH  - tour entries are kept one per lane and stored 32 at a time;
//   TM     - clock64 segment timing (row wait, probe, scan, pick, tail).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false -I../../paper_1709_03187_b200/csrc ub_decision2.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include "device.cuh"
using namespace pacob200;

enum : int { DEFER = 1, RPHIL = 2, BATCH = 4, TM = 8, NOTIE = 16, NOWARM = 32 };

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) { uint32_t v; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr)); return v; }
__device__ __forceinline__ void cp_async16_if(uint32_t dst, const void* src, bool cond) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q cp.async.ca.shared.global [%0], [%1], 16;\n\t}" ::"r"(dst), "l"(src), "r"((uint32_t)cond));
}
__device__ __forceinline__ long long clk_dep(uint32_t dep) {
    long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c) : "r"(dep) : "memory");
    return c;
}

template <int V>
__global__ void __launch_bounds__(32, 1) dec(const uint2* __restrict__ cand, uint32_t n, uint32_t D, uint32_t* tours,
                                             long long* cyc, unsigned long long* seg) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t lane = threadIdx.x, ant = blockIdx.x, nw = (n + 31) / 32;
    uint32_t* vis = reinterpret_cast<uint32_t*>(smem);
    for (uint32_t w = lane; w < nw; w += 32) vis[w] = 0u;
    __syncwarp();
    const uint32_t vis_s = (uint32_t)__cvta_generic_to_shared(vis);
    const uint32_t warm_s = ((vis_s + nw * 4 + 15) & ~15u) + lane * 16;
    uint32_t cur = (ant * 977u) % n;
    if (lane == 0) vis[cur >> 5] |= 1u << (cur & 31);
    __syncwarp();
    uint32_t* out = tours + (size_t)ant * D;
    const uint2 key = make_uint2(7u, 0u);
    uint4 pb;
    uint32_t uw;
    if (V & RPHIL) {
        pb = philox10(make_uint4(1, ant, 0, 0), key);  // block of decisions 0..3 (all lanes)
        uw = pb.x;
    } else {
        pb = philox10(make_uint4(1 + lane, ant, 0, 0), key);
        uw = __shfl_sync(kFull, pb.x, 0);
    }
    const bool lane_in = lane < 16;
    const uint2* row_base = cand + lane;
    uint2 e_pre = ldg_u64_if(row_base + (size_t)cur * 16, lane_in, make_uint2(cur, 0u));
    uint32_t n_fb = 0, n_tie = 0, held = 0;
    long long s1 = 0, s2 = 0, s3 = 0, s4 = 0, s5 = 0;
    const long long t0 = clock64();
    long long tprev = t0;
    for (uint32_t t = 0; t < D; ++t) {
        __syncwarp();
        const uint2 e = e_pre;
        long long ta = 0, tb = 0, tc = 0, td = 0;
        if (V & TM) ta = clk_dep(e.x);
        const uint32_t vw = lds_u32(vis_s + ((e.x >> 5) << 2));
        if (V & DEFER) red_or_shared_if(vis_s + ((cur >> 5) << 2), 1u << (cur & 31), lane == 0);
        const float w = ((vw >> (e.x & 31)) & 1u) ? 0.0f : __uint_as_float(e.y);
        if (V & TM) tb = clk_dep(__float_as_uint(w));
        if (!(V & NOWARM)) {
            const unsigned char* src = reinterpret_cast<const unsigned char*>(cand + (size_t)e.x * 16);
#pragma unroll
            for (int c = 0; c < 4; ++c) cp_async16_if(warm_s, src + 32 * c, w > 0.0f);
        }
        float v = w;
#pragma unroll
        for (int st = 0; st < 4; ++st) {
            const float y = __shfl_up_sync(kFull, v, 1u << st);
            if (lane >= (1u << st)) v = __fadd_rn(v, y);
        }
        const float u = u01_f32(uw);
        const float S = __shfl_sync(kFull, v, 15);
        if (V & TM) tc = clk_dep(__float_as_uint(S));
        uint32_t next;
        if (S > 0.0f) {
            const float target = __fmul_rn(u, S);
            const float tol = __fmul_rn(1e-6f, S);
            const unsigned ball = __ballot_sync(kFull, w > 0.0f && v > target);
            const unsigned feas = __ballot_sync(kFull, w > 0.0f);
            unsigned tie = 0;
            if (!(V & NOTIE)) tie = __ballot_sync(kFull, lane_in && fabsf(__fsub_rn(v, target)) <= tol);
            const int r = ball ? __ffs(ball) - 1 : 31 - __clz(feas);
            next = __shfl_sync(kFull, e.x, r);
            n_tie += tie ? 1u : 0u;
        } else {
            if (V & DEFER) __syncwarp();
            next = (uint32_t)(((uint64_t)(cur + 1) * 2654435761ull) % n);
            ++n_fb;
        }
        if (V & TM) td = clk_dep(next);
        e_pre = ldg_u64_if(row_base + (size_t)next * 16, lane_in, make_uint2(next, 0u));
        if (!(V & DEFER)) red_or_shared_if(vis_s + ((next >> 5) << 2), 1u << (next & 31), lane == 0);
        if (V & BATCH) {
            if (lane == (t & 31)) held = next;
            if ((t & 31) == 31) out[t - 31 + lane] = held;
        } else {
            stg_u32_if(out + t, next, lane == 0);
        }
        cur = next;
        const uint32_t t1 = t + 1;
        if (V & RPHIL) {
            if ((t1 & 3) == 0) pb = philox10(make_uint4(1 + (t1 >> 2), ant, 0, 0), key);
            uw = pick_word(pb, t1 & 3);
        } else {
            if ((t1 & 127) == 0) pb = philox10(make_uint4(1 + (t1 >> 2) + lane, ant, 0, 0), key);
            uw = __shfl_sync(kFull, pick_word(pb, t1 & 3), (t1 & 127) >> 2);
        }
        if (V & TM) {
            const long long te = clk_dep(uw);
            s1 += ta - tprev; s2 += tb - ta; s3 += tc - tb; s4 += td - tc; s5 += te - td;
            tprev = te;
        }
    }
    if (V & BATCH) {
        if ((D & 31) && lane < (D & 31)) out[(D & ~31u) + lane] = held;
    }
    const long long t1 = clock64();
    if (lane == 0) {
        cyc[ant] = t1 - t0;
        atomicAdd(&seg[0], (unsigned long long)n_fb);
        atomicAdd(&seg[1], (unsigned long long)n_tie);
        if (V & TM) {
            atomicAdd(&seg[2], (unsigned long long)s1); atomicAdd(&seg[3], (unsigned long long)s2);
            atomicAdd(&seg[4], (unsigned long long)s3); atomicAdd(&seg[5], (unsigned long long)s4);
            atomicAdd(&seg[6], (unsigned long long)s5);
        }
    }
}

std::vector<uint32_t> g_ref;

template <int V>
void run(const char* name, const uint2* cand, uint32_t n, uint32_t D, uint32_t m, uint32_t* tours, long long* cyc,
         unsigned long long* seg) {
    const size_t smem = ((n + 31) / 32) * 4 + 16 + 512;
    cudaFuncSetAttribute(dec<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(dec<V>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    dec<V><<<m, 32, smem>>>(cand, n, D, tours, cyc, seg);
    cudaMemset(seg, 0, 64);
    cudaEventRecord(a);
    dec<V><<<m, 32, smem>>>(cand, n, D, tours, cyc, seg);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    std::vector<long long> h(m); cudaMemcpy(h.data(), cyc, m * 8, cudaMemcpyDeviceToHost);
    unsigned long long sg[8]; cudaMemcpy(sg, seg, 64, cudaMemcpyDeviceToHost);
    double mean = 0; for (auto v : h) mean += v;
    mean /= m;
    std::vector<uint32_t> got((size_t)m * D);
    cudaMemcpy(got.data(), tours, got.size() * 4, cudaMemcpyDeviceToHost);
    const char* same = "";
    if (m == 1024) {
        if (g_ref.empty()) g_ref = got;
        same = (g_ref == got) ? "same tours" : "TOURS DIFFER";
    }
    const double d = (double)m * D;
    printf("%-26s m=%-4u %6.1f cyc/dec %7.3f ms fb %.3f%% ties %llu %s %s\n", name, m, mean / D, ms, 100.0 * sg[0] / d,
           sg[1], same, cudaGetErrorString(cudaGetLastError()));
    if (V & TM)
        printf("    segments: row-wait %.0f probe %.0f scan+S %.0f pick %.0f tail %.0f\n", sg[2] / d, sg[3] / d, sg[4] / d,
               sg[5] / d, sg[6] / d);
}

int main() {
    const uint32_t n = 200000, m = 1024, D = 20000;
    std::mt19937 rng(5);
    std::vector<uint2> h((size_t)n * 16);
    std::uniform_int_distribution<int> off(-300, 300);
    std::uniform_real_distribution<float> wd(0.1f, 1.0f);
    for (uint32_t i = 0; i < n; ++i)
        for (int r = 0; r < 16; ++r) {
            int o = off(rng); if (o == 0) o = 1;
            const uint32_t c = (uint32_t)(((int64_t)i + o + n) % n);
            h[(size_t)i * 16 + r] = make_uint2(c, __builtin_bit_cast(uint32_t, wd(rng)));
        }
    uint2* cand; uint32_t* tours; long long* cyc; unsigned long long* seg;
    cudaMalloc(&cand, h.size() * 8); cudaMemcpy(cand, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMalloc(&tours, (size_t)m * D * 4); cudaMalloc(&cyc, m * 8); cudaMalloc(&seg, 64);
    printf("n=%u m=%u D=%u\n", n, m, D);
    run<0>("baseline", cand, n, D, m, tours, cyc, seg);
    run<TM>("baseline (timed)", cand, n, D, m, tours, cyc, seg);
    run<DEFER>("defer mark", cand, n, D, m, tours, cyc, seg);
    run<DEFER | TM>("defer mark (timed)", cand, n, D, m, tours, cyc, seg);
    run<RPHIL>("redundant philox", cand, n, D, m, tours, cyc, seg);
    run<BATCH>("batched tour store", cand, n, D, m, tours, cyc, seg);
    run<DEFER | RPHIL>("defer + rphil", cand, n, D, m, tours, cyc, seg);
    run<DEFER | RPHIL | BATCH>("defer + rphil + batch", cand, n, D, m, tours, cyc, seg);
    run<DEFER | RPHIL | BATCH | TM>("all three (timed)", cand, n, D, m, tours, cyc, seg);
    run<DEFER | RPHIL | BATCH | NOWARM>("all three, no warm", cand, n, D, m, tours, cyc, seg);
    run<DEFER | RPHIL | BATCH>("all three", cand, n, D, 1, tours, cyc, seg);
    run<0>("baseline", cand, n, D, 1, tours, cyc, seg);
    return 0;
}
