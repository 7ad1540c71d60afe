// Decision-loop study (third round): the current K2 loop (vote, Hillis-Steele shuffle
// scan, S shuffle, two redux.min picks, winner-lane mark) on a synthetic 200k-city,
// 16-candidate table, against variants that must choose the same tours:
//   ONE  - one redux.min: the last feasible lane (from the feasibility vote, off the
//          chain) is folded into the winner predicate, so "lowest winning lane, else last
//          feasible lane" is a single reduction with no select afterwards;
//   TREE - no shuffle scan: the masked weights go to a zero-padded shared row, and every
//          lane sums its own prefix S_r (and the total S_15) with the same balanced tree
//          the Hillis-Steele scan forms, from 16 lane-shifted LDS (plus 4 broadcast LDS.128);
//   TM   - clock64 segments.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false -I../../paper_1709_03187_b200/csrc ub_decision3.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include "device.cuh"
using namespace pacob200;

enum : int { ONE = 1, TREE = 2, TM = 4, NOWARM = 8, TREE4 = 16 };

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) { uint32_t v; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr)); return v; }
__device__ __forceinline__ float lds_f32(uint32_t addr) { float v; asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr)); return v; }
__device__ __forceinline__ float4 lds_f128(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts_f32(uint32_t addr, float v) { asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory"); }
__device__ __forceinline__ void sts_u32_if(uint32_t addr, uint32_t v, bool cond) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.shared.u32 [%0], %1;\n\t}" ::"r"(addr), "r"(v),
                 "r"((uint32_t)cond) : "memory");
}
__device__ __forceinline__ void cp_async16_if(uint32_t dst, const void* src, bool cond) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q cp.async.ca.shared.global [%0], [%1], 16;\n\t}" ::"r"(dst), "l"(src), "r"((uint32_t)cond));
}
__device__ __forceinline__ long long clk_dep(uint32_t dep) {
    long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c) : "r"(dep) : "memory");
    return c;
}
// balanced pairwise tree over x[0..15] in the Hillis-Steele association:
// ((((x15+x14)+(x13+x12))+((x11+x10)+(x9+x8))) + (((x7+x6)+(x5+x4))+((x3+x2)+(x1+x0))))
__device__ __forceinline__ float tree16(const float (&x)[16]) {
    float a[8], b[4], c[2];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __fadd_rn(x[2 * i + 1], x[2 * i]);
#pragma unroll
    for (int i = 0; i < 4; ++i) b[i] = __fadd_rn(a[2 * i + 1], a[2 * i]);
#pragma unroll
    for (int i = 0; i < 2; ++i) c[i] = __fadd_rn(b[2 * i + 1], b[2 * i]);
    return __fadd_rn(c[1], c[0]);
}

template <int V>
__global__ void __launch_bounds__(32, 1) dec(const uint2* __restrict__ cand, uint32_t n, uint32_t D, uint32_t* tours,
                                             long long* cyc, unsigned long long* seg) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t lane = threadIdx.x, ant = blockIdx.x, nw = (n + 31) / 32;
    uint32_t* vis = reinterpret_cast<uint32_t*>(smem + 1152);
    float* stage = reinterpret_cast<float*>(smem);  // 16 zeros | 16 masked weights | spare
    for (uint32_t w = lane; w < nw; w += 32) vis[w] = 0u;
    for (uint32_t i = lane; i < 1152 / 4; i += 32) stage[i] = 0.0f;
    __syncwarp();
    const uint32_t vis_s = (uint32_t)__cvta_generic_to_shared(vis);
    const uint32_t stage_s = (uint32_t)__cvta_generic_to_shared(stage);
    const uint32_t warm_s = ((vis_s + nw * 4 + 15) & ~15u) + lane * 16;
    uint32_t cur = (ant * 977u) % n;
    if (lane == 0) vis[cur >> 5] |= 1u << (cur & 31);
    __syncwarp();
    uint32_t* out = tours + (size_t)ant * D;
    const uint2 key = make_uint2(7u, 0u);
    const bool lane_in = lane < 16;
    const uint2* row_base = cand + lane;
    uint2 e_pre = ldg_u64_if(row_base + (size_t)cur * 16, lane_in, make_uint2(cur, 0u));
    uint32_t n_fb = 0, n_tie = 0;
    long long s1 = 0, s2 = 0, s3 = 0, s4 = 0;
    const long long t0 = clock64();
    long long tprev = t0;
    for (uint32_t b0 = 0; b0 < D; b0 += 128) {
        const uint4 pb = philox10(make_uint4(1 + (b0 >> 2) + lane, ant, 0, 0), key);
        const uint32_t b1 = b0 + 128 < D ? b0 + 128 : D;
#pragma unroll 2
        for (uint32_t t = b0; t < b1; ++t) {
            __syncwarp();
            const uint2 e = e_pre;
            long long ta = 0, tb = 0, tc = 0, td = 0;
            if (V & TM) ta = clk_dep(e.x);
            const uint32_t vw_addr = vis_s + ((e.x >> 5) << 2);
            const uint32_t vw = lds_u32(vw_addr);
            const uint32_t uw = __shfl_sync(kFull, pick_word(pb, t & 3), (t & 127) >> 2);
            const uint32_t bit = 1u << (e.x & 31);
            const float w = (vw & bit) ? 0.0f : __uint_as_float(e.y);
            if (V & TM) tb = clk_dep(__float_as_uint(w));
            if (!(V & NOWARM)) {
                const unsigned char* src = reinterpret_cast<const unsigned char*>(cand + (size_t)e.x * 16);
#pragma unroll
                for (int c = 0; c < 4; ++c) cp_async16_if(warm_s, src + 32 * c, w > 0.0f);
            }
            const unsigned feas = __ballot_sync(kFull, w > 0.0f);
            float v, S;
            if (V & TREE4) {
                // copy q at stage_s + 284 q (bank offset 7q): lane r reads its window from
                // copy (r+1)&3 as four 16-byte-aligned LDS.128, conflict-free per quarter warp
                if (lane_in) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) sts_f32(stage_s + 284 * q + 64 + 4 * lane, w);
                }
                __syncwarp();
                const uint32_t r = lane_in ? lane : 15u;
                const uint32_t wa = stage_s + 284 * ((r + 1) & 3) + 4 * (r + 1);
                float x[16], y[16];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float4 f = lds_f128(wa + 16 * q);
                    x[4 * q] = f.x; x[4 * q + 1] = f.y; x[4 * q + 2] = f.z; x[4 * q + 3] = f.w;
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float4 f = lds_f128(stage_s + 64 + 16 * q);
                    y[4 * q] = f.x; y[4 * q + 1] = f.y; y[4 * q + 2] = f.z; y[4 * q + 3] = f.w;
                }
                v = tree16(x);
                S = tree16(y);
                if (!lane_in) v = 0.0f;
            } else if (V & TREE) {
                if (lane_in) sts_f32(stage_s + 64 + 4 * lane, w);
                __syncwarp();
                float x[16];
                // lane r: x[j] = w_{r-15+j} (zeros below index 0); lanes >= 16 read lane 15's window
                const uint32_t r = lane_in ? lane : 15u;
#pragma unroll
                for (int j = 0; j < 16; ++j) x[j] = lds_f32(stage_s + 4 * (r + 1 + j));
                float y[16];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float4 f = lds_f128(stage_s + 64 + 16 * q);
                    y[4 * q] = f.x; y[4 * q + 1] = f.y; y[4 * q + 2] = f.z; y[4 * q + 3] = f.w;
                }
                v = tree16(x);
                S = tree16(y);
                if (!lane_in) v = 0.0f;
            } else {
                v = w;
#pragma unroll
                for (int st = 0; st < 4; ++st) {
                    const float y = __shfl_up_sync(kFull, v, 1u << st);
                    if (lane >= (1u << st)) v = __fadd_rn(v, y);
                }
                S = __shfl_sync(kFull, v, 15);
            }
            if (V & TM) tc = clk_dep(__float_as_uint(S));
            uint32_t next;
            if (feas) {
                const float u = u01_f32(uw);
                const float target = __fmul_rn(u, S);
                const float tol = __fmul_rn(1e-6f, S);
                uint32_t r;
                if (V & ONE) {
                    const uint32_t last = 31u - __clz(feas);
                    const uint32_t kw = __reduce_min_sync(kFull, (w > 0.0f && (v > target || lane == last)) ? ((lane << 27) | e.x) : kNone);
                    r = kw >> 27;
                    next = kw & 0x07ffffffu;
                } else {
                    const uint32_t kw = __reduce_min_sync(kFull, (w > 0.0f && v > target) ? ((lane << 27) | e.x) : kNone);
                    const uint32_t kf = __reduce_min_sync(kFull, w > 0.0f ? (((31u - lane) << 27) | e.x) : kNone);
                    r = kw != kNone ? (kw >> 27) : 31u - (kf >> 27);
                    next = (kw != kNone ? kw : kf) & 0x07ffffffu;
                }
                const unsigned tie = __ballot_sync(kFull, lane_in && fabsf(__fsub_rn(v, target)) <= tol);
                sts_u32_if(vw_addr, vw | bit, lane == r);
                n_tie += tie ? 1u : 0u;
            } else {
                next = (uint32_t)(((uint64_t)(cur + 1) * 2654435761ull) % n);
                if (lane == 0) vis[next >> 5] |= 1u << (next & 31);
                ++n_fb;
            }
            if (V & TM) td = clk_dep(next);
            e_pre = ldg_u64_if(row_base + (size_t)next * 16, lane_in, make_uint2(next, 0u));
            stg_u32_if(out + t, next, lane == 0);
            cur = next;
            if (V & TM) {
                s1 += ta - tprev; s2 += tb - ta; s3 += tc - tb; s4 += td - tc;
                tprev = td;
            }
        }
    }
    const long long t1 = clock64();
    if (lane == 0) {
        cyc[ant] = t1 - t0;
        atomicAdd(&seg[0], (unsigned long long)n_fb);
        atomicAdd(&seg[1], (unsigned long long)n_tie);
        if (V & TM) {
            atomicAdd(&seg[2], (unsigned long long)s1); atomicAdd(&seg[3], (unsigned long long)s2);
            atomicAdd(&seg[4], (unsigned long long)s3); atomicAdd(&seg[5], (unsigned long long)s4);
        }
    }
}

std::vector<uint32_t> g_ref;

template <int V>
void run(const char* name, const uint2* cand, uint32_t n, uint32_t D, uint32_t m, uint32_t* tours, long long* cyc,
         unsigned long long* seg) {
    const size_t smem = 1152 + ((n + 31) / 32) * 4 + 16 + 512;
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
        printf("    segments: row-wait %.0f probe %.0f scan+S %.0f pick %.0f\n", sg[2] / d, sg[3] / d, sg[4] / d, sg[5] / d);
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
    cudaMalloc(&tours, (size_t)2048 * D * 4); cudaMalloc(&cyc, 2048 * 8); cudaMalloc(&seg, 64);
    printf("n=%u m=%u D=%u\n", n, m, D);
    for (uint32_t mm : {1024u, 740u, 444u, 296u, 148u, 1u}) {
        run<0>("baseline", cand, n, D, mm, tours, cyc, seg);
        run<ONE>("one redux", cand, n, D, mm, tours, cyc, seg);
        run<TREE | ONE>("tree + one", cand, n, D, mm, tours, cyc, seg);
        run<TREE4 | ONE>("tree4 + one", cand, n, D, mm, tours, cyc, seg);
    }
    run<TREE4 | ONE | TM>("tree4 + one (timed)", cand, n, D, 1024, tours, cyc, seg);
    return 0;
}
