// Decision-loop study (round 2): the K2 loop (byte probe, vote, Hillis-Steele shuffle scan,
// S shuffle, one redux.min pick, deferred tie test) against shuffle-free roulettes in which
// every lane reads the whole candidate row's weights from L1 (uniform-address loads of a
// row the previous decision pulled into L1) and forms its own inclusive prefix S_r and the
// total S with one fixed pairwise tree over the 16 feasibility-masked weights:
//   BASE  - the engine's loop ({city, w} rows, 8 B per lane);
//   ROW2  - split rows [16 cities | 16 weights]: per lane LDG.32 of its city + 4 LDG.128 of
//           the weights; prefix and total as one f32x2 tree (15 packed adds);
//   ROW1  - the same with scalar adds (30);
//   ROWI  - {city, w} rows: 8 LDG.128 per lane, packed tree.
//   WLDG  - L1 warming by four plain 4-byte loads per lane into registers folded into a sink
//           one decision later, instead of cp.async.ca copies into a shared-memory slot;
//   TM    - clock64 segments (the clock read does not wait for its "dependency": the first
//           segment boundary is issue time, so pick->row + row->probe is what is meaningful).
// ROW* choose identical tours among themselves (same association); BASE differs (Hillis-
// Steele association). Results: profiles/r02_ubench_decision4.txt, profiles/README.md
// (round 2). Single file; build:
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false -I../../paper_1709_03187_b200/csrc ub_decision4.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include "device.cuh"
using namespace pacob200;

enum : int { BASE = 0, ROW2 = 1, ROW1 = 2, ROWI = 4, NOWARM = 8, TM = 16, WLDG = 32, WPF = 64, WPF2 = 128 };
__device__ __forceinline__ uint32_t ldg_ca_u32_if(const void* p, bool cond) {
    uint32_t v = 0;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.global.ca.u32 %0, [%1];\n\t}" : "+r"(v) : "l"(p), "r"((uint32_t)cond));
    return v;
}
__device__ __forceinline__ long long clk_dep(uint32_t dep) {
    long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c) : "r"(dep) : "memory");
    return c;
}

__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) { uint32_t v; asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr)); return v; }
__device__ __forceinline__ void sts_u8_if(uint32_t addr, uint32_t v, bool cond) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.shared.u8 [%0], %1;\n\t}" ::"r"(addr), "r"(v),
                 "r"((uint32_t)cond) : "memory");
}
__device__ __forceinline__ void cp_async16_if(uint32_t dst, const void* src, bool cond) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q cp.async.ca.shared.global [%0], [%1], 16;\n\t}" ::"r"(dst), "l"(src), "r"((uint32_t)cond));
}
__device__ __forceinline__ uint32_t ldg_u32_if(const uint32_t* p, bool cond, uint32_t v) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.global.u32 %0, [%1];\n\t}" : "+r"(v) : "l"(p), "r"((uint32_t)cond));
    return v;
}
__device__ __forceinline__ float4 ldg_f128(const void* p) {
    float4 v;
    asm volatile("ld.global.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ unsigned long long pk(float a, float b) {
    unsigned long long x;
    asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a), "f"(b));
    return x;
}
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b) {
    unsigned long long z;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(z) : "l"(a), "l"(b));
    return z;
}
__device__ __forceinline__ void unpk(unsigned long long x, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(x));
}
// fixed pairwise tree: ((((x15+x14)+(x13+x12))+((x11+x10)+(x9+x8))) + (((x7+x6)+(x5+x4))+((x3+x2)+(x1+x0))))
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
__device__ __forceinline__ unsigned long long tree16x2(const unsigned long long (&x)[16]) {
    unsigned long long a[8], b[4], c[2];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = add2(x[2 * i + 1], x[2 * i]);
#pragma unroll
    for (int i = 0; i < 4; ++i) b[i] = add2(a[2 * i + 1], a[2 * i]);
#pragma unroll
    for (int i = 0; i < 2; ++i) c[i] = add2(b[2 * i + 1], b[2 * i]);
    return add2(c[1], c[0]);
}

template <int V>
__global__ void __launch_bounds__(32, 1) dec(const uint2* __restrict__ cand, const uint32_t* __restrict__ split, uint32_t n,
                                             uint32_t D, uint32_t* tours, long long* cyc, unsigned long long* seg) {
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
    const bool lane_in = lane < 16;
    const uint32_t lemask = lane_in ? (2u << lane) - 1u : 0xffffu;
    constexpr bool SPLIT = (V & (ROW1 | ROW2)) != 0;
    constexpr bool ROWV = (V & (ROW1 | ROW2 | ROWI)) != 0;
    const uint2* row_base = cand + lane;
    // current row: per-lane entry (city, w) and, for ROW*, all 16 weights
    uint2 e_pre;
    float wr_pre[16];
    auto load_row = [&](uint32_t c, uint2& e, float (&wr)[16]) {
        if (SPLIT) {
            const uint32_t* r = split + (size_t)c * 32;
            e = make_uint2(ldg_u32_if(r + lane, lane_in, c), 0u);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float4 f = ldg_f128(r + 16 + 4 * q);
                wr[4 * q] = f.x; wr[4 * q + 1] = f.y; wr[4 * q + 2] = f.z; wr[4 * q + 3] = f.w;
            }
        } else {
            e = ldg_u64_if(row_base + (size_t)c * 16, lane_in, make_uint2(c, 0u));
            if (V & ROWI) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const float4 f = ldg_f128(cand + (size_t)c * 16 + 2 * q);
                    wr[2 * q] = f.y; wr[2 * q + 1] = f.w;
                }
            }
        }
    };
    load_row(cur, e_pre, wr_pre);
    uint32_t n_fb = 0, n_tie = 0;
    float tie_v = 0.0f, tie_t = 0.0f, tie_tol = -1.0f;
    const long long t0 = clock64();
    long long cprev = t0, sg[5] = {0, 0, 0, 0, 0};
    uint32_t sink = 0, wd_prev[4] = {0, 0, 0, 0};
    for (uint32_t b0 = 0; b0 < D; b0 += 128) {
        const uint4 pb = philox10(make_uint4(1 + (b0 >> 2) + lane, ant, 0, 0), key);
        const uint32_t b1 = b0 + 128 < D ? b0 + 128 : D;
#pragma unroll 2
        for (uint32_t t = b0; t < b1; ++t) {
            __syncwarp();
            const uint2 e = e_pre;
            long long c0 = 0, c1 = 0, c2 = 0, c3 = 0, c4 = 0;
            if (V & TM) c0 = clk_dep(e.x);
            float wr[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) wr[j] = wr_pre[j];
            n_tie += __ballot_sync(kFull, lane_in && fabsf(__fsub_rn(tie_v, tie_t)) <= tie_tol) ? 1u : 0u;
            const uint32_t vw_addr = vis_s + (e.x >> 3);
            const uint32_t vw = lds_u8(vw_addr);
            const uint32_t uw = __shfl_sync(kFull, pick_word(pb, t & 3), (t & 127) >> 2);
            const uint32_t bit = 1u << (e.x & 7);
            const bool fe = lane_in && !(vw & bit);
            if (V & TM) c1 = clk_dep(vw);
            uint32_t wd[4] = {0, 0, 0, 0};
            if (V & WLDG) {
                const unsigned char* src = SPLIT ? reinterpret_cast<const unsigned char*>(split + (size_t)e.x * 32)
                                                 : reinterpret_cast<const unsigned char*>(cand + (size_t)e.x * 16);
#pragma unroll
                for (int c = 0; c < 4; ++c) wd[c] = ldg_ca_u32_if(src + 32 * c, fe);
            } else if (V & (WPF | WPF2)) {
                const unsigned char* src = SPLIT ? reinterpret_cast<const unsigned char*>(split + (size_t)e.x * 32)
                                                 : reinterpret_cast<const unsigned char*>(cand + (size_t)e.x * 16);
                if (fe) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(src + 32 * c));
                    }
                }
            } else if (!(V & NOWARM)) {
                const unsigned char* src = SPLIT ? reinterpret_cast<const unsigned char*>(split + (size_t)e.x * 32)
                                                 : reinterpret_cast<const unsigned char*>(cand + (size_t)e.x * 16);
#pragma unroll
                for (int c = 0; c < 4; ++c) cp_async16_if(warm_s, src + 32 * c, fe);
            }
            const unsigned feas = __ballot_sync(kFull, ROWV ? fe : (fe && __uint_as_float(e.y) > 0.0f));
            const bool is_last = lane == 31u - __clz(feas);
            const uint32_t pick_key = (lane << 27) | e.x;
            float v, S;
            if (ROWV) {
                const uint32_t P = feas & lemask;
                if (V & ROW1) {
                    float x[16], y[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        x[j] = ((P >> j) & 1u) ? wr[j] : 0.0f;
                        y[j] = ((feas >> j) & 1u) ? wr[j] : 0.0f;
                    }
                    v = tree16(x);
                    S = tree16(y);
                } else {
                    unsigned long long x[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        x[j] = pk(((P >> j) & 1u) ? wr[j] : 0.0f, ((feas >> j) & 1u) ? wr[j] : 0.0f);
                    unpk(tree16x2(x), v, S);
                }
            } else {
                v = fe ? __uint_as_float(e.y) : 0.0f;
#pragma unroll
                for (int st = 0; st < 4; ++st) {
                    const float y = __shfl_up_sync(kFull, v, 1u << st);
                    if (lane >= (1u << st)) v = __fadd_rn(v, y);
                }
                S = __shfl_sync(kFull, v, 15);
            }
            if (V & TM) c2 = clk_dep(__float_as_uint(v));
            if (V & TM) c3 = clk_dep(__float_as_uint(S));
            uint32_t next;
            if (feas) {
                const float u = u01_f32(uw);
                const float target = __fmul_rn(u, S);
                const float tol = __fmul_rn(1e-6f, S);
                const bool win = (fe & (v > target)) | is_last;
                const uint32_t kw = __reduce_min_sync(kFull, win ? pick_key : kNone);
                tie_v = v; tie_t = target; tie_tol = tol;
                const uint32_t r = kw >> 27;
                next = kw & 0x07ffffffu;
                sts_u8_if(vw_addr, vw | bit, lane == r);
                if (V & WLDG) sink ^= wd_prev[0] ^ wd_prev[1] ^ wd_prev[2] ^ wd_prev[3];
            } else {
                next = (uint32_t)(((uint64_t)(cur + 1) * 2654435761ull) % n);
                tie_tol = -1.0f;
                if (lane == 0) vis[next >> 5] |= 1u << (next & 31);
                ++n_fb;
            }
            if (V & TM) {
                c4 = clk_dep(next);
                sg[0] += c0 - cprev; sg[1] += c1 - c0; sg[2] += c2 - c1; sg[3] += c3 - c2; sg[4] += c4 - c3;
                cprev = c4;
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) wd_prev[c] = wd[c];
            load_row(next, e_pre, wr_pre);
            stg_u32_if(out + t, next, lane == 0);
            cur = next;
        }
    }
    const long long t1 = clock64();
    if (lane == 0) {
        cyc[ant] = t1 - t0 + (sink == 0x12345u ? 1 : 0);
        atomicAdd(&seg[0], (unsigned long long)n_fb);
        atomicAdd(&seg[1], (unsigned long long)n_tie);
        if (V & TM)
            for (int q = 0; q < 5; ++q) atomicAdd(&seg[2 + q], (unsigned long long)sg[q]);
    }
}

std::vector<uint32_t> g_ref;

// HELPER: warp 0 builds the tour with no L1-warming copies of its own; warp 1 of the same
// CTA watches the city warp 0 has just moved to (a shared-memory sequence number) and pulls
// the rows of all of that city's candidates into L1 with cp.async.ca. GVIS: the visited
// bitmap in global memory (L1-cached byte loads / stores) instead of shared memory, with
// warp 0's own cp.async warming. Both test whether the bitmap probe (LDS) waits behind the
// same warp's LDGSTS.
template <int V>
__global__ void __launch_bounds__(64, 1) dec_helper(const uint2* __restrict__ cand, uint32_t n, uint32_t D,
                                                    uint32_t* tours, long long* cyc, unsigned char* gvis_all) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, ant = blockIdx.x, nw = (n + 31) / 32;
    constexpr bool GV = (V & 1) != 0;   // global bitmap
    constexpr bool HLP = (V & 2) != 0;  // helper warp warms
    volatile uint32_t* seq = reinterpret_cast<volatile uint32_t*>(smem);  // [0] seq, [1] city, [2] done
    uint32_t* vis = reinterpret_cast<uint32_t*>(smem + 64);
    unsigned char* gvis = gvis_all + (size_t)ant * nw * 4;
    if (warp == 0) {
        for (uint32_t w = lane; w < nw; w += 32) { vis[w] = 0u; if (GV) reinterpret_cast<uint32_t*>(gvis)[w] = 0u; }
    }
    if (threadIdx.x == 0) { seq[0] = 0; seq[1] = 0; seq[2] = 0; }
    __syncthreads();
    const uint32_t vis_s = (uint32_t)__cvta_generic_to_shared(vis);
    const uint32_t warm_s = ((vis_s + nw * 4 + 15) & ~15u) + (threadIdx.x & 63) * 16;
    uint32_t cur = (ant * 977u) % n;
    if (warp == 1) {
        if (!HLP) return;
        uint32_t last = 0;
        for (;;) {
            uint32_t s0;
            do { s0 = seq[0]; } while (s0 == last && !seq[2]);
            if (seq[2]) break;
            last = s0;
            const uint32_t c = seq[1];
            const uint2 e = ldg_u64_if(cand + (size_t)c * 16 + lane, lane < 16, make_uint2(c, 0u));
            const unsigned char* src = reinterpret_cast<const unsigned char*>(cand + (size_t)e.x * 16);
#pragma unroll
            for (int q = 0; q < 4; ++q) cp_async16_if(warm_s, src + 32 * q, lane < 16);
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        return;
    }
    if (lane == 0) { vis[cur >> 5] |= 1u << (cur & 31); if (GV) gvis[cur >> 3] |= 1u << (cur & 7); }
    __syncwarp();
    uint32_t* out = tours + (size_t)ant * D;
    const uint2 key = make_uint2(7u, 0u);
    const bool lane_in = lane < 16;
    const uint2* row_base = cand + lane;
    uint2 e_pre = ldg_u64_if(row_base + (size_t)cur * 16, lane_in, make_uint2(cur, 0u));
    uint32_t n_tie = 0;
    float tie_v = 0.0f, tie_t = 0.0f, tie_tol = -1.0f;
    const long long t0 = clock64();
    for (uint32_t b0 = 0; b0 < D; b0 += 128) {
        const uint4 pb = philox10(make_uint4(1 + (b0 >> 2) + lane, ant, 0, 0), key);
        const uint32_t b1 = b0 + 128 < D ? b0 + 128 : D;
#pragma unroll 2
        for (uint32_t t = b0; t < b1; ++t) {
            __syncwarp();
            const uint2 e = e_pre;
            n_tie += __ballot_sync(kFull, lane_in && fabsf(__fsub_rn(tie_v, tie_t)) <= tie_tol) ? 1u : 0u;
            const uint32_t vw_addr = vis_s + (e.x >> 3);
            uint32_t vw;
            if (GV) {
                asm volatile("ld.global.u8 %0, [%1];" : "=r"(vw) : "l"(gvis + (e.x >> 3)));
            } else {
                vw = lds_u8(vw_addr);
            }
            const uint32_t uw = __shfl_sync(kFull, pick_word(pb, t & 3), (t & 127) >> 2);
            const uint32_t bit = 1u << (e.x & 7);
            const bool fe = lane_in && !(vw & bit);
            if (!HLP) {
                const unsigned char* src = reinterpret_cast<const unsigned char*>(cand + (size_t)e.x * 16);
#pragma unroll
                for (int c = 0; c < 4; ++c) cp_async16_if(warm_s, src + 32 * c, fe);
            }
            const unsigned feas = __ballot_sync(kFull, fe);
            const bool is_last = lane == 31u - __clz(feas);
            const uint32_t pick_key = (lane << 27) | e.x;
            float v = fe ? __uint_as_float(e.y) : 0.0f;
#pragma unroll
            for (int st = 0; st < 4; ++st) {
                const float y = __shfl_up_sync(kFull, v, 1u << st);
                if (lane >= (1u << st)) v = __fadd_rn(v, y);
            }
            const float S = __shfl_sync(kFull, v, 15);
            uint32_t next;
            if (feas) {
                const float u = u01_f32(uw);
                const float target = __fmul_rn(u, S);
                const float tol = __fmul_rn(1e-6f, S);
                const bool win = (fe & (v > target)) | is_last;
                const uint32_t kw = __reduce_min_sync(kFull, win ? pick_key : kNone);
                tie_v = v; tie_t = target; tie_tol = tol;
                const uint32_t r = kw >> 27;
                next = kw & 0x07ffffffu;
                if (GV) {
                    if (lane == r) asm volatile("st.global.u8 [%0], %1;" :: "l"(gvis + (e.x >> 3)), "r"(vw | bit) : "memory");
                } else {
                    sts_u8_if(vw_addr, vw | bit, lane == r);
                }
            } else {
                next = (uint32_t)(((uint64_t)(cur + 1) * 2654435761ull) % n);
                tie_tol = -1.0f;
                if (lane == 0) {
                    vis[next >> 5] |= 1u << (next & 31);
                    if (GV) gvis[next >> 3] |= 1u << (next & 7);
                }
            }
            if (HLP && lane == 0) { seq[1] = next; __threadfence_block(); seq[0] = t + 1; }
            e_pre = ldg_u64_if(row_base + (size_t)next * 16, lane_in, make_uint2(next, 0u));
            stg_u32_if(out + t, next, lane == 0);
            cur = next;
        }
    }
    const long long t1 = clock64();
    if (lane == 0) { seq[2] = 1; cyc[ant] = t1 - t0 + (n_tie == 0xffffffffu); }
    asm volatile("cp.async.wait_all;" ::: "memory");
}

template <int V>
void run_helper(const char* name, const uint2* cand, uint32_t n, uint32_t D, uint32_t m, uint32_t* tours, long long* cyc,
                unsigned char* gvis) {
    const size_t smem = 64 + ((n + 31) / 32) * 4 + 16 + 1024;
    cudaFuncSetAttribute(dec_helper<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(dec_helper<V>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    dec_helper<V><<<m, 64, smem>>>(cand, n, D, tours, cyc, gvis);
    cudaEventRecord(a);
    dec_helper<V><<<m, 64, smem>>>(cand, n, D, tours, cyc, gvis);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    std::vector<long long> h(m); cudaMemcpy(h.data(), cyc, m * 8, cudaMemcpyDeviceToHost);
    double mean = 0, mx = 0; for (auto v : h) { mean += v; mx = v > mx ? v : mx; }
    mean /= m;
    std::vector<uint32_t> got((size_t)m * D);
    cudaMemcpy(got.data(), tours, got.size() * 4, cudaMemcpyDeviceToHost);
    const char* same = "";
    if (m == 1024) same = (g_ref == got) ? "same tours" : "TOURS DIFFER";
    printf("%-22s m=%-4u %6.1f cyc/dec (max ant %6.1f) %8.3f ms %s %s\n", name, m, mean / D, mx / D, ms, same,
           cudaGetErrorString(cudaGetLastError()));
}

template <int V>
void run(const char* name, const uint2* cand, const uint32_t* split, uint32_t n, uint32_t D, uint32_t m, uint32_t* tours,
         long long* cyc, unsigned long long* seg, bool reset_ref) {
    const size_t smem = ((n + 31) / 32) * 4 + 16 + 512;
    cudaFuncSetAttribute(dec<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(dec<V>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    dec<V><<<m, 32, smem>>>(cand, split, n, D, tours, cyc, seg);
    cudaMemset(seg, 0, 64);
    cudaEventRecord(a);
    dec<V><<<m, 32, smem>>>(cand, split, n, D, tours, cyc, seg);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    std::vector<long long> h(m); cudaMemcpy(h.data(), cyc, m * 8, cudaMemcpyDeviceToHost);
    unsigned long long sg[8]; cudaMemcpy(sg, seg, 64, cudaMemcpyDeviceToHost);
    double mean = 0, mx = 0; for (auto v : h) { mean += v; mx = v > mx ? v : mx; }
    mean /= m;
    std::vector<uint32_t> got((size_t)m * D);
    cudaMemcpy(got.data(), tours, got.size() * 4, cudaMemcpyDeviceToHost);
    const char* same = "";
    if (m == 1024) {
        if (reset_ref) g_ref = got;
        same = (g_ref == got) ? "same tours" : "TOURS DIFFER";
    }
    const double d = (double)m * D;
    if (V & TM)
        printf("    segments (cycles/decision): pick->row %.0f  row->probe %.0f  probe->v %.0f  v->S %.0f  S->next %.0f\n",
               sg[2] / d, sg[3] / d, sg[4] / d, sg[5] / d, sg[6] / d);
    printf("%-22s m=%-4u %6.1f cyc/dec (max ant %6.1f) %8.3f ms fb %.3f%% ties %llu %s %s\n", name, m, mean / D, mx / D, ms,
           100.0 * sg[0] / d, sg[1], same, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const uint32_t n = 200000, m = 1024, D = 20000;
    std::mt19937 rng(5);
    std::vector<uint2> h((size_t)n * 16);
    std::vector<uint32_t> hs((size_t)n * 32);
    std::uniform_int_distribution<int> off(-300, 300);
    std::uniform_real_distribution<float> wd(0.1f, 1.0f);
    for (uint32_t i = 0; i < n; ++i)
        for (int r = 0; r < 16; ++r) {
            int o = off(rng); if (o == 0) o = 1;
            const uint32_t c = (uint32_t)(((int64_t)i + o + n) % n);
            const float w = wd(rng);
            h[(size_t)i * 16 + r] = make_uint2(c, __builtin_bit_cast(uint32_t, w));
            hs[(size_t)i * 32 + r] = c;
            hs[(size_t)i * 32 + 16 + r] = __builtin_bit_cast(uint32_t, w);
        }
    uint2* cand; uint32_t* split; uint32_t* tours; long long* cyc; unsigned long long* seg;
    cudaMalloc(&cand, h.size() * 8); cudaMemcpy(cand, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMalloc(&split, hs.size() * 4); cudaMemcpy(split, hs.data(), hs.size() * 4, cudaMemcpyHostToDevice);
    cudaMalloc(&tours, (size_t)2048 * D * 4); cudaMalloc(&cyc, 2048 * 8); cudaMalloc(&seg, 64);
    printf("n=%u m=%u D=%u\n", n, m, D);
    run<BASE | TM>("base timed", cand, split, n, D, 1, tours, cyc, seg, true);
    run<ROW1 | TM>("row f32 timed", cand, split, n, D, 1, tours, cyc, seg, true);
    unsigned char* gvis; cudaMalloc(&gvis, (size_t)2048 * ((n + 31) / 32) * 4);
    for (uint32_t mm : {1u, 148u, 1024u}) {
        run<BASE>("base (engine loop)", cand, split, n, D, mm, tours, cyc, seg, true);
        run_helper<0>("2-warp CTA, own warm", cand, n, D, mm, tours, cyc, gvis);
        run_helper<2>("helper-warp warming", cand, n, D, mm, tours, cyc, gvis);
        run_helper<1>("global bitmap", cand, n, D, mm, tours, cyc, gvis);
        run_helper<3>("global bitmap + helper", cand, n, D, mm, tours, cyc, gvis);
    }
    run<BASE | TM | NOWARM>("base nowarm timed", cand, split, n, D, 1, tours, cyc, seg, true);
    run<BASE | TM | WLDG>("base ldg-warm timed", cand, split, n, D, 1, tours, cyc, seg, true);
    run<BASE | TM>("base timed", cand, split, n, D, 1024, tours, cyc, seg, true);
    run<BASE | TM | WLDG>("base ldg-warm timed", cand, split, n, D, 1024, tours, cyc, seg, false);
    for (uint32_t mm : {1024u, 148u, 1u}) {
        run<BASE>("base (engine loop)", cand, split, n, D, mm, tours, cyc, seg, true);
        run<BASE | WPF>("base prefetch.L1 warm", cand, split, n, D, mm, tours, cyc, seg, false);
        run<BASE | NOWARM>("base no warm", cand, split, n, D, mm, tours, cyc, seg, false);
    }
    for (uint32_t mm : {1024u, 444u, 148u, 1u}) {
        run<BASE>("base (engine loop)", cand, split, n, D, mm, tours, cyc, seg, true);
        run<BASE | WLDG>("base ldg-warm", cand, split, n, D, mm, tours, cyc, seg, false);
        run<ROW1 | WLDG>("row f32 ldg-warm", cand, split, n, D, mm, tours, cyc, seg, true);
    }
    for (uint32_t mm : {1024u, 444u, 148u, 1u}) {
        run<BASE>("base (engine loop)", cand, split, n, D, mm, tours, cyc, seg, true);
        run<ROW2>("row split, f32x2 tree", cand, split, n, D, mm, tours, cyc, seg, true);
        run<ROW1>("row split, f32 tree", cand, split, n, D, mm, tours, cyc, seg, false);
        run<ROWI>("row {c,w}, f32x2 tree", cand, split, n, D, mm, tours, cyc, seg, false);
    }
    return 0;
}
