// Decision-loop anatomy: the K2 inner loop (one warp per ant, bitmap in shared memory,
// 16 candidates per row, shuffle scan + ballots) on a synthetic 200k-city candidate
// table, with pieces switched off one at a time to attribute the per-decision latency.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false -I../../paper_1709_03187_b200/csrc ub_decision.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include "device.cuh"
using namespace pacob200;

enum : int { NOATOM = 1, NOSTG = 2, NOWARM = 4, NOTIE = 8, SMALL = 16, NOSCAN = 32, NOSYNC = 64, NOPHILOX = 128,
             STSMARK = 256, R2 = 512, R2SHFL = 1024, R2FADD2 = 2048, S1 = 4096, S1SEL = 8192, PF = 16384, PFF = 32768 };

__device__ __forceinline__ uint4 ldg_v4(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ void fadd2(float& a0, float& a1, float b0, float b1) {
    unsigned long long x, y, z;
    asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a0), "f"(a1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(y) : "f"(b0), "f"(b1));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(z) : "l"(x), "l"(y));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(z));
}

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) { uint32_t v; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr)); return v; }
__device__ __forceinline__ void cp_async16_if(uint32_t dst, const void* src, bool cond) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q cp.async.ca.shared.global [%0], [%1], 16;\n\t}" ::"r"(dst), "l"(src), "r"((uint32_t)cond));
}
__device__ __forceinline__ void sts_u32_if(uint32_t addr, uint32_t v, bool cond) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.shared.u32 [%0], %1;\n\t}" ::"r"(addr), "r"(v), "r"((uint32_t)cond) : "memory");
}

template <int V>
__global__ void __launch_bounds__(32, 1) dec(const uint2* __restrict__ cand, uint32_t n, uint32_t D, uint32_t* tours,
                                             long long* cyc, unsigned long long* fbs) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t lane = threadIdx.x, ant = blockIdx.x, nw = (n + 31) / 32;
    uint32_t* vis = reinterpret_cast<uint32_t*>(smem);
    for (uint32_t w = lane; w < nw; w += 32) vis[w] = 0u;
    __syncwarp();
    const uint32_t vis_s = (uint32_t)__cvta_generic_to_shared(vis);
    const uint32_t warm_s = ((vis_s + nw * 4 + 15) & ~15u) + lane * 16;
    const uint32_t tab = (V & SMALL) ? 512u : n;
    uint32_t cur = (ant * 977u) % tab;
    if (lane == 0) vis[cur >> 5] |= 1u << (cur & 31);
    __syncwarp();
    uint32_t* out = tours + (size_t)ant * D;
    const uint2 key = make_uint2(7u, 0u);
    uint4 pb = philox10(make_uint4(1 + lane, ant, 0, 0), key);
    uint32_t uw = __shfl_sync(kFull, pb.x, 0);
    const bool lane_in = lane < 16;
    const uint2* row_base = cand + lane;
    uint2 e_pre = ldg_u64_if(row_base + (size_t)cur * 16, lane_in, make_uint2(cur, 0u));
    uint32_t n_fb = 0, n_tie = 0;
    const long long t0 = clock64();
    for (uint32_t t = 0; t < D; ++t) {
        if (!(V & NOSYNC)) __syncwarp();
        const uint2 e = e_pre;
        const uint32_t vw = lds_u32(vis_s + ((e.x >> 5) << 2));
        const float w = ((vw >> (e.x & 31)) & 1u) ? 0.0f : __uint_as_float(e.y);
        float v = w;
        if (!(V & NOWARM)) {
            const unsigned char* src = reinterpret_cast<const unsigned char*>(cand + (size_t)e.x * 16);
#pragma unroll
            for (int c = 0; c < 4; ++c) cp_async16_if(warm_s, src + 32 * c, w > 0.0f);
        }
        if (!(V & NOSCAN)) {
#pragma unroll
            for (int st = 0; st < 4; ++st) {
                const float y = __shfl_up_sync(kFull, v, 1u << st);
                if (lane >= (1u << st)) v = __fadd_rn(v, y);
            }
        }
        const float u = u01_f32(uw);
        const float S = __shfl_sync(kFull, v, 15);
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
            // stand-in fallback: jump to a pseudo-random unvisited-ish city
            next = (uint32_t)(((uint64_t)(cur + 1) * 2654435761ull) % tab);
            ++n_fb;
        }
        e_pre = ldg_u64_if(row_base + (size_t)next * 16, lane_in, make_uint2(next, 0u));
        if (!(V & NOATOM)) {
            if (V & STSMARK) sts_u32_if(vis_s + ((next >> 5) << 2), 1u << (next & 31), lane == 0);
            else red_or_shared_if(vis_s + ((next >> 5) << 2), 1u << (next & 31), lane == 0);
        }
        if (!(V & NOSTG)) stg_u32_if(out + t, next, lane == 0);
        cur = next;
        if (!(V & NOPHILOX)) {
            const uint32_t t1 = t + 1;
            if ((t1 & 127) == 0) pb = philox10(make_uint4(1 + (t1 >> 2) + lane, ant, 0, 0), key);
            uw = __shfl_sync(kFull, pick_word(pb, t1 & 3), (t1 & 127) >> 2);
        } else {
            uw = uw * 1664525u + 1013904223u;
        }
    }
    const long long t1 = clock64();
    asm volatile("cp.async.wait_all;" ::: "memory");
    if (lane == 0) { cyc[ant] = t1 - t0; atomicAdd(fbs, (unsigned long long)n_fb + 0ull * n_tie); out[0] ^= cur; }
}

// Redundant-register roulette: every lane holds the whole 16-entry row (8 broadcast
// 16-byte loads), feasibility is one ballot over the per-lane bitmap probes, and the
// Hillis-Steele scan, the pick and the tie test run in registers with the same f32
// association as the shuffle scan (v_r += v_{r-d}, old values, d = 1, 2, 4, 8).
template <int V>
__global__ void __launch_bounds__(32, 1) dec_r2(const uint2* __restrict__ cand, uint32_t n, uint32_t D, uint32_t* tours,
                                                long long* cyc, unsigned long long* fbs) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t lane = threadIdx.x, ant = blockIdx.x, nw = (n + 31) / 32;
    uint32_t* vis = reinterpret_cast<uint32_t*>(smem);
    for (uint32_t w = lane; w < nw; w += 32) vis[w] = 0u;
    __syncwarp();
    const uint32_t vis_s = (uint32_t)__cvta_generic_to_shared(vis);
    const uint32_t tab = n;
    uint32_t cur = (ant * 977u) % tab;
    if (lane == 0) vis[cur >> 5] |= 1u << (cur & 31);
    __syncwarp();
    uint32_t* out = tours + (size_t)ant * D;
    const uint2 key = make_uint2(7u, 0u);
    uint4 pb = philox10(make_uint4(1 + lane, ant, 0, 0), key);
    uint32_t uw = __shfl_sync(kFull, pb.x, 0);
    const bool lane_in = lane < 16;
    const uint2* row_base = cand + lane;
    const uint4* rowv = reinterpret_cast<const uint4*>(cand);
    uint2 e_pre = ldg_u64_if(row_base + (size_t)cur * 16, lane_in, make_uint2(cur, 0u));
    uint4 rv_pre[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) rv_pre[q] = ldg_v4(rowv + (size_t)cur * 8 + q);
    uint32_t n_fb = 0, n_tie = 0;
    const long long t0 = clock64();
    for (uint32_t t = 0; t < D; ++t) {
        __syncwarp();
        const uint2 e = e_pre;
        uint4 rv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) rv[q] = rv_pre[q];
        const uint32_t vw = lds_u32(vis_s + ((e.x >> 5) << 2));
        const bool feasible = lane_in && !((vw >> (e.x & 31)) & 1u) && __uint_as_float(e.y) > 0.0f;
        const unsigned feas = __ballot_sync(kFull, feasible);
        float v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const uint32_t wb = (r & 1) ? rv[r >> 1].w : rv[r >> 1].y;
            v[r] = ((feas >> r) & 1u) ? __uint_as_float(wb) : 0.0f;
        }
#pragma unroll
        for (int d = 1; d < 16; d <<= 1) {
            if ((V & R2FADD2) && d >= 2) {
#pragma unroll
                for (int r = 14; r >= d; r -= 2) fadd2(v[r], v[r + 1], v[r - d], v[r + 1 - d]);
            } else {
#pragma unroll
                for (int r = 15; r >= d; --r) v[r] = __fadd_rn(v[r], v[r - d]);
            }
        }
        const float u = u01_f32(uw);
        const float S = v[15];
        uint32_t next;
        if (S > 0.0f) {
            const float target = __fmul_rn(u, S);
            const float tol = __fmul_rn(1e-6f, S);
            unsigned mk = 0;
            bool tie = false;
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                mk |= (((feas >> r) & 1u) && v[r] > target) ? (1u << r) : 0u;
                tie |= fabsf(__fsub_rn(v[r], target)) <= tol;
            }
            const int r = mk ? __ffs(mk) - 1 : 31 - __clz(feas);
            if (V & R2SHFL) {
                next = __shfl_sync(kFull, e.x, r);
            } else {
                uint32_t c8[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) c8[q] = (r & 1) ? rv[q].z : rv[q].x;
                uint32_t c4[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) c4[q] = (r & 2) ? c8[2 * q + 1] : c8[2 * q];
                const uint32_t c2a = (r & 4) ? c4[1] : c4[0], c2b = (r & 4) ? c4[3] : c4[2];
                next = (r & 8) ? c2b : c2a;
            }
            n_tie += tie ? 1u : 0u;
        } else {
            next = (uint32_t)(((uint64_t)(cur + 1) * 2654435761ull) % tab);
            ++n_fb;
        }
        e_pre = ldg_u64_if(row_base + (size_t)next * 16, lane_in, make_uint2(next, 0u));
#pragma unroll
        for (int q = 0; q < 8; ++q) rv_pre[q] = ldg_v4(rowv + (size_t)next * 8 + q);
        red_or_shared_if(vis_s + ((next >> 5) << 2), 1u << (next & 31), lane == 0);
        stg_u32_if(out + t, next, lane == 0);
        cur = next;
        const uint32_t t1 = t + 1;
        if ((t1 & 127) == 0) pb = philox10(make_uint4(1 + (t1 >> 2) + lane, ant, 0, 0), key);
        uw = __shfl_sync(kFull, pick_word(pb, t1 & 3), (t1 & 127) >> 2);
    }
    const long long t1 = clock64();
    if (lane == 0) { cyc[ant] = t1 - t0; atomicAdd(fbs, (unsigned long long)n_fb + 0ull * n_tie); out[0] ^= cur; }
}

// Sequential-prefix roulette: every lane holds the whole row (8 broadcast 16-byte loads),
// feasibility is one ballot, and lane r computes its own left-to-right prefix sum
// P_r = (((w_0 + w_1) + w_2) + ... + w_r) over feasible candidates and the total S in two
// interleaved FADD chains (adding 0.0 for masked entries is exact). One vote picks the
// lowest feasible lane with P_r > u*S. No shuffle on the chain except the winner's city.
template <int V>
__global__ void __launch_bounds__(32, 1) dec_s1(const uint2* __restrict__ cand, uint32_t n, uint32_t D, uint32_t* tours,
                                                long long* cyc, unsigned long long* fbs) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t lane = threadIdx.x, ant = blockIdx.x, nw = (n + 31) / 32;
    uint32_t* vis = reinterpret_cast<uint32_t*>(smem);
    for (uint32_t w = lane; w < nw; w += 32) vis[w] = 0u;
    __syncwarp();
    const uint32_t vis_s = (uint32_t)__cvta_generic_to_shared(vis);
    const uint32_t tab = n;
    uint32_t cur = (ant * 977u) % tab;
    if (lane == 0) vis[cur >> 5] |= 1u << (cur & 31);
    __syncwarp();
    uint32_t* out = tours + (size_t)ant * D;
    const uint2 key = make_uint2(7u, 0u);
    uint4 pb = philox10(make_uint4(1 + lane, ant, 0, 0), key);
    uint32_t uw = __shfl_sync(kFull, pb.x, 0);
    const bool lane_in = lane < 16;
    const uint32_t lane_mask = lane_in ? (2u << lane) - 1u : 0xffffu;
    const uint2* row_base = cand + lane;
    const uint4* rowv = reinterpret_cast<const uint4*>(cand);
    uint2 e_pre = ldg_u64_if(row_base + (size_t)cur * 16, lane_in, make_uint2(cur, 0u));
    uint4 rv_pre[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) rv_pre[q] = ldg_v4(rowv + (size_t)cur * 8 + q);
    uint32_t n_fb = 0, n_tie = 0;
    const long long t0 = clock64();
    for (uint32_t t = 0; t < D; ++t) {
        __syncwarp();
        const uint2 e = e_pre;
        uint4 rv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) rv[q] = rv_pre[q];
        const uint32_t vw = lds_u32(vis_s + ((e.x >> 5) << 2));
        const bool feasible = lane_in && !((vw >> (e.x & 31)) & 1u) && __uint_as_float(e.y) > 0.0f;
        const unsigned feas = __ballot_sync(kFull, feasible);
        const unsigned own = feas & lane_mask;
        float P = 0.0f, S = 0.0f;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const float wr = __uint_as_float((r & 1) ? rv[r >> 1].w : rv[r >> 1].y);
            S = __fadd_rn(S, ((feas >> r) & 1u) ? wr : 0.0f);
            P = __fadd_rn(P, ((own >> r) & 1u) ? wr : 0.0f);
        }
        const float u = u01_f32(uw);
        uint32_t next;
        if (S > 0.0f) {
            const float target = __fmul_rn(u, S);
            const float tol = __fmul_rn(1e-6f, S);
            const unsigned ball = __ballot_sync(kFull, feasible && P > target);
            const unsigned tie = __ballot_sync(kFull, lane_in && fabsf(__fsub_rn(P, target)) <= tol);
            const int r = ball ? __ffs(ball) - 1 : 31 - __clz(feas);
            if (!(V & S1SEL)) {
                next = __shfl_sync(kFull, e.x, r);
            } else {
                uint32_t c8[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) c8[q] = (r & 1) ? rv[q].z : rv[q].x;
                uint32_t c4[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) c4[q] = (r & 2) ? c8[2 * q + 1] : c8[2 * q];
                const uint32_t c2a = (r & 4) ? c4[1] : c4[0], c2b = (r & 4) ? c4[3] : c4[2];
                next = (r & 8) ? c2b : c2a;
            }
            n_tie += tie ? 1u : 0u;
        } else {
            next = (uint32_t)(((uint64_t)(cur + 1) * 2654435761ull) % tab);
            ++n_fb;
        }
        e_pre = ldg_u64_if(row_base + (size_t)next * 16, lane_in, make_uint2(next, 0u));
#pragma unroll
        for (int q = 0; q < 8; ++q) rv_pre[q] = ldg_v4(rowv + (size_t)next * 8 + q);
        red_or_shared_if(vis_s + ((next >> 5) << 2), 1u << (next & 31), lane == 0);
        stg_u32_if(out + t, next, lane == 0);
        cur = next;
        const uint32_t t1 = t + 1;
        if ((t1 & 127) == 0) pb = philox10(make_uint4(1 + (t1 >> 2) + lane, ant, 0, 0), key);
        uw = __shfl_sync(kFull, pick_word(pb, t1 & 3), (t1 & 127) >> 2);
    }
    const long long t1 = clock64();
    if (lane == 0) { cyc[ant] = t1 - t0; atomicAdd(fbs, (unsigned long long)n_fb + n_tie); out[0] ^= cur; }
}

// Register prefetch of every candidate's row: as soon as the current row is known, lane r
// loads entry r of each candidate q's row (16 coalesced 8-byte loads, one 128-byte line
// each, candidate ids broadcast by shuffle). The winner's entry is then selected from
// registers (uniform index), so the next decision does not wait for an L2 round trip
// that starts only after the pick.
template <int V>
__global__ void __launch_bounds__(32, 1) dec_pf(const uint2* __restrict__ cand, uint32_t n, uint32_t D, uint32_t* tours,
                                                long long* cyc, unsigned long long* fbs) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t lane = threadIdx.x, ant = blockIdx.x, nw = (n + 31) / 32;
    uint32_t* vis = reinterpret_cast<uint32_t*>(smem);
    for (uint32_t w = lane; w < nw; w += 32) vis[w] = 0u;
    __syncwarp();
    const uint32_t vis_s = (uint32_t)__cvta_generic_to_shared(vis);
    const uint32_t tab = n;
    uint32_t cur = (ant * 977u) % tab;
    if (lane == 0) vis[cur >> 5] |= 1u << (cur & 31);
    __syncwarp();
    uint32_t* out = tours + (size_t)ant * D;
    const uint2 key = make_uint2(7u, 0u);
    uint4 pb = philox10(make_uint4(1 + lane, ant, 0, 0), key);
    uint32_t uw = __shfl_sync(kFull, pb.x, 0);
    const bool lane_in = lane < 16;
    const uint2* row_base = cand + lane;
    uint2 e = ldg_u64_if(row_base + (size_t)cur * 16, lane_in, make_uint2(cur, 0u));
    uint32_t n_fb = 0, n_tie = 0;
    const long long t0 = clock64();
    for (uint32_t t = 0; t < D; ++t) {
        __syncwarp();
        uint2 pf[16];
        if (!(V & PFF)) {
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const uint32_t cq = __shfl_sync(kFull, e.x, q);
                pf[q] = ldg_u64_if(row_base + (size_t)cq * 16, lane_in, make_uint2(cq, 0u));
            }
        }
        const uint32_t vw = lds_u32(vis_s + ((e.x >> 5) << 2));
        const float w = ((vw >> (e.x & 31)) & 1u) ? 0.0f : __uint_as_float(e.y);
        if (V & PFF) {
            const unsigned fm = __ballot_sync(kFull, w > 0.0f);
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const uint32_t cq = __shfl_sync(kFull, e.x, q);
                pf[q] = ldg_u64_if(row_base + (size_t)cq * 16, lane_in && ((fm >> q) & 1u), make_uint2(cq, 0u));
            }
        }
        float v = w;
#pragma unroll
        for (int st = 0; st < 4; ++st) {
            const float y = __shfl_up_sync(kFull, v, 1u << st);
            if (lane >= (1u << st)) v = __fadd_rn(v, y);
        }
        const float u = u01_f32(uw);
        const float S = __shfl_sync(kFull, v, 15);
        uint32_t next;
        if (S > 0.0f) {
            const float target = __fmul_rn(u, S);
            const float tol = __fmul_rn(1e-6f, S);
            const unsigned ball = __ballot_sync(kFull, w > 0.0f && v > target);
            const unsigned feas = __ballot_sync(kFull, w > 0.0f);
            const unsigned tie = __ballot_sync(kFull, lane_in && fabsf(__fsub_rn(v, target)) <= tol);
            const int r = ball ? __ffs(ball) - 1 : 31 - __clz(feas);
            uint2 c8[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) c8[q] = (r & 1) ? pf[2 * q + 1] : pf[2 * q];
            uint2 c4[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) c4[q] = (r & 2) ? c8[2 * q + 1] : c8[2 * q];
            const uint2 c2a = (r & 4) ? c4[1] : c4[0], c2b = (r & 4) ? c4[3] : c4[2];
            next = __shfl_sync(kFull, e.x, r);
            e = (r & 8) ? c2b : c2a;
            n_tie += tie ? 1u : 0u;
        } else {
            next = (uint32_t)(((uint64_t)(cur + 1) * 2654435761ull) % tab);
            e = ldg_u64_if(row_base + (size_t)next * 16, lane_in, make_uint2(next, 0u));
            ++n_fb;
        }
        red_or_shared_if(vis_s + ((next >> 5) << 2), 1u << (next & 31), lane == 0);
        stg_u32_if(out + t, next, lane == 0);
        cur = next;
        const uint32_t t1 = t + 1;
        if ((t1 & 127) == 0) pb = philox10(make_uint4(1 + (t1 >> 2) + lane, ant, 0, 0), key);
        uw = __shfl_sync(kFull, pick_word(pb, t1 & 3), (t1 & 127) >> 2);
    }
    const long long t1 = clock64();
    if (lane == 0) { cyc[ant] = t1 - t0; atomicAdd(fbs, (unsigned long long)n_fb + 0ull * n_tie); out[0] ^= cur; }
}

__device__ __forceinline__ long long clk_dep(uint32_t dep) {
    long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c) : "r"(dep) : "memory");
    return c;
}
// Segment timing of the baseline loop (1 = row arrival, 2 = bitmap probe, 3 = scan,
// 4 = total shuffle, 5 = pick, 6 = bookkeeping up to the next decision).
__global__ void __launch_bounds__(32, 1) dec_tm(const uint2* __restrict__ cand, uint32_t n, uint32_t D, uint32_t* tours,
                                                long long* seg) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t lane = threadIdx.x, ant = blockIdx.x, nw = (n + 31) / 32;
    uint32_t* vis = reinterpret_cast<uint32_t*>(smem);
    for (uint32_t w = lane; w < nw; w += 32) vis[w] = 0u;
    __syncwarp();
    const uint32_t vis_s = (uint32_t)__cvta_generic_to_shared(vis);
    uint32_t cur = (ant * 977u) % n;
    if (lane == 0) vis[cur >> 5] |= 1u << (cur & 31);
    __syncwarp();
    uint32_t* out = tours + (size_t)ant * D;
    const uint2 key = make_uint2(7u, 0u);
    uint4 pb = philox10(make_uint4(1 + lane, ant, 0, 0), key);
    uint32_t uw = __shfl_sync(kFull, pb.x, 0);
    const bool lane_in = lane < 16;
    const uint2* row_base = cand + lane;
    uint2 e_pre = ldg_u64_if(row_base + (size_t)cur * 16, lane_in, make_uint2(cur, 0u));
    long long s1 = 0, s2 = 0, s3 = 0, s4 = 0, s5 = 0, s6 = 0;
    long long tprev = clk_dep(0);
    for (uint32_t t = 0; t < D; ++t) {
        __syncwarp();
        const uint2 e = e_pre;
        const long long ta = clk_dep(e.x);
        const uint32_t vw = lds_u32(vis_s + ((e.x >> 5) << 2));
        const float w = ((vw >> (e.x & 31)) & 1u) ? 0.0f : __uint_as_float(e.y);
        const long long tb = clk_dep(__float_as_uint(w));
        float v = w;
#pragma unroll
        for (int st = 0; st < 4; ++st) {
            const float y = __shfl_up_sync(kFull, v, 1u << st);
            if (lane >= (1u << st)) v = __fadd_rn(v, y);
        }
        const long long tc = clk_dep(__float_as_uint(v));
        const float u = u01_f32(uw);
        const float S = __shfl_sync(kFull, v, 15);
        const long long td = clk_dep(__float_as_uint(S));
        uint32_t next;
        if (S > 0.0f) {
            const float target = __fmul_rn(u, S);
            const unsigned ball = __ballot_sync(kFull, w > 0.0f && v > target);
            const unsigned feas = __ballot_sync(kFull, w > 0.0f);
            const int r = ball ? __ffs(ball) - 1 : 31 - __clz(feas);
            next = __shfl_sync(kFull, e.x, r);
        } else {
            next = (uint32_t)(((uint64_t)(cur + 1) * 2654435761ull) % n);
        }
        const long long te = clk_dep(next);
        e_pre = ldg_u64_if(row_base + (size_t)next * 16, lane_in, make_uint2(next, 0u));
        red_or_shared_if(vis_s + ((next >> 5) << 2), 1u << (next & 31), lane == 0);
        stg_u32_if(out + t, next, lane == 0);
        cur = next;
        const uint32_t t1 = t + 1;
        if ((t1 & 127) == 0) pb = philox10(make_uint4(1 + (t1 >> 2) + lane, ant, 0, 0), key);
        uw = __shfl_sync(kFull, pick_word(pb, t1 & 3), (t1 & 127) >> 2);
        const long long tf = clk_dep(uw);
        s1 += ta - tprev; s2 += tb - ta; s3 += tc - tb; s4 += td - tc; s5 += te - td; s6 += tf - te;
        tprev = tf;
    }
    if (lane == 0) {
        atomicAdd((unsigned long long*)&seg[0], (unsigned long long)s1); atomicAdd((unsigned long long*)&seg[1], (unsigned long long)s2);
        atomicAdd((unsigned long long*)&seg[2], (unsigned long long)s3); atomicAdd((unsigned long long*)&seg[3], (unsigned long long)s4);
        atomicAdd((unsigned long long*)&seg[4], (unsigned long long)s5); atomicAdd((unsigned long long*)&seg[5], (unsigned long long)s6);
        out[0] ^= cur;
    }
}

void run_tm(const uint2* cand, uint32_t n, uint32_t D, uint32_t m, uint32_t* tours, long long* seg) {
    const size_t smem = ((n + 31) / 32) * 4 + 16 + 512;
    cudaFuncSetAttribute(dec_tm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(dec_tm, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaMemset(seg, 0, 64);
    dec_tm<<<m, 32, smem>>>(cand, n, D, tours, seg);
    long long h[6]; cudaMemcpy(h, seg, 48, cudaMemcpyDeviceToHost);
    const double d = (double)m * D;
    printf("segments m=%-5u row-wait %.0f  bitmap %.0f  scan %.0f  S %.0f  pick %.0f  tail %.0f  = %.0f cyc/dec\n", m,
           h[0] / d, h[1] / d, h[2] / d, h[3] / d, h[4] / d, h[5] / d, (h[0] + h[1] + h[2] + h[3] + h[4] + h[5]) / d);
}

template <int V>
void run(const char* name, const uint2* cand, uint32_t n, uint32_t D, uint32_t m, uint32_t* tours, long long* cyc,
         unsigned long long* fbs) {
    const size_t smem = ((n + 31) / 32) * 4 + 16 + 512;
    auto kern = (V & (PF | PFF)) ? dec_pf<V> : (V & S1) ? dec_s1<V> : (V & R2) ? dec_r2<V> : dec<V>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    kern<<<m, 32, smem>>>(cand, n, D, tours, cyc, fbs);  // warm-up
    cudaMemset(fbs, 0, 8);
    cudaEventRecord(a);
    kern<<<m, 32, smem>>>(cand, n, D, tours, cyc, fbs);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    std::vector<long long> h(m); cudaMemcpy(h.data(), cyc, m * 8, cudaMemcpyDeviceToHost);
    unsigned long long f; cudaMemcpy(&f, fbs, 8, cudaMemcpyDeviceToHost);
    double mean = 0, mx = 0; for (auto v : h) { mean += v; mx = v > mx ? v : mx; }
    mean /= m;
    printf("%-28s %7.1f cyc/dec (max ant %7.1f)  %8.3f ms  fb %.3f%%  err=%s\n", name, mean / D, mx / D, ms,
           100.0 * f / ((double)m * D), cudaGetErrorString(cudaGetLastError()));
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
    // the SMALL variant wraps ids into [0, 512): remap rows 0..511 to stay inside
    for (uint32_t i = 0; i < 512; ++i)
        for (int r = 0; r < 16; ++r) h[(size_t)i * 16 + r].x %= 512;
    uint2* cand; uint32_t* tours; long long* cyc; unsigned long long* fbs;
    cudaMalloc(&cand, h.size() * 8); cudaMemcpy(cand, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMalloc(&tours, (size_t)m * D * 4); cudaMalloc(&cyc, m * 8); cudaMalloc(&fbs, 8);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("n=%u m=%u D=%u, SM clock attr %d MHz\n", n, m, D, clk / 1000);
    run<0>("baseline (K2 loop)", cand, n, D, m, tours, cyc, fbs);
    long long* seg; cudaMalloc(&seg, 64);
    run_tm(cand, n, D, 1, tours, seg);
    run_tm(cand, n, D, 148, tours, seg);
    run_tm(cand, n, D, m, tours, seg);
    std::vector<uint32_t> ref((size_t)m * D), got((size_t)m * D);
    cudaMemcpy(ref.data(), tours, ref.size() * 4, cudaMemcpyDeviceToHost);
    auto same = [&](const char* nm) {
        cudaMemcpy(got.data(), tours, got.size() * 4, cudaMemcpyDeviceToHost);
        printf("    %s tours identical to baseline: %s\n", nm, ref == got ? "yes" : "NO");
    };
    run<PF>("PF prefetch all cand rows", cand, n, D, m, tours, cyc, fbs); same("PF");
    run<PFF>("PFF prefetch feasible rows", cand, n, D, m, tours, cyc, fbs); same("PFF");
    run<PF>("PF, 1 warp per SM", cand, n, D, 148, tours, cyc, fbs);
    run<S1>("S1 seq prefix, shfl pick", cand, n, D, m, tours, cyc, fbs);
    run<S1 | S1SEL>("S1 seq prefix, select pick", cand, n, D, m, tours, cyc, fbs);
    run<S1>("S1, 1 warp per SM", cand, n, D, 148, tours, cyc, fbs);
    run<S1 | S1SEL>("S1 select, 1 warp per SM", cand, n, D, 148, tours, cyc, fbs);
    run<0>("baseline, 1 warp per SM", cand, n, D, 148, tours, cyc, fbs);
    run<0>("baseline, 1 warp total", cand, n, D, 1, tours, cyc, fbs);
    run<R2>("R2, 1 warp per SM", cand, n, D, 148, tours, cyc, fbs);
    run<NOWARM | NOATOM | NOSTG | NOTIE | NOPHILOX>("chain only, 1 warp/SM", cand, n, D, 148, tours, cyc, fbs);
    run<NOWARM | NOATOM | NOSTG | NOTIE | NOPHILOX | NOSCAN>("chain -scan, 1 warp/SM", cand, n, D, 148, tours, cyc, fbs);
    run<0>("baseline (again, full)", cand, n, D, m, tours, cyc, fbs);
    run<R2>("R2 redundant, select tree", cand, n, D, m, tours, cyc, fbs); same("R2");
    run<R2 | R2SHFL>("R2 redundant, shfl pick", cand, n, D, m, tours, cyc, fbs); same("R2 shfl");
    run<R2 | R2FADD2>("R2 + f32x2 adds", cand, n, D, m, tours, cyc, fbs); same("R2 fadd2");
    run<NOWARM>("-warm", cand, n, D, m, tours, cyc, fbs);
    run<NOATOM>("-mark", cand, n, D, m, tours, cyc, fbs);
    run<STSMARK>("mark via st.shared", cand, n, D, m, tours, cyc, fbs);
    run<NOSTG>("-tour store", cand, n, D, m, tours, cyc, fbs);
    run<NOTIE>("-tie vote", cand, n, D, m, tours, cyc, fbs);
    run<NOSYNC>("-syncwarp", cand, n, D, m, tours, cyc, fbs);
    run<NOPHILOX>("-philox (LCG)", cand, n, D, m, tours, cyc, fbs);
    run<NOSCAN>("-scan", cand, n, D, m, tours, cyc, fbs);
    run<SMALL>("table in L1 (512 rows)", cand, n, D, m, tours, cyc, fbs);
    run<SMALL | NOWARM>("L1 table -warm", cand, n, D, m, tours, cyc, fbs);
    run<NOWARM | NOATOM | NOSTG | NOTIE | NOPHILOX>("chain only (row,lds,scan,pick)", cand, n, D, m, tours, cyc, fbs);
    run<NOWARM | NOATOM | NOSTG | NOTIE | NOPHILOX | SMALL>("chain only, L1 table", cand, n, D, m, tours, cyc, fbs);
    run<NOWARM | NOATOM | NOSTG | NOTIE | NOPHILOX | NOSCAN>("chain -scan", cand, n, D, m, tours, cyc, fbs);
    return 0;
}
