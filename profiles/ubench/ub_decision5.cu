// Decision-loop study (round 2, part 2): the roulette on integer (fixed-point) weights.
// With q_r = 24-bit fixed-point weights every partial sum is exact, so the association of
// the scan is free and the prefix sums can come from independent integer reductions
// (redux.sync.add) instead of a chain of shuffle levels:
//   BASE - the engine's loop: f32 Hillis-Steele shuffle scan, S shuffle, one redux.min;
//   I16  - E_m = sum of q' over lanes < m for m = 1..16, sixteen independent redux.add;
//          pick = #{m in 1..15 : E_m <= target}, target = (u24 * S) >> 24; the city by one
//          redux.min over (lane == pick ? city : ~0);
//   I44  - two rounds: the four group sums E_4, E_8, E_12, E_16, then three sums inside the
//          chosen group of four;
//   SLOT - the engine's f32 roulette, but the L1-warming copies become real: lanes l and
//          l + 16 stage the two halves of feasible candidate (l & 15)'s row into a
//          shared-memory slot (double-buffered, 2 x 2 KB per ant), and the next decision
//          reads its row with one LDS (after cp.async.wait_all + bar.warp.sync) instead of
//          an L1-hit LDG. Same tours as BASE.
// Results: profiles/r02_ubench_decision5.txt.
// Same synthetic 200K-city table as ub_decision4.cu; I16 and I44 must choose identical
// tours (same integer rule). Build:
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false -I../../paper_1709_03187_b200/csrc ub_decision5.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include "device.cuh"
using namespace pacob200;

enum : int { BASE = 0, I16 = 1, I44 = 2, SLOT = 3 };

__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) { uint32_t v; asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr)); return v; }
__device__ __forceinline__ void sts_u8_if(uint32_t addr, uint32_t v, bool cond) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.shared.u8 [%0], %1;\n\t}" ::"r"(addr), "r"(v),
                 "r"((uint32_t)cond) : "memory");
}
__device__ __forceinline__ void cp_async16_if(uint32_t dst, const void* src, bool cond) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q cp.async.ca.shared.global [%0], [%1], 16;\n\t}" ::"r"(dst), "l"(src), "r"((uint32_t)cond));
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
    // SLOT: two buffers of 16 rows x 128 B after the warm slots; lane l stages half (l >> 4)
    // of candidate (l & 15)'s row
    const uint32_t slot_s = ((vis_s + nw * 4 + 15) & ~15u) + 512;
    const uint32_t r16 = lane & 15u;
    uint32_t cur = (ant * 977u) % n;
    if (lane == 0) vis[cur >> 5] |= 1u << (cur & 31);
    __syncwarp();
    uint32_t* out = tours + (size_t)ant * D;
    const uint2 key = make_uint2(7u, 0u);
    const bool lane_in = lane < 16;
    uint32_t mk[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) mk[m] = lane < (uint32_t)(m + 1) ? ~0u : 0u;  // lanes < m+1
    const uint2* row_base = cand + (V == SLOT ? r16 : lane);
    uint2 e_pre = ldg_u64_if(row_base + (size_t)cur * 16, V == SLOT || lane_in, make_uint2(cur, 0u));
    bool from_slot = false;
    uint32_t slot_j = 0;
    uint32_t n_fb = 0, n_tie = 0;
    float tie_v = 0.0f, tie_t = 0.0f, tie_tol = -1.0f;
    const long long t0 = clock64();
    for (uint32_t b0 = 0; b0 < D; b0 += 128) {
        const uint4 pb = philox10(make_uint4(1 + (b0 >> 2) + lane, ant, 0, 0), key);
        const uint32_t b1 = b0 + 128 < D ? b0 + 128 : D;
#pragma unroll 2
        for (uint32_t t = b0; t < b1; ++t) {
            __syncwarp();
            uint2 e = e_pre;
            const uint32_t buf = slot_s + (t & 1u) * 2048u;
            if (V == SLOT && from_slot) {
                asm volatile("cp.async.wait_all;" ::: "memory");
                __syncwarp();
                const uint32_t a = slot_s + ((t + 1u) & 1u) * 2048u + slot_j * 128u + r16 * 8u;
                asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(e.x), "=r"(e.y) : "r"(a) : "memory");
            }
            if (V == BASE) n_tie += __ballot_sync(kFull, lane_in && fabsf(__fsub_rn(tie_v, tie_t)) <= tie_tol) ? 1u : 0u;
            const uint32_t vw_addr = vis_s + (e.x >> 3);
            const uint32_t vw = lds_u8(vw_addr);
            const uint32_t uw = __shfl_sync(kFull, pick_word(pb, t & 3), (t & 127) >> 2);
            const uint32_t bit = 1u << (e.x & 7);
            const bool fe = (V == SLOT || lane_in) && !(vw & bit);
            if (V == SLOT) {
                const unsigned char* src = reinterpret_cast<const unsigned char*>(cand + (size_t)e.x * 16) + (lane >> 4) * 64;
                const uint32_t dst = buf + r16 * 128u + (lane >> 4) * 64u;
#pragma unroll
                for (int c = 0; c < 4; ++c) cp_async16_if(dst + 16 * c, src + 16 * c, fe);
            } else {
                const unsigned char* src = reinterpret_cast<const unsigned char*>(cand + (size_t)e.x * 16);
#pragma unroll
                for (int c = 0; c < 4; ++c) cp_async16_if(warm_s, src + 32 * c, fe);
            }
            uint32_t next;
            if (V == BASE || V == SLOT) {
                const unsigned feas = __ballot_sync(kFull, lane_in && fe && __uint_as_float(e.y) > 0.0f);
                const bool is_last = lane == 31u - __clz(feas);
                const uint32_t pick_key = (lane << 27) | e.x;
                float v = (lane_in && fe) ? __uint_as_float(e.y) : 0.0f;
#pragma unroll
                for (int st = 0; st < 4; ++st) {
                    const float y = __shfl_up_sync(kFull, v, 1u << st);
                    if (lane >= (1u << st)) v = __fadd_rn(v, y);
                }
                const float S = __shfl_sync(kFull, v, 15);
                from_slot = feas != 0u;
                if (feas) {
                    const float u = u01_f32(uw);
                    const float target = __fmul_rn(u, S);
                    const float tol = __fmul_rn(1e-6f, S);
                    const bool win = (fe & (v > target)) | is_last;
                    const uint32_t kw = __reduce_min_sync(kFull, win ? pick_key : kNone);
                    tie_v = v; tie_t = target; tie_tol = tol;
                    const uint32_t r = kw >> 27;
                    next = kw & 0x07ffffffu;
                    slot_j = r;
                    sts_u8_if(vw_addr, vw | bit, lane == r);
                } else {
                    next = (uint32_t)(((uint64_t)(cur + 1) * 2654435761ull) % n);
                    tie_tol = -1.0f;
                    if (lane == 0) vis[next >> 5] |= 1u << (next & 31);
                    ++n_fb;
                }
            } else {
                const uint32_t q = fe ? e.y : 0u;
                uint32_t S, pick;
                const uint64_t u24 = uw >> 8;
                if (V == I16) {
                    uint32_t E[16];
#pragma unroll
                    for (int m = 0; m < 16; ++m) E[m] = __reduce_add_sync(kFull, q & mk[m]);  // E[m] = sum lanes <= m
                    S = E[15];
                    const uint32_t target = (uint32_t)((u24 * S) >> 24);
                    pick = 0;
#pragma unroll
                    for (int m = 0; m < 15; ++m) pick += E[m] <= target ? 1u : 0u;
                } else {
                    uint32_t G[4];
#pragma unroll
                    for (int g = 0; g < 4; ++g) G[g] = __reduce_add_sync(kFull, q & mk[4 * g + 3]);
                    S = G[3];
                    const uint32_t target = (uint32_t)((u24 * S) >> 24);
                    const uint32_t g = (G[0] <= target ? 1u : 0u) + (G[1] <= target ? 1u : 0u) + (G[2] <= target ? 1u : 0u);
                    const uint32_t base = g ? (g == 1 ? G[0] : (g == 2 ? G[1] : G[2])) : 0u;
                    // sums over lanes 4g .. 4g+j, j = 0..2
                    const uint32_t in_g = (lane >> 2) == g ? q : 0u;
                    uint32_t H[3];
#pragma unroll
                    for (int j = 0; j < 3; ++j) H[j] = __reduce_add_sync(kFull, (lane & 3) <= (uint32_t)j ? in_g : 0u);
                    const uint32_t tt = target - base;
                    pick = 4 * g + (H[0] <= tt ? 1u : 0u) + (H[1] <= tt ? 1u : 0u) + (H[2] <= tt ? 1u : 0u);
                }
                if (S) {
                    next = __reduce_min_sync(kFull, lane == pick ? e.x : kNone);
                    sts_u8_if(vw_addr, vw | bit, lane == pick);
                } else {
                    next = (uint32_t)(((uint64_t)(cur + 1) * 2654435761ull) % n);
                    if (lane == 0) vis[next >> 5] |= 1u << (next & 31);
                    ++n_fb;
                }
            }
            if (V != SLOT || !from_slot) e_pre = ldg_u64_if(row_base + (size_t)next * 16, V == SLOT || lane_in, make_uint2(next, 0u));
            stg_u32_if(out + t, next, lane == 0);
            cur = next;
        }
    }
    const long long t1 = clock64();
    if (lane == 0) {
        cyc[ant] = t1 - t0;
        atomicAdd(&seg[0], (unsigned long long)n_fb);
        atomicAdd(&seg[1], (unsigned long long)n_tie);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
}

std::vector<uint32_t> g_ref;

template <int V>
void run(const char* name, const uint2* cand, uint32_t n, uint32_t D, uint32_t m, uint32_t* tours, long long* cyc,
         unsigned long long* seg, bool reset_ref) {
    const size_t smem = ((n + 31) / 32) * 4 + 16 + 512 + 4096;
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
    double mean = 0, mx = 0; for (auto v : h) { mean += v; mx = v > mx ? v : mx; }
    mean /= m;
    std::vector<uint32_t> got((size_t)m * D);
    cudaMemcpy(got.data(), tours, got.size() * 4, cudaMemcpyDeviceToHost);
    const char* same = "";
    if (reset_ref) g_ref = got;
    same = (g_ref == got) ? "same tours" : "TOURS DIFFER";
    const double d = (double)m * D;
    printf("%-16s m=%-4u %6.1f cyc/dec (max ant %6.1f) %8.3f ms fb %.3f%% ties %llu %s %s\n", name, m, mean / D, mx / D, ms,
           100.0 * sg[0] / d, sg[1], same, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const uint32_t n = 200000, D = 20000;
    std::mt19937 rng(5);
    std::vector<uint2> hf((size_t)n * 16), hi((size_t)n * 16);
    std::uniform_int_distribution<int> off(-300, 300);
    std::uniform_real_distribution<float> wd(0.1f, 1.0f);
    for (uint32_t i = 0; i < n; ++i)
        for (int r = 0; r < 16; ++r) {
            int o = off(rng); if (o == 0) o = 1;
            const uint32_t c = (uint32_t)(((int64_t)i + o + n) % n);
            const float w = wd(rng);
            hf[(size_t)i * 16 + r] = make_uint2(c, __builtin_bit_cast(uint32_t, w));
            hi[(size_t)i * 16 + r] = make_uint2(c, (uint32_t)(w * 16777216.0f));
        }
    uint2 *cf, *ci; uint32_t* tours; long long* cyc; unsigned long long* seg;
    cudaMalloc(&cf, hf.size() * 8); cudaMemcpy(cf, hf.data(), hf.size() * 8, cudaMemcpyHostToDevice);
    cudaMalloc(&ci, hi.size() * 8); cudaMemcpy(ci, hi.data(), hi.size() * 8, cudaMemcpyHostToDevice);
    cudaMalloc(&tours, (size_t)2048 * D * 4); cudaMalloc(&cyc, 2048 * 8); cudaMalloc(&seg, 64);
    printf("n=%u D=%u\n", n, D);
    for (uint32_t mm : {1u, 148u, 444u, 1024u}) {
        run<BASE>("base f32 scan", cf, n, D, mm, tours, cyc, seg, true);
        run<SLOT>("rows in smem slots", cf, n, D, mm, tours, cyc, seg, false);
        run<I16>("int 16 redux", ci, n, D, mm, tours, cyc, seg, true);
        run<I44>("int 4+3 redux", ci, n, D, mm, tours, cyc, seg, false);
    }
    return 0;
}
