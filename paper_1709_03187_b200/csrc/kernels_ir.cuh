// Reference-rule mode: the reference's own selection rule,
// Independent Roulette over every unvisited city (construction.hpp:243-281), with the
// reference's per-ant xoshiro256++ draw streams (rng.hpp:24-74), so a GPU run is
// bit-identical to paco::run in synchronous mode (engine.hpp:245-306): same tours,
// same lengths, same g_best, same comparison count.
//
// This mode exists for parity, not speed: the rule scans O(n) candidates per decision
// and the streams are sequential, so lane 0 generates the draws of each 32-city chunk
// while the warp scores them. Cities are kept in their original order (identity
// internal numbering) because the rule consumes draws in ascending city index.
#pragma once
#include "device.cuh"

namespace pacob200 {

// xoshiro256++ step (rng.hpp:40-50)
__device__ __forceinline__ uint64_t xoshiro_next(uint64_t s[4]) {
    const uint64_t x = s[0] + s[3];
    const uint64_t result = ((x << 23) | (x >> 41)) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = (s[3] << 45) | (s[3] >> 19);
    return result;
}
// Rng::uniform (rng.hpp:53-55)
__device__ __forceinline__ double xo_uniform(uint64_t s[4]) {
    return (double)(xoshiro_next(s) >> 11) * 0x1.0p-53;
}
// Rng::uniform_below (rng.hpp:59-66): mask rejection, variable number of draws
__device__ __forceinline__ uint32_t xo_below(uint64_t s[4], uint32_t bound) {
    const uint32_t mask = bound <= 1 ? 0u : (0xffffffffu >> __clz(bound - 1));
    for (;;) {
        const uint32_t r = (uint32_t)xoshiro_next(s) & mask;
        if (r < bound) return r;
    }
}

struct IrArgs {
    const double2* xy;        // original order
    const uint2* nbr;         // m*n (prev, next) of each ant's l_best (P-ACO)
    const double* ratio;      // m g/l ratios snapshotted for this iteration (0 = no tour)
    const double* T;          // classic: n*n pheromone matrix, else nullptr
    uint64_t* rng;            // m*4 xoshiro256++ states, carried across iterations
    uint32_t* tours;          // m*2*n
    const uint8_t* lb_sel;
    int64_t* new_len;
    uint8_t* partial_flag;
    unsigned long long* counters;  // decisions, fallbacks, ties, forced, full, partial, iter, improv, comparisons
    uint32_t n, m, nwords;
    double alpha, beta, tau0, eff_pp, mmf;
    int seeding, coin_always, eta_table;  // eta_table: reference table path (n <= 5000) rounds eta^beta to f32
    double two_opt_prob;
    uint32_t two_opt_window;
};

// One warp per ant: detail::build_candidate (engine.hpp:129-148) with construct_full /
// construct_partial (construction.hpp:283-365) and select_next (construction.hpp:246-281).
__global__ void __launch_bounds__(32, 1) k_construct_ir(IrArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t lane = threadIdx.x, ant = blockIdx.x, n = a.n, nw = a.nwords;
    double* acc = reinterpret_cast<double*>(smem_raw);              // n (P-ACO): ColonyPheromone::acc_
    uint64_t* dbuf = reinterpret_cast<uint64_t*>(acc + (a.T ? 0 : n)); // 32 draws of the current chunk
    uint32_t* vis = reinterpret_cast<uint32_t*>(dbuf + 32);          // nw
    uint64_t s[4] = {0, 0, 0, 0};  // lane 0 owns the stream
    if (lane == 0)
        for (int q = 0; q < 4; ++q) s[q] = a.rng[(size_t)ant * 4 + q];
    if (!a.T)
        for (uint32_t j = lane; j < n; j += 32) acc[j] = 0.0;
    for (uint32_t w = lane; w < nw; w += 32) vis[w] = 0u;
    __syncwarp();
    if (lane == 0 && (n & 31)) vis[nw - 1] = 0xffffffffu << (n & 31);
    __syncwarp();
    const uint8_t sel = a.lb_sel[ant];
    uint32_t* out = a.tours + ((size_t)ant * 2 + (1 - sel)) * n;
    const uint32_t* lb = a.tours + ((size_t)ant * 2 + sel) * n;

    // lane-0 draws broadcast to the warp
    auto bcast = [&](uint32_t v) { return __shfl_sync(kFull, v, 0); };
    int partial = 0;
    uint32_t start_pos = 0, m_mod = 0, start = 0;
    {
        uint32_t p = 0, sp = 0, mm = 0, st = 0;
        if (lane == 0) {
            if (!a.seeding || a.coin_always) {
                const double coin = xo_uniform(s);  // engine.hpp:137
                p = coin < a.eff_pp ? 1 : 0;
            }
            if (p) {
                sp = xo_below(s, n);  // construction.hpp:358
                double capd = floor(a.mmf * (double)n);
                if (capd < 2.0) capd = 2.0;
                mm = 2 + xo_below(s, (uint32_t)capd - 1);
            } else {
                st = xo_below(s, n);  // construction.hpp:291
            }
        }
        partial = (int)bcast(p); start_pos = bcast(sp); m_mod = bcast(mm); start = bcast(st);
    }
    uint32_t pos, cur, remaining;
    if (!partial) {
        if (lane == 0) { out[0] = start; vis[start >> 5] |= 1u << (start & 31); }
        pos = 1; cur = start; remaining = n - 1;
    } else {
        const uint32_t preserved = n - m_mod;
        for (uint32_t t = lane; t < preserved; t += 32) {
            uint32_t p = start_pos + t; if (p >= n) p -= n;
            const uint32_t city = lb[p];
            out[t] = city;
            atomicOr(&vis[city >> 5], 1u << (city & 31));
        }
        if (preserved == 0) {
            const uint32_t anchor = lb[start_pos];
            if (lane == 0) { out[0] = anchor; vis[anchor >> 5] |= 1u << (anchor & 31); }
            pos = 1;
        } else {
            pos = preserved;
        }
        uint32_t p = start_pos + pos - 1; if (p >= n) p -= n;
        cur = lb[p];
        remaining = n - pos;
    }
    __syncwarp();

    unsigned long long n_dec = 0, n_cmp = 0, n_forced = 0;
    const double tau0_alpha = power(a.alpha, a.tau0);
    (void)tau0_alpha;
    // full constructions score every step (the last one with a single candidate);
    // partial constructions append the final city unscored (construction.hpp:338-348)
    const uint32_t scored = partial ? (remaining > 0 ? remaining - 1 : 0) : remaining;
    for (uint32_t step = 0; step < remaining; ++step) {
        uint32_t next;
        if (step >= scored) {
            // forced append of the single remaining candidate
            next = kNone;
            for (uint32_t base = 0; base < nw; base += 32) {
                const uint32_t w = base + lane;
                const uint32_t fb = w < nw ? ~vis[w] : 0u;
                const unsigned ball = __ballot_sync(kFull, fb != 0);
                if (ball) {
                    const int src = __ffs(ball) - 1;
                    next = (base + src) * 32 + (__ffs(__shfl_sync(kFull, fb, src)) - 1);
                    break;
                }
            }
            ++n_forced;
        } else {
            // ColonyPheromone::begin_step (construction.hpp:121-132): ant order, lane 0
            if (!a.T) {
                if (lane == 0)
                    for (uint32_t q = 0; q < a.m; ++q) {
                        const double r = a.ratio[q];
                        if (r == 0.0) continue;
                        const uint2 pr = a.nbr[(size_t)q * n + cur];
                        acc[pr.x] += r;
                        acc[pr.y] += r;
                    }
                __syncwarp();
            }
            const double2 qc = a.xy[cur];
            const double* trow = a.T ? a.T + (size_t)cur * n : nullptr;
            double best = -1.0;
            uint32_t bj = kNone;
            uint32_t cnt_total = 0;
            for (uint32_t w = 0; w < nw; ++w) {
                const uint32_t free_bits = ~vis[w];
                if (!free_bits) continue;
                const uint32_t cnt = __popc(free_bits);
                cnt_total += cnt;
                if (lane == 0)
                    for (uint32_t q = 0; q < cnt; ++q) dbuf[q] = xoshiro_next(s);  // one draw per candidate
                __syncwarp();
                if ((free_bits >> lane) & 1u) {
                    const uint32_t j = w * 32 + lane;
                    const double u = (double)(dbuf[__popc(free_bits & ((1u << lane) - 1u))] >> 11) * 0x1.0p-53;
                    int32_t d = euc2d(qc, a.xy[j]);
                    if (d < 1) d = 1;
                    double eta = power(a.beta, 1.0 / (double)d);
                    if (a.eta_table) eta = (double)(float)eta;
                    const double ta = trow ? power(a.alpha, trow[j]) : power(a.alpha, __dadd_rn(a.tau0, acc[j]));
                    const double score = __dmul_rn(__dmul_rn(ta, eta), u);
                    if (score > best) { best = score; bj = j; }
                }
                __syncwarp();
            }
            // warp argmax, strict >, lowest city index on equal scores
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const double b2 = __shfl_xor_sync(kFull, best, off);
                const uint32_t j2 = __shfl_xor_sync(kFull, bj, off);
                if (b2 > best || (b2 == best && j2 < bj)) { best = b2; bj = j2; }
            }
            next = bj;
            n_cmp += cnt_total;  // construction.hpp:275
            if (!a.T) {
                // ColonyPheromone::end_step: reset the touched entries
                for (uint32_t q = lane; q < a.m; q += 32) {
                    if (a.ratio[q] == 0.0) continue;
                    const uint2 pr = a.nbr[(size_t)q * n + cur];
                    acc[pr.x] = 0.0;
                    acc[pr.y] = 0.0;
                }
                __syncwarp();
            }
        }
        ++n_dec;
        if (lane == 0) { out[pos] = next; vis[next >> 5] |= 1u << (next & 31); }
        __syncwarp();
        ++pos;
        cur = next;
    }
    // maybe_two_opt consumes exactly one draw (two_opt.hpp:71-76)
    uint32_t do2 = 0;
    if (lane == 0) do2 = xo_uniform(s) < a.two_opt_prob ? 1u : 0u;
    do2 = __shfl_sync(kFull, do2, 0);
    __syncwarp();
    if (do2) two_opt_warp(out, n, a.two_opt_window, a.xy, lane);
    long long len = 0;
    for (uint32_t p = lane; p < n; p += 32) len += euc2d(a.xy[out[p]], a.xy[out[p + 1 < n ? p + 1 : 0]]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) len += __shfl_xor_sync(kFull, len, off);
    if (lane == 0) {
        for (int q = 0; q < 4; ++q) a.rng[(size_t)ant * 4 + q] = s[q];
        a.new_len[ant] = len;
        a.partial_flag[ant] = (uint8_t)partial;
        atomicAdd(&a.counters[0], n_dec);
        atomicAdd(&a.counters[3], n_forced);
        atomicAdd(&a.counters[partial ? 5 : 4], 1ull);
        atomicAdd(&a.counters[8], n_cmp);
        if (do2) atomicAdd(&a.counters[9], 1ull);
    }
}

// ratios snapshot (Colony::snapshot_ratios, colony.hpp:159-167)
__global__ void k_ratios(const int64_t* __restrict__ lb_len, const uint8_t* __restrict__ has_lb,
                         const int64_t* __restrict__ g_len, uint32_t m, double* __restrict__ ratio) {
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= m) return;
    double r = 0.0;
    if (has_lb[q]) { r = (double)*g_len / (double)lb_len[q]; r = r > 1.0 ? 1.0 : r; }
    ratio[q] = r;
}

// classic matrix (construction.hpp:187-207): evaporate every entry, then deposit the built
// tours in tour order; thread per row i, each row's entries receive their deposits in
// ant order (the reference's order for every entry).
__global__ void k_classic_full(const uint2* __restrict__ cur_nbr, const int64_t* __restrict__ new_len, uint32_t n,
                               uint32_t m, double rho, double* __restrict__ T) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double* row = T + (size_t)i * n;
    const double keep = 1.0 - rho;
    for (uint32_t j = 0; j < n; ++j) {
        const double v = __dmul_rn(row[j], keep);
        row[j] = v < 1e-6 ? 1e-6 : v;
    }
    for (uint32_t q = 0; q < m; ++q) {
        const uint2 p = cur_nbr[(size_t)q * n + i];
        const double delta = 1.0 / (double)new_len[q];
        row[p.x] = __dadd_rn(row[p.x], delta);
        if (p.y != p.x) row[p.y] = __dadd_rn(row[p.y], delta);
    }
}

}  // namespace pacob200
