// Reference-rule mode: the reference's own selection rule,
// Independent Roulette over every unvisited city (construction.hpp:243-281), with the
// reference's per-ant xoshiro256++ draw streams (rng.hpp:24-74), so a GPU run is
// bit-identical to paco::run in synchronous mode (engine.hpp:245-306): same tours,
// same lengths, same g_best, same comparison count.
//
// This mode exists for parity, not speed: the rule scans O(n) candidates per decision
// and the streams are sequential, so a generator warp runs each ant's stream ahead while
// the construction warp scores. Cities are kept in their original order (identity
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

// the construction kernel's per-city tau^alpha array in shared memory is padded by one
// slot per 32 cities, so that lanes reading the 32 cities of their own word (stride 32)
// hit different banks
__host__ __device__ inline uint32_t accx(uint32_t j) { return j + (j >> 5); }
__host__ __device__ inline uint32_t ir_acc_slots(uint32_t n) { return n + (n >> 5) + 1; }

struct IrJump;
struct IrArgs {
    const double2* xy;        // original order
    const uint2* nbr;         // m*n (prev, next) of each ant's l_best (P-ACO)
    const double* ratio;      // m g/l ratios snapshotted for this iteration (0 = no tour)
    const uint32_t* tl_city;  // P-ACO: n rows of 2m + 1: the count, then the touched cities of each
                              // city's begin_step (k_ir_touched)
    const double* tl_tau;     // n*2m their tau^alpha
    const double* T;          // classic: n*n pheromone matrix, else nullptr
    const float* eta_tab;     // n*n eta^beta as f32 (the reference's table path, n <= 5000), else nullptr
    uint64_t* rng;            // m*4 xoshiro256++ states, carried across iterations
    uint32_t* tours;          // m*2*n
    const uint8_t* lb_sel;
    int64_t* new_len;
    uint8_t* partial_flag;
    unsigned long long* counters;  // decisions, fallbacks, ties, forced, full, partial, iter, improv, comparisons
    uint32_t n, m, nwords;
    const IrJump* jump;       // generator jump polynomials
    double alpha, beta, tau0, eff_pp, mmf;
    int seeding, coin_always, eta_table;  // eta_table: reference table path (n <= 5000) rounds eta^beta to f32
    double two_opt_prob;
    uint32_t two_opt_window;
};

// acquire / release on shared-memory flags (no full fence between the two warps)
__device__ __forceinline__ uint32_t ld_acquire_cta(const volatile uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared((const void*)p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_cta(volatile uint32_t* p, uint32_t v) {
    asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared((const void*)p)), "r"(v) : "memory");
}

// Draw ring between the generator warp and the construction warp of one ant. The
// generator's 32 lanes each produce chunks of kIrChunk consecutive draws of the ant's one
// stream - lane i chunks i, i + 32, ... - reaching its next chunk with a xoshiro jump
// (the state advanced by 31 chunks: Cayley-Hamilton, the jump polynomial x^J mod the
// transition's characteristic polynomial, computed on the host, ir_jump_polys). A round is
// 32 chunks; the ring holds two rounds.
constexpr uint32_t kIrChunk = 64;                  // draws per chunk
constexpr uint32_t kIrRound = 32 * kIrChunk;       // draws per generator round
constexpr uint32_t kIrRing = 2 * kIrRound;         // u64 draws in flight
constexpr uint32_t kIrCkpt = kIrRing / kIrChunk;   // chunk start states kept
struct IrRing {
    unsigned long long draw[kIrRing];
    unsigned long long ckpt[kIrCkpt][4];    // state before draw kIrChunk * c (slot c % kIrCkpt)
    volatile uint32_t produced, consumed, stop;
};
// ring slot of stream position p: XOR-swizzled inside its chunk, so that the 32 lanes that
// write one step of their chunks at once fall in different bank pairs
__device__ __forceinline__ uint32_t ir_slot(uint32_t p) {
    return ((p & ~(kIrChunk - 1)) | ((p & (kIrChunk - 1)) ^ ((p / kIrChunk) & 15u))) % kIrRing;
}
// Jump polynomials (bit b of word w = coefficient of x^(64w+b)): [0..31] lane offsets
// x^(i * kIrChunk), [32] the step to a lane's next chunk x^(31 * kIrChunk)
struct IrJump {
    unsigned long long p[33][4];
};
// s <- p(M) s for the xoshiro256 transition M (the structure of the published jump()):
// the states M^b s accumulated where p has bit b
__device__ __forceinline__ void xo_jump(uint64_t s[4], const unsigned long long* __restrict__ p) {
    uint64_t t0 = 0, t1 = 0, t2 = 0, t3 = 0;
    for (int w = 0; w < 4; ++w) {
        const uint64_t pw = p[w];
#pragma unroll 8
        for (int b = 0; b < 64; ++b) {
            if ((pw >> b) & 1u) { t0 ^= s[0]; t1 ^= s[1]; t2 ^= s[2]; t3 ^= s[3]; }
            xoshiro_next(s);
        }
    }
    s[0] = t0; s[1] = t1; s[2] = t2; s[3] = t3;
}

// One CTA of two warps per ant: detail::build_candidate (engine.hpp:129-148) with
// construct_full / construct_partial (construction.hpp:283-365) and select_next
// (construction.hpp:246-281).
//  * warp 1, lane 0 runs the ant's xoshiro256++ stream ahead into a shared-memory ring;
//  * warp 0 builds the tour, consuming the draws in the reference's order.
// The stream is inherently sequential; with the generator on its own warp it overlaps
// the scoring instead of alternating with it. The draws a construction actually consumed
// decide the stored stream state: the generator checkpoints its state every 32 draws
// and never runs so far ahead that the checkpoint below the consumption point is
// overwritten; the construction warp replays at most 31 steps from it.
__global__ void __launch_bounds__(64, 1) k_construct_ir(IrArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, ant = blockIdx.x, n = a.n, nw = a.nwords;
    IrRing* ring = reinterpret_cast<IrRing*>(smem_raw);
    double* acc = reinterpret_cast<double*>(ring + 1);  // ir_acc_slots(n) (P-ACO): this step's tau^alpha, negated, at accx(j)
    uint32_t* vis = reinterpret_cast<uint32_t*>(acc + (a.T ? 0 : ir_acc_slots(n)));  // nw
    if (threadIdx.x == 0) { ring->produced = 0; ring->consumed = 0; ring->stop = 0; }
    if (warp == 0) {
        if (!a.T) {  // untouched cities score with tau0^alpha (ColonyPheromone::mult_, construction.hpp:108-111)
            const double t0a = power(a.alpha, a.tau0);
            for (uint32_t j = lane; j < ir_acc_slots(n); j += 32) acc[j] = t0a;
        }
        for (uint32_t w = lane; w < nw; w += 32) vis[w] = 0u;
    }
    __syncthreads();
    if (warp == 1) {
        // the generator warp (rng.hpp:40-50): lane i starts at stream position i * kIrChunk
        // of the ant's stream (state carried across iterations in a.rng), produces its chunk
        // of every round, then jumps 31 chunks ahead
        uint64_t s[4];
        for (int q = 0; q < 4; ++q) s[q] = a.rng[(size_t)ant * 4 + q];
        if (lane) xo_jump(s, a.jump->p[lane]);
        for (uint32_t r = 0;; ++r) {
            // round r reuses round r - 2's slots and checkpoints: wait for them to be consumed
            if (r >= 2) {
                if (lane == 0)
                    while (ld_acquire_cta(&ring->consumed) < (r - 1) * kIrRound && !ring->stop) __nanosleep(64);
                __syncwarp();
            }
            // one lane reads the flag, so that the warp leaves the loop together
            if (__shfl_sync(kFull, lane == 0 ? (uint32_t)ring->stop : 0u, 0)) break;
            const uint32_t c = 32 * r + lane, p0 = c * kIrChunk;
            unsigned long long* ck = ring->ckpt[c % kIrCkpt];
            ck[0] = s[0]; ck[1] = s[1]; ck[2] = s[2]; ck[3] = s[3];
#pragma unroll 16
            for (uint32_t q = 0; q < kIrChunk; ++q) ring->draw[ir_slot(p0 + q)] = xoshiro_next(s);
            xo_jump(s, a.jump->p[32]);
            __syncwarp();
            if (lane == 0) st_release_cta(&ring->produced, (r + 1) * kIrRound);  // the round's draws before the count
        }
        return;
    }
    // ---- warp 0: the construction ----
    if (lane == 0 && (n & 31)) vis[nw - 1] = 0xffffffffu << (n & 31);
    __syncwarp();
    uint32_t cidx = 0;  // draws consumed so far (warp-uniform)
#ifdef PACO_IRSEG
    long long sg_wait = 0, sg_begin = 0, sg_scan = 0, sg_end = 0, sg_stage = 0, sg_group = 0, sg_ld = 0, sg_loop = 0;
#endif
    auto wait_for = [&](uint32_t upto) {  // draws [0, upto) are in the ring
#ifdef PACO_IRSEG
        const long long w0c = clock64();
#endif
        // publish the consumption point first: the generator may be waiting for it to start
        // the round that holds `upto` (after every lane's reads of the earlier draws: lane 0's
        // release covers them through the warp barrier)
        __syncwarp();
        if (lane == 0) {
            // a release: the draws read so far are read before the generator may reuse their slots
            if (ring->consumed != cidx) st_release_cta(&ring->consumed, cidx);
            while (ld_acquire_cta(&ring->produced) < upto) {}
        }
        __syncwarp();
#ifdef PACO_IRSEG
        sg_wait += clock64() - w0c;
#endif
    };
    auto take = [&]() -> uint64_t {  // next draw, lane 0's view (other lanes follow the index)
        wait_for(cidx + 1);
        const uint64_t v = ring->draw[ir_slot(cidx)];
        ++cidx;
        return v;
    };
    auto uniform = [&]() { return (double)(take() >> 11) * 0x1.0p-53; };  // Rng::uniform, rng.hpp:53-55
    auto below = [&](uint32_t bound) {  // Rng::uniform_below, rng.hpp:59-66
        const uint32_t mask = bound <= 1 ? 0u : (0xffffffffu >> __clz(bound - 1));
        for (;;) {
            const uint32_t r = (uint32_t)take() & mask;
            if (r < bound) return r;
        }
    };
    const uint8_t sel = a.lb_sel[ant];
    uint32_t* out = a.tours + ((size_t)ant * 2 + (1 - sel)) * n;
    const uint32_t* lb = a.tours + ((size_t)ant * 2 + sel) * n;

    int partial = 0;
    uint32_t start_pos = 0, m_mod = 0, start = 0;
    if (!a.seeding || a.coin_always) partial = uniform() < a.eff_pp ? 1 : 0;  // engine.hpp:137
    if (partial) {
        start_pos = below(n);  // construction.hpp:358
        double capd = floor(a.mmf * (double)n);
        if (capd < 2.0) capd = 2.0;
        m_mod = 2 + below((uint32_t)capd - 1);
    } else {
        start = below(n);  // construction.hpp:291
    }
    uint32_t pos, cur, remaining;
    if (!partial) {
        if (lane == 0) { out[0] = start; vis[start >> 5] |= 1u << (start & 31); }
        pos = 1; cur = start; remaining = n - 1;
    } else {
        const uint32_t preserved = n - m_mod;
        warp_copy_segment(out, lb, n, start_pos, preserved, vis, lane);
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
    // untouched cities score with tau0^alpha (ColonyPheromone::mult_, construction.hpp:108-111);
    // a touched city always has acc > 0 (contributions are g/l ratios > 0)
    const double tau0_alpha = power(a.alpha, a.tau0);
    // full constructions score every step (the last one with a single candidate);
    // partial constructions append the final city unscored (construction.hpp:338-348)
    const uint32_t scored = partial ? (remaining > 0 ? remaining - 1 : 0) : remaining;
    const uint32_t* lc = nullptr;  // the current step's touched-city list (P-ACO)
    const double* lv = nullptr;
    uint32_t tl0 = 0u, tl_cnt = 0u;  // this lane's first-round slot, the list's length
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
#ifdef PACO_IRSEG
            const long long b0c = clock64();
#endif
            // ColonyPheromone::begin_step (construction.hpp:121-132). The 2m contributions
            // (ant q's prev then next of cur) are fetched at once into a shared staging list,
            // then applied 32 per pass, one lane each: lanes that hit the same city are grouped
            // (match.any) and the group's lowest lane adds them in lane order, so every acc[c]
            // receives its terms in ant order - the fp64 sum order of the reference.
            if (!a.T) {
                // the step's touched cities and their tau^alpha, precomputed for the iteration
                // (k_ir_touched); every other city holds tau0^alpha
                // (k_ir_touched); every other city holds tau0^alpha. One round trip for the count
                // (lane 0) and the first 31 entries (lanes 1..31); longer lists loop.
                lc = a.tl_city + (size_t)cur * (2 * a.m + 1);
                lv = a.tl_tau + (size_t)cur * 2 * a.m;
                tl0 = lane <= 2 * a.m ? lc[lane] : 0u;
                const double v0 = lane >= 1 && lane <= 2 * a.m ? lv[lane - 1] : 0.0;
                tl_cnt = __shfl_sync(kFull, tl0, 0);
                if (lane >= 1 && lane <= tl_cnt) acc[accx(tl0)] = v0;
                for (uint32_t e = 31 + lane; e < tl_cnt; e += 32) acc[accx(lc[e + 1])] = lv[e];
                __syncwarp();
            }
#ifdef PACO_IRSEG
            const long long b1c = clock64();
            sg_begin += b1c - b0c;
#endif
            const double2 qc = a.xy[cur];
            const double* trow = a.T ? a.T + (size_t)cur * n : nullptr;
            double best = -1.0;
            uint32_t bj = kNone;
            uint32_t cnt_total = 0;
            if (a.eta_tab && !trow) {
                // The table path (n <= 5000), P-ACO: words of 32 cities, lane l owning word l of each
                // chunk of 32 words. A lane's draws are the consecutive block after the unvisited
                // cities of the lower words (a warp scan of the words' popcounts), its eta^beta
                // row segment (128 bytes) and tau row segment are loaded at once, and it scores its
                // unvisited cities in ascending order with strict > (the lowest index keeps a tie).
                for (uint32_t w0 = 0; w0 < nw; w0 += 32) {
                    const uint32_t wl = w0 + lane;
                    const uint32_t fbw = wl < nw ? ~vis[wl] : 0u;
                    const uint32_t cw = __popc(fbw);
                    uint32_t incl = cw;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t y = __shfl_up_sync(kFull, incl, o);
                        if (lane >= (uint32_t)o) incl += y;
                    }
                    const uint32_t tot = __shfl_sync(kFull, incl, 31);
                    if (tot == 0) continue;
                    const uint32_t excl = incl - cw;
                    const size_t j0 = (size_t)wl * 32;
                    float ef[32];
                    double tv[32];
                    if (fbw) {
                        const float4* erow = reinterpret_cast<const float4*>(a.eta_tab + (size_t)cur * n + j0);
                        // the table's row stride is n: a 16-byte load needs 4-aligned cities
                        if (((size_t)cur * n + j0) % 4 == 0 && j0 + 32 <= n) {
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                const float4 f = erow[q];
                                ef[4 * q] = f.x; ef[4 * q + 1] = f.y; ef[4 * q + 2] = f.z; ef[4 * q + 3] = f.w;
                            }
                        } else {
                            const float* er = a.eta_tab + (size_t)cur * n + j0;
#pragma unroll
                            for (int q = 0; q < 32; ++q) ef[q] = j0 + q < n ? er[q] : 0.0f;
                        }
#pragma unroll
                        for (int q = 0; q < 32; ++q) tv[q] = ((fbw >> q) & 1u) ? acc[j0 + q + wl] : 0.0;
                    }
#ifndef PACO_IRSEG
                    // the row loads land before the draw wait (left to the compiler they were
                    // issued behind it: 453 against 373 ms for C1's 100 iterations)
#pragma unroll
                    for (int q = 0; q < 32; ++q) asm volatile("" ::"f"(ef[q]), "d"(tv[q]));
#endif
#ifdef PACO_IRSEG
                    const long long q0c = clock64();
                    double tsum = 0.0;
#pragma unroll
                    for (int q = 0; q < 32; ++q) tsum += tv[q] + (double)ef[q];
                    { long long q1c; asm volatile("mov.u64 %0, %%clock64;" : "=l"(q1c) : "d"(tsum)); sg_ld += q1c - q0c; }
#endif
                    wait_for(cidx + tot);
#ifdef PACO_IRSEG
                    const long long q2c = clock64();
#endif
                    // every city's draw address is its rank among the word's unvisited cities (no
                    // dependence between cities), and the lane's best is a tree over the 32 cities
                    // that keeps the lower index on equal scores - the strict > of an ascending scan
                    const uint32_t base = cidx + excl;
                    // branch-free: every city is scored (a visited city reads some ring slot and
                    // gets -1), so the 32 loads, conversions and products overlap. The score is
                    // taken times 2^53: (tau * eta) * ((raw >> 11) * 2^-53) rounds like
                    // (tau * eta) * (raw >> 11) scaled by the exact power of two, so the order of
                    // the scores - all the argmax uses - is the reference's
                    double sc[32];
#pragma unroll
                    for (int q = 0; q < 32; ++q) {
                        const uint64_t raw = ring->draw[ir_slot(base + __popc(fbw & ((1u << q) - 1u)))];
                        const double v = __dmul_rn(__dmul_rn(tv[q], (double)ef[q]), (double)(raw >> 11));
                        sc[q] = ((fbw >> q) & 1u) ? v : -1.0;
                    }
                    uint32_t ix[32];
#pragma unroll
                    for (int q = 0; q < 32; ++q) ix[q] = q;
#pragma unroll
                    for (int st = 1; st < 32; st <<= 1) {
#pragma unroll
                        for (int q = 0; q + st < 32; q += 2 * st) {
                            // left (lower index) wins unless right is strictly larger
                            if (sc[q + st] > sc[q]) { sc[q] = sc[q + st]; ix[q] = ix[q + st]; }
                        }
                    }
                    if (sc[0] > best) { best = sc[0]; bj = (uint32_t)j0 + ix[0]; }  // best is scaled by 2^53 here
#ifdef PACO_IRSEG
                    { long long q3c; asm volatile("mov.u64 %0, %%clock64;" : "=l"(q3c) : "d"(best)); sg_loop += q3c - q2c; }
#endif
                    cidx += tot;
                    cnt_total += tot;
                    __syncwarp();  // every lane's draws are read before the slots are released
                    if (lane == 0) st_release_cta(&ring->consumed, cidx);
                }
            } else {
                // one draw per unvisited city in ascending index; four bitmap words per pass so
                // that four rows of eta / tau loads are in flight per lane
                constexpr uint32_t U = 4;
                const unsigned lt = (1u << lane) - 1u;
                for (uint32_t w0 = 0; w0 < nw; w0 += U) {
                    uint32_t fb[U], cntv[U], tot = 0;
    #pragma unroll
                    for (uint32_t u = 0; u < U; ++u) {
                        fb[u] = w0 + u < nw ? ~vis[w0 + u] : 0u;
                        cntv[u] = __popc(fb[u]);
                        tot += cntv[u];
                    }
                    if (tot == 0) continue;
                    double eta[U], ta[U];
                    if (a.eta_tab) {
                        // every global load of the pass is issued before the first use (predicated
                        // PTX loads; left to the compiler, each conversion sat right behind its load
                        // and a pass made U serial L2 round trips)
                        const size_t j0 = (size_t)w0 * 32 + lane;
                        const float* erow = a.eta_tab + (size_t)cur * n + j0;
                        float ef[U];
                        double tv[U];
    #pragma unroll
                        for (uint32_t u = 0; u < U; ++u) {
                            const bool f = (fb[u] >> lane) & 1u;
                            ef[u] = ldg_f32_if(erow + u * 32, f);
                            tv[u] = trow ? ldg_f64_if(trow + j0 + u * 32, f) : (f ? acc[accx((uint32_t)j0 + u * 32)] : tau0_alpha);
                        }
    #pragma unroll
                        for (uint32_t u = 0; u < U; ++u) {
                            eta[u] = (double)ef[u];
                            ta[u] = trow ? power(a.alpha, tv[u]) : tv[u];
                        }
                    } else
    #pragma unroll
                    for (uint32_t u = 0; u < U; ++u) {
                        eta[u] = 0.0; ta[u] = 0.0;
                        if ((fb[u] >> lane) & 1u) {
                            const uint32_t j = (w0 + u) * 32 + lane;
                            {
                                int32_t d = euc2d(qc, a.xy[j]);
                                if (d < 1) d = 1;
                                eta[u] = power(a.beta, 1.0 / (double)d);
                                if (a.eta_table) eta[u] = (double)(float)eta[u];
                            }
                            if (trow) ta[u] = power(a.alpha, trow[j]);
                            else {
                                ta[u] = acc[accx(j)];
                            }
                        }
                    }
                    wait_for(cidx + tot);
                    uint32_t off = cidx;
    #pragma unroll
                    for (uint32_t u = 0; u < U; ++u) {
                        if ((fb[u] >> lane) & 1u) {
                            const uint64_t raw = ring->draw[ir_slot(off + __popc(fb[u] & lt))];
                            const double uu = (double)(raw >> 11) * 0x1.0p-53;
                            const double score = __dmul_rn(__dmul_rn(ta[u], eta[u]), uu);
                            if (score > best) { best = score; bj = (w0 + u) * 32 + lane; }
                        }
                        off += cntv[u];
                    }
                    cidx += tot;
                    cnt_total += tot;
                    __syncwarp();  // every lane's draws are read before the slots are released
                    if (lane == 0) st_release_cta(&ring->consumed, cidx);
                }
            }
            // warp argmax, strict >, lowest city index on equal scores
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const double b2 = __shfl_xor_sync(kFull, best, off);
                const uint32_t j2 = __shfl_xor_sync(kFull, bj, off);
                if (b2 > best || (b2 == best && j2 < bj)) { best = b2; bj = j2; }
            }
            next = bj;
#ifdef PACO_IRSEG
            const long long b2c = clock64();
            sg_scan += b2c - b1c;
#endif
            n_cmp += cnt_total;  // construction.hpp:275
            if (!a.T) {
                // ColonyPheromone::end_step: reset the touched entries
                if (lane >= 1 && lane <= tl_cnt) acc[accx(tl0)] = tau0_alpha;
                for (uint32_t e = 31 + lane; e < tl_cnt; e += 32) acc[accx(lc[e + 1])] = tau0_alpha;
                __syncwarp();
            }
#ifdef PACO_IRSEG
            sg_end += clock64() - b2c;
#endif
        }
        ++n_dec;
        if (lane == 0) { out[pos] = next; vis[next >> 5] |= 1u << (next & 31); }
        __syncwarp();
        ++pos;
        cur = next;
    }
#ifdef PACO_IRSEG
    if (lane == 0) {
        atomicAdd(&g_timing[0], (unsigned long long)sg_begin); atomicAdd(&g_timing[1], (unsigned long long)sg_scan);
        atomicAdd(&g_timing[2], (unsigned long long)sg_wait); atomicAdd(&g_timing[3], (unsigned long long)sg_end);
        atomicAdd(&g_timing[4], n_dec); atomicAdd(&g_timing[5], n_cmp);
        atomicAdd(&g_timing[6], (unsigned long long)sg_ld); atomicAdd(&g_timing[7], (unsigned long long)sg_loop);
    }
#endif
    // maybe_two_opt consumes exactly one draw (two_opt.hpp:71-76)
    const uint32_t do2 = uniform() < a.two_opt_prob ? 1u : 0u;
    // stop the generator; the stream state after exactly cidx draws: the start state of the
    // chunk holding position cidx (alive: the generator never runs two rounds past the
    // consumption point) advanced by the remainder
    wait_for(cidx + 1);  // the chunk holding position cidx is produced: its start state is kept
    __syncwarp();
    if (lane == 0) {
        st_release_cta(&ring->consumed, cidx);
        ring->stop = 1;
        const unsigned long long* c = ring->ckpt[(cidx / kIrChunk) % kIrCkpt];
        uint64_t s[4] = {c[0], c[1], c[2], c[3]};
        for (uint32_t q = 0; q < cidx % kIrChunk; ++q) xoshiro_next(s);
        for (int q = 0; q < 4; ++q) a.rng[(size_t)ant * 4 + q] = s[q];
    }
    __syncwarp();
    if (do2) two_opt_exact<false>(out, n, a.two_opt_window, a.xy, nullptr, nullptr, nullptr, nullptr);
    const long long len = warp_tour_length(out, n, a.xy, lane);
    if (lane == 0) {
        a.new_len[ant] = len;
        a.partial_flag[ant] = (uint8_t)partial;
        atomicAdd(&a.counters[0], n_dec);
        atomicAdd(&a.counters[3], n_forced);
        atomicAdd(&a.counters[partial ? 5 : 4], 1ull);
        atomicAdd(&a.counters[8], n_cmp);
        if (do2) atomicAdd(&a.counters[9], 1ull);
    }
}

// ColonyPheromone::begin_step (construction.hpp:121-132) of every city, once per synchronous
// iteration: the colony is frozen for the iteration (engine.hpp:246-248), so the touched
// cities of a step at city c and their tau^alpha = Power(alpha)(tau0 + acc) are the same for
// every ant and every decision at c. One warp per city: the 2m contributions (ant q's prev
// then next of c, skipped when ratio q is 0) are staged, then applied 32 per pass - lanes that
// hit the same city are grouped (match.any) and the group's lowest lane adds them in lane
// order, so every acc receives its terms in ant order, the reference's fp64 sum order. The
// list of (touched city, tau^alpha) is written in first-occurrence order.
__global__ void __launch_bounds__(32) k_ir_touched(const uint2* __restrict__ nbr, const double* __restrict__ ratio,
                                                   uint32_t n, uint32_t m, double alpha, double tau0,
                                                   uint32_t* __restrict__ tl_city, double* __restrict__ tl_tau) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* acc = reinterpret_cast<double*>(smem_raw);   // n
    double* stage_r = acc + n;                           // m
    uint32_t* stage_c = reinterpret_cast<uint32_t*>(stage_r + m);  // 2m
    const uint32_t lane = threadIdx.x;
    for (uint32_t j = lane; j < n; j += 32) acc[j] = 0.0;
    for (uint32_t q = lane; q < m; q += 32) stage_r[q] = ratio[q];
    __syncwarp();
    for (uint32_t c = blockIdx.x; c < n; c += gridDim.x) {
        for (uint32_t q = lane; q < m; q += 32) {
            uint2 pr = make_uint2(kNone, kNone);
            if (stage_r[q] != 0.0) pr = nbr[(size_t)q * n + c];
            stage_c[2 * q] = pr.x;
            stage_c[2 * q + 1] = pr.y;
        }
        __syncwarp();
        for (uint32_t e0 = 0; e0 < 2 * m; e0 += 32) {
            const uint32_t e = e0 + lane;
            const uint32_t cc = e < 2 * m ? stage_c[e] : kNone;
            const unsigned live = __ballot_sync(kFull, cc != kNone);
            if (!live) continue;
            const unsigned grp = __match_any_sync(kFull, cc);
            const bool leader = cc != kNone && (int)lane == __ffs(grp) - 1;
            double v = leader ? acc[cc] : 0.0;
            const double* sr = stage_r + (e0 >> 1);
            const uint32_t nt = 2 * m - e0;
#pragma unroll
            for (uint32_t src = 0; src < 32; ++src) {
                const double x = src < nt ? sr[src >> 1] : 0.0;
                if ((grp >> src) & 1u) v = __dadd_rn(v, x);
            }
            if (leader) acc[cc] = v;
            __syncwarp();
        }
        // the list: each touched city once (its first occurrence), tau^alpha, then acc reset
        uint32_t cnt = 0;
        uint32_t* oc = tl_city + (size_t)c * (2 * m + 1) + 1;  // slot 0: the count
        double* ov = tl_tau + (size_t)c * 2 * m;
        for (uint32_t e0 = 0; e0 < 2 * m; e0 += 32) {
            const uint32_t e = e0 + lane;
            const uint32_t cc = e < 2 * m ? stage_c[e] : kNone;
            const unsigned grp = __match_any_sync(kFull, cc);
            const bool first_here = cc != kNone && (int)lane == __ffs(grp) - 1;
            // a city already listed by an earlier pass has acc reset to 0 (acc > 0 otherwise)
            const double a = first_here ? acc[cc] : 0.0;
            const bool emit = first_here && a > 0.0;
            const unsigned ball = __ballot_sync(kFull, emit);
            if (emit) {
                const uint32_t slot = cnt + __popc(ball & ((1u << lane) - 1u));
                oc[slot] = cc;
                ov[slot] = power(alpha, __dadd_rn(tau0, a));
                acc[cc] = 0.0;
            }
            cnt += __popc(ball);
            __syncwarp();
        }
        if (lane == 0) oc[-1] = cnt;
        __syncwarp();
    }
}

// Heuristic's table (construction.hpp:52-61): eta^beta of every pair as f32, the same
// expression the construction would otherwise evaluate per candidate and step
__global__ void k_eta_table(const double2* __restrict__ xy, uint32_t n, double beta, float* __restrict__ tab) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)n * n) return;
    const uint32_t i = (uint32_t)(idx / n), j = (uint32_t)(idx % n);
    int32_t d = euc2d(xy[i], xy[j]);
    if (d < 1) d = 1;
    tab[idx] = (float)power(beta, 1.0 / (double)d);
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
