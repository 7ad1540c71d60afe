// sm_100a kernels of the tour-construction engine. See DESIGN.md §4 for the
// roofline of each kernel and the reference function it replaces.
#pragma once
#include "device.cuh"

namespace pacob200 {

// ============================================================ K0: spatial sort
// key = morton(cell) << 32 | original index; sorted by cub (one-time setup).
__global__ void k_cell_keys(const double* __restrict__ xs, const double* __restrict__ ys, uint32_t n,
                            GridParams g, unsigned long long* __restrict__ keys) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t cx = cell_coord(xs[i], g.x0, g.inv, g.gw);
    const int32_t cy = cell_coord(ys[i], g.y0, g.inv, g.gh);
    keys[i] = ((unsigned long long)morton((uint32_t)cx, (uint32_t)cy) << 32) | i;
}

__global__ void k_scatter(const unsigned long long* __restrict__ keys, const double* __restrict__ xs,
                          const double* __restrict__ ys, uint32_t n, double2* __restrict__ xy,
                          uint32_t* __restrict__ orig_of, uint32_t* __restrict__ int_of,
                          uint32_t* __restrict__ cellm) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const unsigned long long key = keys[p];
    const uint32_t o = (uint32_t)key;
    orig_of[p] = o;
    int_of[o] = p;
    cellm[p] = (uint32_t)(key >> 32);
    xy[p] = make_double2(xs[o], ys[o]);
}

// cell_start[c] = first internal id with cell >= c (ncells + 1 entries)
__global__ void k_cell_start(const uint32_t* __restrict__ cellm, uint32_t n, uint32_t ncells,
                             uint32_t* __restrict__ cell_start) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const uint32_t c = cellm[p];
    const uint32_t lo = p == 0 ? 0 : cellm[p - 1] + 1;
    if (p == 0 || cellm[p - 1] != c)
        for (uint32_t q = lo; q <= c; ++q) cell_start[q] = p;
    if (p == n - 1)
        for (uint32_t q = c + 1; q <= ncells; ++q) cell_start[q] = n;
}

// ============================================================ K1: k-NN lists
// Per city: the k nearest other cities by (d^2, original index). One CTA per
// superblock; the 3x3 superblock neighbourhood is staged in shared memory when it
// fits, and a city whose k-th key is not certified by the staged region's border
// (sparse areas, dense clusters) falls back to an exact ring search over global
// memory. Output rows are in internal ids; eta^beta (construction.hpp:46-61) is
// emitted alongside.
template <int KMAX>
struct TopK {
    double d[KMAX];
    uint32_t o[KMAX], j[KMAX];
    __device__ void init() {
#pragma unroll
        for (int r = 0; r < KMAX; ++r) { d[r] = __longlong_as_double(0x7ff0000000000000LL); o[r] = kNone; j[r] = kNone; }
    }
    __device__ __forceinline__ void offer(double dd, uint32_t oo, uint32_t jj, int k) {
        if (!key_less(dd, oo, d[k - 1], o[k - 1])) return;
#pragma unroll
        for (int r = KMAX - 1; r > 0; --r) {
            if (r < k) {
                if (key_less(dd, oo, d[r - 1], o[r - 1])) { d[r] = d[r - 1]; o[r] = o[r - 1]; j[r] = j[r - 1]; }
                else if (key_less(dd, oo, d[r], o[r])) { d[r] = dd; o[r] = oo; j[r] = jj; }
            }
        }
        if (key_less(dd, oo, d[0], o[0])) { d[0] = dd; o[0] = oo; j[0] = jj; }
    }
};

template <int KMAX>
__device__ void knn_ring_search(uint32_t i, double2 q, const double2* __restrict__ xy,
                                const uint32_t* __restrict__ orig_of, const uint32_t* __restrict__ cell_start,
                                const GridParams& g, int k, TopK<KMAX>& t) {
    t.init();
    const int32_t cx = cell_coord(q.x, g.x0, g.inv, g.gw), cy = cell_coord(q.y, g.y0, g.inv, g.gh);
    const int32_t rmax = g.gw > g.gh ? g.gw : g.gh;
    uint32_t found = 0;
    for (int32_t rho = 0; rho <= rmax; ++rho) {
        if (rho >= 1 && found >= (uint32_t)k) {
            const double lb = ((double)rho - 1.0 - 1e-6) * g.cs;
            if (lb > 0 && lb * lb > t.d[k - 1]) break;
        }
        const int32_t cnt = rho == 0 ? 1 : 8 * rho;
        for (int32_t c = 0; c < cnt; ++c) {
            int32_t x = cx, y = cy;
            if (rho) ring_cell(rho, c, cx, cy, x, y);
            if (x < 0 || y < 0 || x >= g.gw || y >= g.gh) continue;
            const uint32_t m = morton((uint32_t)x, (uint32_t)y);
            const uint32_t s = cell_start[m], e = cell_start[m + 1];
            for (uint32_t jj = s; jj < e; ++jj) {
                if (jj == i) continue;
                ++found;
                t.offer(dist2(q, xy[jj]), orig_of[jj], jj, k);
            }
        }
    }
}

template <int KMAX>
__device__ void knn_emit(uint32_t i, double2 q, const TopK<KMAX>& t, int k, const double2* __restrict__ xy,
                         double beta, uint32_t* __restrict__ knn, float* __restrict__ eta) {
#pragma unroll
    for (int r = 0; r < KMAX; ++r) {
        if (r < k) {
            const uint32_t jj = t.j[r];
            knn[(size_t)i * k + r] = jj;
            int32_t d = euc2d(q, xy[jj]);
            if (d < 1) d = 1;
            eta[(size_t)i * k + r] = (float)power(beta, 1.0 / (double)d);
        }
    }
}

template <int KMAX>
__global__ void __launch_bounds__(128) k_knn(const double2* __restrict__ xy, const uint32_t* __restrict__ orig_of,
                                             const uint32_t* __restrict__ cell_start, GridParams g, uint32_t n,
                                             int k, double beta, uint32_t cap, uint32_t* __restrict__ knn,
                                             float* __restrict__ eta, uint32_t* __restrict__ n_global) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t sb = blockIdx.x;
    const uint32_t s0 = cell_start[sb << 6], e0 = cell_start[(sb + 1) << 6];
    if (s0 >= e0) return;
    const int32_t sbx = (int32_t)compact16(sb), sby = (int32_t)compact16(sb >> 1);
    // staged neighbourhood: up to 9 contiguous id ranges
    __shared__ uint32_t rs[9], re[9], roff[10];
    if (threadIdx.x == 0) {
        uint32_t off = 0;
        for (int q = 0; q < 9; ++q) {
            const int32_t x = sbx + q % 3 - 1, y = sby + q / 3 - 1;
            uint32_t a = 0, b = 0;
            if (x >= 0 && y >= 0 && x < g.gws && y < g.ghs) {
                const uint32_t m = morton((uint32_t)x, (uint32_t)y);
                a = cell_start[m << 6]; b = cell_start[(m + 1) << 6];
            }
            rs[q] = a; re[q] = b; roff[q] = off; off += b - a;
        }
        roff[9] = off;
    }
    __syncthreads();
    const uint32_t C = roff[9];
    const bool staged = C <= cap;
    double2* sxy = reinterpret_cast<double2*>(smem);
    uint32_t* so = reinterpret_cast<uint32_t*>(sxy + (staged ? C : 0));
    uint32_t* sj = so + (staged ? C : 0);
    if (staged) {
        for (int q = 0; q < 9; ++q)
            for (uint32_t p = rs[q] + threadIdx.x; p < re[q]; p += blockDim.x) {
                const uint32_t dst = roff[q] + (p - rs[q]);
                sxy[dst] = xy[p]; so[dst] = orig_of[p]; sj[dst] = p;
            }
    }
    __syncthreads();
    // staged region border (infinite where the region reaches the grid edge)
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    const double span = 8.0 * g.cs;
    const double xlo = sbx >= 2 ? g.x0 + (sbx - 1) * span : -inf;
    const double xhi = sbx + 2 < g.gws ? g.x0 + (sbx + 2) * span : inf;
    const double ylo = sby >= 2 ? g.y0 + (sby - 1) * span : -inf;
    const double yhi = sby + 2 < g.ghs ? g.y0 + (sby + 2) * span : inf;
    for (uint32_t i = s0 + threadIdx.x; i < e0; i += blockDim.x) {
        const double2 q = xy[i];
        TopK<KMAX> t;
        bool ok = false;
        if (staged) {
            t.init();
            for (uint32_t p = 0; p < C; ++p) {
                if (sj[p] == i) continue;
                t.offer(dist2(q, sxy[p]), so[p], sj[p], k);
            }
            double lb = fmin(fmin(q.x - xlo, xhi - q.x), fmin(q.y - ylo, yhi - q.y));
            if (C >= (uint32_t)k + 1) {
                if (lb == inf) ok = true;  // the staged region is the whole instance
                else {
                    lb -= 1e-6 * g.cs;
                    ok = lb > 0 && lb * lb > t.d[k - 1];
                }
            }
        }
        if (!ok) {
            atomicAdd(n_global, 1u);
            knn_ring_search<KMAX>(i, q, xy, orig_of, cell_start, g, k, t);
        }
        knn_emit<KMAX>(i, q, t, k, xy, beta, knn, eta);
    }
}

// ============================================================ K5: weight table
// Per iteration, for every candidate edge (i, c_r): tau = tau0 + sum over ants a in
// ant order of ratio_a * [c_r in {prev_a(i), next_a(i)}]  (fp64, bit-identical to
// ColonyPheromone::begin_step, construction.hpp:121-132, restricted to candidate
// edges; ratios per colony.hpp:159-177), w = f32(Power(alpha)(tau)) * eta^beta (f32).
// Classic mode reads tau from the candidate-edge pheromone table T instead.
// Output: packed {c_r, w} rows, the only table the construction kernel reads.
template <int KMAX>
__global__ void __launch_bounds__(256) k_weights(const uint32_t* __restrict__ knn, const float* __restrict__ eta,
                                                 const uint2* __restrict__ nbr, const int64_t* __restrict__ lb_len,
                                                 const uint8_t* __restrict__ has_lb, const int64_t* __restrict__ g_len,
                                                 const double* __restrict__ T, uint32_t n, uint32_t m, int k,
                                                 double alpha, double tau0, uint2* __restrict__ cand) {
    extern __shared__ double ratio[];
    if (!T) {
        const double g = (double)*g_len;
        for (uint32_t a = threadIdx.x; a < m; a += blockDim.x) {
            double r = 0.0;
            if (has_lb[a]) { r = g / (double)lb_len[a]; r = r > 1.0 ? 1.0 : r; }
            ratio[a] = r;
        }
        __syncthreads();
    }
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t c[KMAX];
    double acc[KMAX];
#pragma unroll
    for (int r = 0; r < KMAX; ++r) { c[r] = r < k ? knn[(size_t)i * k + r] : kNone; acc[r] = 0.0; }
    if (!T) {
        for (uint32_t a = 0; a < m; ++a) {
            const double ra = ratio[a];
            if (ra == 0.0) continue;
            const uint2 p = __ldcs(&nbr[(size_t)a * n + i]);
#pragma unroll
            for (int r = 0; r < KMAX; ++r) {
                if (c[r] == p.x) acc[r] = __dadd_rn(acc[r], ra);
                if (c[r] == p.y) acc[r] = __dadd_rn(acc[r], ra);
            }
        }
    }
#pragma unroll
    for (int r = 0; r < KMAX; ++r) {
        if (r < k) {
            const double tau = T ? T[(size_t)i * k + r] : __dadd_rn(tau0, acc[r]);
            const float w = __fmul_rn((float)power(alpha, tau), eta[(size_t)i * k + r]);
            cand[(size_t)i * k + r] = make_uint2(c[r], __float_as_uint(w));
        }
    }
}

// ============================================================ K2: construction
struct ConstructArgs {
    const uint2* cand;        // n*k {city, f32 weight}
    const double2* xy;        // internal coordinates
    const uint32_t* orig_of;  // internal -> original (fallback tie-break)
    const uint32_t* int_of;   // original -> internal (start city draw)
    const uint32_t* cell_start;
    GridParams g;
    uint32_t* tours;          // m * 2 * n; l_best in half lb_sel[a], new tour in the other
    const uint8_t* lb_sel;
    int64_t* new_len;
    uint8_t* partial_flag;
    unsigned long long* counters; // decisions, fallbacks, ties, forced, full, partial
    const uint32_t* words;    // validation draws: m rows of `stride` words (nullptr = Philox)
    uint64_t stride;
    uint64_t seed, iter;
    uint32_t n, m, k, nwords;
    double eff_pp, mmf;
    int seeding;
    int validate;
    int* err;
    // explicit construct_partial_at (tests): ant = force_ant, params given
    int force;
    uint32_t force_ant, force_start_pos, force_m_mod;
};

// Exact nearest unvisited city by (d^2, original index), warp-cooperative.
// Phase 1: Chebyshev rings of fine cells around cur (radius <= 2). Phase 2: rings
// of 8x8-cell superblocks with rectangle lower bounds, pruning fully visited
// superblocks with the shared-memory bitmap and far cells with the running bound.
__device__ __noinline__ uint32_t nearest_unvisited(const ConstructArgs& a, const uint32_t* vis, uint32_t cur,
                                                   uint32_t lane) {
    const GridParams& g = a.g;
    const double2 q = a.xy[cur];
    const int32_t cx = cell_coord(q.x, g.x0, g.inv, g.gw), cy = cell_coord(q.y, g.y0, g.inv, g.gh);
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    double bd = inf;
    uint32_t bo = kNone, bj = kNone;
    const double slack = 1e-6 * g.cs;
    constexpr int32_t R1 = 2;
    for (int32_t rho = 0; rho <= R1 + 1; ++rho) {
        if (rho >= 1) {
            const double lb = (rho - 1) * g.cs - slack;
            if (lb > 0 && lb * lb > bd) return bj;
        }
        if (rho > R1) break;
        const int32_t cnt = rho == 0 ? 1 : 8 * rho;
        for (int32_t c = lane; c < cnt; c += 32) {
            int32_t x = cx, y = cy;
            if (rho) ring_cell(rho, c, cx, cy, x, y);
            if (x < 0 || y < 0 || x >= g.gw || y >= g.gh) continue;
            const uint32_t m = morton((uint32_t)x, (uint32_t)y);
            const uint32_t s = a.cell_start[m], e = a.cell_start[m + 1];
            for (uint32_t j = s; j < e; ++j) {
                if (is_visited(vis, j)) continue;
                const double d = dist2(q, a.xy[j]);
                const uint32_t o = a.orig_of[j];
                if (key_less(d, o, bd, bo)) { bd = d; bo = o; bj = j; }
            }
        }
        warp_argmin(bd, bo, bj);
    }
    // phase 2: superblock rings
    const int32_t sx = cx >> 3, sy = cy >> 3;
    const int32_t rmax = g.gws > g.ghs ? g.gws : g.ghs;
    const double span = 8.0 * g.cs;
    for (int32_t rho = 0; rho <= rmax; ++rho) {
        if (rho >= 1) {
            const double lb = (rho - 1) * span - slack;
            if (lb > 0 && lb * lb > bd) break;
        }
        const int32_t cnt = rho == 0 ? 1 : 8 * rho;
        for (int32_t base = 0; base < cnt; base += 32) {
            const int32_t c = base + (int32_t)lane;
            bool cand = false;
            uint32_t sbm = 0;
            if (c < cnt) {
                int32_t x = sx, y = sy;
                if (rho) ring_cell(rho, c, sx, sy, x, y);
                if (x >= 0 && y >= 0 && x < g.gws && y < g.ghs) {
                    const double rx0 = g.x0 + x * span, rx1 = rx0 + span;
                    const double ry0 = g.y0 + y * span, ry1 = ry0 + span;
                    const double dx = fmax(0.0, fmax(rx0 - q.x, q.x - rx1));
                    const double dy = fmax(0.0, fmax(ry0 - q.y, q.y - ry1));
                    const double lb = sqrt(dx * dx + dy * dy) - slack;
                    if (!(lb > 0 && lb * lb > bd)) {
                        sbm = morton((uint32_t)x, (uint32_t)y);
                        cand = range_has_unvisited(vis, a.cell_start[sbm << 6], a.cell_start[(sbm + 1) << 6]);
                    }
                }
            }
            unsigned ball = __ballot_sync(kFull, cand);
            while (ball) {
                const int src = __ffs(ball) - 1;
                ball &= ball - 1;
                const uint32_t sb = __shfl_sync(kFull, sbm, src);
                const double bound = bd;  // warp-uniform at this point
                // 64 cells of the superblock, two per lane, pruned by the running bound
                for (uint32_t cc = lane; cc < 64; cc += 32) {
                    const uint32_t cm = (sb << 6) | cc;
                    const uint32_t s = a.cell_start[cm], e = a.cell_start[cm + 1];
                    if (s >= e) continue;
                    const int32_t x = (int32_t)compact16(cm), y = (int32_t)compact16(cm >> 1);
                    const double rx0 = g.x0 + x * g.cs, rx1 = rx0 + g.cs;
                    const double ry0 = g.y0 + y * g.cs, ry1 = ry0 + g.cs;
                    const double dx = fmax(0.0, fmax(rx0 - q.x, q.x - rx1));
                    const double dy = fmax(0.0, fmax(ry0 - q.y, q.y - ry1));
                    const double lb = sqrt(dx * dx + dy * dy) - slack;
                    if (lb > 0 && lb * lb > bound) continue;
                    for (uint32_t j = s; j < e; ++j) {
                        if (is_visited(vis, j)) continue;
                        const double d = dist2(q, a.xy[j]);
                        const uint32_t o = a.orig_of[j];
                        if (key_less(d, o, bd, bo)) { bd = d; bo = o; bj = j; }
                    }
                }
                warp_argmin(bd, bo, bj);
            }
        }
    }
    return bj;
}

// the single remaining unvisited city (forced final step)
__device__ __noinline__ uint32_t last_unvisited(const uint32_t* vis, uint32_t nwords, uint32_t lane) {
    for (uint32_t base = 0; base < nwords; base += 32) {
        const uint32_t w = base + lane;
        const uint32_t free_bits = w < nwords ? ~vis[w] : 0u;
        const unsigned ball = __ballot_sync(kFull, free_bits != 0);
        if (ball) {
            const int src = __ffs(ball) - 1;
            const uint32_t fb = __shfl_sync(kFull, free_bits, src);
            return (base + src) * 32 + (__ffs(fb) - 1);
        }
    }
    return kNone;
}

// One warp per ant (construction.hpp:283-365 with the north-star selection rule,
// engine.hpp:129-148 draw order). The visited bitmap (n bits) lives in shared
// memory; each decision is one coalesced 8-byte-per-lane load of the current
// city's candidate row, a bitmap probe, a warp inclusive scan, a ballot and a
// shuffle. Preserved-segment copy, tour length and the optional permutation
// check are warp-parallel passes fused before/after the dependent chain.
__global__ void __launch_bounds__(32) k_construct(ConstructArgs a) {
    extern __shared__ uint32_t vis[];
    const uint32_t lane = threadIdx.x;
    const uint32_t ant = a.force ? a.force_ant : blockIdx.x;
    const uint32_t n = a.n, k = a.k, nw = a.nwords;
    auto word = [&](uint32_t slot) -> uint32_t {
        if (a.words) return a.words[(a.force ? 0 : (uint64_t)ant * a.stride) + slot];
        const uint4 v = philox10(make_uint4(slot >> 2, ant, (uint32_t)a.iter, (uint32_t)(a.iter >> 32)),
                                 make_uint2((uint32_t)a.seed, (uint32_t)(a.seed >> 32)));
        return pick_word(v, slot & 3);
    };
    for (uint32_t w = lane; w < nw; w += 32) vis[w] = 0u;
    __syncwarp();
    if (lane == 0 && (n & 31)) vis[nw - 1] = 0xffffffffu << (n & 31);  // padding bits count as visited
    __syncwarp();
    const uint8_t sel = a.lb_sel[ant];
    uint32_t* out = a.tours + ((size_t)ant * 2 + (1 - sel)) * n;
    const uint32_t* lb = a.tours + ((size_t)ant * 2 + sel) * n;
    bool partial = false;
    uint32_t start_pos = 0, m_mod = 0;
    if (a.force) { partial = true; start_pos = a.force_start_pos; m_mod = a.force_m_mod; }
    else if (!a.seeding) {
        partial = u01_f64(word(0)) < a.eff_pp;  // engine.hpp:137-138
        if (partial) {
            start_pos = below(word(1), n);       // construction.hpp:358
            double capd = floor(a.mmf * (double)n);
            if (capd < 2.0) capd = 2.0;
            m_mod = 2 + below(word(2), (uint32_t)capd - 1);  // construction.hpp:359-362
        }
    }
    uint32_t pos, cur;
    if (!partial) {
        const uint32_t start = a.int_of[below(word(1), n)];  // construction.hpp:291
        if (lane == 0) { out[0] = start; vis[start >> 5] |= 1u << (start & 31); }
        pos = 1; cur = start;
    } else {
        // construction.hpp:322-333: copy the cyclic preserved segment of l_best
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
            pos = 1; cur = anchor;
        } else {
            pos = preserved;
            uint32_t p = start_pos + preserved - 1; if (p >= n) p -= n;
            cur = lb[p];
        }
    }
    __syncwarp();

    unsigned long long n_dec = 0, n_fb = 0, n_tie = 0, n_forced = 0;
    uint4 pw = make_uint4(0, 0, 0, 0);
    const uint2 key = make_uint2((uint32_t)a.seed, (uint32_t)(a.seed >> 32));
    uint32_t remaining = n - pos;
    for (uint32_t t = 0; remaining > 0; ++t, --remaining) {
        uint32_t next;
        ++n_dec;
        if (remaining == 1) {
            next = last_unvisited(vis, nw, lane);
            ++n_forced;
#ifdef PACO_DEBUG
            {
                uint32_t zeros = 0;
                for (uint32_t w = lane; w < nw; w += 32) zeros += __popc(~vis[w]);
                for (int off = 16; off; off >>= 1) zeros += __shfl_xor_sync(kFull, zeros, off);
                if (lane == 0 && zeros != 1) printf("DBG ant %u pos %u forced: zeros=%u next=%u\n", ant, pos, zeros, next);
            }
#endif
        } else {
            uint32_t uw;
            if (a.words) uw = a.words[(a.force ? 0 : (uint64_t)ant * a.stride) + 4 + t];
            else {
                if ((t & 3) == 0)
                    pw = philox10(make_uint4(1 + (t >> 2), ant, (uint32_t)a.iter, (uint32_t)(a.iter >> 32)), key);
                uw = pick_word(pw, t & 3);
            }
            uint2 e = make_uint2(kNone, 0u);
            if (lane < k) e = __ldg(&a.cand[(size_t)cur * k + lane]);
            float w = 0.0f;
            if (lane < k && !is_visited(vis, e.x)) w = __uint_as_float(e.y);
            // Hillis-Steele inclusive scan over the k candidate lanes
            float v = w;
            for (uint32_t off = 1; off < k; off <<= 1) {
                const float y = __shfl_up_sync(kFull, v, off);
                if (lane >= off) v = __fadd_rn(v, y);
            }
            const float S = __shfl_sync(kFull, v, k - 1);
            if (S > 0.0f) {
                const float target = __fmul_rn(u01_f32(uw), S);
                const float tol = __fmul_rn(1e-6f, S);
                const bool in = lane < k;
                if (__any_sync(kFull, in && fabsf(__fsub_rn(v, target)) <= tol)) ++n_tie;
                // only feasible lanes may win: the tree-shaped scan is not monotone in f32,
                // so an infeasible lane's S_r can exceed its left neighbour's by an ulp
                unsigned ball = __ballot_sync(kFull, in && w > 0.0f && v > target);
                int r;
                if (ball) r = __ffs(ball) - 1;
                else r = 31 - __clz(__ballot_sync(kFull, in && w > 0.0f));
                next = __shfl_sync(kFull, e.x, r);
            } else {
                next = nearest_unvisited(a, vis, cur, lane);
                ++n_fb;
            }
        }
#ifdef PACO_DEBUG
        {
            const uint32_t nx0 = __shfl_sync(kFull, next, 0);
            if (!__all_sync(kFull, nx0 == next) && lane == 0) printf("DBG ant %u pos %u non-uniform next\n", ant, pos);
            if (is_visited(vis, next)) {
                for (uint32_t q = lane; q < pos; q += 32)
                    if (out[q] == next) printf("DBG ant %u pos %u dup next=%u rem=%u earlier at %u (partial=%d start_pos=%u m_mod=%u)\n", ant, pos, next, remaining, q, (int)partial, start_pos, m_mod);
                if (lane == 0) printf("DBG ant %u pos %u dup next=%u word=%08x\n", ant, pos, next, vis[next >> 5]);
            }
        }
#endif
        if (lane == 0) { out[pos] = next; vis[next >> 5] |= 1u << (next & 31); }
        __syncwarp();
        ++pos;
        cur = next;
    }
    __syncwarp();
    // tour length (instance.hpp:120-127), int64, warp-parallel over positions
    long long len = 0;
    for (uint32_t p = lane; p < n; p += 32) {
        const uint32_t c0 = out[p], c1 = out[p + 1 < n ? p + 1 : 0];
        len += euc2d(a.xy[c0], a.xy[c1]);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) len += __shfl_xor_sync(kFull, len, off);
    if (a.validate) {
        // permutation check (instance.hpp:109-117) reusing the bitmap
        for (uint32_t w = lane; w < nw; w += 32) vis[w] = 0u;
        __syncwarp();
        bool bad = false;
        for (uint32_t p = lane; p < n; p += 32) {
            const uint32_t c = out[p];
            if (c >= n) { bad = true; continue; }
            const uint32_t old = atomicOr(&vis[c >> 5], 1u << (c & 31));
            if (old & (1u << (c & 31))) bad = true;
        }
        if (__any_sync(kFull, bad) && lane == 0) atomicExch(a.err, 1);
    }
    if (lane == 0) {
        a.new_len[ant] = len;
        if (!a.force) {
            a.partial_flag[ant] = partial ? 1 : 0;
            atomicAdd(&a.counters[0], n_dec);
            atomicAdd(&a.counters[1], n_fb);
            atomicAdd(&a.counters[2], n_tie);
            atomicAdd(&a.counters[3], n_forced);
            atomicAdd(&a.counters[partial ? 5 : 4], 1ull);
        }
    }
}

// ============================================================ K4: completion step
// engine.hpp:261-265: for every ant in order, update_l_best (strict improvement,
// colony.hpp:117-124) then update_g_best (colony.hpp:127-139). The l_best switch is
// a flip of the ant's double-buffer selector, so no tour is copied.
struct GBest { long long len; int32_t ant; int32_t has; };

__global__ void k_update(uint32_t first, uint32_t count, const int64_t* __restrict__ new_len,
                         int64_t* __restrict__ lb_len, uint8_t* __restrict__ has_lb, uint8_t* __restrict__ lb_sel,
                         uint8_t* __restrict__ improved, GBest* __restrict__ gb, int64_t* __restrict__ g_len,
                         unsigned long long* __restrict__ counters) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    GBest g = *gb;
    unsigned long long imp = 0;
    for (uint32_t a = first; a < first + count; ++a) {
        const int64_t L = new_len[a];
        if (!has_lb[a] || L < lb_len[a]) {
            has_lb[a] = 1; lb_len[a] = L; lb_sel[a] ^= 1; improved[a] = 1; ++imp;
            if (!g.has || L < g.len) { g.len = L; g.ant = (int32_t)a; g.has = 1; }
        } else {
            improved[a] = 0;
        }
    }
    *gb = g;
    *g_len = g.has ? g.len : 0x7fffffffffffffffLL;
    counters[7] += imp;
}

// Ant::publish (colony.hpp:39-52) for the improved ants: neighbour pairs of the new
// l_best, nbr[a][city] = (prev, next). Grid (ceil(n/256), m).
__global__ void k_publish(const uint32_t* __restrict__ tours, const uint8_t* __restrict__ lb_sel,
                          const uint8_t* __restrict__ improved, uint32_t n, int current,
                          uint2* __restrict__ nbr) {
    const uint32_t a = blockIdx.y;
    if (!current && !improved[a]) return;
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const uint8_t half = current ? (uint8_t)(1 - lb_sel[a]) : lb_sel[a];
    const uint32_t* t = tours + ((size_t)a * 2 + half) * n;
    const uint32_t prev = t[p == 0 ? n - 1 : p - 1], next = t[p + 1 == n ? 0 : p + 1];
    nbr[(size_t)a * n + t[p]] = make_uint2(prev, next);
}

// ============================================================ K6: classic mode
// PheromoneMatrix::evaporate + deposit (construction.hpp:187-207) restricted to the
// candidate edges (each entry evolves independently, so the restriction is exact):
// T = max(T (1-rho), 1e-6), then for every built tour in tour order T += 1/C_a when
// the tour contains the edge. cur_nbr holds the built tours' neighbour pairs.
template <int KMAX>
__global__ void __launch_bounds__(256) k_classic(const uint32_t* __restrict__ knn, const uint2* __restrict__ cur_nbr,
                                                 const int64_t* __restrict__ new_len, uint32_t n, uint32_t m, int k,
                                                 double rho, double* __restrict__ T) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t c[KMAX];
    double t[KMAX];
    const double keep = 1.0 - rho;
#pragma unroll
    for (int r = 0; r < KMAX; ++r) {
        c[r] = r < k ? knn[(size_t)i * k + r] : kNone;
        if (r < k) {
            double v = __dmul_rn(T[(size_t)i * k + r], keep);
            t[r] = v < 1e-6 ? 1e-6 : v;
        } else t[r] = 0.0;
    }
    for (uint32_t a = 0; a < m; ++a) {
        const uint2 p = cur_nbr[(size_t)a * n + i];
        const double delta = 1.0 / (double)new_len[a];
#pragma unroll
        for (int r = 0; r < KMAX; ++r)
            if (c[r] == p.x || c[r] == p.y) t[r] = __dadd_rn(t[r], delta);
    }
#pragma unroll
    for (int r = 0; r < KMAX; ++r)
        if (r < k) T[(size_t)i * k + r] = t[r];
}

// reference-order tour -> internal ids (host offers), and internal -> original on readback
__global__ void k_map(const uint32_t* __restrict__ in, const uint32_t* __restrict__ table, size_t count,
                      uint32_t* __restrict__ out) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) out[i] = table[in[i]];
}

__global__ void k_tour_length(const uint32_t* __restrict__ t, const double2* __restrict__ xy, uint32_t n,
                              unsigned long long* __restrict__ out) {
    long long len = 0;
    for (uint32_t p = threadIdx.x; p < n; p += blockDim.x)
        len += euc2d(xy[t[p]], xy[t[p + 1 < n ? p + 1 : 0]]);
    atomicAdd(out, (unsigned long long)len);
}

} // namespace pacob200
