// sm_100a kernels of the tour-construction engine. See DESIGN.md §4 for the
// roofline of each kernel and the reference function it replaces.
#pragma once
#include "device.cuh"

#if defined(PACO_TIMING) || defined(PACO_SPECSTAT) || defined(PACO_PHASES) || defined(PACO_IRSEG) || defined(PACO_ANTPROF)
#define PACO_DEBUG_SYMS
#endif

namespace pacob200 {
#ifdef PACO_DEBUG_SYMS
__device__ unsigned long long g_timing[16];
__device__ unsigned long long g_prof[96];  // ant 0 profile by tour position (20 buckets)
#ifdef PACO_ANTPROF
__device__ unsigned long long g_ant[4096 * 6];  // per ant: start ns, end ns, smid, decisions, fallbacks, partial
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif
#endif

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

// sb_start[b] = first internal id of Morton superblock b (8x8 cells = 64 Morton codes)
__global__ void k_sb_start(const uint32_t* __restrict__ cell_start, uint32_t nsb, uint32_t* __restrict__ sb_start) {
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b <= nsb) sb_start[b] = cell_start[(size_t)b << 6];
}

// ============================================================ K1: k-NN lists
// Per city: the k nearest other cities by (d^2, original index), rows in internal
// ids; eta^beta (construction.hpp:46-61) is emitted alongside.
// Bounded max-heap of the KMAX smallest (d^2, original index) keys seen so far (root =
// current worst), kept in shared memory: element p of thread t at [p * T + t], so that
// threads touching the same heap level hit distinct banks. An accepted candidate costs
// O(log KMAX); the original index (tie-break key) is read only on an exact distance tie.
// (The per-thread arrays in local memory spilled to DRAM: 35 GB per C5 build.)
template <int KMAX, int T>
struct NearHeap {
    double* d;
    uint32_t* j;
    const uint32_t* __restrict__ orig_of;
    int size;
    __device__ __forceinline__ double D(int p) const { return d[p * T]; }
    __device__ __forceinline__ uint32_t J(int p) const { return j[p * T]; }
    __device__ __forceinline__ bool worse(int a, int b) const {  // key[a] > key[b]
        const double da = D(a), db = D(b);
        return da != db ? da > db : orig_of[J(a)] > orig_of[J(b)];
    }
    __device__ __forceinline__ void swap_(int a, int b) {
        const double td = d[a * T]; d[a * T] = d[b * T]; d[b * T] = td;
        const uint32_t tj = j[a * T]; j[a * T] = j[b * T]; j[b * T] = tj;
    }
    __device__ void sift_down(int p, int m) {
        for (;;) {
            const int l = 2 * p + 1, r = l + 1;
            int big = p;
            if (l < m && worse(l, big)) big = l;
            if (r < m && worse(r, big)) big = r;
            if (big == p) return;
            swap_(p, big);
            p = big;
        }
    }
    __device__ void offer(double dd, uint32_t jj, int k) {
        if (size < k) {
            int p = size++;
            d[p * T] = dd; j[p * T] = jj;
            while (p > 0) {
                const int q = (p - 1) / 2;
                if (!worse(p, q)) break;
                swap_(p, q);
                p = q;
            }
            return;
        }
        const double d0 = D(0);
        if (dd > d0 || (dd == d0 && orig_of[jj] >= orig_of[J(0)])) return;
        d[0] = dd; j[0] = jj;
        sift_down(0, size);
    }
    __device__ void sort() {
        for (int m = size - 1; m > 0; --m) { swap_(0, m); sift_down(0, m); }
    }
};

template <int KMAX, int T>
__device__ void near_ring_search(uint32_t i, double2 q, const double2* __restrict__ xy,
                                 const uint32_t* __restrict__ cell_start, const GridParams& g, int k,
                                 NearHeap<KMAX, T>& t) {
    t.size = 0;
    const int32_t cx = cell_coord(q.x, g.x0, g.inv, g.gw), cy = cell_coord(q.y, g.y0, g.inv, g.gh);
    const int32_t rmax = g.gw > g.gh ? g.gw : g.gh;
    for (int32_t rho = 0; rho <= rmax; ++rho) {
        if (rho >= 1 && t.size >= k) {
            const double lb = ((double)rho - 1.0 - 1e-6) * g.cs;
            if (lb > 0 && lb * lb > t.D(0)) break;
        }
        const int32_t cnt = rho == 0 ? 1 : 8 * rho;
        for (int32_t c = 0; c < cnt; ++c) {
            int32_t x = cx, y = cy;
            if (rho) ring_cell(rho, c, cx, cy, x, y);
            if (x < 0 || y < 0 || x >= g.gw || y >= g.gh) continue;
            const uint32_t m = morton((uint32_t)x, (uint32_t)y);
            const uint32_t s = cell_start[m], e = cell_start[m + 1];
            for (uint32_t jj = s; jj < e; ++jj)
                if (jj != i) t.offer(dist2(q, xy[jj]), jj, k);
        }
    }
    t.sort();
}

// One thread per city (internal id order, so a CTA covers a compact patch and its cell
// scans share L1 lines), exact ring search over grid cells until the ring's lower bound
// exceeds the current k-th key. Work per city follows the local density (about 100
// candidates in uniform areas). A superblock-staged variant (3x3 superblocks in shared
// memory, one CTA per superblock) measured 14x slower at C5: in dense clusters every
// city scanned thousands of staged cities, and the 147 KB stage allowed one CTA per SM.
template <int KMAX, int T>
__global__ void __launch_bounds__(T) k_knn_cells(const double2* __restrict__ xy, const uint32_t* __restrict__ orig_of,
                                                 const uint32_t* __restrict__ cell_start, GridParams g, uint32_t n,
                                                 int kk, int k, double beta, uint32_t* __restrict__ knn32,
                                                 float* __restrict__ eta) {
    extern __shared__ __align__(16) unsigned char heap_smem[];  // d[KMAX][T] | j[KMAX][T]
    const uint32_t i = blockIdx.x * T + threadIdx.x;
    if (i >= n) return;
    NearHeap<KMAX, T> t;
    t.d = reinterpret_cast<double*>(heap_smem) + threadIdx.x;
    t.j = reinterpret_cast<uint32_t*>(heap_smem + sizeof(double) * KMAX * T) + threadIdx.x;
    t.orig_of = orig_of;
    const double2 q = xy[i];
    near_ring_search<KMAX, T>(i, q, xy, cell_start, g, kk, t);  // leaves the heap sorted
    for (int r = 0; r < KMAX; ++r) {
        const uint32_t jj = r < kk ? t.J(r) : kNone;
        knn32[(size_t)i * KMAX + r] = jj;
        if (r < k) {
            int32_t d = euc2d(q, xy[jj]);
            if (d < 1) d = 1;
            eta[(size_t)i * k + r] = (float)power(beta, 1.0 / (double)d);
        }
    }
}

// ============================================================ K5: weight table
// Per-city perfect hash of the candidate list (setup, once per instance): the multiplier
// M_i maps the k candidates of city i to distinct slots (c * M_i) >> (32 - B) of 2^B, so
// k_weights finds the candidate index of a neighbour with one shared-memory lookup
// instead of k comparisons. B = hash_slot_bits(k): 32 slots for k <= 16 (success 1.04%
// per trial at k = 16), 64 for k <= 24 (0.8% at k = 24, 5.1% at k = 20), 128 for k <= 32
// (1.5% at k = 32). Trial multipliers are odd SplitMix values of (i, trial), 2^14 trials
// are allowed; a city without one sets *fail and k_weights keeps the comparison loop.
__host__ __device__ constexpr int hash_slot_bits(int kmax) { return kmax <= 16 ? 5 : kmax <= 24 ? 6 : 7; }
template <int B>
__device__ __forceinline__ uint32_t cand_slot(uint32_t c, uint32_t M) { return (c * M) >> (32 - B); }
template <int KMAX>
__global__ void k_cand_hash(const uint32_t* __restrict__ knn32, uint32_t n, int k, uint32_t* __restrict__ mult,
                            int* __restrict__ fail) {
    constexpr int B = hash_slot_bits(KMAX), W = (1 << B) / 32;
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t c[KMAX];
#pragma unroll
    for (int r = 0; r < KMAX; ++r) c[r] = r < k ? knn32[(size_t)i * kNearRow + r] : 0u;
    for (uint32_t t = 0; t < (1u << 14); ++t) {
        unsigned long long z = ((unsigned long long)i << 20 | t) + 0x9e3779b97f4a7c15ull;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        const uint32_t M = (uint32_t)(z ^ (z >> 31)) | 1u;
        uint32_t used[W];
#pragma unroll
        for (int w = 0; w < W; ++w) used[w] = 0;
        bool ok = true;
#pragma unroll
        for (int r = 0; r < KMAX; ++r) {
            if (r < k) {
                const uint32_t sl = cand_slot<B>(c[r], M), bit = 1u << (sl & 31);
                uint32_t u = 0;
#pragma unroll
                for (int w = 0; w < W; ++w) u |= (sl >> 5) == (uint32_t)w ? used[w] : 0u;
                ok &= (u & bit) == 0;
#pragma unroll
                for (int w = 0; w < W; ++w) used[w] |= (sl >> 5) == (uint32_t)w ? bit : 0u;
            }
        }
        if (ok) { mult[i] = M; return; }
    }
    mult[i] = 0;
    atomicExch(fail, 1);
}

// Per iteration, for every candidate edge (i, c_r): tau = tau0 + sum over ants a in
// ant order of ratio_a * [c_r in {prev_a(i), next_a(i)}]  (fp64, bit-identical to
// ColonyPheromone::begin_step, construction.hpp:121-132, restricted to candidate
// edges; ratios per colony.hpp:159-177), w = f32(Power(alpha)(tau)) * eta^beta (f32).
// Classic mode reads tau from the candidate-edge pheromone table T instead.
// Output: packed {c_r, w} rows, the only table the construction kernel reads.
template <int KMAX, bool LIVE, bool HASH>
__global__ void __launch_bounds__(256, KMAX > 16 ? 1 : 2) k_weights(const uint32_t* __restrict__ knn32, const float* __restrict__ eta,
                                                 const uint2* __restrict__ nbr, const int64_t* __restrict__ lb_len,
                                                 const uint8_t* __restrict__ has_lb, const int64_t* __restrict__ g_len,
                                                 const unsigned long long* __restrict__ gkey,
                                                 const double* __restrict__ T, const uint32_t* __restrict__ mult,
                                                 uint32_t n, uint32_t m, int k,
                                                 int kp, double alpha, double tau0, uint2* __restrict__ cand) {
    extern __shared__ double ratio[];  // m ratios | HASH: slot table [2^B][blockDim] u32, acc [KMAX][blockDim] f64
    if (!T) {
        // colony.hpp:159-177 ratios. In async mode (gkey != nullptr) the colony changes under
        // this pass: lengths and g_best are read past L1 (ld.cv), a snapshot at pass start.
        const double g = gkey ? (double)(long long)(__ldcv(gkey) >> 16) : (double)*g_len;
        for (uint32_t a = threadIdx.x; a < m; a += blockDim.x) {
            double r = 0.0;
            if (gkey ? __ldcv(reinterpret_cast<const unsigned char*>(&has_lb[a])) != 0 : has_lb[a] != 0) {
                r = g / (double)(gkey ? __ldcv(reinterpret_cast<const long long*>(&lb_len[a])) : lb_len[a]);
                r = r > 1.0 ? 1.0 : r;
            }
            ratio[a] = r;
        }
        __syncthreads();
    }
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t c[KMAX];
    double acc[KMAX];
#pragma unroll
    for (int r = 0; r < KMAX; ++r) { c[r] = r < k ? knn32[(size_t)i * kNearRow + r] : kNone; acc[r] = 0.0; }
    if (HASH && !T) {
        // The candidate index of a neighbour is one lookup in the city's perfect-hash table
        // (k_cand_hash): slot entries hold (r << 27 | c_r), empty slots kNone, and the
        // per-candidate sums live in shared memory (column t of [KMAX][blockDim]) so the
        // add can address acc[r] with the r found. Every sum still takes its terms in ant
        // order. The comparison loop below was ALU-bound (91% of the ALU pipe, 32 compares
        // per ant and city; profiles/README.md).
        constexpr int B = hash_slot_bits(KMAX);
        const uint32_t t = threadIdx.x, bd = blockDim.x;
        uint32_t* tab = reinterpret_cast<uint32_t*>(ratio + m);
        double* accs = reinterpret_cast<double*>(tab + (1 << B) * bd);
        const uint32_t M = mult[i];
#pragma unroll
        for (int s = 0; s < (1 << B); ++s) tab[s * bd + t] = kNone;
#pragma unroll
        for (int r = 0; r < KMAX; ++r) {
            if (r < k) tab[cand_slot<B>(c[r], M) * bd + t] = ((uint32_t)r << 27) | c[r];
            accs[r * bd + t] = 0.0;
        }
        constexpr uint32_t U = 8;
        auto fetch = [&](uint32_t a0, uint2 (&p)[U], double (&rr)[U]) {
#pragma unroll
            for (uint32_t u = 0; u < U; ++u) {
                const uint32_t a = a0 + u;
                rr[u] = a < m ? ratio[a] : 0.0;
                const uint2* src = &nbr[(size_t)a * n + i];
                p[u] = rr[u] != 0.0 ? (LIVE ? __ldcv(src) : __ldcs(src)) : make_uint2(kNone, kNone);
            }
        };
        uint2 p[U], pn[U];
        double rr[U], rrn[U];
        fetch(0, p, rr);
        for (uint32_t a0 = 0; a0 < m; a0 += U) {
            if (a0 + U < m) fetch(a0 + U, pn, rrn);
#pragma unroll
            for (uint32_t u = 0; u < U; ++u) {
                const uint32_t ex = tab[cand_slot<B>(p[u].x, M) * bd + t], ey = tab[cand_slot<B>(p[u].y, M) * bd + t];
                if ((ex & 0x07ffffffu) == p[u].x) {
                    double* q = accs + (ex >> 27) * bd + t;
                    *q = __dadd_rn(*q, rr[u]);
                }
                if ((ey & 0x07ffffffu) == p[u].y) {
                    double* q = accs + (ey >> 27) * bd + t;
                    *q = __dadd_rn(*q, rr[u]);
                }
            }
#pragma unroll
            for (uint32_t u = 0; u < U; ++u) { p[u] = pn[u]; rr[u] = rrn[u]; }
        }
#pragma unroll
        for (int r = 0; r < KMAX; ++r) acc[r] = accs[r * bd + t];
    } else if (!T) {
        // Pairs of eight ants per batch, accumulated in ant order (the fp64 sum order of
        // ColonyPheromone::begin_step); the next batch's loads are issued before the current
        // batch is accumulated, so eight pairs are always in flight (issuing and then
        // accumulating left the loads idle during the 512 compare/add instructions of a
        // batch: 1.49 -> see profiles/README.md). The slices are streamed once: evict-first
        // in sync mode, read past L1 in async mode (LIVE), where ants rewrite them meanwhile.
        // prev != next for n >= 3 (a tour of distinct cities), so a candidate matches at
        // most one of them and one predicated add per candidate does both tests. Four ants
        // per batch above 16 candidates keep the sums and pairs in registers (no spills).
        constexpr uint32_t U = KMAX > 16 ? 4 : 8;
        auto fetch = [&](uint32_t a0, uint2 (&p)[U], double (&rr)[U]) {
#pragma unroll
            for (uint32_t u = 0; u < U; ++u) {
                const uint32_t a = a0 + u;
                rr[u] = a < m ? ratio[a] : 0.0;
                const uint2* src = &nbr[(size_t)a * n + i];
                p[u] = rr[u] != 0.0 ? (LIVE ? __ldcv(src) : __ldcs(src)) : make_uint2(kNone, kNone);
            }
        };
        uint2 p[U], pn[U];
        double rr[U], rrn[U];
        fetch(0, p, rr);
        for (uint32_t a0 = 0; a0 < m; a0 += U) {
            if (a0 + U < m) fetch(a0 + U, pn, rrn);
#pragma unroll
            for (uint32_t u = 0; u < U; ++u) {
#pragma unroll
                for (int r = 0; r < KMAX; ++r)
                    if ((c[r] == p[u].x) | (c[r] == p[u].y)) acc[r] = __dadd_rn(acc[r], rr[u]);
            }
#pragma unroll
            for (uint32_t u = 0; u < U; ++u) { p[u] = pn[u]; rr[u] = rrn[u]; }
        }
    }
#pragma unroll
    for (int r = 0; r < KMAX; ++r) {
        if (r < k) {
            const double tau = T ? T[(size_t)i * k + r] : __dadd_rn(tau0, acc[r]);
            const float w = __fmul_rn((float)power(alpha, tau), eta[(size_t)i * k + r]);
            cand[(size_t)i * kp + r] = make_uint2(HASH ? knn32[(size_t)i * kNearRow + r] : c[r], __float_as_uint(w));
        }
    }
}

// ============================================================ K2: construction
struct ConstructArgs {
    const uint2* cand;        // n*k {city, f32 weight}
    const uint32_t* order;    // CTA -> ant (k_ant_order), nullptr = identity
    const uint32_t* knn32;    // n*kNearRow nearest cities by (d^2, orig), kNone padded
    const double2* xy;        // internal coordinates
    const uint32_t* orig_of;  // internal -> original (fallback tie-break)
    const uint32_t* int_of;   // original -> internal (start city draw)
    const uint32_t* sb_start;   // first internal id of every Morton superblock
    GridParams g;
    uint32_t* tours;          // m * 2 * n; l_best in half lb_sel[a], new tour in the other
    const uint8_t* lb_sel;
    int64_t* new_len;
    uint8_t* partial_flag;
    unsigned long long* counters; // decisions, fallbacks, ties, forced, full, partial
    const uint32_t* words;    // validation draws: m rows of `stride` words (nullptr = Philox)
    uint64_t stride;
    uint64_t seed, iter;
    uint32_t n, m, k, kp, nwords;  // kp = row stride of cand (k rounded up to even)
    uint32_t sbe_words;            // words of the per-ant "superblock known empty" bitmap (0 = none)
    double eff_pp, mmf;
    int seeding;
    int validate;
    int* err;
    // explicit construct_partial_at (tests): ant = force_ant, params given
    double two_opt_prob;       // maybe_two_opt (two_opt.hpp:71-76), draw slot 3
    uint32_t two_opt_window;
    uint8_t* two_opt_flag;     // non-null: record the draw for k_two_opt instead of searching inline
    int force;
    uint32_t force_ant, force_start_pos, force_m_mod;
    int defer_len;             // synchronous engine: lengths come from k_lengths after this kernel
    uint32_t sb_words;         // words of sb_start staged in shared memory behind the per-ant arrays (0 = read from global)
    unsigned int* qhead;       // non-null: CTAs keep taking the next position of `order` (starts at gridDim.x)
};

// squared lower bound of the distance from q to the square [rx0, rx0+side) x [ry0, ry0+side),
// with the square grown by `slack` on every side (no sqrt: compared against squared bests)
__device__ __forceinline__ double rect_lb2(double2 q, double rx0, double ry0, double side, double slack) {
    const double dx = fmax(0.0, fmax(rx0 - slack - q.x, q.x - (rx0 + side + slack)));
    const double dy = fmax(0.0, fmax(ry0 - slack - q.y, q.y - (ry0 + side + slack)));
    return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
}

struct FbStats {
#ifdef PACO_TIMING
    long long searches = 0, rings = 0, sbs = 0, cities = 0, t_test = 0, t_scan = 0, t_argmin = 0, t_pre = 0;
    long long f0_n = 0, f0_row = 0, f0_probe = 0, f0_redux = 0;  // F0 anatomy: near row, bitmap probes, reduction
#endif
};

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts_u8_if(uint32_t addr, uint32_t v, bool cond) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.shared.u8 [%0], %1;\n\t}" ::"r"(addr), "r"(v),
                 "r"((uint32_t)cond)
                 : "memory");
}
__device__ __forceinline__ void sts_u32_if(uint32_t addr, uint32_t v, bool cond) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.shared.u32 [%0], %1;\n\t}" ::"r"(addr), "r"(v),
                 "r"((uint32_t)cond)
                 : "memory");
}
// predicated 16-byte global->shared async copy (LDGSTS), L1-allocating
__device__ __forceinline__ void cp_async16_if(uint32_t dst, const void* src, bool cond) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q cp.async.ca.shared.global [%0], [%1], 16;\n\t}" ::"r"(dst),
                 "l"(src), "r"((uint32_t)cond));
}
__device__ __forceinline__ void prefetch_l2_if(const void* p, bool cond) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t@q prefetch.global.L2 [%0];\n\t}" ::"l"(p), "r"((uint32_t)cond));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

constexpr uint32_t kFbList = 256;  // per-warp shared-memory list of unvisited city ids (fallback)

// Everything the fallback reads, kept in shared memory so the (rarely executed)
// fallback can be a separate function without an argument struct on the stack.
struct FallbackCtx {
    const uint32_t* knn32;
    const double2* xy;
    const uint32_t* orig_of;
    const uint32_t* sb_start;  // first internal id of every Morton superblock (+ end sentinel)
    GridParams g;
};

__device__ __forceinline__ uint32_t ld_u32(const uint32_t* p) {  // generic address (global or shared)
    uint32_t v;
    asm volatile("ld.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double2 ldg_d2(const double2* p) {
    double2 v;
    asm volatile("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}

// Warp argmin by (d^2, original index). Non-negative doubles order like their bit
// patterns, so the distance minimum is two integer min-reductions (high word, then low
// word among the lanes holding the high minimum). Original indices are fetched only if
// several lanes hold the minimum (o == kNone with j != kNone means "not loaded").
// Leaves (d, j) uniform; o is the winner's original index if it was needed, else kNone.
__device__ __forceinline__ void warp_argmin_redux(double& d, uint32_t& o, uint32_t& j,
                                                  const uint32_t* __restrict__ orig_of, uint32_t lane) {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(d);
    const uint32_t hi = (uint32_t)(bits >> 32), lo = (uint32_t)bits;
    const uint32_t hmin = __reduce_min_sync(kFull, hi);
    const uint32_t lmin = __reduce_min_sync(kFull, hi == hmin ? lo : 0xffffffffu);
    const unsigned holders = __ballot_sync(kFull, j != kNone && hi == hmin && lo == lmin);
    if (holders == 0) return;  // no candidate anywhere (every d is +inf)
    int src;
    if (__popc(holders) == 1) {
        src = __ffs(holders) - 1;
        o = kNone;
    } else {
        uint32_t mine = 0xffffffffu;
        if ((holders >> lane) & 1u) mine = (o == kNone) ? ldg_u32(orig_of + j) : o;
        const uint32_t omin = __reduce_min_sync(kFull, mine);
        src = __ffs(__ballot_sync(kFull, mine == omin)) - 1;
        o = omin;
    }
    j = __shfl_sync(kFull, j, src);
    d = __longlong_as_double((long long)(((unsigned long long)hmin << 32) | lmin));
}

#ifdef PACO_SEG
__device__ __forceinline__ long long seg_clk(uint32_t dep) {
    long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c) : "r"(dep) : "memory");
    return c;
}
#endif

#ifdef PACO_FB_INLINE
#define PACO_FB_ATTR __forceinline__
#else
#define PACO_FB_ATTR __noinline__
#endif

// Exact nearest unvisited city by (d^2, original index), warp-cooperative.
// F0: the 32-nearest list is sorted by the same key, so its first unvisited entry
//     is the answer whenever one exists (one 128-byte row, one ballot).
// F1: rings of 8x8-cell superblocks (each a contiguous id range) around cur with
//     squared rectangle lower bounds. Per ring, each lane tests one superblock (its id
//     range from the compact sb_start table, its free bits from the shared-memory
//     bitmap); the unvisited ids of every surviving superblock are appended to a shared
//     list, and the list is scored once, four coordinate loads per lane in flight - one
//     L2 round trip per ring. A warp argmin closes each ring; its result prunes the
//     superblocks of the next ring (scoring rings 0 and 1 together, unpruned, measured
//     slower).
__device__ __forceinline__ uint32_t lds_u32_if(uint32_t addr, bool cond, uint32_t v) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.shared.u32 %0, [%1];\n\t}" : "+r"(v) : "r"(addr), "r"((uint32_t)cond));
    return v;
}
// any unvisited city in the internal id range [s, e)? (bitmap at shared address vis_s;
// the words are read four at a time, independently)
__device__ __forceinline__ bool range_has_unvisited_s(uint32_t vis_s, uint32_t s, uint32_t e) {
    if (s >= e) return false;
    const uint32_t w0 = s >> 5, w1 = (e - 1) >> 5;
    const uint32_t m0 = 0xffffffffu << (s & 31), m1 = 0xffffffffu >> (31 - ((e - 1) & 31));
    uint32_t any = 0;
    for (uint32_t w = w0; w <= w1; w += 4) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t ww = w + q;
            uint32_t f = ~lds_u32_if(vis_s + 4 * ww, ww <= w1, ~0u);
            if (ww == w0) f &= m0;
            if (ww == w1) f &= m1;
            any |= f;
        }
    }
    return any != 0;
}
// unvisited bits of bitmap word w restricted to the id range [s, e) (0 unless cond)
__device__ __forceinline__ uint32_t free_bits_s(uint32_t vis_s, uint32_t w, uint32_t s, uint32_t e, bool cond) {
    uint32_t fb = ~lds_u32_if(vis_s + 4 * w, cond, ~0u);
    if (w == (s >> 5)) fb &= 0xffffffffu << (s & 31);
    if (w == ((e - 1) >> 5)) fb &= 0xffffffffu >> (31 - ((e - 1) & 31));
    return fb;
}

__device__ PACO_FB_ATTR uint32_t nearest_unvisited(const FallbackCtx& a, uint32_t vis_s, uint32_t cur,
                                                   uint32_t lane, uint32_t list_s, uint32_t sbe_s, bool sbe,
                                                   FbStats& fs) {
    const double2 q = ldg_d2(a.xy + cur);  // issued with the F0 row: F1 needs it first
    {
        // lane l holds entries [E*l, E*l + E) of the sorted near list; the first unvisited
        // entry overall is one integer min-reduction over (entry index, city) keys
        constexpr uint32_t E = kNearRow / 32;
        uint32_t c[E];
#ifdef PACO_TIMING
        const long long f0a = clock64();
#endif
        const uint32_t* row = a.knn32 + (size_t)cur * kNearRow + E * lane;
        if constexpr (E == 1) {
            c[0] = ldg_u32(row);
        } else if constexpr (E == 2) {
            const uint2 v = ldg_u64(reinterpret_cast<const uint2*>(row));
            c[0] = v.x; c[1] = v.y;
        } else if constexpr (E == 4) {
            const uint4 v = ldg_u128(reinterpret_cast<const uint4*>(row));
            c[0] = v.x; c[1] = v.y; c[2] = v.z; c[3] = v.w;
        } else {
            const uint4 v = ldg_u128(reinterpret_cast<const uint4*>(row));
            const uint4 w = ldg_u128(reinterpret_cast<const uint4*>(row) + 1);
            c[0] = v.x; c[1] = v.y; c[2] = v.z; c[3] = v.w;
            c[4] = w.x; c[5] = w.y; c[6] = w.z; c[7] = w.w;
        }
#ifdef PACO_TIMING
        long long f0b; asm volatile("mov.u64 %0, %%clock64;" : "=l"(f0b) : "r"(c[0] ^ c[E - 1]));
#endif
        uint32_t key = kNone;
#pragma unroll
        for (int s = E - 1; s >= 0; --s) {
            const bool ok = c[s] != kNone;
            const uint32_t vw = lds_u32_if(vis_s + ((c[s] >> 5) << 2), ok, ~0u);
            if (ok && !((vw >> (c[s] & 31)) & 1u)) key = ((E * lane + s) << 21) | c[s];
        }
#ifdef PACO_TIMING
        long long f0c; asm volatile("mov.u64 %0, %%clock64;" : "=l"(f0c) : "r"(key));
#endif
        const uint32_t km = __reduce_min_sync(kFull, key);
#ifdef PACO_TIMING
        long long f0d; asm volatile("mov.u64 %0, %%clock64;" : "=l"(f0d) : "r"(km));
        ++fs.f0_n; fs.f0_row += f0b - f0a; fs.f0_probe += f0c - f0b; fs.f0_redux += f0d - f0c;
#endif
        if (km != kNone) return km & 0x1fffffu;
    }
#ifdef PACO_TIMING
    ++fs.searches;
#endif
    const GridParams& g = a.g;
    const double2* __restrict__ xy = a.xy;
    const uint32_t* __restrict__ orig_of = a.orig_of;
    const uint32_t* __restrict__ sb_start = a.sb_start;
    const int32_t cx = cell_coord(q.x, g.x0, g.inv, g.gw), cy = cell_coord(q.y, g.y0, g.inv, g.gh);
    double bd = __longlong_as_double(0x7ff0000000000000LL);
    uint32_t bo = kNone, bj = kNone;  // bo == kNone with bj != kNone: original index not loaded yet
    const double slack = 1e-6 * g.cs;
    const int32_t sx = cx >> 3, sy = cy >> 3;
    const int32_t rmax = g.gws > g.ghs ? g.gws : g.ghs;
    const double span = 8.0 * g.cs;
    const unsigned lt_mask = (1u << lane) - 1u;
    uint32_t n_list = 0;
    // score every listed id against the lane's best, four loads in flight per lane
    auto flush = [&]() {
        __syncwarp();
        for (uint32_t t0 = 0; t0 < n_list; t0 += 128) {
            uint32_t jj[4];
            double2 pp[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t t = t0 + 32 * u + lane;
                jj[u] = lds_u32_if(list_s + 4 * t, t < n_list, kNone);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) pp[u] = jj[u] != kNone ? ldg_d2(xy + jj[u]) : q;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (jj[u] == kNone) continue;
                const double d = dist2(q, pp[u]);
                if (d < bd) { bd = d; bj = jj[u]; bo = kNone; }
                else if (d == bd) {
                    if (bo == kNone && bj != kNone) bo = ldg_u32(orig_of + bj);
                    const uint32_t o = ldg_u32(orig_of + jj[u]);
                    if (o < bo) { bj = jj[u]; bo = o; }
                }
            }
        }
#ifdef PACO_TIMING
        if (lane == 0) fs.cities += n_list;
#endif
        n_list = 0;
        __syncwarp();
    };
    for (int32_t rho = 0; rho <= rmax;) {
        if (rho >= 1) {
            const double lb = (rho - 1) * span - slack;
            if (lb > 0 && lb * lb > bd) break;
        }
#ifdef PACO_TIMING
        ++fs.rings;
#endif
        const double bound = bd;  // warp-uniform (argmin at the end of every pass)
        const int32_t cnt = rho == 0 ? 1 : 8 * rho;
        for (int32_t base = 0; base < cnt; base += 32) {
#ifdef PACO_TIMING
            long long tt0 = clock64();
#endif
            const int32_t c = base + (int32_t)lane;
            bool cand = false;
            uint32_t rs = 0, re = 0;
            if (c < cnt) {
                int32_t x = sx, y = sy;
                if (rho) ring_cell(rho, c, sx, sy, x, y);
                if (x >= 0 && y >= 0 && x < g.gws && y < g.ghs &&
                    (rho == 0 || !(rect_lb2(q, g.x0 + x * span, g.y0 + y * span, span, slack) > bound))) {
                    const uint32_t sbm = morton((uint32_t)x, (uint32_t)y);
                    // a superblock found empty earlier in this construction stays empty (the
                    // visited set only grows): its id range and bitmap words are not read again
                    const bool known_empty = sbe && ((lds_u32(sbe_s + 4 * (sbm >> 5)) >> (sbm & 31)) & 1u);
                    if (!known_empty) {
                        rs = ld_u32(sb_start + sbm);  // generic: global, or the CTA's staged copy
                        re = ld_u32(sb_start + sbm + 1);
                        cand = range_has_unvisited_s(vis_s, rs, re);
                        red_or_shared_if(sbe_s + 4 * (sbm >> 5), 1u << (sbm & 31), sbe && !cand);
                    }
                }
            }
            unsigned ball = __ballot_sync(kFull, cand);
#ifdef PACO_TIMING
            { long long tt1; asm volatile("mov.u64 %0, %%clock64;" : "=l"(tt1) : "r"(ball)); fs.t_test += tt1 - tt0; tt0 = tt1; }
#endif
            while (ball) {
                const int src = __ffs(ball) - 1;
                ball &= ball - 1;
                const uint32_t s = __shfl_sync(kFull, rs, src), e = __shfl_sync(kFull, re, src);
#ifdef PACO_TIMING
                ++fs.sbs;
#endif
                // append the superblock's unvisited ids, 128 ids per step: lane l tests
                // bit l of four broadcast bitmap words
                for (uint32_t j0 = s & ~31u; j0 < e; j0 += 128) {
                    uint32_t fb[4];
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) {
                        const uint32_t w = (j0 >> 5) + q4;
                        fb[q4] = free_bits_s(vis_s, w, s, e, j0 + 32 * q4 < e);
                    }
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) {
                        sts_u32_if(list_s + 4 * (n_list + __popc(fb[q4] & lt_mask)), j0 + 32 * q4 + lane, (fb[q4] >> lane) & 1u);
                        n_list += __popc(fb[q4]);
                    }
                    if (n_list > kFbList - 128) flush();
                }
            }
#ifdef PACO_TIMING
            { long long tt2; asm volatile("mov.u64 %0, %%clock64;" : "=l"(tt2) : "r"(n_list)); fs.t_pre += tt2 - tt0; }
#endif
        }
#ifdef PACO_TIMING
        long long ts0 = clock64();
#endif
        if (n_list) flush();
#ifdef PACO_TIMING
        long long ts1; asm volatile("mov.u64 %0, %%clock64;" : "=l"(ts1) : "l"(__double_as_longlong(bd))); fs.t_scan += ts1 - ts0;
#endif
        warp_argmin_redux(bd, bo, bj, orig_of, lane);
#ifdef PACO_TIMING
        { long long ts2; asm volatile("mov.u64 %0, %%clock64;" : "=l"(ts2) : "r"(bj)); fs.t_argmin += ts2 - ts1; }
#endif
        ++rho;
    }
    return bj;
}

// the single remaining unvisited city (forced final step)
__device__ __forceinline__ uint32_t last_unvisited(const uint32_t* vis, uint32_t nwords, uint32_t lane) {
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
// memory. The dependent chain of one decision is:
//   candidate row of the current city (8 B per lane, one coalesced line at k = 16)
//   -> bitmap byte probe -> warp inclusive scan + total -> one redux.min pick whose key
//   carries the winner's city -> the next row's load.
// Everything else is scheduled around that chain: the visited bit of the new city is
// the winning lane's predicated byte store, ordered for the other lanes by the
// __syncwarp that opens the next decision; Philox draws come 128 at a time (one 4-word
// block per lane) and the next decision's draw is fetched while its row is in flight,
// as is the previous decision's tie test; all lane-divergent bookkeeping is predicated
// PTX. Preserved-segment copy, tour length and the optional permutation check are
// warp-parallel passes around the chain.
//
// KP = row stride (k rounded up to even; 0 = runtime value), STEPS = scan steps
// (ceil(log2 k); extra steps never touch lanes < k), BUF = validation-buffer draws.
// One construction of ant `ant` for iteration `iter` (the draw counter), seeding or not.
// Returns the tour length (every lane); the tour is in the ant's non-l_best half.
// cnt = {decisions, fallbacks, ties, forced, 2-opt runs}.
template <int KP, int STEPS, bool BUF>
__device__ __forceinline__ long long build_one(const ConstructArgs& a, uint32_t ant, uint64_t iter, bool seeding,
                                               unsigned char* smem_raw, const FallbackCtx& fctx, bool& partial_out,
                                               uint32_t (&cnt)[5]) {
    const uint32_t lane = threadIdx.x;
    const uint32_t n = a.n, k = a.k, nw = a.nwords;
    const uint32_t kp = KP ? (uint32_t)KP : a.kp;
    uint32_t* fb_list = reinterpret_cast<uint32_t*>(smem_raw);
    uint32_t* vis = reinterpret_cast<uint32_t*>(smem_raw + kFbList * 4);
    const uint2 key = make_uint2((uint32_t)a.seed, (uint32_t)(a.seed >> 32));
    const uint32_t* wrow = BUF ? a.words + (a.force ? 0 : (uint64_t)ant * a.stride) : nullptr;
    auto word = [&](uint32_t slot) -> uint32_t {
        if (BUF) return wrow[slot];
        const uint4 v = philox10(make_uint4(slot >> 2, ant, (uint32_t)iter, (uint32_t)(iter >> 32)), key);
        return pick_word(v, slot & 3);
    };
#ifdef PACO_PHASES
    const long long ph0 = clock64();
#endif
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
    else if (!seeding) {
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
        warp_copy_segment(out, lb, n, start_pos, preserved, vis, lane);
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

#ifdef PACO_PHASES
    const long long ph1 = clock64();
#endif
    uint32_t n_fb = 0, n_tie = 0;
    // The previous roulette decision's tie test, evaluated while the next row is in flight
    // (between the scan and the next row's load it held seven instructions of the in-order
    // issue stream: C5 construction 52.30 -> 50.98 ms). tie_tol < 0: no pending test.
    float tie_v = 0.0f, tie_t = 0.0f, tie_tol = -1.0f;
    const uint32_t n_dec = n - pos;       // decisions of this construction (the last one forced)
    // shared-window addresses pinned in registers (an opaque move keeps the compiler from
    // re-deriving them from SR_CgaCtaId inside the loop, on the probe's address path)
    uint32_t vis_s, warm_s, fb_s;
    asm volatile("mov.b32 %0, %1;" : "=r"(vis_s) : "r"((uint32_t)__cvta_generic_to_shared(vis)));
    asm volatile("mov.b32 %0, %1;" : "=r"(fb_s) : "r"((uint32_t)__cvta_generic_to_shared(fb_list)));
    asm volatile("mov.b32 %0, %1;" : "=r"(warm_s) : "r"(((vis_s + nw * 4 + 15) & ~15u) + lane * 16));  // L1-warming scratch
    // superblocks known to be empty (F1), after the warming scratch; cleared per construction
    uint32_t sbe_s;
    asm volatile("mov.b32 %0, %1;" : "=r"(sbe_s) : "r"(((vis_s + nw * 4 + 15) & ~15u) + 512));
    for (uint32_t w = lane; w < a.sbe_words; w += 32) sts_u32_if(sbe_s + 4 * w, 0u, true);
    __syncwarp();
    // lanes >= k never load: they hold (cur, 0.0f), and cur is always marked visited
    const bool lane_in = lane < k;
    const uint2* __restrict__ row_base = a.cand + lane;
    const uint32_t iter_lo = (uint32_t)iter, iter_hi = (uint32_t)(iter >> 32);
    FbStats fs;
#ifdef PACO_TIMING
    const long long loop0 = clock64();
    long long fbc = 0;
    long long pb_t = clock64(), pb_fb = 0, pb_s = 0, pb_r = 0;
    uint32_t pb_bucket = 0;
#endif
    // candidate row entry of the current decision
    const uint32_t n_free = n_dec > 0 ? n_dec - 1 : 0;  // roulette / fallback decisions
#ifdef PACO_SEG
    long long sq_tail = 0, sq_probe = 0, sq_scan = 0, sq_pick = 0, sq_n = 0, sq_prev = clock64();
#endif
    uint2 e_pre = ldg_u64_if(row_base + (size_t)cur * kp, lane_in && n_free > 0, make_uint2(cur, 0u));
    // Decisions in batches of 128: each lane holds the Philox block of 4 decisions of the
    // batch (draw slot 4 + t), handed out by shuffle. Inside a batch the only branch is
    // the (warp-uniform, vote-derived) roulette / fallback split.
    for (uint32_t t0 = 0; t0 < n_free; t0 += 128) {
        uint4 pb = make_uint4(0, 0, 0, 0);
        if (!BUF) pb = philox10(make_uint4(1 + (t0 >> 2) + lane, ant, iter_lo, iter_hi), key);
        const uint32_t t1 = t0 + 128 < n_free ? t0 + 128 : n_free;
        // two decisions per loop body give the scheduler room around the back edge
        // (C5: 58.0 -> 56.8 ms; 3 and 4 measured the same as 2)
#pragma unroll 2
        for (uint32_t t = t0; t < t1; ++t) {
            __syncwarp();  // orders the previous decision's visited-bit update for every lane
            const uint2 e = e_pre;  // requested at the end of the previous decision
            n_tie += __ballot_sync(kFull, lane_in && fabsf(__fsub_rn(tie_v, tie_t)) <= tie_tol) ? 1u : 0u;
#ifdef PACO_SEG
            const long long sg0 = seg_clk(e.x);
#endif
            // feasibility from the bitmap
            // the probe reads the bitmap byte holding the candidate's bit: its address is one
            // LEA.HI of the city id (the word address took a shift, a mask and an add on the
            // chain; C5 construction 53.31 -> 52.31 ms)
            const uint32_t vw_addr = vis_s + (e.x >> 3);
            const uint32_t vw = lds_u8(vw_addr);
            const uint32_t uw = BUF ? wrow[4 + t] : __shfl_sync(kFull, pick_word(pb, t & 3), (t & 127) >> 2);
            const uint32_t bit = 1u << (e.x & 7);
            const float w = (vw & bit) ? 0.0f : __uint_as_float(e.y);
#ifdef PACO_SEG
            const long long sg1 = seg_clk(__float_as_uint(w));
#endif
            // Pull every feasible candidate's row into L1 with predicated cp.async.ca (one
            // 16-byte copy per 32-byte sector into a per-lane scratch slot that is never
            // read): the winner's row is then an L1 hit for the next decision.
            // prefetch.global.L1 has no measurable effect on B200 (profiles/README.md).
#ifndef PACO_NO_WARM
            {
                const bool cp = w > 0.0f;
                const unsigned char* src = reinterpret_cast<const unsigned char*>(a.cand + (size_t)e.x * kp);
                if (KP) {
#pragma unroll
                    for (int c = 0; c < (KP * 8 + 31) / 32; ++c) cp_async16_if(warm_s, src + 32 * c, cp);
                } else {
                    for (uint32_t c = 0; c < (kp * 8 + 31) / 32; ++c) cp_async16_if(warm_s, src + 32 * c, cp);
                }
            }
#endif
            // S > 0 exactly when some candidate is feasible (a sum of non-negative f32 is at
            // least its largest term), so the split is decided by a vote the compiler knows
            // to be warp-uniform
            const unsigned feas = __ballot_sync(kFull, w > 0.0f);
            // the highest feasible lane (feasible by construction), while the scan runs
            const bool is_last = lane == 31u - __clz(feas);
            const uint32_t pick_key = (lane << 27) | e.x;
            // Hillis-Steele inclusive scan over the candidate lanes; S = S_{k-1}. (Forming S
            // from the two last-level terms by broadcast, or every lane summing its own prefix
            // from a shared-memory row, measured slower: the chain is sensitive to how the MIO
            // operations interleave, profiles/README.md.)
            float v = w;
#pragma unroll
            for (int st = 0; st < STEPS; ++st) {
                const float y = __shfl_up_sync(kFull, v, 1u << st);
                if (lane >= (1u << st)) v = __fadd_rn(v, y);
            }
            const float S = __shfl_sync(kFull, v, k - 1);
#ifdef PACO_SEG
            const long long sg2 = seg_clk(__float_as_uint(S));
#endif
            uint32_t next;
            if (feas) {
                const float u = u01_f32(uw);
                const float target = __fmul_rn(u, S);
                const float tol = __fmul_rn(1e-6f, S);
                // Only feasible lanes (w > 0; lanes >= k have w = 0) may win: the tree-shaped
                // scan is not monotone in f32, so an infeasible lane's S_r can exceed its left
                // neighbour's by an ulp. The pick is one integer min-reduction over (lane, city)
                // key - lowest winning lane, else highest feasible lane - which delivers the
                // city itself (ids < 2^21: the bitmap fits in shared memory), no ffs, no shuffle.
                // The highest feasible lane comes from the feasibility vote, off the chain, and
                // is folded into the predicate: if no lane wins, it is the only candidate left
                // (one reduction instead of two plus a select; C5 construction 54.40 -> 54.18
                // ms, profiles/README.md).
                const bool win = ((w > 0.0f) & (v > target)) | is_last;
                const uint32_t kw = __reduce_min_sync(kFull, win ? pick_key : kNone);
                tie_v = v; tie_t = target; tie_tol = tol;
                const uint32_t r = kw >> 27;
                next = kw & 0x07ffffffu;
                // the visit of next: the winning lane already holds next's bitmap word (nothing
                // has written the bitmap since it was read), so a predicated plain store does
                // it - no atomic, no branch. No candidate of next is next itself, so the next
                // decision's probe does not depend on it.
                sts_u8_if(vw_addr, vw | bit, lane == r);
#ifdef PACO_SPECSTAT
                {
                    const uint32_t mx = __reduce_max_sync(kFull, lane_in ? e.y : 0u);
                    const int tl = __ffs(__ballot_sync(kFull, lane_in && e.y == mx)) - 1;
                    const uint32_t top = __shfl_sync(kFull, e.x, tl);
                    const uint32_t mx2 = __reduce_max_sync(kFull, (lane_in && lane != (uint32_t)tl) ? e.y : 0u);
                    const int tl2 = __ffs(__ballot_sync(kFull, lane_in && lane != (uint32_t)tl && e.y == mx2)) - 1;
                    const uint32_t top2 = __shfl_sync(kFull, e.x, tl2);
                    const uint32_t mf = __reduce_max_sync(kFull, __float_as_uint(w));
                    const int fl = __ffs(__ballot_sync(kFull, w > 0.0f && __float_as_uint(w) == mf)) - 1;
                    const uint32_t topf = __shfl_sync(kFull, e.x, fl);
                    if (lane == 0) {
                        atomicAdd(&g_timing[4], 1ull);
                        if (next == top) atomicAdd(&g_timing[5], 1ull);
                        if (next == top || next == top2) atomicAdd(&g_timing[6], 1ull);
                        if (next == topf) atomicAdd(&g_timing[7], 1ull);
                        if (!partial) {
                            atomicAdd(&g_timing[8], 1ull);
                            if (next == top) atomicAdd(&g_timing[9], 1ull);
                        }
                    }
                }
#endif
#ifdef PACO_SEG
                const long long sg3 = seg_clk(next);
                sq_tail += sg0 - sq_prev; sq_probe += sg1 - sg0; sq_scan += sg2 - sg1; sq_pick += sg3 - sg2; ++sq_n;
                sq_prev = sg3;
#endif
            } else {
#ifdef PACO_TIMING
                const long long c0 = clock64();
#endif
                next = nearest_unvisited(fctx, vis_s, cur, lane, fb_s, sbe_s, a.sbe_words != 0, fs);
                tie_tol = -1.0f;
                if (lane == 0) vis[next >> 5] |= 1u << (next & 31);
                // fallbacks come in runs: pull the new city's near row from HBM into L2 now,
                // while its candidate row is probed (C5 construction 53.61 -> 53.26 ms; doing
                // it also after decisions with one or two feasible candidates measured slower)
                prefetch_l2_if(a.knn32 + (size_t)next * kNearRow + 32 * lane, lane < kNearRow / 32);  // 128-byte lines
#ifdef PACO_SEG
                sq_prev = seg_clk(next);
#endif
#ifdef PACO_TIMING
                fbc += clock64() - c0;
#endif
                ++n_fb;
            }
#ifdef PACO_TIMING
            if (blockIdx.x == 0 && !partial && lane == 0) {
                const uint32_t bk = (uint32_t)(((uint64_t)pos * 20) / n);
                if (bk != pb_bucket || t + 1 == n_free) {
                    const long long now = clock64();
                    g_prof[pb_bucket] = now - pb_t; g_prof[24 + pb_bucket] = n_fb - pb_fb;
                    g_prof[48 + pb_bucket] = fs.searches - pb_s; g_prof[72 + pb_bucket] = fs.rings - pb_r;
                    pb_t = now; pb_fb = n_fb; pb_s = fs.searches; pb_r = fs.rings; pb_bucket = bk;
                }
            }
#endif
            // head of the next decision's dependent chain, issued before any bookkeeping
            e_pre = ldg_u64_if(row_base + (size_t)next * kp, lane_in, make_uint2(next, 0u));
            stg_u32_if(out + pos, next, lane == 0);
            ++pos;
            cur = next;
        }
    }
    n_tie += __ballot_sync(kFull, lane_in && fabsf(__fsub_rn(tie_v, tie_t)) <= tie_tol) ? 1u : 0u;
    if (n_dec > 0) {  // the single remaining city is appended unscored (construction.hpp:342-348)
        __syncwarp();
        const uint32_t last = last_unvisited(vis, nw, lane);
        if (lane == 0) out[pos] = last;
        ++pos;
    }
    const uint32_t n_forced = n_dec > 0 ? 1u : 0u;
#ifdef PACO_SEG
    if (lane == 0 && sq_n > 1) {
        atomicAdd(&g_timing[4], (unsigned long long)sq_tail); atomicAdd(&g_timing[5], (unsigned long long)sq_probe);
        atomicAdd(&g_timing[6], (unsigned long long)sq_scan); atomicAdd(&g_timing[7], (unsigned long long)sq_pick);
        atomicAdd(&g_timing[8], (unsigned long long)sq_n);
    }
#endif
    cp_async_wait_all();
    __syncwarp();
#ifdef PACO_TIMING
    if (lane == 0) {
        atomicAdd(&g_timing[0], (unsigned long long)(clock64() - loop0));
        atomicAdd(&g_timing[4], (unsigned long long)fs.f0_n); atomicAdd(&g_timing[5], (unsigned long long)fs.f0_row);
        atomicAdd(&g_timing[6], (unsigned long long)fs.f0_probe); atomicAdd(&g_timing[7], (unsigned long long)fs.f0_redux);
        atomicAdd(&g_timing[1], (unsigned long long)fbc);
        atomicAdd(&g_timing[2], (unsigned long long)n_dec);
    }
    {
        long long c = fs.cities;
        for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
        if (lane == 0) {
            atomicAdd(&g_timing[9], (unsigned long long)fs.searches); atomicAdd(&g_timing[10], (unsigned long long)fs.rings);
            atomicAdd(&g_timing[11], (unsigned long long)fs.sbs); atomicAdd(&g_timing[12], (unsigned long long)c);
            atomicAdd(&g_timing[13], (unsigned long long)fs.t_test); atomicAdd(&g_timing[14], (unsigned long long)fs.t_scan);
            atomicAdd(&g_timing[15], (unsigned long long)fs.t_argmin); atomicAdd(&g_timing[3], (unsigned long long)fs.t_pre);
        }
    }
#endif
#ifdef PACO_PHASES
    const long long ph2 = clock64();
#endif
    // maybe_two_opt (two_opt.hpp:71-76): draw slot 3. The synchronous engine defers the
    // search to k_two_opt (a whole CTA per tour, after this kernel; the length computed
    // below is then corrected by the search's delta); the asynchronous one runs it here.
    uint32_t n_2opt = 0;
    if (!a.force && a.two_opt_prob > 0.0 && u01_f64(word(3)) < a.two_opt_prob) {
        if (a.two_opt_flag) {
            if (lane == 0) a.two_opt_flag[ant] = 1;
        } else {
            two_opt_exact<false>(out, n, a.two_opt_window, a.xy, nullptr, nullptr, nullptr, nullptr);
        }
        n_2opt = 1;
    }
    // tour length (instance.hpp:120-127), int64, warp-parallel over positions
    // The synchronous engine sums the lengths of all m tours in one grid-wide kernel after
    // this one (k_lengths): one warp's pass over a C5 tour is a chain of ~780 dependent L2
    // round-trip pairs at the tail of the longest ant, on the iteration's critical path.
    const long long len = a.defer_len ? 0 : warp_tour_length(out, n, a.xy, lane);
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
#ifdef PACO_PHASES
    if (lane == 0) {
        const long long ph3 = clock64();
        const int o = partial ? 5 : 0;
        atomicAdd(&g_timing[o + 0], (unsigned long long)(ph1 - ph0));
        atomicAdd(&g_timing[o + 1], (unsigned long long)(ph2 - ph1));
        atomicAdd(&g_timing[o + 2], (unsigned long long)(ph3 - ph2));
        atomicAdd(&g_timing[o + 3], (unsigned long long)n_dec);
        atomicAdd(&g_timing[o + 4], 1ull);
    }
#endif
    partial_out = partial;
    cnt[0] = n_dec; cnt[1] = n_fb; cnt[2] = n_tie; cnt[3] = n_forced; cnt[4] = n_2opt;
    return len;
}

__device__ __forceinline__ void init_fallback_ctx(const ConstructArgs& a, FallbackCtx& fctx) {
    if (threadIdx.x == 0) {
        fctx.knn32 = a.knn32; fctx.xy = a.xy; fctx.orig_of = a.orig_of; fctx.sb_start = a.sb_start; fctx.g = a.g;
    }
    __syncwarp();
}

// Synchronous construction: every ant once against the frozen colony (engine.hpp:245-306);
// the completion step (k_update, k_publish) runs after it in ant order.
template <int KP, int STEPS, bool BUF>
__global__ void __launch_bounds__(32, 1) k_construct(ConstructArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];  // fallback list | visited bitmap | warm scratch
    __shared__ FallbackCtx fctx;
    init_fallback_ctx(a, fctx);
    if (a.sb_words) {
        // The superblock-start table (6.4 KB at C5) staged behind the per-ant arrays when the
        // launch leaves the shared memory for it (persistent CTAs, five per SM): a ring search
        // reads two entries per superblock it tests, an L2 round trip each from global memory
        // (C5 construction 46.79 -> 46.63 ms).
        uint32_t* sb = reinterpret_cast<uint32_t*>(smem_raw + kFbList * 4 + ((a.nwords * 4 + 15) & ~15u) + 512 + a.sbe_words * 4);
        for (uint32_t i = threadIdx.x; i < a.sb_words; i += 32) sb[i] = a.sb_start[i];
        if (threadIdx.x == 0) fctx.sb_start = sb;
        __syncwarp();
    }
    uint32_t slot = blockIdx.x;
    // one ant per CTA, or (qhead) the next position of the launch order until none is left
    for (;;) {
        const uint32_t ant = a.force ? a.force_ant : (a.order ? a.order[slot] : slot);
        bool partial;
        uint32_t cnt[5];
#ifdef PACO_ANTPROF
        const unsigned long long pt0 = gtimer();
#endif
        const long long len = build_one<KP, STEPS, BUF>(a, ant, a.iter, a.seeding != 0, smem_raw, fctx, partial, cnt);
#ifdef PACO_ANTPROF
        if (threadIdx.x == 0 && ant < 4096) {
            uint32_t smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            unsigned long long* g = g_ant + 6 * ant;
            uint32_t wid;
            asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
            g[0] = pt0; g[1] = gtimer(); g[2] = smid | (wid << 16); g[3] = cnt[0]; g[4] = cnt[1]; g[5] = partial;
        }
#endif
        if (threadIdx.x == 0) {
            a.new_len[ant] = len;
            if (!a.force) {
                a.partial_flag[ant] = partial ? 1 : 0;
                atomicAdd(&a.counters[0], (unsigned long long)cnt[0]);
                atomicAdd(&a.counters[1], (unsigned long long)cnt[1]);
                atomicAdd(&a.counters[2], (unsigned long long)cnt[2]);
                atomicAdd(&a.counters[3], (unsigned long long)cnt[3]);
                atomicAdd(&a.counters[partial ? 5 : 4], 1ull);
                if (cnt[4]) atomicAdd(&a.counters[9], 1ull);
            }
        }
        if (!a.qhead) break;
        uint32_t nxt = 0;
        if (threadIdx.x == 0) nxt = atomicAdd(a.qhead, 1u);
        nxt = __shfl_sync(kFull, nxt, 0);
        if (nxt >= a.m) break;
        slot = nxt;
        __syncwarp();
    }
}

// Colony state the asynchronous mode updates from inside the construction kernel.
struct AsyncState {
    uint2* nbr;                   // m*n published (prev, next) of every l_best
    int64_t* lb_len;
    uint8_t* has_lb;
    uint8_t* lb_sel;
    unsigned long long* gkey;     // g_best as (length << 16 | ant), atomicMin
    uint8_t* improved;            // of the ant's latest construction (readback)
};

// Asynchronous mode (engine.hpp:213-244, the reference's default): each ant's warp runs
// `count` constructions back to back with no barrier and applies its own update
// immediately - update_l_best (strict improvement, colony.hpp:117-124) with the
// publish of its neighbour slice (colony.hpp:39-52), then update_g_best
// (colony.hpp:127-139) as an atomic minimum. The candidate weights are rebuilt by
// k_weights passes running concurrently on another stream, so constructions see other
// ants' improvements with a delay, as the reference's workers see them whenever they
// next gather. Not deterministic (the reference's async mode is not either).
template <int KP, int STEPS>
__global__ void __launch_bounds__(32, 1) k_construct_async(ConstructArgs a, uint32_t count, AsyncState st) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ FallbackCtx fctx;
    init_fallback_ctx(a, fctx);
    const uint32_t lane = threadIdx.x, ant = blockIdx.x, n = a.n;
    unsigned long long tot[5] = {0, 0, 0, 0, 0}, fulls = 0, parts = 0, imps = 0;
    for (uint32_t it = 0; it < count; ++it) {
        bool partial;
        uint32_t cnt[5];
        // gpu-scope fence per construction: the SM's L1 drops lines cached before it, so the
        // rows this construction reads (k_weights rewrites them from other SMs) are at most
        // one construction older than the latest pass, whatever the L1 hit rate
        __threadfence();
        const long long len = build_one<KP, STEPS, false>(a, ant, a.iter + it, a.seeding != 0 && it == 0, smem_raw,
                                                          fctx, partial, cnt);
#pragma unroll
        for (int q = 0; q < 5; ++q) tot[q] += cnt[q];
        if (partial) ++parts; else ++fulls;
        const bool imp = !st.has_lb[ant] || len < st.lb_len[ant];
        if (lane == 0) {
            a.new_len[ant] = len;
            a.partial_flag[ant] = partial ? 1 : 0;
            st.improved[ant] = imp ? 1 : 0;
        }
        if (imp) {
            const uint8_t ns = (uint8_t)(1 - st.lb_sel[ant]);
            const uint32_t* t = a.tours + ((size_t)ant * 2 + ns) * n;
            uint2* nb = st.nbr + (size_t)ant * n;
            // Ant::publish (colony.hpp:39-52): eight positions per lane per pass, all loads
            // issued before the scattered stores
            constexpr int U = 8;
            for (uint32_t b = 0; b < n; b += 32 * U) {
                uint32_t c[U], pv[U], nx[U];
#pragma unroll
                for (int j = 0; j < U; ++j) {
                    const uint32_t p = b + 32 * j + lane;
                    const bool in = p < n;
                    c[j] = in ? t[p] : 0u;
                    pv[j] = in ? t[p == 0 ? n - 1 : p - 1] : 0u;
                    nx[j] = in ? t[p + 1 == n ? 0 : p + 1] : 0u;
                }
#pragma unroll
                for (int j = 0; j < U; ++j)
                    if (b + 32 * j + lane < n) nb[c[j]] = make_uint2(pv[j], nx[j]);
            }
            __syncwarp();
            if (lane == 0) {
                __threadfence();  // the slice before the length that makes it count
                st.lb_sel[ant] = ns;
                st.has_lb[ant] = 1;
                *(volatile int64_t*)&st.lb_len[ant] = len;
                __threadfence();
                // update_g_best (colony.hpp:127-139): CAS loop with strict '<', so an equal
                // length never displaces the incumbent
                const unsigned long long mine = ((unsigned long long)len << 16) | ant;
                unsigned long long cur = *(volatile unsigned long long*)st.gkey;
                while (cur == ~0ull || (mine >> 16) < (cur >> 16)) {
                    const unsigned long long seen = atomicCAS(st.gkey, cur, mine);
                    if (seen == cur) break;
                    cur = seen;
                }
            }
            ++imps;
            __syncwarp();
        }
    }
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) atomicAdd(&a.counters[q], tot[q]);
        atomicAdd(&a.counters[9], tot[4]);
        atomicAdd(&a.counters[4], fulls);
        atomicAdd(&a.counters[5], parts);
        atomicAdd(&a.counters[7], imps);
    }
}

// g_best between the two encodings: the sync path's GBest, the async path's atomic key
struct GBest { long long len; int32_t ant; int32_t has; };
__global__ void k_gkey_from_gbest(const GBest* __restrict__ gb, unsigned long long* __restrict__ gkey) {
    *gkey = gb->has ? (((unsigned long long)gb->len << 16) | (uint32_t)gb->ant) : ~0ull;
}
__global__ void k_gbest_from_gkey(const unsigned long long* __restrict__ gkey, GBest* __restrict__ gb,
                                  int64_t* __restrict__ g_len) {
    const unsigned long long k = *gkey;
    if (k == ~0ull) return;
    gb->len = (long long)(k >> 16); gb->ant = (int32_t)(k & 0xffffu); gb->has = 1;
    *g_len = (int64_t)(k >> 16);
}

// ============================================================ K4: completion step
// engine.hpp:261-265: for every ant in order, update_l_best (strict improvement,
// colony.hpp:117-124) then update_g_best (colony.hpp:127-139). The l_best switch is
// a flip of the ant's double-buffer selector, so no tour is copied.

// The ants' l_best updates are independent; the g_best update sequence in ant order with
// strict improvement ends at the lexicographic minimum (length, ant) of the improved ants
// when that beats the incumbent, so it is one block-wide argmin. One CTA.
__global__ void __launch_bounds__(1024) k_update(uint32_t first, uint32_t count, const int64_t* __restrict__ new_len,
                                                 int64_t* __restrict__ lb_len, uint8_t* __restrict__ has_lb,
                                                 uint8_t* __restrict__ lb_sel, uint8_t* __restrict__ improved,
                                                 GBest* __restrict__ gb, int64_t* __restrict__ g_len,
                                                 unsigned long long* __restrict__ counters) {
    __shared__ long long s_len[32];
    __shared__ int32_t s_ant[32];
    __shared__ unsigned s_imp[32];
    long long bl = 0x7fffffffffffffffLL;
    int32_t ba = -1;
    unsigned imp = 0;
    for (uint32_t a = first + threadIdx.x; a < first + count; a += blockDim.x) {
        const int64_t L = new_len[a];
        if (!has_lb[a] || L < lb_len[a]) {
            has_lb[a] = 1; lb_len[a] = L; lb_sel[a] ^= 1; improved[a] = 1; ++imp;
            if (L < bl) { bl = L; ba = (int32_t)a; }  // ants visited in increasing order per thread
        } else {
            improved[a] = 0;
        }
    }
    auto better = [](long long l1, int32_t a1, long long l2, int32_t a2) {
        return a1 >= 0 && (a2 < 0 || l1 < l2 || (l1 == l2 && a1 < a2));
    };
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const long long l2 = __shfl_xor_sync(kFull, bl, off);
        const int32_t a2 = __shfl_xor_sync(kFull, ba, off);
        imp += __shfl_xor_sync(kFull, imp, off);
        if (better(l2, a2, bl, ba)) { bl = l2; ba = a2; }
    }
    const uint32_t w = threadIdx.x >> 5, nwarps = (blockDim.x + 31) >> 5;
    if ((threadIdx.x & 31) == 0) { s_len[w] = bl; s_ant[w] = ba; s_imp[w] = imp; }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long tot = 0;
        for (uint32_t q = 0; q < nwarps; ++q) {
            tot += s_imp[q];
            if (better(s_len[q], s_ant[q], bl, ba)) { bl = s_len[q]; ba = s_ant[q]; }
        }
        GBest g = *gb;
        if (ba >= 0 && (!g.has || bl < g.len)) { g.len = bl; g.ant = ba; g.has = 1; }
        *gb = g;
        *g_len = g.has ? g.len : 0x7fffffffffffffffLL;
        counters[7] += tot;
    }
}

// Ant::publish (colony.hpp:39-52) for the improved ants: neighbour pairs of the new
// l_best, nbr[a][city] = (prev, next). Grid (ceil(n/256), count) covers ants first..
__global__ void k_publish(const uint32_t* __restrict__ tours, const uint8_t* __restrict__ lb_sel,
                          const uint8_t* __restrict__ improved, uint32_t n, int current,
                          uint2* __restrict__ nbr, uint32_t first = 0) {
    const uint32_t a = first + blockIdx.y;
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
__global__ void __launch_bounds__(256) k_classic(const uint32_t* __restrict__ knn32, const uint2* __restrict__ cur_nbr,
                                                 const int64_t* __restrict__ new_len, uint32_t n, uint32_t m, int k,
                                                 double rho, double* __restrict__ T) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t c[KMAX];
    double t[KMAX];
    const double keep = 1.0 - rho;
#pragma unroll
    for (int r = 0; r < KMAX; ++r) {
        c[r] = r < k ? knn32[(size_t)i * kNearRow + r] : kNone;
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

// Readback of one tour per ant in original ids: l_best (lbest = 1), or the tour built by
// the last iteration - the half that is not l_best unless it improved, in which case the
// selector already flipped onto it. Grid (ceil(n/256), count) over ants first.. ; out is
// count x n.
__global__ void k_gather_tours(const uint32_t* __restrict__ tours, const uint8_t* __restrict__ lb_sel,
                               const uint8_t* __restrict__ improved, const uint32_t* __restrict__ orig_of,
                               uint32_t n, uint32_t first, int lbest, uint32_t* __restrict__ out) {
    const uint32_t a = first + blockIdx.y;
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const uint8_t sel = lb_sel[a];
    const uint8_t half = (lbest || improved[a]) ? sel : (uint8_t)(1 - sel);
    out[(size_t)blockIdx.y * n + p] = orig_of[tours[((size_t)a * 2 + half) * n + p]];
}

// maybe_two_opt's search for the synchronous engine (two_opt.hpp:28-67): one CTA per
// flagged tour (the new tour in the ant's non-l_best half, before k_update), the CTA-wide
// exact first-improvement search of two_opt_exact, the length corrected by its delta.
// CTAs loop over the ants; `edges` holds one n-entry edge cache per CTA.
__global__ void __launch_bounds__(512, 1) k_two_opt(uint32_t* __restrict__ tours, const uint8_t* __restrict__ lb_sel,
                                                  uint8_t* __restrict__ flag, int64_t* __restrict__ new_len,
                                                  uint32_t n, uint32_t m, uint32_t window,
                                                  const double2* __restrict__ xy, int32_t* __restrict__ edges,
                                                  double2* __restrict__ txy, unsigned long long* __restrict__ moves) {
    __shared__ unsigned long long s_key[33];
    int32_t* e = edges + (size_t)blockIdx.x * n;
    double2* tx = txy + (size_t)blockIdx.x * n;
    for (uint32_t a = blockIdx.x; a < m; a += gridDim.x) {
        if (!flag[a]) continue;  // CTA-uniform
        uint32_t* o = tours + ((size_t)a * 2 + (1 - lb_sel[a])) * n;
        uint32_t mv = 0;
        const long long d = two_opt_block(o, n, window, xy, e, tx, s_key, &mv);
        __syncthreads();
        if (threadIdx.x == 0) { new_len[a] += d; flag[a] = 0; atomicAdd(moves, (unsigned long long)mv); }
        __syncthreads();
    }
}

// maybe_two_opt's searches when few tours are flagged (the paper's p = 0.001: about one
// search per iteration): one thread-block cluster of CS CTAs per flagged tour
// (two_opt_cluster), clusters striding over the ants. Same moves as k_two_opt.
__global__ void __launch_bounds__(512, 1) k_two_opt_cluster(uint32_t* __restrict__ tours, const uint8_t* __restrict__ lb_sel,
                                                          uint8_t* __restrict__ flag, int64_t* __restrict__ new_len,
                                                          uint32_t n, uint32_t m, uint32_t window,
                                                          const double2* __restrict__ xy, int32_t* __restrict__ edges,
                                                          double2* __restrict__ txy, unsigned long long* __restrict__ moves,
                                                          uint32_t stage_cap) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    __shared__ TwoOptShared sh;
    extern __shared__ __align__(16) unsigned char stage_raw[];  // stage_cap double2 | int32 | u32
    double2* s_txy = reinterpret_cast<double2*>(stage_raw);
    int32_t* s_edge = reinterpret_cast<int32_t*>(stage_raw + (size_t)stage_cap * sizeof(double2));
    uint32_t* s_o = reinterpret_cast<uint32_t*>(s_edge + stage_cap);
    const uint32_t CS = cl.num_blocks();
    const uint32_t cid = blockIdx.x / CS, ncl = gridDim.x / CS;
    int32_t* e = edges + (size_t)cid * n;
    double2* tx = txy + (size_t)cid * n;
    for (uint32_t a = cid; a < m; a += ncl) {
        if (!flag[a]) continue;  // cluster-uniform
        uint32_t* o = tours + ((size_t)a * 2 + (1 - lb_sel[a])) * n;
        uint32_t mv = 0;
        const long long d = two_opt_cluster(cl, o, n, window, xy, e, tx, sh, s_txy, s_edge, s_o, stage_cap, &mv);
        if (cl.block_rank() == 0 && threadIdx.x == 0) {  // every CTA read flag[a] before the search
            new_len[a] += d;
            flag[a] = 0;
            atomicAdd(moves, (unsigned long long)mv);
        }
        cl.sync();  // the caches are reused for the cluster's next tour
    }
}

// Launch order of the synchronous construction (K2): every ant's decision count this
// iteration follows from its draws alone (coin, start_pos, m_mod: slots 0-2), so the ants
// are sorted by it, longest first. CTAs are handed out in index order, so the longest
// ants land on distinct SMs and share them with ever shorter ones, which finish early:
// the critical ant runs most of its construction with fewer co-resident warps. Results do
// not depend on the order. One CTA of 1024 threads, bitonic sort of (decisions, ant)
// keys over the next power of two >= m (m <= 4096; larger colonies keep the identity).
__global__ void __launch_bounds__(1024) k_ant_order(const uint32_t* __restrict__ words, uint64_t stride,
                                                    uint64_t seed, uint64_t iter, uint32_t n, uint32_t m,
                                                    double eff_pp, double mmf, int seeding, uint32_t* __restrict__ order,
                                                    unsigned int* qhead, unsigned int qstart) {
    __shared__ unsigned long long key[4096];
    if (qhead && threadIdx.x == 0) *qhead = qstart;
    uint32_t P = 1;
    while (P < m) P <<= 1;
    const uint2 k2 = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    for (uint32_t a = threadIdx.x; a < P; a += blockDim.x) {
        unsigned long long kk = 0ull;  // padding sorts last
        if (a < m) {
            uint32_t w0, w2;
            if (words) { w0 = words[(size_t)a * stride]; w2 = words[(size_t)a * stride + 2]; }
            else {
                const uint4 v = philox10(make_uint4(0u, a, (uint32_t)iter, (uint32_t)(iter >> 32)), k2);
                w0 = v.x; w2 = v.z;
            }
            uint32_t dec = n - 1;
            if (!seeding && u01_f64(w0) < eff_pp) {  // partial: m_mod decisions (construction.hpp:354-362)
                double capd = floor(mmf * (double)n);
                if (capd < 2.0) capd = 2.0;
                dec = 2 + below(w2, (uint32_t)capd - 1);
            }
            kk = ((unsigned long long)dec << 32) | (0xffffffffu - a);  // longest first, then lower ant
        }
        key[a] = kk;
    }
    __syncthreads();
    for (uint32_t k = 2; k <= P; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
                const uint32_t l = i ^ j;
                if (l > i) {
                    const bool desc = (i & k) == 0;
                    const unsigned long long x = key[i], y = key[l];
                    if (desc ? x < y : x > y) { key[i] = y; key[l] = x; }
                }
            }
            __syncthreads();
        }
    }
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) order[i] = 0xffffffffu - (uint32_t)key[i];
}

// reference-order tour -> internal ids (host offers), and internal -> original on readback
__global__ void k_map(const uint32_t* __restrict__ in, const uint32_t* __restrict__ table, size_t count,
                      uint32_t* __restrict__ out) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) out[i] = table[in[i]];
}

// Tour lengths (instance.hpp:120-127) of the m tours a synchronous k_construct launch wrote
// (half 1 - lb_sel[a] of each ant's pair), exact int64 sums of EUC_2D distances added to
// new_len[a] (k_construct left 0 there): kLenPos positions per 256-thread CTA, all loads of
// a thread issued before its first distance. Integer sums, so the order of the atomic adds
// does not matter.
constexpr uint32_t kLenU = 8, kLenPos = 256 * kLenU;
__global__ void __launch_bounds__(256) k_lengths(const uint32_t* __restrict__ tours, const uint8_t* __restrict__ lb_sel,
                                                 const double2* __restrict__ xy, uint32_t n, int64_t* __restrict__ new_len) {
    const uint32_t ant = blockIdx.y;
    const uint32_t* __restrict__ out = tours + ((size_t)ant * 2 + (1 - lb_sel[ant])) * n;
    // kLenU consecutive positions per thread: position p's second city is position p + 1's
    // first, so a thread gathers kLenU + 1 coordinates for kLenU distances
    const uint32_t p0 = (blockIdx.x * 256 + threadIdx.x) * kLenU;
    uint32_t c[kLenU + 1];
    if ((n & 3u) == 0 && p0 + kLenU <= n) {  // 16-byte aligned rows: two vector loads
        const uint4 v0 = *reinterpret_cast<const uint4*>(out + p0), v1 = *reinterpret_cast<const uint4*>(out + p0 + 4);
        c[0] = v0.x; c[1] = v0.y; c[2] = v0.z; c[3] = v0.w; c[4] = v1.x; c[5] = v1.y; c[6] = v1.z; c[7] = v1.w;
        c[kLenU] = out[p0 + kLenU < n ? p0 + kLenU : 0];
    } else {
#pragma unroll
        for (uint32_t j = 0; j <= kLenU; ++j) {
            const uint32_t p = p0 + j;
            c[j] = p < n ? out[p] : (p == n ? out[0] : 0u);
        }
    }
    double2 x[kLenU + 1];
#pragma unroll
    for (uint32_t j = 0; j <= kLenU; ++j) x[j] = xy[c[j]];
    double d2[kLenU];
    bool ok = true;
#pragma unroll
    for (uint32_t j = 0; j < kLenU; ++j) {
        d2[j] = p0 + j < n ? sq_dist(x[j], x[j + 1]) : 0.0;
        ok &= sqrt_fast_ok(d2[j]);
    }
    long long len = 0;
    if (__all_sync(kFull, ok)) {
#pragma unroll
        for (uint32_t j = 0; j < kLenU; ++j) len += (int32_t)__dadd_rn(sqrt_rn_fast(d2[j]), 0.5);
    } else {
#pragma unroll
        for (uint32_t j = 0; j < kLenU; ++j) len += (int32_t)__dadd_rn(__dsqrt_rn(d2[j]), 0.5);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) len += __shfl_xor_sync(kFull, len, off);
    __shared__ long long part[8];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = len;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) t += part[w];
        atomicAdd(reinterpret_cast<unsigned long long*>(new_len + ant), (unsigned long long)t);
    }
}

__global__ void k_tour_length(const uint32_t* __restrict__ t, const double2* __restrict__ xy, uint32_t n,
                              unsigned long long* __restrict__ out) {
    long long len = 0;
    for (uint32_t p = threadIdx.x; p < n; p += blockDim.x)
        len += euc2d(xy[t[p]], xy[t[p + 1 < n ? p + 1 : 0]]);
    atomicAdd(out, (unsigned long long)len);
}

} // namespace pacob200
