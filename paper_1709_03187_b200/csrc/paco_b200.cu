// Host side of the B200 tour-construction engine and its C ABI (include/paco_b200.h).
// One handle = one instance + one colony resident in HBM + one CUDA stream (two in
// asynchronous mode). A synchronous iteration is these launches on that stream
// (DESIGN.md §4):
//   K5 k_weights  -> K2 k_construct -> [K6 classic deposit] -> K4 k_update -> k_publish
// which together replace one barrier-synchronous iteration of paco::run
// (/root/reference/proj/include/paco/engine.hpp:245-306). Asynchronous calls
// (engine.hpp:213-244) are one k_construct_async launch with k_weights passes running
// beside it on the second stream.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/paco_b200.h"
#include "kernels.cuh"
#include "kernels_ir.cuh"

using namespace pacob200;

namespace {

thread_local std::string g_last_error;

paco_status fail(paco_status s, const std::string& msg) {
    g_last_error = msg;
    return s;
}

#define CU(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(PACO_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));     \
    } while (0)

// Device memory comes from the engine's own stream-ordered pool, one per device and
// process (cudaMallocFromPoolAsync on the legacy stream, then a synchronize so every
// stream may use it), and returns to it on free: the pool keeps it (release threshold at
// the maximum) for the next handle instead of handing it back to the driver. The device's
// default pool, which other cudaMallocAsync users share, is left alone. Measured on a
// fresh process after another engine process: create + destroy of a C4 handle took
// 114-127 ms + 336-591 ms through cudaMalloc/cudaFree, 11-21 ms + 3-5 ms when warm
// (profiles/README.md). paco_release_cached_memory() trims the pool.
constexpr int kMaxDevices = 64;
cudaMemPool_t g_pool[kMaxDevices] = {};
std::mutex g_pool_mu;

cudaError_t engine_pool(int dev, cudaMemPool_t* out) {
    if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (!g_pool[dev]) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaError_t e = cudaMemPoolCreate(&g_pool[dev], &props);
        if (e != cudaSuccess) { g_pool[dev] = nullptr; return e; }
        uint64_t threshold = UINT64_MAX;
        cudaMemPoolSetAttribute(g_pool[dev], cudaMemPoolAttrReleaseThreshold, &threshold);
    }
    *out = g_pool[dev];
    return cudaSuccess;
}

template <class T>
cudaError_t dalloc(T** p, size_t count) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    cudaMemPool_t pool = nullptr;
    if (e == cudaSuccess) e = engine_pool(dev, &pool);
    if (e == cudaSuccess)
        e = cudaMallocFromPoolAsync(reinterpret_cast<void**>(p), sizeof(T) * (count ? count : 1), pool, 0);
    return e != cudaSuccess ? e : cudaStreamSynchronize(0);
}
// callers make sure no stream still uses p
inline void dfree(void* p) {
    if (p) cudaFreeAsync(p, 0);
}

int kmax_for(uint32_t k) { return k <= 8 ? 8 : k <= 16 ? 16 : k <= 24 ? 24 : 32; }

} // namespace

struct paco_handle {
    int dev = 0;
    int num_sms = 148;
    cudaStream_t st = nullptr;
    paco_config cfg{};
    int mode = 0;
    uint32_t n = 0, m = 0, k = 0, kp = 0, nwords = 0;
    GridParams g{};
    std::vector<double> hx, hy;
    std::vector<uint32_t> h_orig, h_int;
    // device
    double2* xy = nullptr;
    uint32_t *orig_of = nullptr, *int_of = nullptr, *cell_start = nullptr, *sb_start = nullptr;
    uint32_t* knn = nullptr;
    // synchronous 2-opt (k_two_opt): per-ant request flags and one edge cache per CTA
    uint8_t* two_opt_flag = nullptr;
    int32_t* two_opt_edges = nullptr;
    double2* two_opt_txy = nullptr;
    uint32_t two_opt_ctas = 0;
    uint32_t two_opt_cs = 0, two_opt_clusters = 0;  // k_two_opt_cluster: cluster size, clusters (0 = unavailable)
    uint32_t two_opt_stage = 0;                      // positions staged in shared memory per round (0 = none)
    bool two_opt_use_cluster = false;
    float* eta = nullptr;
    uint2* cand = nullptr;
    uint32_t* order = nullptr;  // CTA -> ant launch order of K2 (k_ant_order), m <= 4096
    unsigned int* qhead = nullptr;  // next position of `order` to hand out (persistent K2 CTAs)
    uint32_t* tours = nullptr;
    uint8_t *lb_sel = nullptr, *has_lb = nullptr, *improved = nullptr, *partial = nullptr;
    int64_t *new_len = nullptr, *lb_len = nullptr, *g_len = nullptr;
    uint2* nbr = nullptr;
    uint32_t* cand_mult = nullptr;       // per-city candidate perfect-hash multipliers (k <= 16)
    uint2* cur_nbr = nullptr;
    double* T = nullptr;
    GBest* gb = nullptr;
    unsigned long long* gkey = nullptr;  // async mode: g_best as (length << 16 | ant)
    cudaStream_t st2 = nullptr;          // async mode: concurrent weight rebuilds
    bool async_mode = false;
    unsigned long long* counters = nullptr;
    int* err = nullptr;
    uint32_t* words = nullptr;
    uint64_t words_stride = 0, words_cap = 0;
    bool words_ready = false;
    uint32_t* scratch_u32 = nullptr;  // n-sized staging for offers / construct_at
    unsigned long long* scratch_u64 = nullptr;
    uint64_t iter = 0, weight_passes = 0;
    double construct_ms = 0, update_ms = 0, setup_ms = 0;
    std::vector<cudaEvent_t> evpool;
    // reference-rule (IR) mode
    bool ir = false;
    uint64_t* rng = nullptr;   // m*4 xoshiro256++ states
    double* ratio = nullptr;   // m
    uint32_t* tl_city = nullptr;   // reference rule, P-ACO: n rows of 2m + 1 (count, touched cities; k_ir_touched)
    double* tl_tau = nullptr;      // n*2m their tau^alpha
    IrJump* ir_jump = nullptr;     // reference rule: the generator's jump polynomials
    double* Tfull = nullptr;   // classic: n*n
    float* eta_tab = nullptr;  // n*n eta^beta f32 (n <= 5000)

    ~paco_handle() {
        if (dev >= 0) cudaSetDevice(dev);
        if (st) cudaStreamSynchronize(st);  // nothing may still use the buffers returned below
        if (st2) cudaStreamSynchronize(st2);
        void* ptrs[] = {xy, orig_of, int_of, cell_start, sb_start, knn, eta, cand, tours, lb_sel, has_lb, improved,
                        partial, new_len, lb_len, g_len, nbr, cur_nbr, T, gb, gkey, counters, err, words, order, qhead, two_opt_flag, two_opt_edges, two_opt_txy,
                        scratch_u32, scratch_u64, rng, ratio, tl_city, tl_tau, ir_jump, Tfull, eta_tab, cand_mult};
        for (void* p : ptrs) dfree(p);
        for (auto e : evpool) cudaEventDestroy(e);
        if (st) cudaStreamDestroy(st);
        if (st2) cudaStreamDestroy(st2);
    }
};

extern "C" {

const char* paco_last_error(void) { return g_last_error.c_str(); }
int paco_version(void) { return 1; }

paco_status paco_release_cached_memory(int device) {
    int dev = device;
    if (dev < 0) CU(cudaGetDevice(&dev));
    CU(cudaSetDevice(dev));
    cudaMemPool_t pool;
    CU(engine_pool(dev, &pool));
    CU(cudaStreamSynchronize(0));  // frees of destroyed handles complete in stream order
    CU(cudaMemPoolTrimTo(pool, 0));
    return PACO_OK;
}

paco_status paco_config_default(paco_config* c) {
    if (!c) return fail(PACO_E_INVALID, "null config");
    *c = paco_config{};
    // RunConfig defaults, engine.hpp:43-59
    c->ants = 16; c->iterations = 100000; c->alpha = 5.0; c->beta = 5.0;
    c->partial_prob = 0.95; c->max_mod_frac = 1.0; c->two_opt_prob = 0.0; c->two_opt_window = 0;
    c->workers = 8; c->seed = 1; c->rho = 0.1; c->tau_max = 1.0; c->tau0 = 1.0;
    c->time_budget_s = 0.0; c->convergence_interval_s = 1.0;
    c->synchronous = 1;  // the reference defaults to async; the GPU engine defaults to the deterministic path
    c->validate_tours = 0;
    c->candidates = 16; c->draws = PACO_DRAWS_PHILOX; c->device = -1;
    return PACO_OK;
}

paco_status paco_config_validate(const paco_config* c, uint32_t n, int mode) {
    if (!c) return fail(PACO_E_INVALID, "null config");
    // RunConfig::validate, engine.hpp:61-75 (same messages)
    if (c->ants < 1) return fail(PACO_E_INVALID, "ants must be >= 1");
    if (c->iterations < 1) return fail(PACO_E_INVALID, "iterations must be >= 1");
    if (c->workers < 1) return fail(PACO_E_INVALID, "workers must be >= 1");
    if (!(c->partial_prob >= 0.0 && c->partial_prob <= 1.0))
        return fail(PACO_E_INVALID, "partial_prob must be in [0,1]");
    if (!(c->max_mod_frac > 0.0 && c->max_mod_frac <= 1.0))
        return fail(PACO_E_INVALID, "max_mod_frac must be in (0,1]");
    if (!(c->two_opt_prob >= 0.0 && c->two_opt_prob <= 1.0))
        return fail(PACO_E_INVALID, "two_opt_prob must be in [0,1]");
    if (!(c->rho >= 0.0 && c->rho <= 1.0)) return fail(PACO_E_INVALID, "rho must be in [0,1]");
    if (!(c->tau0 > 0.0)) return fail(PACO_E_INVALID, "tau0 must be positive");
    if (!(c->tau_max > 0.0)) return fail(PACO_E_INVALID, "tau_max must be positive");
    if (!(c->time_budget_s >= 0.0)) return fail(PACO_E_INVALID, "time budget must be >= 0");
    if (mode < 0 || mode > 2) return fail(PACO_E_INVALID, "unknown mode");
    // engine.hpp:158-160
    if (mode == PACO_MODE_CLASSIC && n > 5000)
        return fail(PACO_E_INVALID, "classic mode requires n <= 5000");
    if (n < 3) return fail(PACO_E_INVALID, "instance needs at least 3 cities, got " + std::to_string(n));
    if (c->candidates < 1 || c->candidates > 32) return fail(PACO_E_INVALID, "candidates must be in [1,32]");
    if (c->draws > 1) return fail(PACO_E_INVALID, "unknown draw source");
    if (c->rule > 1) return fail(PACO_E_INVALID, "unknown selection rule");
    if (c->rule == PACO_RULE_INDEPENDENT_ROULETTE && c->draws != PACO_DRAWS_PHILOX)
        return fail(PACO_E_INVALID, "the reference rule draws from its own xoshiro256++ streams");
    // classic mode always runs barriered iterations (engine.hpp:213); the reference rule is
    // kept synchronous, its purpose being bit-identity with paco::run
    if (!c->synchronous && mode != PACO_MODE_CLASSIC && c->rule == PACO_RULE_INDEPENDENT_ROULETTE)
        return fail(PACO_E_UNSUPPORTED, "the reference-rule engine is synchronous only");
    if (!c->synchronous && mode != PACO_MODE_CLASSIC && c->ants > 65535)
        return fail(PACO_E_UNSUPPORTED, "asynchronous mode supports at most 65535 ants");
    return PACO_OK;
}

// Shared memory of the kernels a handle will launch, checked before anything is
// allocated: the launch-time dynamic size plus the kernel's static shared memory.
static size_t static_smem(const void* kern) {
    cudaFuncAttributes fa{};
    return cudaFuncGetAttributes(&fa, kern) == cudaSuccess ? fa.sharedSizeBytes : 0;
}
// fallback list | visited bitmap | warming scratch | superblocks known to be empty (F1): the
// grid has at most 16 n + 4096 cells (setup_grid), so at most n / 4 + 64 superblocks
static uint32_t sbe_words_bound(uint32_t n) { return (n / 4 + 64 + 31) / 32; }
static size_t construct_dyn_smem(uint32_t nwords, uint32_t sbe_words) {
    return kFbList * 4 + (size_t)nwords * 4 + 512 + 16 + (size_t)sbe_words * 4;
}
static size_t construct_smem_need(uint32_t kp, uint32_t nwords, bool async_mode) {
    const void* kerns[4];
    int nk = 0;
    if (kp == 16) {
        kerns[nk++] = (const void*)k_construct<16, 4, false>; kerns[nk++] = (const void*)k_construct<16, 4, true>;
        if (async_mode) kerns[nk++] = (const void*)k_construct_async<16, 4>;
    } else if (kp == 20) {
        kerns[nk++] = (const void*)k_construct<20, 5, false>; kerns[nk++] = (const void*)k_construct<20, 5, true>;
        if (async_mode) kerns[nk++] = (const void*)k_construct_async<20, 5>;
    } else {
        kerns[nk++] = (const void*)k_construct<0, 5, false>; kerns[nk++] = (const void*)k_construct<0, 5, true>;
        if (async_mode) kerns[nk++] = (const void*)k_construct_async<0, 5>;
    }
    size_t st = 0;
    for (int q = 0; q < nk; ++q) st = std::max(st, static_smem(kerns[q]));
    return construct_dyn_smem(nwords, sbe_words_bound(nwords * 32)) + st;
}
// k_weights: ratios (8 B per ant) plus, on the hashed path, per thread 2^B slots and km sums
static int weights_block(int km, bool hash) { return hash && km > 16 ? 128 : 256; }
static size_t weights_dyn_smem(uint32_t m, int km, bool hash) {
    return sizeof(double) * m +
           (hash ? (sizeof(uint32_t) * (1u << hash_slot_bits(km)) + sizeof(double) * km) * weights_block(km, true) : 0);
}

static paco_status build_grid(paco_handle* h) {
    const uint32_t n = h->n;
    double x0 = h->hx[0], x1 = x0, y0 = h->hy[0], y1 = y0;
    for (uint32_t i = 1; i < n; ++i) {
        x0 = std::min(x0, h->hx[i]); x1 = std::max(x1, h->hx[i]);
        y0 = std::min(y0, h->hy[i]); y1 = std::max(y1, h->hy[i]);
    }
    const double w = std::max(x1 - x0, 1e-9), hh = std::max(y1 - y0, 1e-9);
    double cs = std::sqrt(w * hh * 2.0 / n);
    if (!(cs > 0) || !std::isfinite(cs)) cs = 1.0;
    int32_t gw = 0, gh = 0;
    uint32_t L = 3;
    for (;;) {
        const double fw = w / cs + 1.0, fh = hh / cs + 1.0;
        if (fw < 32768.0 && fh < 32768.0) {
            gw = (int32_t)(w / cs) + 1; gh = (int32_t)(hh / cs) + 1;
            L = 3;
            while ((1 << L) < std::max(gw, gh)) ++L;
            if ((uint64_t)gw * gh <= 4ull * n + 16 && (1ull << (2 * L)) <= 16ull * n + 4096) break;
        }
        cs *= 1.25;
    }
    h->g.x0 = x0; h->g.y0 = y0; h->g.cs = cs; h->g.inv = 1.0 / cs;
    h->g.gw = gw; h->g.gh = gh; h->g.gws = (gw + 7) / 8; h->g.ghs = (gh + 7) / 8;
    h->g.L = L; h->g.ncells = 1u << (2 * L);
    return PACO_OK;
}

// reference rule: [draw ring] [acc n doubles (P-ACO)] [bitmap]
// k_ir_touched: acc[n] (fp64) | ratios[m] (fp64) | the step's 2m contributions (u32)
static size_t ir_touched_smem(uint32_t n, uint32_t m) { return (size_t)8 * n + (size_t)8 * m + (size_t)8 * m; }
static size_t ir_smem_bytes(uint32_t n, uint32_t m, uint32_t nwords, int mode) {
    (void)m;
    return sizeof(IrRing) + (mode == PACO_MODE_CLASSIC ? 0 : (size_t)8 * ir_acc_slots(n)) + (size_t)nwords * 4;
}

// colony state shared by both selection rules
// k_two_opt_cluster's shape: the largest cluster (16 CTAs of 512 threads, non-portable,
// else 8) the device can co-schedule, as many clusters as fit at once (at most the cache
// slots). The searches go to clusters when the expected number of flagged tours per
// iteration (m * two_opt_prob) is at most the number of clusters - the paper's setting,
// p = 0.001 - and to one CTA per tour (k_two_opt) otherwise. PACO_TWO_OPT_PATH=cta|cluster
// overrides the choice (tests).
constexpr uint32_t kTwoOptStageMax = 2048;  // 48 KB of shared memory per CTA
static void pick_two_opt_cluster(paco_handle* h) {
    h->two_opt_cs = 0; h->two_opt_clusters = 0; h->two_opt_use_cluster = false;
    if (cudaFuncSetAttribute(k_two_opt_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess ||
        cudaFuncSetAttribute(k_two_opt_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(kTwoOptStageMax * (sizeof(double2) + sizeof(int32_t) + sizeof(uint32_t)))) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    uint32_t sizes[2] = {16u, 8u};
    if (const char* e = std::getenv("PACO_TWO_OPT_CS")) sizes[0] = sizes[1] = (uint32_t)std::atoi(e);
    for (uint32_t cs : sizes) {
        cudaLaunchConfig_t lc = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        lc.gridDim = dim3(cs); lc.blockDim = dim3(512); lc.attrs = at; lc.numAttrs = 1;
        lc.dynamicSmemBytes = (size_t)kTwoOptStageMax * (sizeof(double2) + sizeof(int32_t) + sizeof(uint32_t));
        int nc = 0;
        if (cudaOccupancyMaxActiveClusters(&nc, k_two_opt_cluster, &lc) == cudaSuccess && nc >= 1) {
            h->two_opt_cs = cs;
            h->two_opt_clusters = std::min<uint32_t>((uint32_t)nc, h->two_opt_ctas);
            break;
        }
        cudaGetLastError();
    }
    if (!h->two_opt_clusters) return;
    // a round reads at most 2W + R + 2 positions (R forward rows, about two cells per thread)
    const uint64_t weff = h->cfg.two_opt_window == 0 ? h->n - 1 : h->cfg.two_opt_window;
    const uint64_t G = (uint64_t)h->two_opt_cs * 512, R = weff >= 2 * G ? 1 : 2 * G / weff;
    const uint64_t span = 2 * weff + R + 2;
    uint32_t cap = 256;
    while (cap < span) cap *= 2;
    h->two_opt_stage = cap <= kTwoOptStageMax ? cap : 0u;  // a power of two (ring slots)
    h->two_opt_use_cluster = (double)h->m * h->cfg.two_opt_prob <= (double)h->two_opt_clusters;
    if (const char* e = std::getenv("PACO_TWO_OPT_PATH")) {
        if (!std::strcmp(e, "cta")) h->two_opt_use_cluster = false;
        if (!std::strcmp(e, "cluster")) h->two_opt_use_cluster = true;
        if (!std::strcmp(e, "verbose") || std::getenv("PACO_TWO_OPT_VERBOSE"))
            std::fprintf(stderr, "k_two_opt_cluster: %u CTAs per cluster, %u clusters, stage %u, in use: %d\n",
                         h->two_opt_cs, h->two_opt_clusters, h->two_opt_stage, (int)h->two_opt_use_cluster);
    }
}

static paco_status alloc_colony(paco_handle* h) {
    const uint32_t n = h->n, m = h->m;
    cudaStream_t st = h->st;
    CU(dalloc(&h->xy, n)); CU(dalloc(&h->orig_of, n)); CU(dalloc(&h->int_of, n));
    CU(dalloc(&h->tours, (size_t)m * 2 * n));
    CU(dalloc(&h->lb_sel, m)); CU(dalloc(&h->has_lb, m)); CU(dalloc(&h->improved, m)); CU(dalloc(&h->partial, m));
    CU(dalloc(&h->new_len, m)); CU(dalloc(&h->lb_len, m)); CU(dalloc(&h->g_len, 1));
    CU(dalloc(&h->nbr, (size_t)m * n));
    CU(dalloc(&h->gb, 1)); CU(dalloc(&h->gkey, 1)); CU(dalloc(&h->counters, 16)); CU(dalloc(&h->err, 1));
    CU(dalloc(&h->scratch_u32, (size_t)n + 64)); CU(dalloc(&h->scratch_u64, 4));
    CU(cudaMemsetAsync(h->lb_sel, 0, m, st)); CU(cudaMemsetAsync(h->has_lb, 0, m, st));
    CU(cudaMemsetAsync(h->improved, 0, m, st)); CU(cudaMemsetAsync(h->partial, 0, m, st));
    CU(cudaMemsetAsync(h->lb_len, 0, sizeof(int64_t) * m, st));
    CU(cudaMemsetAsync(h->nbr, 0, sizeof(uint2) * (size_t)m * n, st));
    CU(cudaMemsetAsync(h->tours, 0, sizeof(uint32_t) * (size_t)m * 2 * n, st));
    GBest g0{0, -1, 0};
    const int64_t gmax = std::numeric_limits<int64_t>::max();
    CU(cudaMemcpyAsync(h->gb, &g0, sizeof g0, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(h->g_len, &gmax, sizeof gmax, cudaMemcpyHostToDevice, st));
    CU(cudaMemsetAsync(h->counters, 0, 16 * sizeof(unsigned long long), st));
    CU(cudaMemsetAsync(h->err, 0, sizeof(int), st));
    if (h->mode == PACO_MODE_CLASSIC) CU(dalloc(&h->cur_nbr, (size_t)m * n));
#ifndef PACO_NO_ORDER
    if (!h->ir && !h->async_mode && m <= 4096) { CU(dalloc(&h->order, m)); CU(dalloc(&h->qhead, 1)); }
#endif
    if (!h->ir && !h->async_mode && h->cfg.two_opt_prob > 0.0) {
        h->two_opt_ctas = std::min<uint32_t>(m, 64);
        pick_two_opt_cluster(h);
        CU(dalloc(&h->two_opt_flag, m));
        CU(dalloc(&h->two_opt_edges, (size_t)h->two_opt_ctas * n));
        CU(dalloc(&h->two_opt_txy, (size_t)h->two_opt_ctas * n));
        CU(cudaMemsetAsync(h->two_opt_flag, 0, m, st));
    }
    CU(cudaStreamSynchronize(st));
    return PACO_OK;
}

// SplitMix64 + Rng::for_stream (rng.hpp:10-38), restated to seed the reference-rule
// streams exactly as Colony does for ant k (colony.hpp:93-95).
static uint64_t splitmix_next(uint64_t& s) {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
static void rng_for_stream(uint64_t master, uint64_t stream, uint64_t out[4]) {
    uint64_t sm = master;
    const uint64_t a = splitmix_next(sm);
    uint64_t mix = a ^ (stream * 0x9e3779b97f4a7c15ULL + 0x2545f4914f6cdd1dULL);
    uint64_t seed = splitmix_next(mix);
    for (int q = 0; q < 4; ++q) out[q] = splitmix_next(seed);
}

// ---- xoshiro256 jump polynomials (the reference-rule generator, kernels_ir.cuh) ----
// The state update of xoshiro256++ (rng.hpp:40-50) is linear over GF(2)^256; by
// Cayley-Hamilton, advancing J steps is p(M) with p = x^J mod P, P the characteristic
// polynomial of M. P is the minimal polynomial of a state-bit sequence (Berlekamp-Massey;
// degree 256), x^J mod P by square-and-multiply.
using Poly = std::array<uint64_t, 8>;  // up to degree 511
static void xo_host_step(uint64_t s[4]) {
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t;
    s[3] = (s[3] << 45) | (s[3] >> 19);
}
static bool pbit(const Poly& a, int i) { return (a[i >> 6] >> (i & 63)) & 1u; }
static void pflip(Poly& a, int i) { a[i >> 6] ^= 1ull << (i & 63); }
static bool xo_char_poly(Poly& P) {
    // the sequence: bit 0 of s[0] along the orbit of a fixed nonzero state
    uint64_t s[4] = {0x9e3779b97f4a7c15ull, 0xbf58476d1ce4e5b9ull, 0x94d049bb133111ebull, 0x2545f4914f6cdd1dull};
    const int N = 1024;
    std::vector<uint8_t> seq(N);
    for (int i = 0; i < N; ++i) { seq[i] = (uint8_t)(s[0] & 1u); xo_host_step(s); }
    std::vector<uint8_t> C(N + 1, 0), B(N + 1, 0), T;
    C[0] = B[0] = 1;
    int L = 0, m = 1;
    for (int n = 0; n < N; ++n) {
        uint8_t d = seq[n];
        for (int i = 1; i <= L; ++i) d ^= (uint8_t)(C[i] & seq[n - i]);
        if (!d) { ++m; continue; }
        T = C;
        for (int i = 0; i + m <= N; ++i) C[i + m] ^= B[i];
        if (2 * L <= n) { L = n + 1 - L; B = T; m = 1; } else ++m;
    }
    if (L != 256) return false;
    P.fill(0);
    for (int k = 0; k <= L; ++k) if (C[L - k]) pflip(P, k);  // reciprocal of the connection polynomial
    return true;
}
static Poly pmulmod(const Poly& a, const Poly& b, const Poly& P) {
    Poly r{};
    for (int i = 0; i < 256; ++i)
        if (pbit(a, i))
            for (int j = 0; j < 256; ++j) if (pbit(b, j)) pflip(r, i + j);
    for (int k = 510; k >= 256; --k)
        if (pbit(r, k))
            for (int j = 0; j <= 256; ++j) if (pbit(P, j)) pflip(r, k - 256 + j);
    return r;
}
static Poly pxpow(uint64_t J, const Poly& P) {  // x^J mod P
    Poly r{}; r[0] = 1;
    for (int b = 63; b >= 0; --b) {
        r = pmulmod(r, r, P);
        if ((J >> b) & 1u) {  // multiply by x
            Poly t{};
            for (int i = 0; i < 256; ++i) if (pbit(r, i)) pflip(t, i + 1);
            if (pbit(t, 256)) for (int j = 0; j <= 256; ++j) if (pbit(P, j)) pflip(t, j);
            r = t;
        }
    }
    return r;
}
static void xo_host_jump(uint64_t s[4], const Poly& p) {
    uint64_t t[4] = {0, 0, 0, 0};
    for (int b = 0; b < 256; ++b) {
        if (pbit(p, b)) for (int q = 0; q < 4; ++q) t[q] ^= s[q];
        xo_host_step(s);
    }
    for (int q = 0; q < 4; ++q) s[q] = t[q];
}
// the table the generator uses, checked against direct stepping once per process
static bool ir_jump_table(IrJump& J) {
    static std::mutex mu;
    static bool done = false, ok = false;
    static IrJump cached;
    std::lock_guard<std::mutex> lk(mu);
    if (!done) {
        done = true;
        Poly P;
        if (xo_char_poly(P)) {
            for (uint32_t i = 0; i < 33; ++i) {
                const Poly q = pxpow(i < 32 ? (uint64_t)i * kIrChunk : 31ull * kIrChunk, P);
                for (int w = 0; w < 4; ++w) cached.p[i][w] = q[w];
            }
            ok = true;
            for (uint32_t i : {1u, 7u, 31u, 32u}) {
                uint64_t a[4] = {1, 2, 3, 0xdeadbeefcafef00dull}, b[4];
                std::memcpy(b, a, sizeof a);
                Poly q{};
                for (int w = 0; w < 4; ++w) q[w] = cached.p[i][w];
                xo_host_jump(a, q);
                const uint64_t steps = i < 32 ? (uint64_t)i * kIrChunk : 31ull * kIrChunk;
                for (uint64_t k = 0; k < steps; ++k) xo_host_step(b);
                ok = ok && std::memcmp(a, b, sizeof a) == 0;
            }
        }
    }
    J = cached;
    return ok;
}

// C ABI (declared extern "C" in paco_b200.h)
paco_status paco_rng_jump(const uint64_t state_in[4], uint64_t steps, uint64_t state_out[4]) {
    if (!state_in || !state_out) return fail(PACO_E_INVALID, "null state");
    static std::mutex mu;
    static bool have = false;
    static Poly P;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (!have) have = xo_char_poly(P);
        if (!have) return fail(PACO_E_RUNTIME, "xoshiro256 characteristic polynomial not found");
    }
    uint64_t s[4] = {state_in[0], state_in[1], state_in[2], state_in[3]};
    xo_host_jump(s, pxpow(steps, P));
    for (int q = 0; q < 4; ++q) state_out[q] = s[q];
    return PACO_OK;
}

// Reference-rule mode: cities stay in their original order (the rule consumes draws
// in ascending city index), no candidate lists.
static paco_status setup_ir(paco_handle* h) {
    const uint32_t n = h->n, m = h->m;
    paco_status s = alloc_colony(h);
    if (s != PACO_OK) return s;
    std::vector<double2> xy(n);
    std::vector<uint32_t> ident(n);
    for (uint32_t i = 0; i < n; ++i) { xy[i] = make_double2(h->hx[i], h->hy[i]); ident[i] = i; }
    // every copy is ordered on the handle's (non-blocking) stream and completes before
    // setup returns: a pageable cudaMemcpy may return before its DMA lands
    CU(cudaMemcpyAsync(h->xy, xy.data(), sizeof(double2) * n, cudaMemcpyHostToDevice, h->st));
    CU(cudaMemcpyAsync(h->orig_of, ident.data(), sizeof(uint32_t) * n, cudaMemcpyHostToDevice, h->st));
    CU(cudaMemcpyAsync(h->int_of, ident.data(), sizeof(uint32_t) * n, cudaMemcpyHostToDevice, h->st));
    h->h_orig = ident;
    h->h_int = ident;
    std::vector<uint64_t> st((size_t)m * 4);
    for (uint32_t a = 0; a < m; ++a) rng_for_stream(h->cfg.seed, a, &st[(size_t)a * 4]);
    CU(dalloc(&h->rng, (size_t)m * 4));
    CU(cudaMemcpyAsync(h->rng, st.data(), sizeof(uint64_t) * st.size(), cudaMemcpyHostToDevice, h->st));
    CU(dalloc(&h->ratio, m));
    CU(cudaMemsetAsync(h->ratio, 0, sizeof(double) * m, h->st));
    {
        IrJump J;
        if (!ir_jump_table(J)) return fail(PACO_E_RUNTIME, "xoshiro256 jump polynomials failed their self-check");
        CU(dalloc(&h->ir_jump, 1));
        CU(cudaMemcpyAsync(h->ir_jump, &J, sizeof J, cudaMemcpyHostToDevice, h->st));
        CU(cudaStreamSynchronize(h->st));  // before J goes out of scope
    }
    if (h->mode != PACO_MODE_CLASSIC) {
        CU(dalloc(&h->tl_city, (size_t)n * (2 * m + 1)));
        CU(dalloc(&h->tl_tau, (size_t)n * 2 * m));
    }
    if (n <= 5000) {  // the reference keeps eta^beta in an f32 table for these sizes
        CU(dalloc(&h->eta_tab, (size_t)n * n));
        k_eta_table<<<(unsigned)(((size_t)n * n + 255) / 256), 256, 0, h->st>>>(h->xy, n, h->cfg.beta, h->eta_tab);
        CU(cudaGetLastError());
    }
    if (h->mode == PACO_MODE_CLASSIC) {  // PheromoneMatrix(n, rho, tau_max), construction.hpp:165-175
        CU(dalloc(&h->Tfull, (size_t)n * n));
        std::vector<double> init((size_t)n * n, h->cfg.tau_max);
        CU(cudaMemcpyAsync(h->Tfull, init.data(), sizeof(double) * init.size(), cudaMemcpyHostToDevice, h->st));
        CU(cudaStreamSynchronize(h->st));  // before `init` goes out of scope
    }
    CU(cudaStreamSynchronize(h->st));
    h->setup_ms = 0.0;
    return PACO_OK;
}

static paco_status setup(paco_handle* h) {
    if (h->ir) return setup_ir(h);
    const uint32_t n = h->n, k = h->k;
    cudaStream_t st = h->st;
    if (build_grid(h) != PACO_OK) return PACO_E_RUNTIME;
    paco_status s0 = alloc_colony(h);
    if (s0 != PACO_OK) return s0;
    double *dx = nullptr, *dy = nullptr;
    unsigned long long *keys = nullptr, *keys2 = nullptr;
    uint32_t* cellm = nullptr;
    CU(dalloc(&dx, n)); CU(dalloc(&dy, n));
    CU(dalloc(&keys, n)); CU(dalloc(&keys2, n)); CU(dalloc(&cellm, n));
    CU(dalloc(&h->cell_start, (size_t)h->g.ncells + 1));
    CU(dalloc(&h->sb_start, (size_t)(h->g.ncells >> 6) + 1));
    CU(dalloc(&h->knn, (size_t)n * kNearRow)); CU(dalloc(&h->eta, (size_t)n * k)); CU(dalloc(&h->cand, (size_t)n * h->kp));
    CU(cudaMemsetAsync(h->cand, 0, sizeof(uint2) * (size_t)n * h->kp, st));
    if (h->mode == PACO_MODE_CLASSIC) {
        CU(dalloc(&h->T, (size_t)n * k));
        std::vector<double> init((size_t)n * k, h->cfg.tau_max);
        CU(cudaMemcpyAsync(h->T, init.data(), sizeof(double) * init.size(), cudaMemcpyHostToDevice, st));
        CU(cudaStreamSynchronize(st));
    }

    cudaEvent_t e0, e1;
    CU(cudaEventCreate(&e0)); CU(cudaEventCreate(&e1));
    CU(cudaEventRecord(e0, st));
    CU(cudaMemcpyAsync(dx, h->hx.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(dy, h->hy.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
    const uint32_t tb = 256, nb = (n + tb - 1) / tb;
    k_cell_keys<<<nb, tb, 0, st>>>(dx, dy, n, h->g, keys);
    CU(cudaGetLastError());
    size_t tmp_bytes = 0;
    const int end_bit = 32 + 2 * (int)h->g.L;
    CU(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, keys, keys2, (int)n, 0, end_bit, st));
    void* tmp = nullptr;
    CU(dalloc(reinterpret_cast<unsigned char**>(&tmp), tmp_bytes ? tmp_bytes : 1));
    CU(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, keys, keys2, (int)n, 0, end_bit, st));
    k_scatter<<<nb, tb, 0, st>>>(keys2, dx, dy, n, h->xy, h->orig_of, h->int_of, cellm);
    k_cell_start<<<nb, tb, 0, st>>>(cellm, n, h->g.ncells, h->cell_start);
    {
        const uint32_t nsb = h->g.ncells >> 6;
        k_sb_start<<<(nsb + 1 + 255) / 256, 256, 0, st>>>(h->cell_start, nsb, h->sb_start);
    }
    CU(cudaGetLastError());
    // K1: k-NN lists, one thread per city, exact ring search over grid cells
    const int kk = (int)std::min<uint32_t>(kNearRow, n - 1);
    {
        constexpr int T = kNearRow >= 256 ? 32 : 64;  // threads per CTA; the heaps take 12 B x kNearRow x T of shared memory
        const size_t hsm = (size_t)(sizeof(double) + sizeof(uint32_t)) * kNearRow * T;
        CU(cudaFuncSetAttribute(k_knn_cells<kNearRow, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm));
        k_knn_cells<kNearRow, T><<<(n + T - 1) / T, T, hsm, st>>>(h->xy, h->orig_of, h->cell_start, h->g, n, kk,
                                                                 (int)k, h->cfg.beta, h->knn, h->eta);
    }
    CU(cudaGetLastError());
    int dev_optin = 0;
    CU(cudaDeviceGetAttribute(&dev_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->dev));
    if (h->mode != PACO_MODE_CLASSIC &&
        weights_dyn_smem(h->m, kmax_for(k), true) <= (size_t)dev_optin) {  // candidate perfect hashes for k_weights
        int* dfail = nullptr;
        CU(dalloc(&h->cand_mult, n)); CU(dalloc(&dfail, 1));
        CU(cudaMemsetAsync(dfail, 0, sizeof(int), st));
        const int km = kmax_for(k);
        if (km == 8) k_cand_hash<8><<<nb, tb, 0, st>>>(h->knn, n, (int)k, h->cand_mult, dfail);
        else if (km == 16) k_cand_hash<16><<<nb, tb, 0, st>>>(h->knn, n, (int)k, h->cand_mult, dfail);
        else if (km == 24) k_cand_hash<24><<<nb, tb, 0, st>>>(h->knn, n, (int)k, h->cand_mult, dfail);
        else k_cand_hash<32><<<nb, tb, 0, st>>>(h->knn, n, (int)k, h->cand_mult, dfail);
        CU(cudaGetLastError());
        int hf = 0;
        CU(cudaMemcpyAsync(&hf, dfail, sizeof(int), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        dfree(dfail);
        if (hf) { dfree(h->cand_mult); h->cand_mult = nullptr; }  // keep the comparison loop
    }
    CU(cudaEventRecord(e1, st));
    CU(cudaStreamSynchronize(st));
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, e0, e1));
    h->setup_ms = ms;
    cudaEventDestroy(e0); cudaEventDestroy(e1);
    h->h_orig.resize(n); h->h_int.resize(n);
    CU(cudaMemcpyAsync(h->h_orig.data(), h->orig_of, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    for (uint32_t p = 0; p < n; ++p) h->h_int[h->h_orig[p]] = p;
    dfree(tmp); dfree(dx); dfree(dy); dfree(keys); dfree(keys2); dfree(cellm);
    return PACO_OK;
}

paco_status paco_create(const double* xs, const double* ys, uint32_t n, const paco_config* cfg, int mode,
                        paco_handle** out) {
    if (!out) return fail(PACO_E_INVALID, "null output handle");
    *out = nullptr;
    if (!xs || !ys) return fail(PACO_E_INVALID, "null coordinates");
    paco_status s = paco_config_validate(cfg, n, mode);
    if (s != PACO_OK) return s;
    for (uint32_t i = 0; i < n; ++i)
        if (!std::isfinite(xs[i]) || !std::isfinite(ys[i])) return fail(PACO_E_INVALID, "non-finite coordinate");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(PACO_E_CUDA, "no CUDA device visible (the B200 engine has no CPU fallback)");
    int dev = cfg->device;
    if (dev < 0) CU(cudaGetDevice(&dev));
    CU(cudaSetDevice(dev));
    cudaDeviceProp prop{};
    CU(cudaGetDeviceProperties(&prop, dev));
    if (prop.major != 10) return fail(PACO_E_CUDA, std::string("device is not sm_100 (Blackwell): ") + prop.name);
    const uint32_t nwords = (n + 31) / 32;
    const uint32_t kk = std::min<uint32_t>(cfg->candidates, n - 1), kpp = (kk + 1) & ~1u;
    const bool ir = cfg->rule == PACO_RULE_INDEPENDENT_ROULETTE;
    const bool want_async = !cfg->synchronous && mode != PACO_MODE_CLASSIC;
    const size_t optin = (size_t)prop.sharedMemPerBlockOptin;
    if (!ir && n >= (1u << 21))  // the pick packs city ids into 21 bits (implied by the bitmap bound below)
        return fail(PACO_E_UNSUPPORTED, "visited bitmap exceeds shared memory (n too large)");
    if (ir) {
        if (ir_smem_bytes(n, cfg->ants, nwords, mode) + static_smem((const void*)k_construct_ir) > optin)
            return fail(PACO_E_UNSUPPORTED, "reference-rule per-ant state exceeds shared memory (n too large)");
        if (mode != PACO_MODE_CLASSIC && ir_touched_smem(n, cfg->ants) > optin)
            return fail(PACO_E_UNSUPPORTED, "reference-rule pheromone staging exceeds shared memory (n or ants too large)");
    } else {
        if (construct_smem_need(kpp, nwords, want_async) > optin)
            return fail(PACO_E_UNSUPPORTED, "visited bitmap exceeds shared memory (n too large)");
        if (mode != PACO_MODE_CLASSIC && weights_dyn_smem(cfg->ants, kmax_for(kk), false) > optin)
            return fail(PACO_E_UNSUPPORTED, "per-ant ratios of the weight rebuild exceed shared memory (too many ants)");
    }
    auto* h = new (std::nothrow) paco_handle();
    if (!h) return fail(PACO_E_RUNTIME, "out of host memory");
    h->ir = ir;
    h->dev = dev;
    h->num_sms = prop.multiProcessorCount;
    h->cfg = *cfg;
    h->mode = mode;
    h->n = n; h->m = cfg->ants; h->k = std::min<uint32_t>(cfg->candidates, n - 1); h->nwords = nwords;
    h->kp = (h->k + 1) & ~1u;
    h->hx.assign(xs, xs + n); h->hy.assign(ys, ys + n);
    if (cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking) != cudaSuccess) {
        delete h;
        return fail(PACO_E_CUDA, "stream creation failed");
    }
    h->async_mode = !cfg->synchronous && mode != PACO_MODE_CLASSIC;
    if (h->async_mode) {
        // g_best key packs the length into 48 bits: bound it by n x the bounding-box diagonal
        double x0 = xs[0], x1 = xs[0], y0 = ys[0], y1 = ys[0];
        for (uint32_t i = 1; i < n; ++i) {
            x0 = std::min(x0, xs[i]); x1 = std::max(x1, xs[i]); y0 = std::min(y0, ys[i]); y1 = std::max(y1, ys[i]);
        }
        if ((double)n * (std::sqrt((x1 - x0) * (x1 - x0) + (y1 - y0) * (y1 - y0)) + 1.0) >= 0x1p48) {
            delete h;
            return fail(PACO_E_UNSUPPORTED, "asynchronous mode needs tour lengths below 2^48");
        }
        if (cudaStreamCreateWithFlags(&h->st2, cudaStreamNonBlocking) != cudaSuccess) {
            delete h;
            return fail(PACO_E_CUDA, "stream creation failed");
        }
    }
    s = setup(h);
    if (s != PACO_OK) { delete h; return s; }
    *out = h;
    return PACO_OK;
}

void paco_destroy(paco_handle* h) { delete h; }

static cudaEvent_t ev(paco_handle* h, size_t i) {
    while (h->evpool.size() <= i) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        h->evpool.push_back(e);
    }
    return h->evpool[i];
}

static paco_status launch_weights(paco_handle* h, cudaStream_t stream = nullptr, const unsigned long long* gkey = nullptr) {
    const uint32_t n = h->n;
    if (!stream) stream = h->st;
    const double* T = h->mode == PACO_MODE_CLASSIC ? h->T : nullptr;
    const int km = kmax_for(h->k);
    const bool hash = !T && h->cand_mult != nullptr;  // perfect-hash lookup (k_cand_hash)
    const uint32_t tb = (uint32_t)weights_block(km, hash);
    const size_t smem = T ? 0 : weights_dyn_smem(h->m, km, hash);
#define LAUNCH_W3(KM, LIVE, HASH)                                                                          \
    do {                                                                                                   \
        if (smem > 48 * 1024)                                                                              \
            CU(cudaFuncSetAttribute(k_weights<KM, LIVE, HASH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
        k_weights<KM, LIVE, HASH><<<(n + tb - 1) / tb, tb, smem, stream>>>(h->knn, h->eta, h->nbr, h->lb_len,  \
                                                            h->has_lb, h->g_len, gkey, T, h->cand_mult, n, h->m, \
                                                            (int)h->k, (int)h->kp, h->cfg.alpha, h->cfg.tau0, h->cand); \
    } while (0)
#define LAUNCH_W2(KM, LIVE) do { if (hash) LAUNCH_W3(KM, LIVE, true); else LAUNCH_W3(KM, LIVE, false); } while (0)
#define LAUNCH_W(KM) do { if (gkey) LAUNCH_W2(KM, true); else LAUNCH_W2(KM, false); } while (0)
    if (km == 8) LAUNCH_W(8); else if (km == 16) LAUNCH_W(16); else if (km == 24) LAUNCH_W(24); else LAUNCH_W(32);
#undef LAUNCH_W
#undef LAUNCH_W2
#undef LAUNCH_W3
    CU(cudaGetLastError());
    return PACO_OK;
}

static paco_status launch_ratios(paco_handle* h) {
    if (h->mode == PACO_MODE_CLASSIC) return PACO_OK;
    k_ratios<<<(h->m + 127) / 128, 128, 0, h->st>>>(h->lb_len, h->has_lb, h->g_len, h->m, h->ratio);
    // every city's begin_step for the iteration (the colony is frozen until the completion step)
    const size_t smem = ir_touched_smem(h->n, h->m);
    if (smem > 48 * 1024)
        CU(cudaFuncSetAttribute(k_ir_touched, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const uint32_t grid = std::min<uint32_t>(h->n, 8 * (uint32_t)h->num_sms);
    k_ir_touched<<<grid, 32, smem, h->st>>>(h->nbr, h->ratio, h->n, h->m, h->cfg.alpha, h->cfg.tau0, h->tl_city,
                                            h->tl_tau);
    CU(cudaGetLastError());
    return PACO_OK;
}

static paco_status launch_construct_ir(paco_handle* h, bool seeding) {
    IrArgs a{};
    a.xy = h->xy; a.nbr = h->nbr; a.ratio = h->ratio;
    a.tl_city = h->tl_city; a.tl_tau = h->tl_tau;
    a.jump = h->ir_jump;
    a.T = h->mode == PACO_MODE_CLASSIC ? h->Tfull : nullptr;
    a.rng = h->rng; a.tours = h->tours; a.lb_sel = h->lb_sel; a.new_len = h->new_len;
    a.partial_flag = h->partial; a.counters = h->counters;
    a.n = h->n; a.m = h->m; a.nwords = h->nwords;
    a.alpha = h->cfg.alpha; a.beta = h->cfg.beta; a.tau0 = h->cfg.tau0;
    a.eff_pp = h->mode == PACO_MODE_PARTIAL ? h->cfg.partial_prob : 0.0;  // engine.hpp:164-165
    a.mmf = h->cfg.max_mod_frac;
    a.seeding = seeding ? 1 : 0;
    a.coin_always = 0;
    a.eta_table = h->n <= 5000 ? 1 : 0;  // Heuristic keeps an f32 table iff the instance has a matrix
    a.eta_tab = h->eta_tab;
    a.two_opt_prob = h->cfg.two_opt_prob; a.two_opt_window = h->cfg.two_opt_window;
    const size_t smem = ir_smem_bytes(h->n, h->m, h->nwords, h->mode);
    if (smem > 48 * 1024)
        CU(cudaFuncSetAttribute(k_construct_ir, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_construct_ir<<<h->m, 64, smem, h->st>>>(a);
    CU(cudaGetLastError());
    return PACO_OK;
}

static ConstructArgs construct_args(paco_handle* h, bool seeding) {
    ConstructArgs a{};
    a.cand = h->cand; a.knn32 = h->knn; a.xy = h->xy; a.orig_of = h->orig_of; a.int_of = h->int_of;
    a.sb_start = h->sb_start; a.g = h->g; a.tours = h->tours; a.lb_sel = h->lb_sel;
    a.new_len = h->new_len; a.partial_flag = h->partial; a.counters = h->counters;
    a.words = h->cfg.draws == PACO_DRAWS_BUFFER ? h->words : nullptr;
    a.stride = h->words_stride; a.seed = h->cfg.seed; a.iter = h->iter;
    a.n = h->n; a.m = h->m; a.k = h->k; a.kp = h->kp; a.nwords = h->nwords;
#ifndef PACO_NO_SB_EMPTY
    a.sbe_words = ((h->g.ncells >> 6) + 31) / 32;
    if (a.sbe_words > sbe_words_bound(h->n)) a.sbe_words = 0;
#endif
    a.eff_pp = h->mode == PACO_MODE_PARTIAL ? h->cfg.partial_prob : 0.0;  // engine.hpp:164-165
    a.mmf = h->cfg.max_mod_frac;
    a.seeding = seeding ? 1 : 0;
    a.validate = h->cfg.validate_tours ? 1 : 0;
    a.err = h->err;
    a.two_opt_prob = h->cfg.two_opt_prob; a.two_opt_window = h->cfg.two_opt_window;
    a.two_opt_flag = h->async_mode ? nullptr : h->two_opt_flag;  // async: inline search
    return a;
}

static paco_status launch_construct(paco_handle* h, const ConstructArgs& a, uint32_t blocks) {
    // shared memory: double-buffered stage of k candidate rows + the n-bit visited bitmap
    const size_t smem = construct_dyn_smem(h->nwords, a.sbe_words) + (size_t)a.sb_words * 4;
    const bool buf = a.words != nullptr;
    // Shared-memory carveout: just enough for the CTAs one SM must host to run every ant at
    // once (ceil(m / #SMs) warps), so the rest of the unified L1 caches candidate rows.
    const int per_sm = (int)((blocks + h->num_sms - 1) / h->num_sms);
    int carve = (int)std::min<size_t>(100, (size_t)per_sm * (smem + 1024) * 100 / (228 * 1024) + 1);
#ifdef PACO_CARVE_ENV
    if (const char* e = getenv("PACO_CARVE")) carve = atoi(e);
#endif
    auto launch = [&](auto kern) -> paco_status {
        if (smem > 48 * 1024)
            CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CU(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
        kern<<<blocks, 32, smem, h->st>>>(a);
        CU(cudaGetLastError());
        return PACO_OK;
    };
    if (h->kp == 16) return buf ? launch(k_construct<16, 4, true>) : launch(k_construct<16, 4, false>);
    if (h->kp == 20) return buf ? launch(k_construct<20, 5, true>) : launch(k_construct<20, 5, false>);
    // generic k: runtime row stride, five scan steps (extra steps never touch lanes < k)
    return buf ? launch(k_construct<0, 5, true>) : launch(k_construct<0, 5, false>);
}

static paco_status launch_construct_async(paco_handle* h, const ConstructArgs& a, uint32_t count) {
    const size_t smem = construct_dyn_smem(h->nwords, a.sbe_words);
    const int per_sm = (int)((h->m + h->num_sms - 1) / h->num_sms);
    const int carve = (int)std::min<size_t>(100, (size_t)per_sm * (smem + 1024) * 100 / (228 * 1024) + 1);
    const AsyncState st{h->nbr, h->lb_len, h->has_lb, h->lb_sel, h->gkey, h->improved};
    auto launch = [&](auto kern) -> paco_status {
        if (smem > 48 * 1024)
            CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CU(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
        kern<<<h->m, 32, smem, h->st>>>(a, count, st);
        CU(cudaGetLastError());
        return PACO_OK;
    };
    if (h->kp == 16) return launch(k_construct_async<16, 4>);
    if (h->kp == 20) return launch(k_construct_async<20, 5>);
    return launch(k_construct_async<0, 5>);
}

static paco_status check_err(paco_handle* h);
constexpr int kWeightPassIntervalUs = 2000;  // minimum spacing of asynchronous weight passes

// Asynchronous iterations (engine.hpp:213-244): one persistent launch in which every ant
// runs `count` constructions with immediate updates, while k_weights passes rebuild the
// candidate weights from the live colony on a second stream until it finishes.
static paco_status iterate_async(paco_handle* h, uint64_t count) {
    if (count == 0) return PACO_OK;
    if (count > 0xffffffffull) return fail(PACO_E_INVALID, "too many iterations for one call");
    const bool seeding = h->iter == 0;
    k_gkey_from_gbest<<<1, 1, 0, h->st>>>(h->gb, h->gkey);
    CU(cudaGetLastError());
    paco_status s = launch_weights(h, h->st, h->gkey);
    if (s != PACO_OK) return s;
    cudaEvent_t e0 = ev(h, 0), e1 = ev(h, 1);
    CU(cudaEventRecord(e0, h->st));
    s = launch_construct_async(h, construct_args(h, seeding), (uint32_t)count);
    if (s != PACO_OK) return s;
    CU(cudaEventRecord(e1, h->st));
    uint64_t passes = 0;
    for (;;) {
        const cudaError_t q = cudaEventQuery(e1);
        if (q == cudaSuccess) break;
        if (q != cudaErrorNotReady) return fail(PACO_E_CUDA, cudaGetErrorString(q));
        const auto p0 = std::chrono::steady_clock::now();
        s = launch_weights(h, h->st2, h->gkey);
        if (s != PACO_OK) return s;
        CU(cudaStreamSynchronize(h->st2));
        ++passes;
        // Passes start at most every kWeightPassIntervalUs: a pass takes ~0.5 ms at C5, and
        // back-to-back passes took SM time from the constructions (C5 async 2.55e9 -> 2.64e9
        // decisions/s with 2 ms; profiles/README.md). Staleness stays about one interval.
        while (std::chrono::steady_clock::now() - p0 < std::chrono::microseconds(kWeightPassIntervalUs)) {
            if (cudaEventQuery(e1) != cudaErrorNotReady) break;
        }
    }
    k_gbest_from_gkey<<<1, 1, 0, h->st>>>(h->gkey, h->gb, h->g_len);
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(h->st));
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, e0, e1));
    h->construct_ms = ms;
    h->update_ms = 0.0;  // the updates run inside the construction kernel
    h->weight_passes += passes;
    h->iter += count;
    if (h->cfg.validate_tours) return check_err(h);
    return PACO_OK;
}

static paco_status check_err(paco_handle* h) {
    int err = 0;
    CU(cudaMemcpyAsync(&err, h->err, sizeof(int), cudaMemcpyDeviceToHost, h->st));
    CU(cudaStreamSynchronize(h->st));
    if (err) return fail(PACO_E_INVALID, "candidate tour is not a permutation");
    return PACO_OK;
}

paco_status paco_iterate(paco_handle* h, uint64_t count) {
    if (!h) return fail(PACO_E_INVALID, "null handle");
    CU(cudaSetDevice(h->dev));
    if (h->cfg.draws == PACO_DRAWS_BUFFER && count > 1)
        return fail(PACO_E_INVALID, "buffer draws feed one iteration per paco_set_draws call");
    if (h->async_mode) {
        if (h->cfg.draws == PACO_DRAWS_BUFFER)
            return fail(PACO_E_INVALID, "validation (buffer) draws need synchronous iterations");
        return iterate_async(h, count);
    }
    const uint32_t n = h->n, m = h->m;
    // Per-iteration timing from a bounded ring of events: every kTimedRing iterations the
    // stream is synchronized and the elapsed times folded, so a long call (the reference's
    // default is 100000 iterations) never holds more than 4 x kTimedRing events.
    constexpr size_t kTimedRing = 64;
    std::vector<std::pair<size_t, size_t>> marks;
    size_t e = 0;
    double c_ms = 0, u_ms = 0;
    auto fold = [&]() -> paco_status {
        if (marks.empty()) return PACO_OK;
        CU(cudaEventSynchronize(ev(h, marks.back().second)));
        for (auto& mk : marks) {
            float a = 0, b = 0, c = 0;
            CU(cudaEventElapsedTime(&a, ev(h, mk.first), ev(h, mk.first + 1)));
            CU(cudaEventElapsedTime(&b, ev(h, mk.first + 1), ev(h, mk.first + 2)));
            CU(cudaEventElapsedTime(&c, ev(h, mk.first + 2), ev(h, mk.second)));
            c_ms += b; u_ms += a + c;
        }
        marks.clear();
        e = 0;
        return PACO_OK;
    };
    for (uint64_t it = 0; it < count; ++it) {
        if (marks.size() == kTimedRing) {
            paco_status sf = fold();
            if (sf != PACO_OK) return sf;
        }
        if (h->cfg.draws == PACO_DRAWS_BUFFER && !h->words_ready)
            return fail(PACO_E_INVALID, "no draw buffer set for this iteration");
        const bool seeding = h->mode != PACO_MODE_CLASSIC && h->iter == 0;
        const size_t e0 = e++, e1 = e++, e2 = e++;
        CU(cudaEventRecord(ev(h, e0), h->st));
        paco_status s = h->ir ? launch_ratios(h) : launch_weights(h);
        if (s != PACO_OK) return s;
        CU(cudaEventRecord(ev(h, e1), h->st));
        if (h->ir) {
            s = launch_construct_ir(h, seeding);
        } else {
            ConstructArgs ca = construct_args(h, seeding);
            uint32_t blocks = m;
            if (h->order && !seeding && h->mode == PACO_MODE_PARTIAL) {  // longest ants first (k_ant_order)
                // Persistent CTAs: with more than kQueueSlots ants per SM, only kQueueSlots CTAs per
                // SM are launched and each takes the next-longest ant when its own is done. The
                // chain of a decision slows by ~4 ns per co-resident warp and by ~13 ns when two
                // warps share a scheduler (profiles/README.md); five resident warps instead of
                // seven-decaying-to-one measured best (C5 47.42 -> 46.86 ms; 4: 47.2 and uneven,
                // 6: 47.09, 3: 60.6).
                constexpr uint32_t kQueueSlots = 5;
                uint32_t qstart = m >= (kQueueSlots + 1) * (uint32_t)h->num_sms ? kQueueSlots * (uint32_t)h->num_sms : 0;
#ifdef PACO_NO_QUEUE
                qstart = 0;
#endif
#ifdef PACO_QUEUE_ENV
                if (const char* e = getenv("PACO_SLOTS")) qstart = std::min<uint32_t>(m, (uint32_t)atoi(e) * (uint32_t)h->num_sms);
#endif
                k_ant_order<<<1, 1024, 0, h->st>>>(ca.words, ca.stride, h->cfg.seed, h->iter, n, m, ca.eff_pp, ca.mmf,
                                                   0, h->order, qstart ? h->qhead : nullptr, qstart);
                CU(cudaGetLastError());
                ca.order = h->order;
                if (qstart) { ca.qhead = h->qhead; blocks = qstart; }
                // the superblock-start table rides in the shared memory five CTAs per SM leave free
                if (qstart) {
                    const size_t sbw = (size_t)(h->g.ncells >> 6) + 1;
                    const size_t per_cta = construct_dyn_smem(h->nwords, ca.sbe_words) + sbw * 4 + 1024 + 256;
                    if (sbw <= 3072 && per_cta * kQueueSlots <= 227 * 1024) ca.sb_words = (uint32_t)sbw;
                }
            }
#ifndef PACO_NO_DEFER_LEN
            // tour lengths in one grid-wide kernel after the constructions instead of one warp's
            // pass at the tail of the longest ant (C5 construction 49.85 -> 48.55 ms, C4 22.10 ->
            // 21.43; at n = 1000 the extra launch costs more than the pass)
            ca.defer_len = n >= 4096 ? 1 : 0;
#endif
            s = launch_construct(h, ca, blocks);
            if (s == PACO_OK && ca.defer_len) {  // new_len[a] += the length of ant a's new tour
                k_lengths<<<dim3((n + kLenPos - 1) / kLenPos, m), 256, 0, h->st>>>(h->tours, h->lb_sel, h->xy, n, h->new_len);
                CU(cudaGetLastError());
            }
        }
        if (s != PACO_OK) return s;
        if (h->two_opt_flag && h->two_opt_use_cluster) {  // maybe_two_opt's searches, a cluster per tour
            cudaLaunchConfig_t lc = {};
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = h->two_opt_cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            lc.gridDim = dim3(h->two_opt_cs * h->two_opt_clusters); lc.blockDim = dim3(512);
            lc.dynamicSmemBytes = (size_t)h->two_opt_stage * (sizeof(double2) + sizeof(int32_t) + sizeof(uint32_t));
            lc.stream = h->st; lc.attrs = at; lc.numAttrs = 1;
            CU(cudaLaunchKernelEx(&lc, k_two_opt_cluster, h->tours, (const uint8_t*)h->lb_sel, h->two_opt_flag,
                                  h->new_len, n, m, h->cfg.two_opt_window, (const double2*)h->xy, h->two_opt_edges,
                                  h->two_opt_txy, h->counters + 10, h->two_opt_stage));
        } else if (h->two_opt_flag) {  // maybe_two_opt's searches, one CTA per flagged tour (k_two_opt)
            k_two_opt<<<h->two_opt_ctas, 512, 0, h->st>>>(h->tours, h->lb_sel, h->two_opt_flag, h->new_len, n, m,
                                                          h->cfg.two_opt_window, h->xy, h->two_opt_edges,
                                                          h->two_opt_txy, h->counters + 10);
            CU(cudaGetLastError());
        }
        CU(cudaEventRecord(ev(h, e2), h->st));
        if (h->ir && h->mode == PACO_MODE_CLASSIC) {
            // full-matrix evaporate + deposit (construction.hpp:187-207), engine.hpp:253-259
            dim3 grid((n + 255) / 256, m);
            k_publish<<<grid, 256, 0, h->st>>>(h->tours, h->lb_sel, h->improved, n, 1, h->cur_nbr);
            k_classic_full<<<(n + 127) / 128, 128, 0, h->st>>>(h->cur_nbr, h->new_len, n, m, h->cfg.rho, h->Tfull);
            CU(cudaGetLastError());
        } else if (h->mode == PACO_MODE_CLASSIC) {
            // evaporate + deposit on the built tours before the l_best updates (engine.hpp:253-259)
            dim3 grid((n + 255) / 256, m);
            k_publish<<<grid, 256, 0, h->st>>>(h->tours, h->lb_sel, h->improved, n, 1, h->cur_nbr);
            const int km = kmax_for(h->k);
            const uint32_t nb = (n + 255) / 256;
            if (km == 8) k_classic<8><<<nb, 256, 0, h->st>>>(h->knn, h->cur_nbr, h->new_len, n, m, (int)h->k, h->cfg.rho, h->T);
            else if (km == 16) k_classic<16><<<nb, 256, 0, h->st>>>(h->knn, h->cur_nbr, h->new_len, n, m, (int)h->k, h->cfg.rho, h->T);
            else if (km == 24) k_classic<24><<<nb, 256, 0, h->st>>>(h->knn, h->cur_nbr, h->new_len, n, m, (int)h->k, h->cfg.rho, h->T);
            else k_classic<32><<<nb, 256, 0, h->st>>>(h->knn, h->cur_nbr, h->new_len, n, m, (int)h->k, h->cfg.rho, h->T);
            CU(cudaGetLastError());
        }
        k_update<<<1, std::min<uint32_t>(1024, (m + 31) & ~31u), 0, h->st>>>(0, m, h->new_len, h->lb_len, h->has_lb, h->lb_sel, h->improved, h->gb,
                                      h->g_len, h->counters);
        dim3 grid((n + 255) / 256, m);
        k_publish<<<grid, 256, 0, h->st>>>(h->tours, h->lb_sel, h->improved, n, 0, h->nbr);
        CU(cudaGetLastError());
        const size_t e3 = e++;
        CU(cudaEventRecord(ev(h, e3), h->st));
        marks.push_back({e0, e3});
        ++h->iter;
        h->words_ready = false;
        if (h->cfg.validate_tours) {
            paco_status s2 = check_err(h);
            if (s2 != PACO_OK) return s2;
        }
    }
    CU(cudaStreamSynchronize(h->st));
    paco_status sf = fold();
    if (sf != PACO_OK) return sf;
    h->construct_ms = c_ms; h->update_ms = u_ms;
    return PACO_OK;
}

paco_status paco_set_draws(paco_handle* h, const uint32_t* words, uint64_t stride) {
    if (!h || !words) return fail(PACO_E_INVALID, "null argument");
    if (h->cfg.draws != PACO_DRAWS_BUFFER) return fail(PACO_E_INVALID, "handle was not created with buffer draws");
    if (stride < 4ull + h->n) return fail(PACO_E_INVALID, "stride must be >= n + 4 words");
    CU(cudaSetDevice(h->dev));
    const uint64_t need = stride * h->m;
    if (need > h->words_cap) {
        if (h->words) dfree(h->words);
        h->words = nullptr;
        CU(dalloc(&h->words, need));
        h->words_cap = need;
    }
    CU(cudaMemcpyAsync(h->words, words, sizeof(uint32_t) * need, cudaMemcpyHostToDevice, h->st));
    CU(cudaStreamSynchronize(h->st));
    h->words_stride = stride;
    h->words_ready = true;
    return PACO_OK;
}

// Tours of every ant in original ids: a gather kernel picks each ant's half and maps the
// ids on the device, then one copy per chunk of ants (at most 256 MB of staging).
static paco_status read_half(paco_handle* h, bool lbest, uint32_t* tours, int64_t* lengths) {
    const uint32_t n = h->n, m = h->m;
    CU(cudaSetDevice(h->dev));
    if (tours) {
        const uint32_t chunk = (uint32_t)std::max<size_t>(1, std::min<size_t>(m, (size_t)(64u << 20) / n));
        uint32_t* stage = nullptr;
        CU(dalloc(&stage, (size_t)chunk * n));
        paco_status s = PACO_OK;
        for (uint32_t a0 = 0; a0 < m && s == PACO_OK; a0 += chunk) {
            const uint32_t c = std::min(chunk, m - a0);
            k_gather_tours<<<dim3((n + 255) / 256, c), 256, 0, h->st>>>(h->tours, h->lb_sel, h->improved, h->orig_of,
                                                                        n, a0, lbest ? 1 : 0, stage);
            cudaError_t e = cudaGetLastError();
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(tours + (size_t)a0 * n, stage, sizeof(uint32_t) * n * c, cudaMemcpyDeviceToHost,
                                    h->st);
            if (e == cudaSuccess) e = cudaStreamSynchronize(h->st);
            if (e != cudaSuccess) s = fail(PACO_E_CUDA, std::string("tour readback: ") + cudaGetErrorString(e));
        }
        cudaStreamSynchronize(h->st);
        dfree(stage);
        if (s != PACO_OK) return s;
    }
    if (lengths) {
        CU(cudaMemcpyAsync(lengths, lbest ? h->lb_len : h->new_len, sizeof(int64_t) * m, cudaMemcpyDeviceToHost, h->st));
        CU(cudaStreamSynchronize(h->st));
    }
    return PACO_OK;
}

paco_status paco_get_tours(paco_handle* h, uint32_t* tours, int64_t* lengths) {
    if (!h) return fail(PACO_E_INVALID, "null handle");
    return read_half(h, false, tours, lengths);
}

paco_status paco_get_l_best(paco_handle* h, uint32_t* tours, int64_t* lengths) {
    if (!h) return fail(PACO_E_INVALID, "null handle");
    return read_half(h, true, tours, lengths);
}

paco_status paco_get_g_best(paco_handle* h, uint32_t* tour, int64_t* length) {
    if (!h) return fail(PACO_E_INVALID, "null handle");
    CU(cudaSetDevice(h->dev));
    GBest g{};
    CU(cudaMemcpyAsync(&g, h->gb, sizeof g, cudaMemcpyDeviceToHost, h->st));
    CU(cudaStreamSynchronize(h->st));
    if (!g.has) { if (length) *length = -1; return PACO_OK; }
    if (length) *length = g.len;
    if (tour) {  // g_best is the holder ant's l_best (strict-improvement invariant)
        uint32_t* stage = nullptr;
        CU(dalloc(&stage, h->n));
        k_gather_tours<<<dim3((h->n + 255) / 256, 1), 256, 0, h->st>>>(h->tours, h->lb_sel, h->improved, h->orig_of,
                                                                       h->n, (uint32_t)g.ant, 1, stage);
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(tour, stage, sizeof(uint32_t) * h->n, cudaMemcpyDeviceToHost, h->st);
        cudaStreamSynchronize(h->st);
        dfree(stage);
        if (e != cudaSuccess) return fail(PACO_E_CUDA, std::string("g_best readback: ") + cudaGetErrorString(e));
    }
    return PACO_OK;
}

paco_status paco_get_counters(paco_handle* h, paco_counters* c) {
    if (!h || !c) return fail(PACO_E_INVALID, "null argument");
    CU(cudaSetDevice(h->dev));
    unsigned long long v[16];
    CU(cudaMemcpyAsync(v, h->counters, sizeof v, cudaMemcpyDeviceToHost, h->st));
    CU(cudaStreamSynchronize(h->st));
    c->decisions = v[0]; c->fallbacks = v[1]; c->ties = v[2]; c->forced = v[3];
    c->full_builds = v[4]; c->partial_builds = v[5]; c->iterations = h->iter; c->improvements = v[7];
    c->comparisons = h->ir ? v[8] : v[0];
    c->two_opts = v[9];
    c->two_opt_moves = v[10];
    return PACO_OK;
}

paco_status paco_get_build_flags(paco_handle* h, uint8_t* partial, uint8_t* improved) {
    if (!h) return fail(PACO_E_INVALID, "null handle");
    CU(cudaSetDevice(h->dev));
    if (partial) CU(cudaMemcpyAsync(partial, h->partial, h->m, cudaMemcpyDeviceToHost, h->st));
    if (improved) CU(cudaMemcpyAsync(improved, h->improved, h->m, cudaMemcpyDeviceToHost, h->st));
    CU(cudaStreamSynchronize(h->st));
    return PACO_OK;
}

paco_status paco_get_candidates(paco_handle* h, uint32_t* knn, float* weights, uint32_t* k_out) {
    if (!h) return fail(PACO_E_INVALID, "null handle");
    if (h->ir) return fail(PACO_E_UNSUPPORTED, "the reference rule has no candidate lists");
    CU(cudaSetDevice(h->dev));
    const uint32_t n = h->n, k = h->k;
    if (k_out) *k_out = k;
    std::vector<uint2> c((size_t)n * h->kp);
    std::vector<uint32_t> kn((size_t)n * kNearRow);
    CU(cudaMemcpyAsync(kn.data(), h->knn, sizeof(uint32_t) * kn.size(), cudaMemcpyDeviceToHost, h->st));
    CU(cudaMemcpyAsync(c.data(), h->cand, sizeof(uint2) * c.size(), cudaMemcpyDeviceToHost, h->st));
    CU(cudaStreamSynchronize(h->st));
    for (uint32_t o = 0; o < n; ++o) {
        const uint32_t i = h->h_int[o];
        for (uint32_t r = 0; r < k; ++r) {
            if (knn) knn[(size_t)o * k + r] = h->h_orig[kn[(size_t)i * kNearRow + r]];
            if (weights) std::memcpy(&weights[(size_t)o * k + r], &c[(size_t)i * h->kp + r].y, 4);
        }
    }
    return PACO_OK;
}

#ifdef PACO_2OPT_PROF
extern "C" void paco_debug_2opt(unsigned long long* out) { cudaMemcpyFromSymbol(out, g_2opt_prof, sizeof(unsigned long long) * 8); }
#endif
#ifdef PACO_DEBUG_SYMS
#ifdef PACO_ANTPROF
extern "C" void paco_debug_ant(unsigned long long* out) { cudaMemcpyFromSymbol(out, g_ant, sizeof(unsigned long long) * 4096 * 6); }
#endif
extern "C" void paco_debug_prof(unsigned long long* out) { cudaMemcpyFromSymbol(out, g_prof, sizeof(unsigned long long) * 96); }
extern "C" void paco_debug_timing(unsigned long long* out, int reset) {
    cudaMemcpyFromSymbol(out, g_timing, sizeof(unsigned long long) * 16);
    if (reset) { unsigned long long z[16] = {0}; cudaMemcpyToSymbol(g_timing, z, sizeof z); }
}
#endif

paco_status paco_get_timing(paco_handle* h, double* c, double* u, double* s) {
    if (!h) return fail(PACO_E_INVALID, "null handle");
    if (c) *c = h->construct_ms;
    if (u) *u = h->update_ms;
    if (s) *s = h->setup_ms;
    return PACO_OK;
}

static int64_t host_length(const paco_handle* h, const uint32_t* order) {
    auto d = [&](uint32_t a, uint32_t b) {
        const double dx = h->hx[a] - h->hx[b], dy = h->hy[a] - h->hy[b];
        return (int64_t)(int32_t)(std::sqrt(dx * dx + dy * dy) + 0.5);
    };
    int64_t t = 0;
    for (uint32_t i = 0; i + 1 < h->n; ++i) t += d(order[i], order[i + 1]);
    return t + d(order[h->n - 1], order[0]);
}

paco_status paco_offer_tour(paco_handle* h, uint32_t ant, const uint32_t* order, int* improved) {
    if (!h || !order) return fail(PACO_E_INVALID, "null argument");
    if (ant >= h->m) return fail(PACO_E_INVALID, "ant out of range");
    const uint32_t n = h->n;
    std::vector<uint8_t> seen(n, 0);
    for (uint32_t i = 0; i < n; ++i) {  // colony.hpp:118-119
        if (order[i] >= n || seen[order[i]]) return fail(PACO_E_INVALID, "candidate tour is not a permutation");
        seen[order[i]] = 1;
    }
    CU(cudaSetDevice(h->dev));
    std::vector<uint32_t> in(n);
    for (uint32_t i = 0; i < n; ++i) in[i] = h->h_int[order[i]];
    // every transfer is ordered on the handle's stream (pageable copies may return before
    // their DMA lands) and `in` / `L` outlive them (synchronize below)
    uint8_t sel = 0;
    CU(cudaMemcpyAsync(&sel, h->lb_sel + ant, 1, cudaMemcpyDeviceToHost, h->st));
    CU(cudaStreamSynchronize(h->st));
    CU(cudaMemcpyAsync(h->tours + ((size_t)ant * 2 + (1 - sel)) * n, in.data(), sizeof(uint32_t) * n,
                       cudaMemcpyHostToDevice, h->st));
    const int64_t L = host_length(h, order);
    CU(cudaMemcpyAsync(h->new_len + ant, &L, sizeof L, cudaMemcpyHostToDevice, h->st));
    k_update<<<1, 32, 0, h->st>>>(ant, 1, h->new_len, h->lb_len, h->has_lb, h->lb_sel, h->improved, h->gb,
                                  h->g_len, h->counters);
    // publish only this ant's slice (grid.y = 1 at ant offset `ant`)
    k_publish<<<dim3((n + 255) / 256, 1), 256, 0, h->st>>>(h->tours, h->lb_sel, h->improved, n, 0, h->nbr, ant);
    CU(cudaGetLastError());
    uint8_t imp = 0;
    CU(cudaMemcpyAsync(&imp, h->improved + ant, 1, cudaMemcpyDeviceToHost, h->st));
    CU(cudaStreamSynchronize(h->st));
    if (improved) *improved = imp;
    return PACO_OK;
}

paco_status paco_construct_at(paco_handle* h, uint32_t ant, uint32_t start_pos, uint32_t m_mod,
                              const uint32_t* words, uint64_t nwords, uint32_t* out_order, int64_t* out_length) {
    if (!h || !words || !out_order) return fail(PACO_E_INVALID, "null argument");
    if (ant >= h->m) return fail(PACO_E_INVALID, "ant out of range");
    const uint32_t n = h->n;
    if (m_mod > n) return fail(PACO_E_INVALID, "m_mod exceeds city count");  // construction.hpp:318
    if (start_pos >= n) return fail(PACO_E_INVALID, "start_pos out of range");
    if (nwords < 4ull + n) return fail(PACO_E_INVALID, "need n + 4 draw words");
    if (h->ir) return fail(PACO_E_UNSUPPORTED, "construct_at is defined for the candidate-list rule");
    CU(cudaSetDevice(h->dev));
    uint8_t has = 0;
    CU(cudaMemcpyAsync(&has, h->has_lb + ant, 1, cudaMemcpyDeviceToHost, h->st));
    CU(cudaStreamSynchronize(h->st));
    if (!has) return fail(PACO_E_INVALID, "ant has no l_best");
    uint32_t* dw = nullptr;
    CU(dalloc(&dw, nwords));
    CU(cudaMemcpyAsync(dw, words, sizeof(uint32_t) * nwords, cudaMemcpyHostToDevice, h->st));
    paco_status s = launch_weights(h);
    if (s != PACO_OK) { dfree(dw); return s; }
    ConstructArgs a = construct_args(h, false);
    a.words = dw; a.stride = nwords; a.force = 1; a.force_ant = ant; a.force_start_pos = start_pos;
    a.force_m_mod = m_mod; a.validate = 1;
    int64_t saved_len = 0;
    CU(cudaMemcpyAsync(&saved_len, h->new_len + ant, sizeof saved_len, cudaMemcpyDeviceToHost, h->st));
    CU(cudaStreamSynchronize(h->st));
    CU(cudaMemsetAsync(h->err, 0, sizeof(int), h->st));
    s = launch_construct(h, a, 1);
    if (s != PACO_OK) { dfree(dw); return s; }
    CU(cudaStreamSynchronize(h->st));
    dfree(dw);
    s = check_err(h);
    if (s != PACO_OK) return s;
    uint8_t sel = 0;
    CU(cudaMemcpyAsync(&sel, h->lb_sel + ant, 1, cudaMemcpyDeviceToHost, h->st));
    CU(cudaStreamSynchronize(h->st));
    std::vector<uint32_t> buf(n);
    CU(cudaMemcpyAsync(buf.data(), h->tours + ((size_t)ant * 2 + (1 - sel)) * n, sizeof(uint32_t) * n,
                       cudaMemcpyDeviceToHost, h->st));
    CU(cudaMemcpyAsync(out_length, h->new_len + ant, sizeof(int64_t), cudaMemcpyDeviceToHost, h->st));
    CU(cudaMemcpyAsync(h->new_len + ant, &saved_len, sizeof saved_len, cudaMemcpyHostToDevice, h->st));
    CU(cudaStreamSynchronize(h->st));  // saved_len outlives its copy
    for (uint32_t p = 0; p < n; ++p) out_order[p] = h->h_orig[buf[p]];
    return PACO_OK;
}

paco_status paco_run_traced(const double* xs, const double* ys, uint32_t n, const paco_config* cfg, int mode,
                            int64_t optimum, paco_report* rep, uint32_t* best_tour, paco_sample* samples,
                            uint32_t cap, uint32_t* n_samples) {
    if (!rep) return fail(PACO_E_INVALID, "null report");
    if (cfg && cfg->draws == PACO_DRAWS_BUFFER) return fail(PACO_E_INVALID, "paco_run uses Philox draws");
    if (n_samples) *n_samples = 0;
    const auto t0 = std::chrono::steady_clock::now();
    auto since = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
    paco_handle* h = nullptr;
    paco_status s = paco_create(xs, ys, n, cfg, mode, &h);
    if (s != PACO_OK) return s;
    double c_ms = 0, u_ms = 0;
    uint64_t done = 0;
    // Convergence monitor (engine.hpp:186-205): a sample of (elapsed, g_best, iterations)
    // each time another convergence_interval_s of wall time has passed, taken between
    // chunks of iterations sized from the measured iteration time. Synchronous results do
    // not depend on the chunking; the last slot is kept for the final sample.
    const double interval = cfg->convergence_interval_s;
    const bool sampling = interval > 0.0 && samples && cap > 1;
    uint32_t ns = 0;
    double next_t = interval;
    const bool budgeted = cfg->time_budget_s > 0.0;
    uint64_t chunk = (sampling || budgeted) ? 1 : cfg->iterations;
    while (done < cfg->iterations && s == PACO_OK) {
        const uint64_t c = std::min<uint64_t>(chunk, cfg->iterations - done);
        s = paco_iterate(h, c);
        c_ms += h->construct_ms; u_ms += h->update_ms;
        done += c;
        const double t = since();
        if (s == PACO_OK && sampling && t >= next_t && ns + 1 < cap) {
            GBest g{};
            if (cudaMemcpyAsync(&g, h->gb, sizeof g, cudaMemcpyDeviceToHost, h->st) == cudaSuccess &&
                cudaStreamSynchronize(h->st) == cudaSuccess && g.has)
                samples[ns++] = paco_sample{t, g.len, done};
            while (next_t <= t) next_t += interval;
        }
        if (budgeted && t >= cfg->time_budget_s) break;  // engine.hpp:270-272: the in-flight iteration completes
        if (sampling && !budgeted) {
            const double per_iter = t / (double)done;
            chunk = (uint64_t)std::max(1.0, std::floor((next_t - t) / std::max(per_iter, 1e-9)));
        }
    }
    if (s == PACO_OK && n_samples) *n_samples = ns;
    if (s != PACO_OK) { paco_destroy(h); return s; }
    std::vector<uint32_t> tour(n);
    int64_t len = 0;
    s = paco_get_g_best(h, tour.data(), &len);
    if (s == PACO_OK) s = paco_get_counters(h, &rep->counters);
    if (s == PACO_OK && host_length(h, tour.data()) != len)  // check_tour, engine.hpp:322
        s = fail(PACO_E_LOGIC, "tour length cache does not match recomputation");
    rep->setup_ms = h->setup_ms;
    paco_destroy(h);
    if (s != PACO_OK) return s;
    rep->best_length = len;
    rep->pct_error = optimum > 0 ? 100.0 * ((double)len - (double)optimum) / (double)optimum
                                 : std::numeric_limits<double>::quiet_NaN();
    rep->iterations_done = done;
    rep->comparisons_total = rep->counters.comparisons;
    rep->construct_ms = c_ms; rep->update_ms = u_ms;
    if (best_tour) std::memcpy(best_tour, tour.data(), sizeof(uint32_t) * n);
    rep->wall_time_s = since();
    if (samples && cap > 0 && n_samples) {  // engine.hpp:327: the final sample
        samples[ns] = paco_sample{rep->wall_time_s, len, done};
        *n_samples = ns + 1;
    }
    return PACO_OK;
}

paco_status paco_run(const double* xs, const double* ys, uint32_t n, const paco_config* cfg, int mode,
                     int64_t optimum, paco_report* rep, uint32_t* best_tour) {
    return paco_run_traced(xs, ys, n, cfg, mode, optimum, rep, best_tour, nullptr, 0, nullptr);
}

} // extern "C"
