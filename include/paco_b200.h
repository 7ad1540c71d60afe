/*
 * paco_b200 -- C ABI of the B200 tour-construction engine (drop-in boundary).
 *
 * The reference's public solver entry point is
 *     RunReport paco::run(const Instance&, const RunConfig&, Mode)
 *     (/root/reference/proj/include/paco/engine.hpp:156)
 * with RunConfig at engine.hpp:42-76, RunReport at engine.hpp:84-92 and Mode at
 * engine.hpp:24. Its per-candidate plugin seam (PheromoneSource,
 * construction.hpp:236-241) is too fine-grained to cross a C ABI, so this
 * library replaces whole iterations per call. Synchronous (engine.hpp:245-306):
 * every ant constructs against a frozen colony on the GPU, then the completion
 * step applies l_best / g_best updates in ant order. Asynchronous
 * (engine.hpp:213-244, the reference's default): every ant runs its
 * constructions back to back and applies its own updates at once.
 *
 * Conventions: plain pointers and sizes, no C++ types; every function returns a
 * paco_status (0 = ok); paco_last_error() returns a thread-local message. The
 * caller owns host buffers; the library owns device memory. One CUDA stream per
 * handle; a handle is single-threaded, distinct handles may run concurrently.
 * City indices at this boundary are the caller's (original) indices.
 */
#ifndef PACO_B200_H
#define PACO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum paco_status {
    PACO_OK = 0,
    PACO_E_RUNTIME = -1,     /* std::runtime_error analogue */
    PACO_E_INVALID = -2,     /* std::invalid_argument analogue (RunConfig::validate, engine.hpp:61-75) */
    PACO_E_CUDA = -3,        /* CUDA failure or no usable sm_100 device */
    PACO_E_UNSUPPORTED = -4, /* valid reference option not provided by this engine */
    PACO_E_LOGIC = -5        /* std::logic_error analogue (length cache mismatch, engine.hpp:110-113) */
} paco_status;

/* Mode, engine.hpp:24 */
typedef enum paco_mode { PACO_MODE_PARTIAL = 0, PACO_MODE_PACO = 1, PACO_MODE_CLASSIC = 2 } paco_mode;

/* Draw source: counter-based Philox (production) or a caller-supplied word buffer
 * (validation mode, shared with the CPU oracle). */
typedef enum paco_draws { PACO_DRAWS_PHILOX = 0, PACO_DRAWS_BUFFER = 1 } paco_draws;

/* Selection rule. CANDIDATE_ROULETTE is the north-star rule (k-NN candidate list,
 * roulette wheel, exact nearest-unvisited fallback; Philox or buffer draws).
 * INDEPENDENT_ROULETTE is the reference's own rule (construction.hpp:243-281) with
 * the reference's xoshiro256++ streams (rng.hpp:24-74): a run is bit-identical to
 * paco::run in synchronous mode. It scans every unvisited city per decision and is
 * provided for parity, not speed. */
typedef enum paco_rule { PACO_RULE_CANDIDATE_ROULETTE = 0, PACO_RULE_INDEPENDENT_ROULETTE = 1 } paco_rule;

/* RunConfig, engine.hpp:42-76, field for field, plus the north-star additions at the end. */
typedef struct paco_config {
    uint32_t ants;                 /* m */
    uint32_t workers;              /* accepted for API parity; the GPU ignores it */
    uint64_t iterations;
    double alpha, beta;
    double partial_prob;           /* engine.hpp:47 */
    double max_mod_frac;           /* engine.hpp:48 */
    double two_opt_prob;           /* engine.hpp:49, first-improvement 2-opt after construction */
    uint32_t two_opt_window;       /* engine.hpp:50, 0 = unbounded (two_opt.hpp:33-35) */
    uint32_t synchronous;          /* engine.hpp:57; 0 = asynchronous (not with the reference rule) */
    uint64_t seed;
    double rho, tau_max, tau0;
    double time_budget_s;          /* 0 = run all iterations (engine.hpp:56) */
    double convergence_interval_s; /* host-side sampling between iterations */
    uint32_t validate_tours;       /* device permutation check + host length re-check */
    /* north-star additions */
    uint32_t candidates;           /* k of the k-NN candidate list, 1..32 (clamped to n-1) */
    uint32_t draws;                /* paco_draws */
    int32_t device;                /* CUDA device ordinal, -1 = current */
    uint32_t rule;                 /* paco_rule */
} paco_config;

typedef struct paco_counters {
    uint64_t decisions;      /* cities placed by the selection rule (incl. forced last city) */
    uint64_t fallbacks;      /* decisions where every candidate was visited */
    uint64_t ties;           /* roulette boundary ties |S_r - u*S| <= 1e-6*S (logged, not resolved) */
    uint64_t forced;         /* single-candidate appends (construction.hpp:342-348) */
    uint64_t full_builds;
    uint64_t partial_builds;
    uint64_t iterations;
    uint64_t improvements;   /* successful update_l_best calls */
    uint64_t comparisons;    /* candidate scores evaluated (IR rule: the reference's comparison count) */
    uint64_t two_opts;       /* constructions that ran 2-opt (maybe_two_opt, two_opt.hpp:71-76) */
    uint64_t two_opt_moves;  /* accepted 2-opt moves (synchronous engine) */
} paco_counters;

/* RunReport, engine.hpp:84-92 (+ counters and device-time breakdown) */
typedef struct paco_report {
    int64_t best_length;
    double pct_error;          /* NaN when no optimum was supplied */
    double wall_time_s;
    uint64_t iterations_done;
    uint64_t comparisons_total;/* IR rule: the reference's count; candidate rule: decisions */
    paco_counters counters;
    double construct_ms;       /* device time in the construction kernel (CUDA events) */
    double update_ms;          /* weights + completion-step kernels */
    double setup_ms;           /* grid + k-NN build */
} paco_report;

/* ConvergenceSample (engine.hpp:79-83) */
typedef struct paco_sample {
    double elapsed_s;
    int64_t g_best_length;
    uint64_t iterations_done;
} paco_sample;

typedef struct paco_handle paco_handle;

const char* paco_last_error(void);
int paco_version(void);
/* Device memory of destroyed handles stays cached in the device's stream-ordered pool for
 * the next handle; this returns it to the driver (device < 0: the current device). */
paco_status paco_release_cached_memory(int device);
/* Advance a xoshiro256++ state (rng.hpp:40-50; the reference's per-ant stream, Rng::for_stream)
 * by `steps` draws with a jump polynomial (x^steps mod the transition's characteristic
 * polynomial) - the jump the reference-rule generator's lanes use. Host-only arithmetic, no
 * device; fails if the characteristic polynomial cannot be found. */
paco_status paco_rng_jump(const uint64_t state_in[4], uint64_t steps, uint64_t state_out[4]);

/* defaults of RunConfig (engine.hpp:42-59) except synchronous = 1 (deterministic per
 * seed; the reference defaults to asynchronous), plus candidates = 16 */
paco_status paco_config_default(paco_config* cfg);
/* RunConfig::validate (engine.hpp:61-75) + classic n <= 5000 (engine.hpp:158-160) */
paco_status paco_config_validate(const paco_config* cfg, uint32_t n, int mode);

/* Instance + colony on the device. xs/ys: n coordinates (Instance, instance.hpp:41-71). */
paco_status paco_create(const double* xs, const double* ys, uint32_t n, const paco_config* cfg,
                        int mode, paco_handle** out);
void paco_destroy(paco_handle* h);

/* `count` iterations; the first iteration of a P-ACO run seeds every l_best with a
 * full construction (engine.hpp:290-292). Asynchronous handles run them as one
 * barrier-free launch in which each ant makes `count` constructions. */
paco_status paco_iterate(paco_handle* h, uint64_t count);

/* Validation mode: words for the NEXT iteration, m rows of `stride` u32 words
 * (row = ant; slot layout in DESIGN.md §3.4). */
paco_status paco_set_draws(paco_handle* h, const uint32_t* words, uint64_t stride);

/* Readbacks (original city indices). tours: m*n, lengths: m. */
paco_status paco_get_tours(paco_handle* h, uint32_t* tours, int64_t* lengths);
paco_status paco_get_l_best(paco_handle* h, uint32_t* tours, int64_t* lengths);
paco_status paco_get_g_best(paco_handle* h, uint32_t* tour, int64_t* length);
paco_status paco_get_counters(paco_handle* h, paco_counters* c);
paco_status paco_get_build_flags(paco_handle* h, uint8_t* partial, uint8_t* improved);
/* k-NN candidate lists (n*k, original indices) and the current weight table (n*k f32) */
paco_status paco_get_candidates(paco_handle* h, uint32_t* knn, float* weights, uint32_t* k_out);
/* device time of the last paco_iterate call, per kernel family (ms) */
paco_status paco_get_timing(paco_handle* h, double* construct_ms, double* update_ms, double* setup_ms);

/* update_l_best + update_g_best for one ant (colony.hpp:115-139). improved may be NULL. */
paco_status paco_offer_tour(paco_handle* h, uint32_t ant, const uint32_t* order, int* improved);
/* construct_partial_at (construction.hpp:312-350) for one ant with explicit start_pos and
 * m_mod (0..n) against the current colony; words[slot] supplies draws (slot 4+t for decision t). */
paco_status paco_construct_at(paco_handle* h, uint32_t ant, uint32_t start_pos, uint32_t m_mod,
                              const uint32_t* words, uint64_t nwords, uint32_t* out_order,
                              int64_t* out_length);

/* paco::run (engine.hpp:156-333): create, iterate to cfg->iterations or the time budget,
 * read g_best back, destroy. best_tour may be NULL; optimum <= 0 means none. */
paco_status paco_run(const double* xs, const double* ys, uint32_t n, const paco_config* cfg,
                     int mode, int64_t optimum, paco_report* report, uint32_t* best_tour);

/* paco_run plus RunReport::convergence (engine.hpp:186-205, 327): a sample each time
 * another cfg->convergence_interval_s of wall time has passed (taken between chunks of
 * iterations), then the final sample. At most `cap` samples, the final one always kept;
 * *n_samples receives the count. */
paco_status paco_run_traced(const double* xs, const double* ys, uint32_t n, const paco_config* cfg,
                            int mode, int64_t optimum, paco_report* report, uint32_t* best_tour,
                            paco_sample* samples, uint32_t cap, uint32_t* n_samples);

#ifdef __cplusplus
}
#endif
#endif /* PACO_B200_H */
