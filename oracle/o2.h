/*
 * O2 -- CPU restatement of the north-star construction rule (TEST INFRASTRUCTURE).
 *
 * This library is the checker for the B200 engine. Only tests/, the smoke()
 * entry point and bench.py's cpu_baseline leg may load it; the product path in
 * paper_1709_03187_b200/ never links or calls anything under oracle/.
 *
 * What it restates (reference paths relative to /root/reference):
 *   - EUC_2D distance and cycle length        proj/include/paco/instance.hpp:33-37, 120-127
 *   - Power (repeated squaring)                proj/include/paco/construction.hpp:19-44
 *   - eta^beta = Power(beta)(1/max(d,1)) -> f32 proj/include/paco/construction.hpp:46-61
 *   - tau = tau0 + sum_k min(g/l_k,1), summed  proj/include/paco/construction.hpp:121-132,
 *     in ant order, then Power(alpha)          proj/include/paco/colony.hpp:159-177
 *   - full / partial construction structure    proj/include/paco/construction.hpp:283-365
 *   - build_candidate coin + seeding           proj/include/paco/engine.hpp:129-148
 *   - sync completion step, strict l/g update  proj/include/paco/engine.hpp:245-306,
 *                                              proj/include/paco/colony.hpp:115-139
 *   - classic evaporate/deposit (edge-local)   proj/include/paco/construction.hpp:187-207
 *   - first-improvement (windowed) 2-opt       proj/include/paco/two_opt.hpp:28-76
 * North-star additions (no reference code; defined in DESIGN.md §3):
 *   - k-NN candidate lists ordered by (d^2, original index)
 *   - roulette over the list: f32 weights, 32-lane Hillis-Steele inclusive scan
 *     simulated lane by lane, pick = lowest feasible lane with S_r > u*S (ballot), clamp
 *     to last feasible lane
 *   - exact nearest-unvisited fallback, key (d^2, original index)
 *   - counter-based Philox4x32-10 draw schedule (slot layout in DESIGN.md)
 * Parity pins: tests/golden/* (generated from the unmodified reference by
 * oracle/make_golden.py through oracle/_ref) and the reference's own KATs
 * re-hosted in tests/test_oracle_*.py.
 */
#ifndef PACO_O2_H
#define PACO_O2_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct o2_params {
    uint32_t n, m, k;
    uint32_t threads;
    double alpha, beta, tau0, partial_prob, max_mod_frac, rho, tau_max;
    double two_opt_prob;     /* maybe_two_opt (two_opt.hpp:71-76), draw slot 3 */
    uint32_t two_opt_window; /* 0 = unbounded */
    uint32_t pad2_;
    uint64_t seed;
    int32_t mode;           /* 0 partial, 1 paco (always full), 2 classic */
    int32_t draw_source;    /* 0 philox, 1 caller buffer per iteration */
    int32_t fallback_brute; /* 1: O(n) brute-force fallback (cross-check of the grid search) */
    int32_t pad_;
} o2_params;

typedef struct o2_counters {
    uint64_t decisions, fallbacks, ties, forced, full_builds, partial_builds, iterations, two_opts;
} o2_counters;

typedef struct o2_state o2_state;

/* primitives */
void o2_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
uint32_t o2_draw_word(uint64_t seed, uint32_t ant, uint64_t iter, uint32_t slot);
int32_t o2_euc2d(double x1, double y1, double x2, double y2);
double o2_power(double e, double x);
int64_t o2_cycle_length(const double* xs, const double* ys, uint32_t n, const uint32_t* order);
/* first-improvement 2-opt to a local optimum (two_opt.hpp:28-67); returns the length delta */
int64_t o2_two_opt(const double* xs, const double* ys, uint32_t n, uint32_t* order, uint32_t window);
void o2_knn_brute(const double* xs, const double* ys, uint32_t n, uint32_t k, uint32_t* out);
void o2_knn_rows(const double* xs, const double* ys, uint32_t n, uint32_t k,
                 const uint32_t* rows, uint32_t nrows, uint32_t* out);
/* roulette primitive: w[k] effective weights (0 = infeasible); returns lane, -1 = fallback */
int32_t o2_roulette(const float* w, uint32_t k, uint32_t word, int32_t* tie);

/* engine */
o2_state* o2_create(const double* xs, const double* ys, const o2_params* p);
void o2_destroy(o2_state* s);
/* one synchronous iteration; words (draw_source==1) = m * stride u32 for this iteration */
int o2_iterate(o2_state* s, const uint32_t* words, uint64_t stride);
void o2_get_knn(const o2_state* s, uint32_t* out);
void o2_tau_row(const o2_state* s, uint32_t i, double* out); /* tau^alpha over all j */
void o2_get_T(const o2_state* s, double* out);               /* classic: n*k candidate-edge tau */
/* classic: one evaporate + deposit of the given tours (construction.hpp:187-207) */
int o2_classic_apply(o2_state* s, const uint32_t* tours, const int64_t* lens, uint32_t ntours);
void o2_get_weights(const o2_state* s, float* out); /* n*k weights of the last iteration */
void o2_get_tours(const o2_state* s, uint32_t* tours, int64_t* lens);
void o2_get_lbest(const o2_state* s, uint32_t* tours, int64_t* lens);
int64_t o2_get_gbest(const o2_state* s, uint32_t* tour);
void o2_get_counters(const o2_state* s, o2_counters* c);
void o2_get_build_flags(const o2_state* s, uint8_t* partial, uint8_t* improved);
/* install an l_best for ant k as update_l_best would (strict improvement + g_best) */
int o2_offer_tour(o2_state* s, uint32_t ant, const uint32_t* order);
/* explicit-parameter partial construction for ant `ant` (construct_partial_at analogue);
   words[slot] supplies the roulette draws (slot 4+t for decision t). */
int o2_construct_at(o2_state* s, uint32_t ant, uint32_t start_pos, uint32_t m_mod,
                    const uint32_t* words, uint64_t nwords, uint32_t* out, int64_t* len);
const char* o2_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
