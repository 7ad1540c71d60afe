/*
 * O2 -- CPU restatement of the north-star construction rule. TEST INFRASTRUCTURE:
 * see o2.h for the contract and the reference lines each piece follows.
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off; never -ffast-math).
 */
#include "o2.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];
const char* o2_last_error(void) { return g_err; }
#define FAIL(...) do { snprintf(g_err, sizeof g_err, __VA_ARGS__); return -1; } while (0)

/* ---------------------------------------------------------------- primitives */

/* Philox4x32-10 (Salmon et al., SC'11), the published round function. */
void o2_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        c0 = hi1 ^ c1 ^ k0; c1 = lo1; c2 = hi0 ^ c3 ^ k1; c3 = lo0;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Draw slot layout: slot 0 coin, 1 start / start_pos, 2 m_mod,
 * 3 two-opt, 4+t roulette draw of decision t. Counter = (slot/4, ant, iter lo, iter hi). */
uint32_t o2_draw_word(uint64_t seed, uint32_t ant, uint64_t iter, uint32_t slot) {
    const uint32_t ctr[4] = {slot >> 2, ant, (uint32_t)iter, (uint32_t)(iter >> 32)};
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t o[4];
    o2_philox4x32_10(ctr, key, o);
    return o[slot & 3];
}

static inline uint32_t below(uint32_t w, uint32_t bound) {
    return (uint32_t)(((uint64_t)w * bound) >> 32);
}
static inline double u01_f64(uint32_t w) { return (double)w * 0x1.0p-32; }
static inline float u01_f32(uint32_t w) { return (float)(w >> 8) * 0x1.0p-24f; }

/* instance.hpp:33-37 */
int32_t o2_euc2d(double x1, double y1, double x2, double y2) {
    const double dx = x1 - x2, dy = y1 - y2;
    return (int32_t)(sqrt(dx * dx + dy * dy) + 0.5);
}

/* construction.hpp:19-44 */
double o2_power(double e, double x) {
    const double r = round(e);
    if (!(r == e && r >= 0.0 && r <= 64.0)) return pow(x, e);
    double result = 1.0, base = x;
    for (unsigned ie = (unsigned)r; ie != 0; ie >>= 1) {
        if (ie & 1) result *= base;
        base *= base;
    }
    return result;
}

/* instance.hpp:120-127 */
int64_t o2_cycle_length(const double* xs, const double* ys, uint32_t n, const uint32_t* o) {
    int64_t t = 0;
    for (uint32_t i = 0; i + 1 < n; ++i) t += o2_euc2d(xs[o[i]], ys[o[i]], xs[o[i + 1]], ys[o[i + 1]]);
    t += o2_euc2d(xs[o[n - 1]], ys[o[n - 1]], xs[o[0]], ys[o[0]]);
    return t;
}

static inline double d2_of(const double* xs, const double* ys, uint32_t i, uint32_t j) {
    const double dx = xs[i] - xs[j], dy = ys[i] - ys[j];
    return dx * dx + dy * dy;
}

/* two_opt_scan (two_opt.hpp:28-51): first improving reversal in lexicographic (i, j)
 * order, window bounds j - i on the linear order; returns the length delta (0 = none). */
static int64_t two_opt_scan(const double* xs, const double* ys, uint32_t n, uint32_t* o, uint32_t window) {
#define D(p, q) ((int64_t)o2_euc2d(xs[p], ys[p], xs[q], ys[q]))
    for (uint32_t i = 0; i + 1 < n; ++i) {
        const uint32_t a = o[i], b = o[i + 1];
        const int64_t d_ab = D(a, b);
        const uint32_t j_end = window == 0 ? n - 1 : (n - 1 < i + window ? n - 1 : i + window);
        for (uint32_t j = i + 1; j <= j_end; ++j) {
            if (i == 0 && j == n - 1) continue;
            const uint32_t c = o[j], d = o[(j + 1) % n];
            const int64_t before = d_ab + D(c, d), after = D(a, c) + D(b, d);
            if (after < before) {
                for (uint32_t l = i + 1, r = j; l < r; ++l, --r) { const uint32_t t = o[l]; o[l] = o[r]; o[r] = t; }
                return after - before;
            }
        }
    }
    return 0;
#undef D
}

/* two_opt (two_opt.hpp:58-67): restart the scan after every accepted move */
int64_t o2_two_opt(const double* xs, const double* ys, uint32_t n, uint32_t* order, uint32_t window) {
    int64_t total = 0;
    for (;;) {
        const int64_t d = two_opt_scan(xs, ys, n, order, window);
        if (d == 0) break;
        total += d;
    }
    return total;
}

/* top-k by (d^2, index) -- brute force over all j != i */
static void knn_row(const double* xs, const double* ys, uint32_t n, uint32_t k, uint32_t i,
                    uint32_t* out, double* kd) {
    uint32_t cnt = 0;
    for (uint32_t j = 0; j < n; ++j) {
        if (j == i) continue;
        const double d = d2_of(xs, ys, i, j);
        if (cnt == k && !(d < kd[k - 1])) continue; /* equal d: larger j loses */
        uint32_t p = cnt < k ? cnt++ : k - 1;
        while (p > 0 && (d < kd[p - 1])) { kd[p] = kd[p - 1]; out[p] = out[p - 1]; --p; }
        kd[p] = d; out[p] = j;
    }
}

void o2_knn_brute(const double* xs, const double* ys, uint32_t n, uint32_t k, uint32_t* out) {
    double* kd = (double*)malloc(sizeof(double) * (k ? k : 1));
    for (uint32_t i = 0; i < n; ++i) knn_row(xs, ys, n, k, i, out + (size_t)i * k, kd);
    free(kd);
}

void o2_knn_rows(const double* xs, const double* ys, uint32_t n, uint32_t k,
                 const uint32_t* rows, uint32_t nrows, uint32_t* out) {
    double* kd = (double*)malloc(sizeof(double) * (k ? k : 1));
    for (uint32_t r = 0; r < nrows; ++r) knn_row(xs, ys, n, k, rows[r], out + (size_t)r * k, kd);
    free(kd);
}

/* Roulette over one candidate list, as one warp computes it: lane l holds w[l]
 * (0 for lanes >= k), five Hillis-Steele steps v[l] += v[l-off] in f32, total
 * S = v[k-1], target = u*S, pick = lowest feasible lane with v > target, else the last
 * lane with w > 0. Returns -1 when S == 0 (every candidate visited). */
int32_t o2_roulette(const float* w, uint32_t k, uint32_t word, int32_t* tie) {
    float v[32], nv[32];
    for (uint32_t l = 0; l < 32; ++l) v[l] = l < k ? w[l] : 0.0f;
    for (uint32_t off = 1; off < 32; off <<= 1) {
        for (uint32_t l = 0; l < 32; ++l) nv[l] = l >= off ? v[l] + v[l - off] : v[l];
        memcpy(v, nv, sizeof v);
    }
    const float S = v[k - 1];
    *tie = 0;
    if (!(S > 0.0f)) return -1;
    const float target = u01_f32(word) * S;
    const float tol = 1e-6f * S;
    for (uint32_t l = 0; l < k; ++l)
        if (fabsf(v[l] - target) <= tol) { *tie = 1; break; }
    /* feasible lanes only: the tree-shaped f32 scan is not monotone, so an
       infeasible lane (w = 0) can carry S_r one ulp above S_{r-1} */
    for (uint32_t l = 0; l < k; ++l)
        if (w[l] > 0.0f && v[l] > target) return (int32_t)l;
    for (int32_t l = (int32_t)k - 1; l >= 0; --l)
        if (w[l] > 0.0f) return l;
    return -1;
}

/* ---------------------------------------------------------------- engine */

struct o2_state {
    o2_params p;
    uint32_t n, m, k;
    double *xs, *ys;
    uint32_t* knn;  /* n*k original ids */
    float* eta;     /* n*k eta^beta (f32) */
    float* W;       /* n*k weights for the current iteration */
    double* T;      /* classic: n*k pheromone on candidate edges */
    uint32_t* lbest; int64_t* lbest_len; uint8_t* has_lbest;
    uint32_t* nbr;  /* m*n*2 (prev, next) of each ant's l_best */
    uint32_t* tours; int64_t* lens; uint8_t* partial_flag; uint8_t* improved;
    uint32_t* gbest; int64_t g_len; int has_g;
    uint64_t iter;
    o2_counters cnt;
    /* grid for the exact fallback */
    double gx0, gy0, cs;
    int32_t gw, gh;
    uint32_t *cell_start, *cell_items, *cell_of;
};

static void set_err_ok(void) { g_err[0] = 0; }

static void build_grid(o2_state* s) {
    const uint32_t n = s->n;
    double x0 = s->xs[0], x1 = x0, y0 = s->ys[0], y1 = y0;
    for (uint32_t i = 1; i < n; ++i) {
        if (s->xs[i] < x0) x0 = s->xs[i];
        if (s->xs[i] > x1) x1 = s->xs[i];
        if (s->ys[i] < y0) y0 = s->ys[i];
        if (s->ys[i] > y1) y1 = s->ys[i];
    }
    double w = x1 - x0, h = y1 - y0;
    if (w <= 0) w = 1; if (h <= 0) h = 1;
    double cs = sqrt(w * h * 2.0 / n);
    if (cs <= 0) cs = 1;
    int32_t gw = (int32_t)(w / cs) + 1, gh = (int32_t)(h / cs) + 1;
    while ((int64_t)gw * gh > 4LL * n + 16) { cs *= 1.5; gw = (int32_t)(w / cs) + 1; gh = (int32_t)(h / cs) + 1; }
    s->gx0 = x0; s->gy0 = y0; s->cs = cs; s->gw = gw; s->gh = gh;
    const size_t nc = (size_t)gw * gh;
    s->cell_start = (uint32_t*)calloc(nc + 1, sizeof(uint32_t));
    s->cell_items = (uint32_t*)malloc(sizeof(uint32_t) * n);
    s->cell_of = (uint32_t*)malloc(sizeof(uint32_t) * n);
    for (uint32_t i = 0; i < n; ++i) {
        int32_t cx = (int32_t)floor((s->xs[i] - x0) / cs), cy = (int32_t)floor((s->ys[i] - y0) / cs);
        if (cx < 0) cx = 0; if (cx >= gw) cx = gw - 1;
        if (cy < 0) cy = 0; if (cy >= gh) cy = gh - 1;
        s->cell_of[i] = (uint32_t)cy * gw + cx;
        s->cell_start[s->cell_of[i] + 1]++;
    }
    for (size_t c = 0; c < nc; ++c) s->cell_start[c + 1] += s->cell_start[c];
    uint32_t* fill = (uint32_t*)malloc(sizeof(uint32_t) * nc);
    memcpy(fill, s->cell_start, sizeof(uint32_t) * nc);
    for (uint32_t i = 0; i < n; ++i) s->cell_items[fill[s->cell_of[i]]++] = i; /* ascending ids */
    free(fill);
}

static inline void consider(const o2_state* s, uint32_t cur, uint32_t j, const uint8_t* vis,
                            double* bd, uint32_t* bj) {
    if (vis[j]) return;
    const double d = d2_of(s->xs, s->ys, cur, j);
    if (d < *bd || (d == *bd && j < *bj)) { *bd = d; *bj = j; }
}

/* exact argmin over unvisited j of (d^2(cur, j), j) */
static uint32_t nearest_unvisited(const o2_state* s, uint32_t cur, const uint8_t* vis) {
    double bd = INFINITY;
    uint32_t bj = UINT32_MAX;
    if (s->p.fallback_brute) {
        for (uint32_t j = 0; j < s->n; ++j) consider(s, cur, j, vis, &bd, &bj);
        return bj;
    }
    const int32_t cx = (int32_t)(s->cell_of[cur] % (uint32_t)s->gw);
    const int32_t cy = (int32_t)(s->cell_of[cur] / (uint32_t)s->gw);
    const int32_t rmax = s->gw > s->gh ? s->gw : s->gh;
    for (int32_t rho = 0; rho <= rmax; ++rho) {
        if (rho >= 1) {
            const double lb = ((double)rho - 1.0 - 1e-6) * s->cs;
            if (lb > 0 && lb * lb > bd) break;
        }
        for (int32_t y = cy - rho; y <= cy + rho; ++y) {
            if (y < 0 || y >= s->gh) continue;
            const int32_t step = (y == cy - rho || y == cy + rho) ? 1 : 2 * rho;
            for (int32_t x = cx - rho; x <= cx + rho; x += (step ? step : 1)) {
                if (x >= 0 && x < s->gw) {
                    const uint32_t c = (uint32_t)y * s->gw + x;
                    for (uint32_t q = s->cell_start[c]; q < s->cell_start[c + 1]; ++q)
                        consider(s, cur, s->cell_items[q], vis, &bd, &bj);
                }
                if (rho == 0) break;
            }
        }
    }
    return bj;
}

typedef struct scratch { uint8_t* vis; } scratch;

static inline uint32_t word_of(const o2_state* s, uint32_t ant, uint32_t slot,
                               const uint32_t* words, uint64_t stride, int* err) {
    if (s->p.draw_source == 1) {
        if (slot >= stride) { *err = 1; return 0; }
        return words[(uint64_t)ant * stride + slot];
    }
    return o2_draw_word(s->p.seed, ant, s->iter, slot);
}

/* Places the remaining unvisited cities after order[0..pos-1]; decision t uses slot 4+t.
 * construction.hpp:283-304 / 312-350 with the north-star selection rule. */
static int complete_tour(const o2_state* s, uint32_t ant, uint32_t* order, uint32_t pos,
                         uint8_t* vis, const uint32_t* words, uint64_t stride,
                         o2_counters* c) {
    const uint32_t n = s->n, k = s->k;
    uint32_t cur = order[pos - 1];
    uint32_t remaining = n - pos;
    float w[32];
    int err = 0;
    for (uint32_t t = 0; remaining > 0; ++t, --remaining) {
        uint32_t next;
        c->decisions++;
        if (remaining == 1) {
            /* final city is forced, no score evaluated (construction.hpp:342-348) */
            next = UINT32_MAX;
            for (uint32_t j = 0; j < n; ++j) if (!vis[j]) { next = j; break; }
            c->forced++;
        } else {
            const uint32_t* row = s->knn + (size_t)cur * k;
            const float* wr = s->W + (size_t)cur * k;
            for (uint32_t r = 0; r < k; ++r) w[r] = vis[row[r]] ? 0.0f : wr[r];
            const uint32_t uw = word_of(s, ant, 4 + t, words, stride, &err);
            if (err) return -1;
            int32_t tie = 0;
            const int32_t lane = o2_roulette(w, k, uw, &tie);
            c->ties += (uint64_t)tie;
            if (lane < 0) { next = nearest_unvisited(s, cur, vis); c->fallbacks++; }
            else next = row[lane];
        }
        vis[next] = 1;
        order[pos++] = next;
        cur = next;
    }
    return 0;
}

static int build_one(o2_state* s, uint32_t ant, int seeding, const uint32_t* words,
                     uint64_t stride, uint8_t* vis, o2_counters* c) {
    const uint32_t n = s->n;
    uint32_t* order = s->tours + (size_t)ant * n;
    memset(vis, 0, n);
    int err = 0;
    const double eff_pp = (s->p.mode == 0) ? s->p.partial_prob : 0.0;
    int partial = 0;
    if (!seeding) {
        const double coin = u01_f64(word_of(s, ant, 0, words, stride, &err)); /* engine.hpp:137 */
        partial = coin < eff_pp;
    }
    uint32_t pos = 0;
    if (!partial) {
        const uint32_t start = below(word_of(s, ant, 1, words, stride, &err), n);
        order[pos++] = start; vis[start] = 1;
        c->full_builds++;
    } else {
        /* construction.hpp:354-365 */
        const uint32_t start_pos = below(word_of(s, ant, 1, words, stride, &err), n);
        double capd = floor(s->p.max_mod_frac * (double)n);
        if (capd < 2.0) capd = 2.0;
        const uint32_t cap = (uint32_t)capd;
        const uint32_t m_mod = 2 + below(word_of(s, ant, 2, words, stride, &err), cap - 1);
        const uint32_t* lb = s->lbest + (size_t)ant * n;
        const uint32_t preserved = n - m_mod;
        for (uint32_t t = 0; t < preserved; ++t) {
            const uint32_t city = lb[(start_pos + t) % n];
            order[pos++] = city; vis[city] = 1;
        }
        if (preserved == 0) { order[pos++] = lb[start_pos]; vis[lb[start_pos]] = 1; }
        c->partial_builds++;
    }
    if (err) return -1;
    s->partial_flag[ant] = (uint8_t)partial;
    if (complete_tour(s, ant, order, pos, vis, words, stride, c)) return -1;
    /* maybe_two_opt (two_opt.hpp:71-76): draw slot 3 */
    const double u2 = u01_f64(word_of(s, ant, 3, words, stride, &err));
    if (err) return -1;
    if (u2 < s->p.two_opt_prob) { o2_two_opt(s->xs, s->ys, n, order, s->p.two_opt_window); c->two_opts++; }
    s->lens[ant] = o2_cycle_length(s->xs, s->ys, n, order);
    return 0;
}

/* -------- weights: tau on candidate edges, frozen colony (construction.hpp:119-132) */

static void weights_rows(o2_state* s, uint32_t i0, uint32_t i1, const double* ratios) {
    const uint32_t n = s->n, k = s->k, m = s->m;
    double acc[32];
    for (uint32_t i = i0; i < i1; ++i) {
        const uint32_t* row = s->knn + (size_t)i * k;
        if (s->p.mode == 2) {
            for (uint32_t r = 0; r < k; ++r) {
                const double ta = o2_power(s->p.alpha, s->T[(size_t)i * k + r]);
                s->W[(size_t)i * k + r] = (float)ta * s->eta[(size_t)i * k + r];
            }
            continue;
        }
        for (uint32_t r = 0; r < k; ++r) acc[r] = 0.0;
        for (uint32_t a = 0; a < m; ++a) {
            const double ra = ratios[a];
            if (ra == 0.0) continue;
            const uint32_t pa = s->nbr[((size_t)a * n + i) * 2], pb = s->nbr[((size_t)a * n + i) * 2 + 1];
            for (uint32_t r = 0; r < k; ++r) {
                if (row[r] == pa) acc[r] += ra;
                if (row[r] == pb) acc[r] += ra;
            }
        }
        for (uint32_t r = 0; r < k; ++r) {
            const double ta = o2_power(s->p.alpha, s->p.tau0 + acc[r]);
            s->W[(size_t)i * k + r] = (float)ta * s->eta[(size_t)i * k + r];
        }
    }
}

/* --------- tiny parallel-for over [0, total) */
typedef struct job {
    o2_state* s; int kind; uint32_t lo, hi; const double* ratios;
    int seeding; const uint32_t* words; uint64_t stride; int rc; o2_counters c;
} job;

static void* run_job(void* arg) {
    job* j = (job*)arg;
    if (j->kind == 0) { weights_rows(j->s, j->lo, j->hi, j->ratios); return NULL; }
    uint8_t* vis = (uint8_t*)malloc(j->s->n);
    for (uint32_t a = j->lo; a < j->hi && j->rc == 0; ++a)
        j->rc = build_one(j->s, a, j->seeding, j->words, j->stride, vis, &j->c);
    free(vis);
    return NULL;
}

static int par_for(o2_state* s, int kind, uint32_t total, const double* ratios, int seeding,
                   const uint32_t* words, uint64_t stride) {
    uint32_t T = s->p.threads ? s->p.threads : 1;
    if (T > total) T = total ? total : 1;
    job* jobs = (job*)calloc(T, sizeof(job));
    pthread_t* th = (pthread_t*)calloc(T, sizeof(pthread_t));
    for (uint32_t t = 0; t < T; ++t) {
        jobs[t] = (job){s, kind, (uint32_t)((uint64_t)total * t / T), (uint32_t)((uint64_t)total * (t + 1) / T),
                        ratios, seeding, words, stride, 0, {0}};
        if (T > 1) pthread_create(&th[t], NULL, run_job, &jobs[t]); else run_job(&jobs[t]);
    }
    int rc = 0;
    for (uint32_t t = 0; t < T; ++t) {
        if (T > 1) pthread_join(th[t], NULL);
        rc |= jobs[t].rc;
        s->cnt.decisions += jobs[t].c.decisions; s->cnt.fallbacks += jobs[t].c.fallbacks;
        s->cnt.ties += jobs[t].c.ties; s->cnt.forced += jobs[t].c.forced;
        s->cnt.full_builds += jobs[t].c.full_builds; s->cnt.partial_builds += jobs[t].c.partial_builds;
        s->cnt.two_opts += jobs[t].c.two_opts;
    }
    free(jobs); free(th);
    return rc;
}

static void compute_weights(o2_state* s) {
    double* ratios = (double*)calloc(s->m, sizeof(double));
    const double g = (double)s->g_len; /* colony.hpp:159-167 */
    for (uint32_t a = 0; a < s->m; ++a)
        if (s->has_lbest[a]) { const double r = g / (double)s->lbest_len[a]; ratios[a] = r > 1.0 ? 1.0 : r; }
    par_for(s, 0, s->n, ratios, 0, NULL, 0);
    free(ratios);
}

static void publish(o2_state* s, uint32_t a) { /* colony.hpp:39-52 */
    const uint32_t n = s->n;
    const uint32_t* t = s->lbest + (size_t)a * n;
    for (uint32_t p = 0; p < n; ++p) {
        s->nbr[((size_t)a * n + t[p]) * 2] = t[(p + n - 1) % n];
        s->nbr[((size_t)a * n + t[p]) * 2 + 1] = t[(p + 1) % n];
    }
}

static int is_perm(uint32_t n, const uint32_t* o) {
    uint8_t* seen = (uint8_t*)calloc(n, 1);
    int ok = 1;
    for (uint32_t i = 0; i < n && ok; ++i) { if (o[i] >= n || seen[o[i]]) ok = 0; else seen[o[i]] = 1; }
    free(seen);
    return ok;
}

/* update_l_best + update_g_best, colony.hpp:115-139 */
static int offer(o2_state* s, uint32_t a, const uint32_t* order, int64_t len) {
    const uint32_t n = s->n;
    if (s->has_lbest[a] && len >= s->lbest_len[a]) return 0;
    memcpy(s->lbest + (size_t)a * n, order, sizeof(uint32_t) * n);
    s->lbest_len[a] = len; s->has_lbest[a] = 1;
    publish(s, a);
    if (!s->has_g || len < s->g_len) {
        s->g_len = len; s->has_g = 1;
        memcpy(s->gbest, order, sizeof(uint32_t) * n);
    }
    return 1;
}

int o2_offer_tour(o2_state* s, uint32_t a, const uint32_t* order) {
    if (a >= s->m) FAIL("ant out of range");
    if (!is_perm(s->n, order)) FAIL("candidate tour is not a permutation");
    return offer(s, a, order, o2_cycle_length(s->xs, s->ys, s->n, order));
}

o2_state* o2_create(const double* xs, const double* ys, const o2_params* p) {
    set_err_ok();
    if (p->n < 3) { snprintf(g_err, sizeof g_err, "instance needs at least 3 cities"); return NULL; }
    if (p->m < 1) { snprintf(g_err, sizeof g_err, "ants must be >= 1"); return NULL; }
    o2_state* s = (o2_state*)calloc(1, sizeof(o2_state));
    s->p = *p;
    s->n = p->n; s->m = p->m;
    s->k = p->k < p->n - 1 ? p->k : p->n - 1;
    if (s->k > 32) s->k = 32;
    if (s->k < 1) s->k = 1;
    const uint32_t n = s->n, m = s->m, k = s->k;
    s->xs = (double*)malloc(sizeof(double) * n); memcpy(s->xs, xs, sizeof(double) * n);
    s->ys = (double*)malloc(sizeof(double) * n); memcpy(s->ys, ys, sizeof(double) * n);
    s->knn = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n * k);
    s->eta = (float*)malloc(sizeof(float) * (size_t)n * k);
    s->W = (float*)malloc(sizeof(float) * (size_t)n * k);
    o2_knn_brute(s->xs, s->ys, n, k, s->knn);
    for (uint32_t i = 0; i < n; ++i)
        for (uint32_t r = 0; r < k; ++r) {
            const uint32_t j = s->knn[(size_t)i * k + r];
            int32_t d = o2_euc2d(xs[i], ys[i], xs[j], ys[j]);
            if (d < 1) d = 1;
            s->eta[(size_t)i * k + r] = (float)o2_power(p->beta, 1.0 / (double)d); /* construction.hpp:59 */
        }
    if (p->mode == 2) {
        s->T = (double*)malloc(sizeof(double) * (size_t)n * k);
        for (size_t q = 0; q < (size_t)n * k; ++q) s->T[q] = p->tau_max;
    }
    s->lbest = (uint32_t*)calloc((size_t)m * n, sizeof(uint32_t));
    s->lbest_len = (int64_t*)calloc(m, sizeof(int64_t));
    s->has_lbest = (uint8_t*)calloc(m, 1);
    s->nbr = (uint32_t*)calloc((size_t)m * n * 2, sizeof(uint32_t));
    s->tours = (uint32_t*)calloc((size_t)m * n, sizeof(uint32_t));
    s->lens = (int64_t*)calloc(m, sizeof(int64_t));
    s->partial_flag = (uint8_t*)calloc(m, 1);
    s->improved = (uint8_t*)calloc(m, 1);
    s->gbest = (uint32_t*)calloc(n, sizeof(uint32_t));
    s->g_len = INT64_MAX;
    build_grid(s);
    return s;
}

void o2_destroy(o2_state* s) {
    if (!s) return;
    free(s->xs); free(s->ys); free(s->knn); free(s->eta); free(s->W); free(s->T);
    free(s->lbest); free(s->lbest_len); free(s->has_lbest); free(s->nbr); free(s->tours);
    free(s->lens); free(s->partial_flag); free(s->improved); free(s->gbest);
    free(s->cell_start); free(s->cell_items); free(s->cell_of);
    free(s);
}

/* evaporate then deposit every built tour in tour order (engine.hpp:253-259,
   construction.hpp:187-207) -- restricted to candidate edges, which evolve
   independently of every other matrix entry */
static void classic_update(o2_state* s, const uint32_t* tours, const int64_t* lens, uint32_t ntours) {
    const uint32_t n = s->n, k = s->k;
    const double keep = 1.0 - s->p.rho;
    for (size_t q = 0; q < (size_t)n * k; ++q) { double t = s->T[q] * keep; if (t < 1e-6) t = 1e-6; s->T[q] = t; }
    uint32_t* pos = (uint32_t*)malloc(sizeof(uint32_t) * n);
    for (uint32_t a = 0; a < ntours; ++a) {
        const uint32_t* t = tours + (size_t)a * n;
        const double delta = 1.0 / (double)lens[a];
        for (uint32_t p = 0; p < n; ++p) pos[t[p]] = p;
        for (uint32_t i = 0; i < n; ++i) {
            const uint32_t pi = pos[i];
            const uint32_t pv = t[(pi + n - 1) % n], nx = t[(pi + 1) % n];
            for (uint32_t r = 0; r < k; ++r) {
                const uint32_t c = s->knn[(size_t)i * k + r];
                if (c == pv || c == nx) s->T[(size_t)i * k + r] += delta;
            }
        }
    }
    free(pos);
}

int o2_classic_apply(o2_state* s, const uint32_t* tours, const int64_t* lens, uint32_t ntours) {
    if (!s->T) FAIL("not a classic-mode state");
    classic_update(s, tours, lens, ntours);
    return 0;
}

int o2_iterate(o2_state* s, const uint32_t* words, uint64_t stride) {
    set_err_ok();
    if (s->p.draw_source == 1 && !words) FAIL("draw buffer required");
    const int seeding = (s->p.mode != 2) && s->iter == 0;
    compute_weights(s);
    if (par_for(s, 1, s->m, NULL, seeding, words, stride)) FAIL("draw buffer too short");
    const uint32_t n = s->n, m = s->m, k = s->k;
    if (s->p.mode == 2) classic_update(s, s->tours, s->lens, m);
    for (uint32_t a = 0; a < m; ++a) /* engine.hpp:261-265, ant order */
        s->improved[a] = (uint8_t)offer(s, a, s->tours + (size_t)a * n, s->lens[a]);
    s->iter++;
    s->cnt.iterations++;
    return 0;
}

int o2_construct_at(o2_state* s, uint32_t ant, uint32_t start_pos, uint32_t m_mod,
                    const uint32_t* words, uint64_t nwords, uint32_t* out, int64_t* len) {
    set_err_ok();
    const uint32_t n = s->n;
    if (ant >= s->m || !s->has_lbest[ant]) FAIL("ant has no l_best");
    if (m_mod > n) FAIL("m_mod exceeds city count");
    if (start_pos >= n) FAIL("start_pos out of range");
    compute_weights(s);
    uint8_t* vis = (uint8_t*)calloc(n, 1);
    const uint32_t* lb = s->lbest + (size_t)ant * n;
    const uint32_t preserved = n - m_mod;
    uint32_t pos = 0;
    for (uint32_t t = 0; t < preserved; ++t) { out[pos++] = lb[(start_pos + t) % n]; vis[out[pos - 1]] = 1; }
    if (preserved == 0) { out[pos++] = lb[start_pos]; vis[lb[start_pos]] = 1; }
    o2_counters c = {0};
    const int32_t saved = s->p.draw_source;
    s->p.draw_source = 1;
    /* words index = slot; the ant index must map to row 0 */
    int rc = 0;
    {
        /* complete_tour reads words[ant*stride + slot]; pass a shifted base */
        const uint32_t* base = words - (uint64_t)ant * nwords;
        rc = complete_tour(s, ant, out, pos, vis, base, nwords, &c);
    }
    s->p.draw_source = saved;
    free(vis);
    if (rc) FAIL("draw buffer too short");
    *len = o2_cycle_length(s->xs, s->ys, n, out);
    return 0;
}

/* tau^alpha(i, j) for every j, exactly as ColonyPheromone::begin_step + tau_alpha
 * (construction.hpp:121-134): acc summed in ant order, Power(alpha)(tau0 + acc). */
void o2_tau_row(const o2_state* s, uint32_t i, double* out) {
    const uint32_t n = s->n;
    double* acc = (double*)calloc(n, sizeof(double));
    const double g = (double)s->g_len;
    for (uint32_t a = 0; a < s->m; ++a) {
        if (!s->has_lbest[a]) continue;
        double r = g / (double)s->lbest_len[a];
        r = r > 1.0 ? 1.0 : r;
        acc[s->nbr[((size_t)a * n + i) * 2]] += r;
        acc[s->nbr[((size_t)a * n + i) * 2 + 1]] += r;
    }
    for (uint32_t j = 0; j < n; ++j) out[j] = o2_power(s->p.alpha, s->p.tau0 + acc[j]);
    free(acc);
}

void o2_get_T(const o2_state* s, double* out) {
    if (s->T) memcpy(out, s->T, sizeof(double) * (size_t)s->n * s->k);
}

void o2_get_knn(const o2_state* s, uint32_t* out) { memcpy(out, s->knn, sizeof(uint32_t) * (size_t)s->n * s->k); }
void o2_get_weights(const o2_state* s, float* out) { memcpy(out, s->W, sizeof(float) * (size_t)s->n * s->k); }
void o2_get_tours(const o2_state* s, uint32_t* t, int64_t* l) {
    memcpy(t, s->tours, sizeof(uint32_t) * (size_t)s->m * s->n);
    memcpy(l, s->lens, sizeof(int64_t) * s->m);
}
void o2_get_lbest(const o2_state* s, uint32_t* t, int64_t* l) {
    memcpy(t, s->lbest, sizeof(uint32_t) * (size_t)s->m * s->n);
    memcpy(l, s->lbest_len, sizeof(int64_t) * s->m);
}
int64_t o2_get_gbest(const o2_state* s, uint32_t* t) {
    if (t) memcpy(t, s->gbest, sizeof(uint32_t) * s->n);
    return s->has_g ? s->g_len : -1;
}
void o2_get_counters(const o2_state* s, o2_counters* c) { *c = s->cnt; }
void o2_get_build_flags(const o2_state* s, uint8_t* partial, uint8_t* improved) {
    if (partial) memcpy(partial, s->partial_flag, s->m);
    if (improved) memcpy(improved, s->improved, s->m);
}
