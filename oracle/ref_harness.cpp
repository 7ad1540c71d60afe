// O1 harness -- TEST INFRASTRUCTURE. Exposes the UNMODIFIED reference library
// (header-only C++20 under /root/reference/proj/include, compiled in place by
// oracle/Makefile into oracle/_ref/libpaco_ref.so) through a small C ABI so the
// tests can pin the O2 restatement against the reference's own arithmetic and so
// bench.py can time the reference's CPU path. Nothing here re-implements the
// reference: every computation below is a call into paco::*.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "paco/colony.hpp"
#include "paco/construction.hpp"
#include "paco/engine.hpp"
#include "paco/instance.hpp"
#include "paco/rng.hpp"
#include "paco/two_opt.hpp"

namespace {
thread_local std::string g_err;

paco::Instance make_instance(const double* xs, const double* ys, uint32_t n) {
    std::vector<std::pair<double, double>> c(n);
    for (uint32_t i = 0; i < n; ++i) c[i] = {xs[i], ys[i]};
    return paco::Instance("h", std::move(c));
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return -2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}
} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int32_t ref_euc2d(double x1, double y1, double x2, double y2) {
    return paco::euc2d(x1, y1, x2, y2);
}

double ref_power(double e, double x) { return paco::Power(e)(x); }

// tour_length (instance.hpp:130-135); -2 when the order is not a permutation
int ref_tour_length(const double* xs, const double* ys, uint32_t n, const uint32_t* order,
                    uint32_t len, int64_t* out) {
    return guarded([&] {
        const auto inst = make_instance(xs, ys, n);
        *out = paco::tour_length(inst, std::span<const uint32_t>(order, len));
    });
}

// eta^beta through the reference Heuristic (table path when n <= 5000)
int ref_eta_beta(const double* xs, const double* ys, uint32_t n, double beta,
                 const uint32_t* pairs, uint32_t npairs, double* out) {
    return guarded([&] {
        const auto inst = make_instance(xs, ys, n);
        paco::Heuristic h(inst, beta);
        for (uint32_t q = 0; q < npairs; ++q) out[q] = h.eta_beta(pairs[2 * q], pairs[2 * q + 1]);
    });
}

// Install m l_best tours in ant order (update_l_best, then update_g_best when it
// improved -- engine.hpp:207-211), then read tau^alpha through ColonyPheromone
// (construction.hpp:104-158) for every (row, j). out is nrows x n. Also returns
// Colony::pheromone(row, j) (colony.hpp:145-155) in out_direct when non-null.
int ref_colony_tau(const double* xs, const double* ys, uint32_t n, uint32_t m,
                   const uint32_t* tours, double tau0, double alpha, const uint32_t* rows,
                   uint32_t nrows, double* out, double* out_direct, int64_t* g_len) {
    return guarded([&] {
        const auto inst = make_instance(xs, ys, n);
        paco::Colony colony(inst, m, tau0, 1);
        for (uint32_t a = 0; a < m; ++a) {
            std::vector<uint32_t> o(tours + size_t(a) * n, tours + size_t(a + 1) * n);
            auto& ant = colony.ant(a);
            if (colony.update_l_best(ant, paco::make_tour(inst, std::move(o))))
                colony.update_g_best(ant.l_best());
        }
        *g_len = colony.g_best_length();
        paco::ColonyPheromone ph(colony, alpha);
        ph.begin_construction();
        for (uint32_t r = 0; r < nrows; ++r) {
            ph.begin_step(rows[r]);
            for (uint32_t j = 0; j < n; ++j) out[size_t(r) * n + j] = ph.tau_alpha(j);
            ph.end_step();
            if (out_direct)
                for (uint32_t j = 0; j < n; ++j)
                    out_direct[size_t(r) * n + j] = (j == rows[r]) ? 0.0 : colony.pheromone(rows[r], j);
        }
    });
}

// Offer `count` candidate tours to ants[q] in order (the sync completion step,
// engine.hpp:261-265). flags[q] = update_l_best result; g_after[q] = g_best length.
int ref_offer_sequence(const double* xs, const double* ys, uint32_t n, uint32_t m,
                       const uint32_t* tours, const uint32_t* ants, uint32_t count,
                       uint8_t* flags, int64_t* g_after) {
    return guarded([&] {
        const auto inst = make_instance(xs, ys, n);
        paco::Colony colony(inst, m, 1.0, 1);
        for (uint32_t q = 0; q < count; ++q) {
            std::vector<uint32_t> o(tours + size_t(q) * n, tours + size_t(q + 1) * n);
            auto& ant = colony.ant(ants[q]);
            const bool imp = colony.update_l_best(ant, paco::make_tour(inst, std::move(o)));
            if (imp) colony.update_g_best(ant.l_best());
            flags[q] = imp ? 1 : 0;
            g_after[q] = colony.g_best_length();
        }
    });
}

// two_opt (two_opt.hpp:58-67) on a given order; returns the new order and length.
int ref_two_opt(const double* xs, const double* ys, uint32_t n, const uint32_t* order, uint32_t window,
                uint32_t* out, int64_t* length) {
    return guarded([&] {
        const auto inst = make_instance(xs, ys, n);
        paco::Tour t = paco::make_tour(inst, std::vector<uint32_t>(order, order + n));
        paco::TwoOptParams prm{1.0, window};
        const paco::Tour r = paco::two_opt(inst, t, prm);
        std::memcpy(out, r.order.data(), sizeof(uint32_t) * n);
        *length = r.length;
    });
}

// Rng::for_stream(seed, stream) raw u64 outputs (rng.hpp:33-50)
void ref_stream_u64(uint64_t seed, uint64_t stream, uint64_t count, uint64_t* out) {
    auto r = paco::Rng::for_stream(seed, stream);
    for (uint64_t i = 0; i < count; ++i) out[i] = r.next_u64();
}

// Classic PheromoneMatrix evaporate + deposit (construction.hpp:160-213): `rounds`
// rounds, round r evaporates then deposits tours[r][0..ntours) with lens[r][..].
int ref_classic_update(uint32_t n, double rho, double tau_init, const uint32_t* tours,
                       const int64_t* lens, uint32_t ntours, uint32_t rounds, double* out) {
    return guarded([&] {
        paco::PheromoneMatrix pm(n, rho, tau_init);
        for (uint32_t r = 0; r < rounds; ++r) {
            std::vector<paco::Tour> ts(ntours);
            for (uint32_t t = 0; t < ntours; ++t) {
                const uint32_t* src = tours + (size_t(r) * ntours + t) * n;
                ts[t].order.assign(src, src + n);
                ts[t].length = lens[size_t(r) * ntours + t];
            }
            pm.evaporate();
            pm.deposit(ts);
        }
        for (uint32_t i = 0; i < n; ++i)
            for (uint32_t j = 0; j < n; ++j) out[size_t(i) * n + j] = pm.tau(i, j);
    });
}

struct ref_run_params {
    uint32_t ants, workers;
    uint64_t iterations, seed;
    double alpha, beta, partial_prob, max_mod_frac, two_opt_prob;
    uint32_t two_opt_window, synchronous;
    double rho, tau_max, tau0, time_budget_s;
    int32_t mode; // 0 partial, 1 paco, 2 classic
    int32_t pad_;
};

// paco::run (engine.hpp:156-333), unmodified.
int ref_run(const double* xs, const double* ys, uint32_t n, const ref_run_params* p,
            int64_t* best_len, uint32_t* best_tour, uint64_t* iterations_done,
            uint64_t* comparisons, double* wall_s) {
    return guarded([&] {
        const auto inst = make_instance(xs, ys, n);
        paco::RunConfig cfg;
        cfg.ants = p->ants; cfg.iterations = p->iterations; cfg.alpha = p->alpha; cfg.beta = p->beta;
        cfg.partial_prob = p->partial_prob; cfg.max_mod_frac = p->max_mod_frac;
        cfg.two_opt_prob = p->two_opt_prob; cfg.two_opt_window = p->two_opt_window;
        cfg.workers = p->workers; cfg.seed = p->seed; cfg.rho = p->rho; cfg.tau_max = p->tau_max;
        cfg.tau0 = p->tau0; cfg.time_budget_s = p->time_budget_s; cfg.convergence_interval_s = 0.0;
        cfg.synchronous = p->synchronous != 0;
        const paco::Mode mode = p->mode == 0 ? paco::Mode::partial_aco
                                : p->mode == 1 ? paco::Mode::paco_full
                                               : paco::Mode::classic_aco;
        const auto rep = paco::run(inst, cfg, mode);
        *best_len = rep.best_length;
        if (best_tour) std::memcpy(best_tour, rep.best_tour.order.data(), sizeof(uint32_t) * n);
        *iterations_done = rep.iterations_done;
        *comparisons = rep.comparisons_total;
        *wall_s = rep.wall_time_s;
    });
}

// Bounded sample of the reference's hot loop on a given workload shape, for the
// CPU baseline: a colony of m ants with random l_best tours, then on `threads`
// threads repeatedly: draw a construction like build_candidate does
// (full with prob 1-partial_prob, else m_mod ~ U{2..cap}), draw the decision's
// position uniformly inside it (remaining candidates r ~ U{1..M}), prepare the
// scratch with that many unvisited cities and time one paco::select_next
// (construction.hpp:246-281) with the reference's ColonyPheromone and Heuristic.
// Stops after `seconds`. Returns decisions, comparisons and the summed seconds
// spent inside select_next over all threads.
int ref_sample_select(const double* xs, const double* ys, uint32_t n, uint32_t m,
                      double alpha, double beta, double partial_prob, double max_mod_frac,
                      uint64_t seed, uint32_t threads, double seconds, uint64_t* decisions,
                      uint64_t* comparisons, double* busy_s) {
    return guarded([&] {
        const auto inst = make_instance(xs, ys, n);
        paco::Colony colony(inst, m, 1.0, seed);
        {
            std::mt19937_64 gen(seed);
            std::vector<uint32_t> o(n);
            for (uint32_t i = 0; i < n; ++i) o[i] = i;
            for (uint32_t a = 0; a < m; ++a) {
                std::shuffle(o.begin(), o.end(), gen);
                auto t = paco::Tour{o, paco::cycle_length(inst, o)};
                if (colony.update_l_best(colony.ant(a), std::move(t)))
                    colony.update_g_best(colony.ant(a).l_best());
            }
        }
        paco::Heuristic heur(inst, beta);
        std::vector<uint64_t> dec(threads, 0), cmp(threads, 0);
        std::vector<double> busy(threads, 0.0);
        const auto t0 = std::chrono::steady_clock::now();
        auto worker = [&](uint32_t w) {
            std::mt19937_64 gen(seed * 7919 + w);
            paco::Rng rng = paco::Rng::for_stream(seed, w);
            paco::ConstructionScratch sc;
            paco::ColonyPheromone ph(colony, alpha);
            const uint32_t cap = std::max<uint32_t>(2, uint32_t(max_mod_frac * n));
            while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() <
                   seconds) {
                const bool full = std::uniform_real_distribution<double>(0, 1)(gen) >= partial_prob;
                const uint32_t M = full ? n - 1 : 2 + uint32_t(gen() % (cap - 1));
                const uint32_t r = 1 + uint32_t(gen() % M);
                // unvisited set: a random set of r cities (excluding `cur`)
                sc.prepare(n);
                ph.begin_construction();
                std::vector<uint32_t> perm(n);
                for (uint32_t i = 0; i < n; ++i) perm[i] = i;
                for (uint32_t i = 0; i < r + 1; ++i) std::swap(perm[i], perm[i + gen() % (n - i)]);
                const uint32_t cur = perm[r];
                for (uint32_t c = 0; c < n; ++c) sc.visited[c] = 1;
                for (uint32_t i = 0; i < r; ++i) sc.visited[perm[i]] = 0;
                for (uint32_t c = 0; c < n; ++c)
                    if (!sc.visited[c]) sc.candidates.push_back(c);
                const uint64_t before = sc.comparisons;
                const auto s0 = std::chrono::steady_clock::now();
                (void)paco::select_next(cur, sc, ph, heur, rng);
                busy[w] += std::chrono::duration<double>(std::chrono::steady_clock::now() - s0).count();
                cmp[w] += sc.comparisons - before;
                dec[w] += 1;
            }
        };
        std::vector<std::thread> th;
        for (uint32_t w = 0; w < threads; ++w) th.emplace_back(worker, w);
        for (auto& t : th) t.join();
        *decisions = 0; *comparisons = 0; *busy_s = 0;
        for (uint32_t w = 0; w < threads; ++w) {
            *decisions += dec[w]; *comparisons += cmp[w]; *busy_s += busy[w];
        }
    });
}

} // extern "C"
