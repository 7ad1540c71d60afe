// Drop-in on the reference's OWN types: one translation unit includes the unmodified
// reference headers (/root/reference/proj/include) and include/paco_b200/paco.hpp, builds a
// paco::Instance with paco::parse_tsplib, and calls paco_b200::run(const paco::Instance&,
// const paco::RunConfig&, paco::Mode) -> paco::RunReport next to paco::run itself.
// With the reference's Independent Roulette rule (Options::rule) and synchronous iterations
// the GPU's report must equal the reference's: best length, best tour, comparisons.
// Usage: ref_drop_in [expect-gpu 0|1]. Exit code 0 = pass.
#include <cstdio>
#include <sstream>
#include <stdexcept>
#include <string>

#include <paco/engine.hpp>
#include <paco/instance.hpp>

#include "paco_b200/paco.hpp"

#ifndef PACO_B200_REFERENCE_TYPES
#error "the reference headers must be on the include path"
#endif

#define CHECK(c) do { if (!(c)) { std::fprintf(stderr, "CHECK failed: %s (line %d)\n", #c, __LINE__); return 1; } } while (0)

static std::string grid_tsplib(int w, int h) {  // 26 x 17 lattice, spacing 10 (data/README.md:7-10)
    std::ostringstream o;
    o << "NAME : grid" << w * h << "\nTYPE : TSP\nDIMENSION : " << w * h << "\nEDGE_WEIGHT_TYPE : EUC_2D\nNODE_COORD_SECTION\n";
    for (int r = 0, id = 1; r < h; ++r)
        for (int c = 0; c < w; ++c) o << id++ << " " << 10 * c << " " << 10 * r << "\n";
    o << "EOF\n";
    return o.str();
}

int main(int argc, char** argv) {
    const bool gpu = argc > 1 && std::string(argv[1]) == "1";
    std::istringstream in(grid_tsplib(26, 17));
    paco::Instance inst = paco::parse_tsplib(in);
    inst.set_optimum(4420);
    // the reference's own validation runs first: identical exception and message
    paco::RunConfig bad;
    bad.ants = 0;
    bool threw = false;
    try { paco_b200::run(inst, bad, paco::Mode::partial_aco); }
    catch (const std::invalid_argument& e) { threw = std::string(e.what()) == "ants must be >= 1"; }
    CHECK(threw);

    paco::RunConfig cfg;  // the reference's defaults (synchronous = false, workers = 8, ...)
    cfg.ants = 16; cfg.iterations = 30; cfg.alpha = 5.0; cfg.beta = 5.0; cfg.seed = 7;
    cfg.convergence_interval_s = 0.0;
    try {
        // 1. the reference's default (asynchronous) engine, north-star rule
        const paco::RunReport a = paco_b200::run(inst, cfg, paco::Mode::partial_aco);
        CHECK(gpu);
        CHECK(a.best_length >= 4420 && a.best_tour.order.size() == 442);
        CHECK(paco::tour_length(inst, a.best_tour.order) == a.best_length);
        CHECK(a.pct_error && *a.pct_error >= 0.0 && a.iterations_done == 30);
        // 2. synchronous, the reference's own rule: bit-identical to paco::run in this process
        paco::RunConfig s = cfg;
        s.synchronous = true;
        paco_b200::Options ir;
        ir.rule = PACO_RULE_INDEPENDENT_ROULETTE;
        const paco::RunReport g = paco_b200::run(inst, s, paco::Mode::partial_aco, ir);
        const paco::RunReport r = paco::run(inst, s, paco::Mode::partial_aco);
        CHECK(g.best_length == r.best_length);
        CHECK(g.best_tour.order == r.best_tour.order);
        CHECK(g.comparisons_total == r.comparisons_total);
        CHECK(g.iterations_done == r.iterations_done);
        CHECK(g.pct_error && r.pct_error && *g.pct_error == *r.pct_error);
        // 3. run_timed_baseline: P-ACO full constructions until the budget expires
        const paco::RunReport t = paco_b200::run_timed_baseline(inst, cfg, 0.05);
        CHECK(t.iterations_done >= 1 && paco::tour_length(inst, t.best_tour.order) == t.best_length);
        std::printf("ref_drop_in ok: async best %lld, sync IR best %lld == paco::run %lld, comparisons %llu\n",
                    (long long)a.best_length, (long long)g.best_length, (long long)r.best_length,
                    (unsigned long long)g.comparisons_total);
    } catch (const std::invalid_argument& e) {
        std::fprintf(stderr, "unexpected invalid_argument: %s\n", e.what());
        return 1;
    } catch (const std::runtime_error& e) {
        if (gpu) { std::fprintf(stderr, "unexpected: %s\n", e.what()); return 1; }
        std::printf("no GPU: %s\n", e.what());  // the engine has no CPU fallback
    }
    // classic mode keeps the reference's size limit and message (engine.hpp:158-160)
    std::vector<std::pair<double, double>> big;
    for (int i = 0; i < 5001; ++i) big.emplace_back(i % 100, i / 100);
    threw = false;
    try { paco_b200::run(paco::Instance("big", big), cfg, paco::Mode::classic_aco); }
    catch (const std::invalid_argument& e) { threw = std::string(e.what()) == "classic mode requires n <= 5000"; }
    catch (const std::runtime_error&) { threw = !gpu; }  // without a GPU the device check may come first
    CHECK(threw);
    return 0;
}
