// Drop-in check: the reference's calling convention (Instance, RunConfig, Mode -> RunReport)
// against the B200 engine through include/paco_b200/paco.hpp. Exit code 0 = pass.
// Usage: drop_in [expect-gpu 0|1]
#include <cstdio>
#include <cstdlib>
#include <sstream>
#include <stdexcept>
#include <string>

#include "paco_b200/paco.hpp"

#define CHECK(c) do { if (!(c)) { std::fprintf(stderr, "CHECK failed: %s (line %d)\n", #c, __LINE__); return 1; } } while (0)

int main(int argc, char** argv) {
    const bool gpu = argc > 1 && std::string(argv[1]) == "1";
    // config validation mirrors RunConfig::validate (engine.hpp:61-75)
    paco_b200::RunConfig bad;
    bad.ants = 0;
    bool threw = false;
    try { bad.validate(); } catch (const std::invalid_argument& e) { threw = std::string(e.what()) == "ants must be >= 1"; }
    CHECK(threw);
    CHECK(paco_b200::mode_from_name("partial") == paco_b200::Mode::partial_aco);
    CHECK(!paco_b200::RunConfig{}.synchronous);  // engine.hpp:58 default: the asynchronous engine
    // parse_tsplib / parse_tsplib_file (instance.hpp:164-249): rules and messages
    {
        std::istringstream ok("NAME : tri\nTYPE : TSP\nDIMENSION : 3\nEDGE_WEIGHT_TYPE : EUC_2D\n"
                              "NODE_COORD_SECTION\n1 0 0\n2 3 0\n3 3 4\nEOF\n");
        const auto tri = paco_b200::parse_tsplib(ok);
        CHECK(tri.name() == "tri" && tri.n() == 3 && tri.dist(0, 2) == 5);
        std::istringstream geo("NAME : x\nDIMENSION : 3\nEDGE_WEIGHT_TYPE : GEO\n");
        threw = false;
        try { paco_b200::parse_tsplib(geo); }
        catch (const paco_b200::ParseError& e) { threw = std::string(e.what()) == "line 3: unsupported EDGE_WEIGHT_TYPE: 'GEO' (only EUC_2D)"; }
        CHECK(threw);
        std::istringstream shortf("DIMENSION : 4\nEDGE_WEIGHT_TYPE : EUC_2D\nNODE_COORD_SECTION\n1 0 0\n2 1 1\n3 2 2\nEOF\n");
        threw = false;
        try { paco_b200::parse_tsplib(shortf); }
        catch (const paco_b200::ParseError& e) { threw = std::string(e.what()) == "line 7: DIMENSION is 4 but 3 coordinate lines were read"; }
        CHECK(threw);
        threw = false;
        try { paco_b200::parse_tsplib_file("/nonexistent/x.tsp"); }
        catch (const std::runtime_error& e) { threw = std::string(e.what()) == "cannot open instance file: /nonexistent/x.tsp"; }
        CHECK(threw);
    }

    // grid442 (26 x 17 lattice, spacing 10, optimum 4420)
    std::vector<std::pair<double, double>> pts;
    for (int r = 0; r < 17; ++r) for (int c = 0; c < 26; ++c) pts.emplace_back(10.0 * c, 10.0 * r);
    paco_b200::Instance inst("grid442", pts, 4420);
    paco_b200::RunConfig cfg;
    cfg.ants = 16; cfg.iterations = 50; cfg.alpha = 1.0; cfg.beta = 2.0; cfg.candidates = 12; cfg.seed = 3;
    cfg.synchronous = true;
    try {
        const auto rep = paco_b200::run(inst, cfg, paco_b200::Mode::partial_aco);
        CHECK(gpu);
        CHECK(rep.best_length >= 4420);
        CHECK(rep.best_tour.order.size() == 442);
        std::vector<int> seen(442, 0);
        for (auto c : rep.best_tour.order) { CHECK(c < 442); CHECK(!seen[c]); seen[c] = 1; }
        std::int64_t len = 0;
        for (size_t i = 0; i < 442; ++i) len += inst.dist(rep.best_tour.order[i], rep.best_tour.order[(i + 1) % 442]);
        CHECK(len == rep.best_length);
        CHECK(rep.pct_error && *rep.pct_error >= 0.0);
        CHECK(rep.iterations_done == 50);
        std::printf("drop_in ok: best %lld (%.2f%% over optimum) decisions %llu wall %.3fs\n",
                    (long long)rep.best_length, *rep.pct_error, (unsigned long long)rep.counters.decisions,
                    rep.wall_time_s);
        // the reference's default engine: asynchronous (engine.hpp:213-244)
        paco_b200::RunConfig acfg = cfg;
        acfg.synchronous = false;
        const auto arep = paco_b200::run(inst, acfg, paco_b200::Mode::partial_aco);
        CHECK(arep.best_length >= 4420 && arep.best_tour.order.size() == 442);
        std::int64_t alen = 0;
        for (size_t i = 0; i < 442; ++i) alen += inst.dist(arep.best_tour.order[i], arep.best_tour.order[(i + 1) % 442]);
        CHECK(alen == arep.best_length);
        CHECK(arep.iterations_done == 50);
        std::printf("drop_in async ok: best %lld\n", (long long)arep.best_length);
        // classic mode refuses n > 5000 with the reference's message (engine.hpp:158-160)
        std::vector<std::pair<double, double>> big;
        for (int i = 0; i < 5001; ++i) big.emplace_back(i % 100, i / 100);
        threw = false;
        try { paco_b200::run(paco_b200::Instance("big", big), cfg, paco_b200::Mode::classic_aco); }
        catch (const std::invalid_argument& e) { threw = std::string(e.what()).find("n <= 5000") != std::string::npos; }
        CHECK(threw);
        paco_b200::release_cached_memory();  // hand the pooled device memory back
    } catch (const std::runtime_error& e) {
        if (gpu) { std::fprintf(stderr, "unexpected: %s\n", e.what()); return 1; }
        std::printf("no GPU: %s\n", e.what());  // the engine has no CPU fallback
    }
    return 0;
}
