// paco_b200/paco.hpp -- C++ drop-in for the reference solver interface.
//
// Two ways in:
//
// 1. On the reference's own types. When the reference headers are on the include path
//    (proj/include, so that <paco/engine.hpp> resolves), this header adds
//        paco::RunReport paco_b200::run(const paco::Instance&, const paco::RunConfig&, paco::Mode)
//        paco::RunReport paco_b200::run_timed_baseline(const paco::Instance&, paco::RunConfig, double)
//    (engine.hpp:156, 339-344), so bench.hpp:351, 402, 415 and paco_cli.cpp:32 switch to
//    the GPU by changing `paco::run` to `paco_b200::run`: same Instance (from
//    paco::parse_tsplib_file, instance.hpp:240), same RunConfig and its defaults
//    (synchronous = false: the asynchronous engine), same RunReport and exceptions.
// 2. Stand-alone look-alikes of the same types (no reference headers needed): Mode,
//    mode_name / mode_from_name (engine.hpp:24-40), RunConfig (:42-76), ConvergenceSample
//    (:78-82), RunReport (:84-92), run / run_timed_baseline, Instance / Tour
//    (instance.hpp:41-107) and parse_tsplib / parse_tsplib_file (instance.hpp:164-249).
//
// Everything below is a thin header-only layer over the C ABI in paco_b200.h
// (link with -lpaco_b200); status codes are rethrown as the reference's
// exception types (std::invalid_argument, std::logic_error, std::runtime_error).
// RunConfig::workers is validated (>= 1) and otherwise has no effect on the GPU: the
// synchronous engine's results do not depend on it (test_engine.cpp:75-95), and the
// asynchronous engine runs every ant concurrently.
#pragma once

#include <cmath>
#include <cstdint>
#include <fstream>
#include <istream>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../paco_b200.h"

namespace paco_b200 {

enum class Mode { partial_aco, paco_full, classic_aco };

inline const char* mode_name(Mode m) {
    switch (m) {
        case Mode::partial_aco: return "partial";
        case Mode::paco_full: return "paco";
        case Mode::classic_aco: return "classic";
    }
    return "?";
}

inline std::optional<Mode> mode_from_name(const std::string& s) {
    if (s == "partial") return Mode::partial_aco;
    if (s == "paco") return Mode::paco_full;
    if (s == "classic") return Mode::classic_aco;
    return std::nullopt;
}

inline void check(paco_status s) {
    if (s == PACO_OK) return;
    const std::string msg = paco_last_error();
    if (s == PACO_E_INVALID) throw std::invalid_argument(msg);
    if (s == PACO_E_LOGIC) throw std::logic_error(msg);
    throw std::runtime_error(msg);
}

// RunConfig, engine.hpp:42-76 (same fields and defaults) + the north-star knob.
struct RunConfig {
    std::uint32_t ants = 16;
    std::uint64_t iterations = 100000;
    double alpha = 5.0;
    double beta = 5.0;
    double partial_prob = 0.95;
    double max_mod_frac = 1.0;
    double two_opt_prob = 0.0;
    std::uint32_t two_opt_window = 0;
    std::uint32_t workers = 8;
    std::uint64_t seed = 1;
    double rho = 0.1;
    double tau_max = 1.0;
    double tau0 = 1.0;
    double time_budget_s = 0.0;
    double convergence_interval_s = 1.0;
    bool synchronous = false;  // engine.hpp:58: the asynchronous engine by default; true = barriered, deterministic
    bool validate_tours = false;
    std::uint32_t candidates = 16;  // k of the k-NN candidate list
    int device = -1;
    paco_rule rule = PACO_RULE_CANDIDATE_ROULETTE;  // INDEPENDENT_ROULETTE = the reference's rule, bit-exact

    paco_config to_c() const {
        paco_config c{};
        check(paco_config_default(&c));
        c.ants = ants; c.iterations = iterations; c.alpha = alpha; c.beta = beta;
        c.partial_prob = partial_prob; c.max_mod_frac = max_mod_frac; c.two_opt_prob = two_opt_prob;
        c.two_opt_window = two_opt_window; c.workers = workers; c.seed = seed; c.rho = rho;
        c.tau_max = tau_max; c.tau0 = tau0; c.time_budget_s = time_budget_s;
        c.convergence_interval_s = convergence_interval_s; c.synchronous = synchronous ? 1u : 0u;
        c.validate_tours = validate_tours ? 1u : 0u; c.candidates = candidates;
        c.draws = PACO_DRAWS_PHILOX; c.device = device; c.rule = rule;
        return c;
    }

    // RunConfig::validate (engine.hpp:61-75)
    void validate() const {
        const paco_config c = to_c();
        check(paco_config_validate(&c, 3, 0));
    }
};

struct Tour {
    std::vector<std::uint32_t> order;
    std::int64_t length = 0;
};

// Immutable city set (instance.hpp:41-101): coordinates plus EUC_2D.
class Instance {
public:
    Instance(std::string name, std::vector<std::pair<double, double>> coords,
             std::optional<std::int64_t> optimum = std::nullopt)
        : name_(std::move(name)), optimum_(optimum) {
        if (coords.size() < 3)
            throw std::invalid_argument("instance needs at least 3 cities, got " + std::to_string(coords.size()));
        if (optimum_ && *optimum_ <= 0) throw std::invalid_argument("known optimum must be positive");
        xs_.reserve(coords.size());
        ys_.reserve(coords.size());
        for (const auto& [x, y] : coords) {
            if (!std::isfinite(x) || !std::isfinite(y)) throw std::invalid_argument("non-finite coordinate");
            xs_.push_back(x);
            ys_.push_back(y);
        }
    }
    const std::string& name() const { return name_; }
    std::uint32_t n() const { return static_cast<std::uint32_t>(xs_.size()); }
    double x(std::uint32_t i) const { return xs_[i]; }
    double y(std::uint32_t i) const { return ys_[i]; }
    const double* xs() const { return xs_.data(); }
    const double* ys() const { return ys_.data(); }
    std::optional<std::int64_t> optimum() const { return optimum_; }
    std::int32_t dist(std::uint32_t i, std::uint32_t j) const {  // instance.hpp:33-37
        const double dx = xs_[i] - xs_[j], dy = ys_[i] - ys_[j];
        return static_cast<std::int32_t>(std::sqrt(dx * dx + dy * dy) + 0.5);
    }

private:
    std::string name_;
    std::vector<double> xs_, ys_;
    std::optional<std::int64_t> optimum_;
};

// TSPLIB EUC_2D reader with the reference's rules and messages (instance.hpp:164-249):
// headers until NODE_COORD_SECTION, "id x y" lines, EOF optional. Errors carry the line
// number ("line N: ..."); parse_tsplib_file prefixes the path and throws runtime_error.
struct ParseError : std::runtime_error {
    int line;
    ParseError(int line_no, const std::string& what)
        : std::runtime_error("line " + std::to_string(line_no) + ": " + what), line(line_no) {}
};

inline Instance parse_tsplib(std::istream& in) {
    auto trim = [](const std::string& t) {
        const auto b = t.find_first_not_of(" \t\r\n");
        if (b == std::string::npos) return std::string();
        return t.substr(b, t.find_last_not_of(" \t\r\n") - b + 1);
    };
    std::string name = "unnamed", raw;
    std::optional<std::uint32_t> dim;
    bool euc2d = false, coords_started = false;
    std::vector<std::pair<double, double>> pts;
    int ln = 0;
    while (std::getline(in, raw)) {
        ++ln;
        const std::string line = trim(raw);
        if (line.empty()) continue;
        if (line == "EOF") break;
        if (coords_started) {
            if (pts.size() == *dim)
                throw ParseError(ln, "more coordinate lines than DIMENSION " + std::to_string(*dim));
            std::istringstream f(line);
            std::string id, extra;
            double x = 0.0, y = 0.0;
            if (!(f >> id >> x >> y)) throw ParseError(ln, "expected 'id x y', got '" + line + "'");
            if (f >> extra) throw ParseError(ln, "trailing content after coordinates: '" + extra + "'");
            if (!std::isfinite(x) || !std::isfinite(y)) throw ParseError(ln, "non-finite coordinate");
            pts.emplace_back(x, y);
            continue;
        }
        if (line == "NODE_COORD_SECTION") {
            if (!dim) throw ParseError(ln, "NODE_COORD_SECTION before DIMENSION");
            if (!euc2d) throw ParseError(ln, "missing EDGE_WEIGHT_TYPE header");
            coords_started = true;
            pts.reserve(*dim);
            continue;
        }
        const auto colon = line.find(':');
        const std::string key = colon == std::string::npos ? std::string() : trim(line.substr(0, colon));
        if (key.empty()) throw ParseError(ln, "malformed header line: '" + line + "'");
        const std::string value = trim(line.substr(colon + 1));
        if (key == "NAME") {
            name = value;
        } else if (key == "DIMENSION") {
            long long d = 0;
            try {
                d = std::stoll(value);
            } catch (const std::exception&) {
                throw ParseError(ln, "non-numeric DIMENSION: '" + value + "'");
            }
            if (d < 3) throw ParseError(ln, "DIMENSION must be at least 3");
            dim = static_cast<std::uint32_t>(d);
        } else if (key == "EDGE_WEIGHT_TYPE") {
            if (value != "EUC_2D") throw ParseError(ln, "unsupported EDGE_WEIGHT_TYPE: '" + value + "' (only EUC_2D)");
            euc2d = true;
        }  // other headers (TYPE, COMMENT, ...) are ignored
    }
    if (!coords_started) throw ParseError(ln, "missing NODE_COORD_SECTION");
    if (pts.size() != *dim)
        throw ParseError(ln, "DIMENSION is " + std::to_string(*dim) + " but " + std::to_string(pts.size()) +
                                 " coordinate lines were read");
    return Instance(name, std::move(pts));
}

inline Instance parse_tsplib_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open instance file: " + path);
    try {
        return parse_tsplib(in);
    } catch (const ParseError& e) {
        throw std::runtime_error(path + ": " + e.what());
    }
}

struct ConvergenceSample {
    double elapsed_s;
    std::int64_t g_best_length;
    std::uint64_t iterations_done;
};

// RunReport, engine.hpp:84-92, plus the engine's counters and device timings.
struct RunReport {
    std::int64_t best_length = 0;
    Tour best_tour;
    std::optional<double> pct_error;
    double wall_time_s = 0.0;
    std::uint64_t iterations_done = 0;
    std::uint64_t comparisons_total = 0;
    std::vector<ConvergenceSample> convergence;
    paco_counters counters{};
    double construct_ms = 0.0, update_ms = 0.0, setup_ms = 0.0;
};

inline paco_mode to_c(Mode m) {
    return m == Mode::partial_aco ? PACO_MODE_PARTIAL : m == Mode::paco_full ? PACO_MODE_PACO : PACO_MODE_CLASSIC;
}

// paco::run (engine.hpp:156-333) on the B200 engine.
inline RunReport run(const Instance& inst, const RunConfig& cfg, Mode mode) {
    const paco_config c = cfg.to_c();
    paco_report rep{};
    RunReport out;
    out.best_tour.order.resize(inst.n());
    std::vector<paco_sample> samples(4096);
    std::uint32_t ns = 0;
    check(paco_run_traced(inst.xs(), inst.ys(), inst.n(), &c, to_c(mode), inst.optimum().value_or(0), &rep,
                          out.best_tour.order.data(), samples.data(), (std::uint32_t)samples.size(), &ns));
    out.best_length = rep.best_length;
    out.best_tour.length = rep.best_length;
    if (inst.optimum()) out.pct_error = rep.pct_error;
    out.wall_time_s = rep.wall_time_s;
    out.iterations_done = rep.iterations_done;
    out.comparisons_total = rep.comparisons_total;
    out.counters = rep.counters;
    out.construct_ms = rep.construct_ms;
    out.update_ms = rep.update_ms;
    out.setup_ms = rep.setup_ms;
    for (std::uint32_t i = 0; i < ns; ++i)
        out.convergence.push_back({samples[i].elapsed_s, samples[i].g_best_length, samples[i].iterations_done});
    return out;
}

// engine.hpp:339-344
// Device memory of finished runs stays cached in the device's memory pool for the next
// run; this hands it back to the driver (device < 0: the current device).
inline void release_cached_memory(int device = -1) { check(paco_release_cached_memory(device)); }

inline RunReport run_timed_baseline(const Instance& inst, RunConfig cfg, double budget_s) {
    if (budget_s <= 0.0) throw std::invalid_argument("budget must be positive");
    cfg.time_budget_s = budget_s;
    return run(inst, cfg, Mode::paco_full);
}

}  // namespace paco_b200

#if defined(__has_include)
#if __has_include(<paco/engine.hpp>)
#include <paco/engine.hpp>
#define PACO_B200_REFERENCE_TYPES 1

namespace paco_b200 {

// The north-star knobs the reference's RunConfig does not have.
struct Options {
    std::uint32_t candidates = 16;                  // k of the k-NN candidate list (1..32)
    paco_rule rule = PACO_RULE_CANDIDATE_ROULETTE;  // INDEPENDENT_ROULETTE: the reference's own rule, bit-exact
    int device = -1;                                // CUDA device ordinal, -1 = current
};

inline paco_mode to_c(paco::Mode m) {
    return m == paco::Mode::partial_aco ? PACO_MODE_PARTIAL
         : m == paco::Mode::paco_full  ? PACO_MODE_PACO
                                       : PACO_MODE_CLASSIC;
}

inline paco_config to_c(const paco::RunConfig& cfg, const Options& opt) {
    paco_config c{};
    check(paco_config_default(&c));
    c.ants = cfg.ants; c.iterations = cfg.iterations; c.alpha = cfg.alpha; c.beta = cfg.beta;
    c.partial_prob = cfg.partial_prob; c.max_mod_frac = cfg.max_mod_frac; c.two_opt_prob = cfg.two_opt_prob;
    c.two_opt_window = cfg.two_opt_window; c.workers = cfg.workers; c.seed = cfg.seed; c.rho = cfg.rho;
    c.tau_max = cfg.tau_max; c.tau0 = cfg.tau0; c.time_budget_s = cfg.time_budget_s;
    c.convergence_interval_s = cfg.convergence_interval_s; c.synchronous = cfg.synchronous ? 1u : 0u;
    c.validate_tours = cfg.validate_tours ? 1u : 0u;
    c.candidates = opt.candidates; c.draws = PACO_DRAWS_PHILOX; c.device = opt.device; c.rule = opt.rule;
    return c;
}

// paco::run (engine.hpp:156-333) on the B200 engine, on the reference's own types:
// RunConfig::validate and the classic-mode size check throw exactly as the reference does
// (the reference's own validate() runs first), then one C-ABI call runs the whole job.
inline paco::RunReport run(const paco::Instance& inst, const paco::RunConfig& cfg, paco::Mode mode,
                           const Options& opt = {}) {
    cfg.validate();
    const std::uint32_t n = inst.n();
    std::vector<double> xs(n), ys(n);
    for (std::uint32_t i = 0; i < n; ++i) { xs[i] = inst.x(i); ys[i] = inst.y(i); }
    const paco_config c = to_c(cfg, opt);
    paco_report rep{};
    paco::RunReport out;
    out.best_tour.order.resize(n);
    std::vector<paco_sample> samples(4096);
    std::uint32_t ns = 0;
    check(paco_run_traced(xs.data(), ys.data(), n, &c, to_c(mode), inst.optimum().value_or(0), &rep,
                          out.best_tour.order.data(), samples.data(), (std::uint32_t)samples.size(), &ns));
    out.best_length = rep.best_length;
    out.best_tour.length = rep.best_length;
    if (inst.optimum()) {  // engine.hpp:322-325
        const double o = static_cast<double>(*inst.optimum());
        out.pct_error = 100.0 * (static_cast<double>(rep.best_length) - o) / o;
    }
    out.wall_time_s = rep.wall_time_s;
    out.iterations_done = rep.iterations_done;
    out.comparisons_total = rep.comparisons_total;
    for (std::uint32_t i = 0; i < ns; ++i)
        out.convergence.push_back({samples[i].elapsed_s, samples[i].g_best_length, samples[i].iterations_done});
    return out;
}

// run_timed_baseline (engine.hpp:339-344)
inline paco::RunReport run_timed_baseline(const paco::Instance& inst, paco::RunConfig cfg, double budget_s,
                                          const Options& opt = {}) {
    if (budget_s <= 0.0) throw std::invalid_argument("budget must be positive");
    cfg.time_budget_s = budget_s;
    return run(inst, cfg, paco::Mode::paco_full, opt);
}

}  // namespace paco_b200
#endif
#endif
