// Test infrastructure (O1): drives the UNMODIFIED reference bench.hpp / config.hpp
// formatting and parsing code on scripted inputs, so that
// paper_1709_03187_b200/experiment.py can be pinned byte for byte
// (tests/test_experiment.py, fixtures written by oracle/make_golden.py).
//
//   ref_bench_tool rows    < script   (ROW/REC/SPEEDUP/LABEL lines, see make_golden.py)
//   ref_bench_tool config  < text     (parse_experiment_config, fields dumped)
//   ref_bench_tool preset NAME        (table_preset, fields dumped)
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "paco/config.hpp"

using namespace paco;

static std::string g(double v) { return detail::fmt_double(v); }

static void dump_spec(const ExperimentSpec& s) {
    std::cout << "label=" << s.label << "\n";
    for (const auto& p : s.instance_paths) std::cout << "instance=" << p << "\n";
    std::cout << "optima=" << s.optima_path << "\nmode=" << mode_name(s.mode) << "\ntrials=" << s.trials
              << "\nants=" << s.base.ants << "\niterations=" << s.base.iterations << "\nalpha=" << g(s.base.alpha)
              << "\nbeta=" << g(s.base.beta) << "\nworkers=" << s.base.workers << "\nseed=" << s.base.seed
              << "\nrho=" << g(s.base.rho) << "\ntau_max=" << g(s.base.tau_max) << "\ntau0=" << g(s.base.tau0)
              << "\ntwo_opt_window=" << s.base.two_opt_window
              << "\nconvergence_interval=" << g(s.base.convergence_interval_s)
              << "\nvalidate_tours=" << s.base.validate_tours << "\nbaseline=" << s.include_baseline
              << "\ntimed_baseline=" << s.timed_baseline << "\nout_dir=" << s.out_dir << "\n";
    for (const auto& p : s.grid())
        std::cout << "grid=" << g(p.max_mod_frac) << "," << g(p.partial_prob) << "," << g(p.two_opt_prob) << "\n";
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const std::string mode = argv[1];
    if (mode == "config") {
        std::stringstream ss;
        ss << std::cin.rdbuf();
        try {
            ExperimentSpec s = parse_experiment_config(ss);
            dump_spec(s);
            std::cout << "synchronous=" << s.base.synchronous << "\n";
        } catch (const ParseError& e) {
            std::cout << "ParseError: " << e.what() << "\n";
        }
        return 0;
    }
    if (mode == "preset") {
        try {
            dump_spec(table_preset(argv[2], "data", "data/optima.txt"));
        } catch (const std::exception& e) {
            std::cout << "error: " << e.what() << "\n";
        }
        return 0;
    }
    // rows
    std::vector<AggregateStats> rows;
    std::vector<std::vector<RunRecord>> recs;
    std::vector<std::string> labels;
    std::string line;
    while (std::getline(std::cin, line)) {
        std::istringstream in(line);
        std::string tag;
        in >> tag;
        if (tag == "ROW") {
            AggregateStats r;
            std::string pairing, error;
            in >> r.label >> r.instance >> r.mode >> r.iterations >> r.max_mod_frac >> r.partial_prob >>
                r.two_opt_prob >> r.two_opt_window >> pairing >> error;
            r.pairing = pairing == "time_budget" ? Pairing::time_budget : Pairing::equal_iterations;
            r.error = error == "-" ? "" : error;
            rows.push_back(r);
            recs.emplace_back();
        } else if (tag == "REC") {
            RunRecord r;
            std::string pe;
            in >> r.instance >> r.row_label >> r.trial >> r.seed >> r.best_length >> pe >> r.wall_s >>
                r.iterations >> r.comparisons;
            r.pct_error = pe == "nan" ? std::numeric_limits<double>::quiet_NaN() : std::stod(pe);
            recs.back().push_back(r);
        } else if (tag == "SPEEDUP") {
            std::size_t i = 0, j = 0;
            in >> i >> j;
            try {
                rows[i].speedup = report_speedup(rows[i], rows[j]);
            } catch (const std::exception& e) {
                labels.push_back(std::string("speedup error: ") + e.what());
            }
        } else if (tag == "AGG") {
            for (std::size_t i = 0; i < rows.size(); ++i) {
                const AggregateStats a = aggregate_stats(recs[i]);
                rows[i].trials = a.trials; rows[i].err_mean = a.err_mean; rows[i].err_sd = a.err_sd;
                rows[i].err_best = a.err_best; rows[i].err_worst = a.err_worst;
                rows[i].time_mean_s = a.time_mean_s; rows[i].time_sd_s = a.time_sd_s;
                rows[i].iters_mean = a.iters_mean;
            }
        } else if (tag == "LABEL") {
            GridPoint gp;
            std::string m;
            in >> m >> gp.max_mod_frac >> gp.partial_prob >> gp.two_opt_prob;
            labels.push_back(detail::row_label(gp, m.c_str()));
        }
    }
    std::ostringstream summary;
    write_summary_csv(rows, summary);
    std::cout << "== summary\n" << summary.str();
    std::vector<RunRecord> all;
    for (const auto& v : recs) all.insert(all.end(), v.begin(), v.end());
    std::cout << "== runs\n";
    write_runs_csv(all, std::cout);
    std::cout << "== table\n";
    render_table(rows, std::cout);
    std::cout << "== reread\n";
    std::istringstream back(summary.str());
    write_summary_csv(read_summary_csv(back), std::cout);
    std::cout << "== labels\n";
    for (const auto& l : labels) std::cout << l << "\n";
    return 0;
}
