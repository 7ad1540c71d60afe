"""Sweeps, presets and CSV outputs against the unmodified reference.

tests/golden/bench_golden.json holds the output of oracle/ref_bench_tool (the reference's
bench.hpp / config.hpp compiled in place) on scripted inputs; the same scripts run through
paper_1709_03187_b200/experiment.py must give byte-identical text. CPU only, except the
end-to-end sweep at the bottom.
"""
import io
import json
import math
import os

import pytest

from paper_1709_03187_b200 import ParseError, emit_tsplib, grid_instance
from paper_1709_03187_b200 import experiment as X

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "bench_golden.json")))


def run_rows(script: str) -> str:
    """Python side of `ref_bench_tool rows` (oracle/ref_bench_tool.cpp)."""
    rows, recs, labels = [], [], []
    for line in script.split("\n"):
        f = line.split()
        if not f:
            continue
        if f[0] == "ROW":
            rows.append(X.AggregateStats(label=f[1], instance=f[2], mode=f[3], iterations=int(f[4]),
                                         max_mod_frac=float(f[5]), partial_prob=float(f[6]), two_opt_prob=float(f[7]),
                                         two_opt_window=int(f[8]),
                                         pairing=X.TIME_BUDGET if f[9] == "time_budget" else X.EQUAL_ITERATIONS,
                                         error="" if f[10] == "-" else f[10]))
            recs.append([])
        elif f[0] == "REC":
            recs[-1].append(X.RunRecord(f[1], f[2], int(f[3]), int(f[4]), int(f[5]),
                                        math.nan if f[6] == "nan" else float(f[6]), float(f[7]), int(f[8]),
                                        int(f[9])))
        elif f[0] == "SPEEDUP":
            i, j = int(f[1]), int(f[2])
            try:
                rows[i].speedup = X.report_speedup(rows[i], rows[j])
            except ValueError as e:
                labels.append(f"speedup error: {e}")
        elif f[0] == "AGG":
            for r, rs in zip(rows, recs):
                a = X.aggregate_stats(rs)
                for k in ("trials", "err_mean", "err_sd", "err_best", "err_worst", "time_mean_s", "time_sd_s",
                          "iters_mean"):
                    setattr(r, k, getattr(a, k))
        elif f[0] == "LABEL":
            labels.append(X.row_label(X.GridPoint(float(f[2]), float(f[3]), float(f[4])), f[1]))
    out = io.StringIO()
    summary = io.StringIO()
    X.write_summary_csv(rows, summary)
    out.write("== summary\n" + summary.getvalue())
    out.write("== runs\n")
    X.write_runs_csv([r for rs in recs for r in rs], out)
    out.write("== table\n")
    X.render_table(rows, out)
    out.write("== reread\n")
    X.write_summary_csv(X.read_summary_csv(summary.getvalue()), out)
    out.write("== labels\n")
    for l in labels:
        out.write(l + "\n")
    return out.getvalue()


def dump_spec(s: X.ExperimentSpec) -> str:
    g = X.fmt_double
    b = s.base
    lines = [f"label={s.label}"] + [f"instance={p}" for p in s.instance_paths]
    lines += [f"optima={s.optima_path}", f"mode={X.mode_name(s.mode)}", f"trials={s.trials}", f"ants={b.ants}",
              f"iterations={b.iterations}", f"alpha={g(b.alpha)}", f"beta={g(b.beta)}", f"workers={b.workers}",
              f"seed={b.seed}", f"rho={g(b.rho)}", f"tau_max={g(b.tau_max)}", f"tau0={g(b.tau0)}",
              f"two_opt_window={b.two_opt_window}", f"convergence_interval={g(b.convergence_interval_s)}",
              f"validate_tours={int(b.validate_tours)}", f"baseline={int(s.include_baseline)}",
              f"timed_baseline={int(s.timed_baseline)}", f"out_dir={s.out_dir}"]
    lines += [f"grid={g(p.max_mod_frac)},{g(p.partial_prob)},{g(p.two_opt_prob)}" for p in s.grid()]
    return "\n".join(lines) + "\n"


@pytest.mark.parametrize("case", range(len(GOLD["rows"])))
def test_tables_and_csv_match_reference(case):
    """aggregate_stats, report_speedup, write_summary_csv / read_summary_csv round trip,
    write_runs_csv, render_table and row_label (bench.hpp:116-297), byte for byte."""
    c = GOLD["rows"][case]
    assert run_rows(c["input"]) == c["output"]


@pytest.mark.parametrize("case", range(len(GOLD["config"])))
def test_experiment_config_matches_reference(case):
    """parse_experiment_config (config.hpp:19-185): values, grids, and every error message."""
    c = GOLD["config"][case]
    try:
        spec = X.parse_experiment_config(c["input"])
        got = dump_spec(spec)
        ref = c["output"].split("synchronous=")[0]
        assert got == ref
        # the reference's RunConfig defaults to asynchronous; the GPU engine keeps its own
        # default unless the file sets it
        if "synchronous" in c["input"]:
            assert f"synchronous={int(spec.base.synchronous)}" in c["output"]
    except ParseError as e:
        assert c["output"] == f"ParseError: {e}\n"


@pytest.mark.parametrize("case", range(len(GOLD["preset"])))
def test_presets_match_reference(case):
    """table_preset (config.hpp:190-252)"""
    c = GOLD["preset"][case]
    try:
        got = dump_spec(X.table_preset(c["input"], "data", "data/optima.txt"))
    except ValueError as e:
        got = f"error: {e}\n"
    assert got == c["output"]


def test_fmt_double_is_setprecision_17():
    assert X.fmt_double(0.1) == "0.10000000000000001"
    assert X.fmt_double(1.0) == "1" and X.fmt_double(1.0 / 3.0) == "0.33333333333333331"
    assert X.fmt_double(math.nan) == "nan"


@pytest.mark.gpu
def test_sweep_end_to_end(tmp_path):
    """run_experiment on the GPU engine: a 2-point grid with a paco_full baseline over two
    trials, the summary / runs CSVs written and read back, errors recorded per row."""
    inst = grid_instance(12, 9, 10.0, "grid108")
    p = tmp_path / "grid108.tsp"
    p.write_text(emit_tsplib(inst))
    (tmp_path / "optima.txt").write_text("grid108 1080\n")
    cfg = (f'label = smoke\ninstances = ["{p}"]\noptima = {tmp_path / "optima.txt"}\ntrials = 2\nants = 8\n'
           f'iterations = 30\nalpha = 1\nbeta = 2\nmax_mod = [1.0, 0.3]\npartial_prob = [1.0]\nout_dir = {tmp_path}\n')
    spec = X.parse_experiment_config(cfg)
    log = io.StringIO()
    res = X.run_experiment(spec, log)
    assert [r.mode for r in res.rows] == ["paco", "partial", "partial"]
    assert all(r.trials == 2 and not r.error for r in res.rows)
    assert all(r.err_best >= 0.0 for r in res.rows)  # 1080 is the optimum of the grid
    assert all(r.speedup > 0 for r in res.rows[1:])
    assert len(res.records) == 6 and all(rec.iterations == 30 for rec in res.records)
    back = X.read_summary_csv((tmp_path / "smoke_summary.csv").read_text())
    assert [r.mode for r in back] == ["paco", "partial", "partial"]
    assert (tmp_path / "smoke_runs.csv").read_text().count("\n") == 7
    assert "baseline (paco_full)" in log.getvalue()


# ------------------------------------------------------------------ test_bench.cpp:217-346, case for case

def write_instance(tmp_path, inst) -> str:
    p = tmp_path / f"{inst.name}.tsp"
    p.write_text(emit_tsplib(inst))
    return str(p)


@pytest.mark.gpu
def test_run_experiment_sweeps_a_grid_and_writes_reports(tmp_path):
    """test_bench.cpp:217-271, on the same 16-city instance (tests/refgen.py) with its Held–Karp optimum."""
    from refgen import MT19937_64, held_karp, random_instance
    inst = random_instance(MT19937_64(5), 16, 300.0, "mini")
    path = write_instance(tmp_path, inst)
    (tmp_path / "optima.txt").write_text(f"mini {held_karp(inst)}\n")
    spec = X.ExperimentSpec(label="smoke", instance_paths=[path], optima_path=str(tmp_path / "optima.txt"), trials=2,
                            max_mod_grid=[1.0, 0.5], partial_prob_grid=[1.0], out_dir=str(tmp_path / "out"))
    spec.base.ants, spec.base.iterations, spec.base.workers, spec.base.seed = 4, 60, 1, 42
    spec.base.convergence_interval_s = 0.001
    res = X.run_experiment(spec, io.StringIO())
    assert len(res.rows) == 3 and res.rows[0].mode == "paco"  # 1 baseline row + 2 grid rows
    assert len(res.records) == 6
    for row in res.rows:
        assert not row.error and row.trials == 2 and not math.isnan(row.err_mean)
        assert row.err_best <= row.err_mean <= row.err_worst and row.err_sd >= 0.0
        assert row.err_best >= 0.0  # Held–Karp is exact
    assert res.rows[1].speedup > 0.0
    out = tmp_path / "out"
    assert (out / "smoke_summary.csv").exists() and (out / "smoke_runs.csv").exists() and (out / "conv").is_dir()
    back = X.read_summary_csv((out / "smoke_summary.csv").read_text())
    assert len(back) == 3
    for b, r in zip(back, res.rows):  # %.17g round trip is exact
        assert b.err_mean == r.err_mean and b.time_mean_s == r.time_mean_s and b.speedup == r.speedup


@pytest.mark.gpu
@pytest.mark.parametrize("rule", ["roulette", "independent"])
def test_sweeps_are_deterministic_for_a_fixed_master_seed(tmp_path, rule):
    """test_bench.cpp:273-306"""
    from refgen import MT19937_64, random_instance
    path = write_instance(tmp_path, random_instance(MT19937_64(7), 18, 400.0, "det"))
    spec = X.ExperimentSpec(label="det", instance_paths=[path], trials=3, include_baseline=False,
                            max_mod_grid=[1.0, 0.3])
    spec.base.ants, spec.base.iterations, spec.base.workers, spec.base.seed, spec.base.rule = 4, 80, 1, 7, rule
    a = X.run_experiment(spec, io.StringIO())
    b = X.run_experiment(spec, io.StringIO())
    assert len(a.records) == len(b.records) == 6
    for x, y in zip(a.records, b.records):
        assert (x.best_length, x.comparisons, x.seed) == (y.best_length, y.comparisons, y.seed)
    spec.base.seed = 8  # fresh seeds shift results
    c = X.run_experiment(spec, io.StringIO())
    assert any(x.comparisons != z.comparisons for x, z in zip(a.records, c.records))


@pytest.mark.gpu
def test_timed_baseline_pairing_produces_a_time_budget_row(tmp_path):
    """test_bench.cpp:308-333"""
    from refgen import MT19937_64, random_instance
    path = write_instance(tmp_path, random_instance(MT19937_64(9), 20, 400.0, "timed"))
    spec = X.ExperimentSpec(label="timed", instance_paths=[path], trials=1, include_baseline=False,
                            timed_baseline=True)
    spec.base.ants, spec.base.iterations, spec.base.workers, spec.base.seed = 2, 300, 1, 3
    res = X.run_experiment(spec, io.StringIO())
    assert len(res.rows) == 2
    assert res.rows[0].pairing == X.EQUAL_ITERATIONS and res.rows[1].pairing == X.TIME_BUDGET
    assert res.rows[1].mode == "paco_timed"
    assert res.rows[1].iters_mean >= 1.0 and res.rows[1].speedup > 0.0


def test_experiment_validation_catches_bad_specs():
    """test_bench.cpp:335-346"""
    spec = X.ExperimentSpec(instance_paths=["/definitely/not/here.tsp"])
    with pytest.raises(ValueError):
        spec.validate()
    spec.instance_paths = []
    with pytest.raises(ValueError):
        spec.validate()
    spec.trials = 0
    with pytest.raises(ValueError):
        spec.validate()
