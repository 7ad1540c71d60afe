"""Experiment sweeps, presets and CSV outputs wired to the B200 engine.

Mirrors the reference's bench.hpp (GridPoint, ExperimentSpec, RunRecord,
AggregateStats, aggregate_stats, report_speedup, the summary / runs CSV writers and
reader, render_table, run_experiment) and config.hpp (the flat `key = value`
experiment config and the table1..table8 presets), with `run` /
`run_timed_baseline` being the GPU engine's. The CSV and table text is
byte-identical to the reference's for the same records
(tests/test_experiment.py against fixtures written by oracle/ref_bench_tool.cpp).
"""
from __future__ import annotations

import math
import os
import re
import sys
from dataclasses import dataclass, field, replace
from typing import Dict, List, Optional, TextIO

from .engine import Mode, RunConfig, mode_from_name, mode_name, run, run_timed_baseline
from .instances import ParseError, load_optima, parse_tsplib

NAN = float("nan")


# ------------------------------------------------------------------ formatting helpers
def fmt_double(v: float) -> str:
    """detail::fmt_double (bench.hpp:144-148): ostream with setprecision(17)."""
    return _fmt_g(v, 17)


def _fmt_g(v: float, prec: int) -> str:
    """ostream << double with the given precision in default float format (%g)."""
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "-inf" if v < 0 else "inf"
    return "%.*g" % (prec, v)


def _fmt_fixed(v: float, prec: int) -> str:
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "-inf" if v < 0 else "inf"
    return "%.*f" % (prec, v)


# ------------------------------------------------------------------ bench.hpp types
@dataclass
class GridPoint:
    """bench.hpp:21-25"""
    max_mod_frac: float = 1.0
    partial_prob: float = 1.0
    two_opt_prob: float = 0.0


@dataclass
class ExperimentSpec:
    """bench.hpp:27-66"""
    label: str = "experiment"
    instance_paths: List[str] = field(default_factory=list)
    optima_path: str = ""
    mode: Mode = Mode.partial_aco
    trials: int = 10
    base: RunConfig = field(default_factory=RunConfig)
    max_mod_grid: List[float] = field(default_factory=lambda: [1.0])
    partial_prob_grid: List[float] = field(default_factory=list)
    two_opt_prob_grid: List[float] = field(default_factory=list)
    include_baseline: bool = True
    timed_baseline: bool = False
    out_dir: str = ""

    def grid(self) -> List[GridPoint]:
        pps = self.partial_prob_grid or [self.base.partial_prob]
        tops = self.two_opt_prob_grid or [self.base.two_opt_prob]
        return [GridPoint(f, pp, top) for f in self.max_mod_grid for pp in pps for top in tops]

    def validate(self) -> None:
        if self.trials < 1:
            raise ValueError("trials must be >= 1")
        if not self.instance_paths:
            raise ValueError("experiment needs at least one instance")
        if not self.max_mod_grid:
            raise ValueError("parameter grid must be non-empty")
        for p in self.instance_paths:
            if not os.path.exists(p):
                raise ValueError("instance file not found: " + p)
        self.base.validate()


EQUAL_ITERATIONS, TIME_BUDGET = "equal_iterations", "time_budget"  # Pairing, bench.hpp:68


@dataclass
class RunRecord:
    """bench.hpp:70-81"""
    instance: str = ""
    row_label: str = ""
    trial: int = 0
    seed: int = 0
    best_length: int = 0
    pct_error: float = NAN
    wall_s: float = 0.0
    iterations: int = 0
    comparisons: int = 0


@dataclass
class AggregateStats:
    """bench.hpp:83-104"""
    label: str = ""
    instance: str = ""
    mode: str = ""
    trials: int = 0
    iterations: int = 0
    max_mod_frac: float = 1.0
    partial_prob: float = 1.0
    two_opt_prob: float = 0.0
    two_opt_window: int = 0
    err_mean: float = NAN
    err_sd: float = NAN
    err_best: float = NAN
    err_worst: float = NAN
    time_mean_s: float = 0.0
    time_sd_s: float = 0.0
    iters_mean: float = 0.0
    speedup: float = 0.0
    pairing: str = EQUAL_ITERATIONS
    error: str = ""


def _mean_sd(xs: List[float]):
    """detail::mean_sd (bench.hpp:116-137): sample sd, accumulated in input order."""
    if not xs:
        return 0.0, 0.0, 0.0, 0.0
    s = 0.0
    lo = hi = xs[0]
    for x in xs:
        s += x
        lo = min(lo, x)
        hi = max(hi, x)
    mean = s / len(xs)
    sd = 0.0
    if len(xs) > 1:
        ss = 0.0
        for x in xs:
            ss += (x - mean) * (x - mean)
        sd = math.sqrt(ss / (len(xs) - 1))
    return mean, sd, lo, hi


def aggregate_stats(records: List[RunRecord]) -> AggregateStats:
    """bench.hpp:152-175: %-error fields stay NaN when any record lacks a known optimum."""
    out = AggregateStats(trials=len(records))
    have = bool(records) and not any(math.isnan(r.pct_error) for r in records)
    if have:
        out.err_mean, out.err_sd, out.err_best, out.err_worst = _mean_sd([r.pct_error for r in records])
    out.time_mean_s, out.time_sd_s, _, _ = _mean_sd([r.wall_s for r in records])
    out.iters_mean = _mean_sd([float(r.iterations) for r in records])[0]
    return out


def report_speedup(reference: AggregateStats, baseline: AggregateStats) -> float:
    """bench.hpp:177-190"""
    if reference.pairing != baseline.pairing:
        raise ValueError("speedup requires rows with the same pairing basis")
    if reference.instance != baseline.instance:
        raise ValueError("speedup requires rows on the same instance")
    if reference.pairing == EQUAL_ITERATIONS:
        if reference.iterations != baseline.iterations:
            raise ValueError("equal-iteration pairing needs matching counts")
        return baseline.time_mean_s / reference.time_mean_s
    return reference.iters_mean / baseline.iters_mean


SUMMARY_HEADER = ("label,instance,mode,trials,iterations,max_mod,partial_prob,two_opt_prob,"
                  "two_opt_window,err_mean,err_sd,err_best,err_worst,time_mean_s,time_sd_s,"
                  "iters_mean,speedup,pairing,error\n")
RUNS_HEADER = "instance,row,trial,seed,best_length,pct_error,wall_s,iterations,comparisons\n"


def write_summary_csv(rows: List[AggregateStats], out: TextIO) -> None:
    """bench.hpp:192-211"""
    out.write(SUMMARY_HEADER)
    for r in rows:
        out.write(",".join([r.label, r.instance, r.mode, str(r.trials), str(r.iterations), fmt_double(r.max_mod_frac),
                            fmt_double(r.partial_prob), fmt_double(r.two_opt_prob), str(r.two_opt_window),
                            fmt_double(r.err_mean), fmt_double(r.err_sd), fmt_double(r.err_best),
                            fmt_double(r.err_worst), fmt_double(r.time_mean_s), fmt_double(r.time_sd_s),
                            fmt_double(r.iters_mean), fmt_double(r.speedup), r.pairing, r.error]) + "\n")


def read_summary_csv(text: str) -> List[AggregateStats]:
    """bench.hpp:213-248"""
    rows = []
    lines = text.split("\n")
    for line in lines[1:]:
        if not line:
            continue
        f = line.split(",")
        if f and f[-1] == "":
            f = f[:-1]  # std::getline on ',' drops a trailing empty field
        f += [""] * (19 - len(f))
        rows.append(AggregateStats(
            label=f[0], instance=f[1], mode=f[2], trials=_stoull(f[3]), iterations=_stoull(f[4]),
            max_mod_frac=_stod(f[5]), partial_prob=_stod(f[6]), two_opt_prob=_stod(f[7]),
            two_opt_window=_stoull(f[8]), err_mean=_stod(f[9]), err_sd=_stod(f[10]), err_best=_stod(f[11]),
            err_worst=_stod(f[12]), time_mean_s=_stod(f[13]), time_sd_s=_stod(f[14]), iters_mean=_stod(f[15]),
            speedup=_stod(f[16]), pairing=TIME_BUDGET if f[17] == "time_budget" else EQUAL_ITERATIONS,
            error=f[18]))
    return rows


def write_runs_csv(records: List[RunRecord], out: TextIO) -> None:
    """bench.hpp:250-258"""
    out.write(RUNS_HEADER)
    for r in records:
        out.write(",".join([r.instance, r.row_label, str(r.trial), str(r.seed), str(r.best_length),
                            fmt_double(r.pct_error), fmt_double(r.wall_s), str(r.iterations),
                            str(r.comparisons)]) + "\n")


def render_table(rows: List[AggregateStats], out: TextIO) -> None:
    """bench.hpp:261-285, the aligned human-readable table."""
    out.write("instance".ljust(16) + "mode".ljust(9) + "maxmod".ljust(8) + "pp".ljust(7) + "2opt".ljust(8)
              + "err_mean".rjust(10) + "err_sd".rjust(9) + "best".rjust(9) + "worst".rjust(9)
              + "time_s".rjust(11) + "speedup".rjust(10) + "\n")
    for r in rows:
        s = (r.instance.ljust(16) + r.mode.ljust(9) + _fmt_g(r.max_mod_frac, 3).ljust(8)
             + _fmt_g(r.partial_prob, 3).ljust(7) + _fmt_g(r.two_opt_prob, 3).ljust(8))
        if math.isnan(r.err_mean):
            s += "-".rjust(10) + "-".rjust(9) + "-".rjust(9) + "-".rjust(9)
        else:
            s += (_fmt_fixed(r.err_mean, 2).rjust(10) + _fmt_fixed(r.err_sd, 2).rjust(9)
                  + _fmt_fixed(r.err_best, 2).rjust(9) + _fmt_fixed(r.err_worst, 2).rjust(9))
        s += _fmt_fixed(r.time_mean_s, 2).rjust(11)
        s += (_fmt_fixed(r.speedup, 2).rjust(9) + "x") if r.speedup > 0.0 else "-".rjust(10)
        if r.error:
            s += "  ERROR: " + r.error
        out.write(s + "\n")


def row_label(g: GridPoint, mode: str) -> str:
    """detail::row_label (bench.hpp:292-297): default stream precision (6, %g)."""
    return f"{mode}_mm{_fmt_g(g.max_mod_frac, 6)}_pp{_fmt_g(g.partial_prob, 6)}_ls{_fmt_g(g.two_opt_prob, 6)}"


def convergence_csv(report, out: TextIO) -> None:
    """engine.hpp:94-100"""
    out.write("elapsed_s,g_best_length,iterations_done\n")
    for s in report.convergence:
        out.write(f"{s.elapsed_s:.6f},{s.g_best_length},{s.iterations_done}\n")


# ------------------------------------------------------------------ the sweep
@dataclass
class ExperimentResult:
    rows: List[AggregateStats] = field(default_factory=list)
    records: List[RunRecord] = field(default_factory=list)


def _record(inst, row, t, seed, rep) -> RunRecord:
    return RunRecord(inst.name, row, t, seed, rep.best_length, NAN if rep.pct_error is None else rep.pct_error,
                     rep.wall_time_s, rep.iterations_done, rep.comparisons_total)


def _fill(row: AggregateStats, agg: AggregateStats) -> None:
    for f in ("trials", "err_mean", "err_sd", "err_best", "err_worst", "time_mean_s", "time_sd_s", "iters_mean"):
        setattr(row, f, getattr(agg, f))


def _write_convergence(out_dir: str, instance: str, row: str, trial: int, rep) -> None:
    if not out_dir or not rep.convergence:
        return
    d = os.path.join(out_dir, "conv")
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, f"{instance}_{row}_t{trial}.csv"), "w") as f:
        convergence_csv(rep, f)


def run_experiment(spec: ExperimentSpec, log: TextIO = sys.stdout) -> ExperimentResult:
    """bench.hpp:319-487: every instance x grid point, `trials` seeded GPU runs (seed = base
    seed + trial), one aggregated row each; per-run failures are recorded on their row."""
    spec.validate()
    result = ExperimentResult()
    optima: Dict[str, int] = {}
    if spec.optima_path:
        try:
            with open(spec.optima_path) as f:
                optima = load_optima(f.read())
        except OSError:
            raise RuntimeError("cannot open optima file: " + spec.optima_path) from None
    if spec.out_dir:
        os.makedirs(spec.out_dir, exist_ok=True)
    for path in spec.instance_paths:
        with open(path) as f:
            inst = parse_tsplib(f.read())
        if inst.name in optima:
            inst.optimum = optima[inst.name]
        baseline: Optional[AggregateStats] = None
        if spec.include_baseline and spec.mode != Mode.paco_full and not spec.timed_baseline:
            row = AggregateStats(label=spec.label, instance=inst.name, mode=mode_name(Mode.paco_full),
                                 iterations=spec.base.iterations, two_opt_window=spec.base.two_opt_window)
            records = []
            for t in range(spec.trials):
                cfg = replace(spec.base, seed=spec.base.seed + t)
                try:
                    rep = run(inst, cfg, Mode.paco_full)
                    records.append(_record(inst, "baseline", t, cfg.seed, rep))
                    _write_convergence(spec.out_dir, inst.name, "baseline", t, rep)
                except Exception as e:  # noqa: BLE001 - recorded on the row, as the reference does
                    row.error = str(e)
                    break
            _fill(row, aggregate_stats(records))
            result.rows.append(row)
            result.records.extend(records)
            if not row.error:
                baseline = row
            log.write(f"[{spec.label}] {inst.name} baseline (paco_full): {_fmt_g(row.time_mean_s, 6)} s mean\n")
        for g in spec.grid():
            row = AggregateStats(label=spec.label, instance=inst.name, mode=mode_name(spec.mode),
                                 iterations=spec.base.iterations, max_mod_frac=g.max_mod_frac,
                                 partial_prob=g.partial_prob, two_opt_prob=g.two_opt_prob,
                                 two_opt_window=spec.base.two_opt_window)
            label = row_label(g, mode_name(spec.mode))
            records, timed = [], []
            for t in range(spec.trials):
                cfg = replace(spec.base, seed=spec.base.seed + t, max_mod_frac=g.max_mod_frac,
                              partial_prob=g.partial_prob, two_opt_prob=g.two_opt_prob)
                try:
                    rep = run(inst, cfg, spec.mode)
                    records.append(_record(inst, label, t, cfg.seed, rep))
                    _write_convergence(spec.out_dir, inst.name, label, t, rep)
                    if spec.timed_baseline:
                        bcfg = replace(spec.base, seed=spec.base.seed + 7777 + t)
                        brep = run_timed_baseline(inst, bcfg, rep.wall_time_s)
                        timed.append(_record(inst, "timed_baseline", t, bcfg.seed, brep))
                        _write_convergence(spec.out_dir, inst.name, "timed_baseline", t, brep)
                except Exception as e:  # noqa: BLE001
                    row.error = str(e)
            _fill(row, aggregate_stats(records))
            if baseline is not None:
                row.pairing = EQUAL_ITERATIONS
                row.speedup = report_speedup(row, baseline)
            result.rows.append(row)
            result.records.extend(records)
            if spec.timed_baseline and timed:
                brow = AggregateStats(label=spec.label, instance=inst.name, mode="paco_timed",
                                      iterations=spec.base.iterations, pairing=TIME_BUDGET)
                _fill(brow, aggregate_stats(timed))
                ref = replace(row, pairing=TIME_BUDGET, iters_mean=float(spec.base.iterations))
                brow.speedup = report_speedup(ref, brow)
                result.rows.append(brow)
                result.records.extend(timed)
            msg = f"[{spec.label}] {inst.name} {label}: "
            if not math.isnan(row.err_mean):
                msg += f"{_fmt_g(row.err_mean, 6)}% mean err, "
            msg += f"{_fmt_g(row.time_mean_s, 6)} s mean"
            if row.speedup > 0.0:
                msg += f", {_fmt_g(row.speedup, 6)}x"
            if row.error:
                msg += " ERROR: " + row.error
            log.write(msg + "\n")
    if spec.out_dir:
        with open(os.path.join(spec.out_dir, spec.label + "_summary.csv"), "w") as f:
            write_summary_csv(result.rows, f)
        with open(os.path.join(spec.out_dir, spec.label + "_runs.csv"), "w") as f:
            write_runs_csv(result.records, f)
    return result


# ------------------------------------------------------------------ config.hpp
_NUM = re.compile(r"[ \t\n\v\f\r]*[+-]?(?:inf(?:inity)?|nan|(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?)", re.I)
_INT = re.compile(r"[ \t\n\v\f\r]*([+-]?)(\d+)")


def _stod(s: str) -> float:
    """std::stod: the longest numeric prefix; no prefix raises."""
    m = _NUM.match(s)
    if not m:
        raise ValueError(s)
    return float(m.group(0))


def _stoull(s: str) -> int:
    """std::stoull: base-10 prefix, a leading '-' negates modulo 2^64; no prefix raises."""
    m = _INT.match(s)
    if not m:
        raise ValueError(s)
    v = int(m.group(2))
    if v >= 1 << 64:
        raise OverflowError(s)
    return (-v) % (1 << 64) if m.group(1) == "-" else v


def _trim(s: str) -> str:
    return s.strip(" \t\r\n")


@dataclass
class _Value:
    items: List[str]
    is_list: bool
    line: int

    def scalar(self) -> str:
        if len(self.items) != 1:
            raise ParseError(self.line, "expected a single value, got a list")
        return self.items[0]

    def number(self) -> float:
        s = self.scalar()
        try:
            return _stod(s)
        except (ValueError, OverflowError):
            raise ParseError(self.line, f"expected a number, got '{s}'") from None

    def integer(self) -> int:
        s = self.scalar()
        try:
            return _stoull(s)
        except (ValueError, OverflowError):
            raise ParseError(self.line, f"expected an integer, got '{s}'") from None

    def boolean(self) -> bool:
        s = self.scalar()
        if s == "true":
            return True
        if s == "false":
            return False
        raise ParseError(self.line, f"expected true/false, got '{s}'")

    def numbers(self) -> List[float]:
        out = []
        for s in self.items:
            try:
                out.append(_stod(s))
            except (ValueError, OverflowError):
                raise ParseError(self.line, f"expected a number, got '{s}'") from None
        return out


def _strip_comment(line: str) -> str:
    quoted = False
    for i, c in enumerate(line):
        if c == '"':
            quoted = not quoted
        if c == "#" and not quoted:
            return line[:i]
    return line


def _split_list(body: str, line_no: int) -> List[str]:
    out, cur, quoted = [], "", False
    for c in body:
        if c == '"':
            quoted = not quoted
            continue
        if c == "," and not quoted:
            t = _trim(cur)
            if t:
                out.append(t)
            cur = ""
            continue
        cur += c
    if quoted:
        raise ParseError(line_no, "unterminated string")
    t = _trim(cur)
    if t:
        out.append(t)
    return out


def _parse_keyvals(text: str) -> Dict[str, _Value]:
    out: Dict[str, _Value] = {}
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    for line_no, raw in enumerate(lines, 1):
        line = _trim(_strip_comment(raw))
        if not line:
            continue
        eq = line.find("=")
        if eq < 0:
            raise ParseError(line_no, f"expected 'key = value', got '{line}'")
        key, body = _trim(line[:eq]), _trim(line[eq + 1:])
        if not key or not body:
            raise ParseError(line_no, f"expected 'key = value', got '{line}'")
        if body[0] == "[":
            if body[-1] != "]":
                raise ParseError(line_no, "unterminated list")
            v = _Value(_split_list(body[1:-1], line_no), True, line_no)
        else:
            v = _Value(_split_list(body, line_no), False, line_no)
            if len(v.items) != 1:
                raise ParseError(line_no, "unexpected comma outside a list")
        out[key] = v
    return out


_KNOWN = ("label", "instances", "optima", "mode", "trials", "ants", "iterations", "alpha", "beta", "workers", "seed",
          "rho", "tau_max", "tau0", "two_opt_window", "convergence_interval", "synchronous", "validate_tours",
          "baseline", "timed_baseline", "out_dir", "max_mod", "partial_prob", "two_opt_prob")


def parse_experiment_config(text: str) -> ExperimentSpec:
    """config.hpp:126-185: flat `key = value` config (quoted strings, numbers, booleans,
    [lists]; '#' comments); unknown keys are errors."""
    kv = _parse_keyvals(text)
    spec = ExperimentSpec(max_mod_grid=[])
    b = spec.base
    v = kv.get
    if v("label"): spec.label = kv["label"].scalar()
    if v("instances"): spec.instance_paths = list(kv["instances"].items)
    if v("optima"): spec.optima_path = kv["optima"].scalar()
    if v("mode"):
        m = mode_from_name(kv["mode"].scalar())
        if m is None:
            raise ParseError(kv["mode"].line, f"unknown mode '{kv['mode'].scalar()}'")
        spec.mode = m
    if v("trials"): spec.trials = kv["trials"].integer() & 0xFFFFFFFF
    if v("ants"): b.ants = kv["ants"].integer() & 0xFFFFFFFF
    if v("iterations"): b.iterations = kv["iterations"].integer()
    if v("alpha"): b.alpha = kv["alpha"].number()
    if v("beta"): b.beta = kv["beta"].number()
    if v("workers"): b.workers = kv["workers"].integer() & 0xFFFFFFFF
    if v("seed"): b.seed = kv["seed"].integer()
    if v("rho"): b.rho = kv["rho"].number()
    if v("tau_max"): b.tau_max = kv["tau_max"].number()
    if v("tau0"): b.tau0 = kv["tau0"].number()
    if v("two_opt_window"): b.two_opt_window = kv["two_opt_window"].integer() & 0xFFFFFFFF
    if v("convergence_interval"): b.convergence_interval_s = kv["convergence_interval"].number()
    if v("synchronous"): b.synchronous = kv["synchronous"].boolean()
    if v("validate_tours"): b.validate_tours = kv["validate_tours"].boolean()
    if v("baseline"): spec.include_baseline = kv["baseline"].boolean()
    if v("timed_baseline"): spec.timed_baseline = kv["timed_baseline"].boolean()
    if v("out_dir"): spec.out_dir = kv["out_dir"].scalar()
    if v("max_mod"): spec.max_mod_grid = kv["max_mod"].numbers()
    if not spec.max_mod_grid:
        spec.max_mod_grid.append(1.0)
    if v("partial_prob"): spec.partial_prob_grid = kv["partial_prob"].numbers()
    if v("two_opt_prob"): spec.two_opt_prob_grid = kv["two_opt_prob"].numbers()
    for key in sorted(kv):  # std::map iterates in key order
        if key not in _KNOWN:
            raise ParseError(kv[key].line, f"unknown key '{key}'")
    return spec


_MIDSIZE = ["pcb442", "d657", "rat783", "pr1002", "pr2392"]
_ART = ["mona-lisa100K", "vangogh120K", "venus140K", "earring200K"]


def table_preset(name: str, instance_dir: str, optima_path: str) -> ExperimentSpec:
    """config.hpp:187-252: tables 1-6 sweep five mid-size TSPLIB instances (16 ants, 100k
    iterations, alpha = beta = 5); tables 7-8 the four art instances with a 1% cap and
    windowed 2-opt (table8 pairs against a time-budget baseline)."""
    spec = ExperimentSpec(label=name, optima_path=optima_path, trials=10)
    spec.base = RunConfig(ants=16, iterations=100000, alpha=5.0, beta=5.0, workers=8, seed=1000,
                          convergence_interval_s=1.0)

    def use(names):
        spec.instance_paths += [os.path.join(instance_dir, n + ".tsp") for n in names]

    caps = [0.5, 0.4, 0.3, 0.2, 0.1]
    if name == "table1":
        use(_MIDSIZE); spec.mode = Mode.paco_full; spec.include_baseline = False
    elif name == "table2":
        use(_MIDSIZE); spec.partial_prob_grid = [1.0]
    elif name == "table3":
        use(_MIDSIZE); spec.max_mod_grid = caps; spec.partial_prob_grid = [1.0]
    elif name == "table4":
        use(_MIDSIZE); spec.max_mod_grid = caps; spec.partial_prob_grid = [0.95]
    elif name == "table5":
        use(_MIDSIZE); spec.partial_prob_grid = [1.0]; spec.two_opt_prob_grid = [0.001]
    elif name == "table6":
        use(_MIDSIZE); spec.max_mod_grid = caps; spec.partial_prob_grid = [1.0]; spec.two_opt_prob_grid = [0.001]
    elif name in ("table7", "table8"):
        use(_ART)
        spec.max_mod_grid = [0.01]
        spec.partial_prob_grid = [1.0]
        spec.two_opt_prob_grid = [0.001]
        spec.base.two_opt_window = 500
        spec.include_baseline = False
        spec.timed_baseline = name == "table8"
    else:
        raise ValueError(f"unknown preset '{name}' (expected table1..table8)")
    return spec
