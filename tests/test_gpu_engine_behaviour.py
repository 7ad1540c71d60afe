"""The reference's engine test suite (tests/test_engine.cpp:25-241), case for case, on the GPU engine.

Each TEST_CASE of test_engine.cpp becomes one test here, on the same instances: tests/refgen.py
reproduces oracles.hpp:123-131's std::mt19937_64 draws exactly. The reference's assertions are
kept as written. Where an assertion is a closed form of the reference's comparison counter
(n(n-1)/2 per full build, construction.hpp:243-281), it is checked with rule="independent", the
reference's own selection rule. The north-star candidate rule counts one comparison per
decision, n-1 per full build, and is checked against that form.

The reference runs most of these cases asynchronously with one worker (small_cfg leaves
RunConfig::synchronous at false, engine.hpp:58). The GPU engine's asynchronous mode is the
candidate rule's persistent kernel. Reference-rule runs are therefore
synchronous. When oracle/_ref is built, they are also compared bit for bit with paco::run in
synchronous mode on the same instance.
"""
import itertools

import numpy as np
import pytest

import oracle
from paper_1709_03187_b200 import (InvalidArgument, Mode, RunConfig, cycle_length, grid_instance, is_permutation_of_n,
                                   run, run_timed_baseline, tour_length)
from refgen import MT19937_64, random_instance

pytestmark = pytest.mark.gpu

RULES = ["roulette", "independent"]
needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


def small_cfg(seed: int, rule: str, **kw) -> RunConfig:
    """test_engine.cpp:12-21"""
    base = dict(ants=4, iterations=50, workers=1, seed=seed, partial_prob=0.9, validate_tours=True, rule=rule,
                synchronous=True)
    base.update(kw)
    return RunConfig(**base)


def full_build_comparisons(n: int, rule: str) -> int:
    return n * (n - 1) // 2 if rule == "independent" else n - 1


def check_against_reference(inst, cfg: RunConfig, mode: Mode, rep):
    """paco::run (synchronous, one worker) on the same instance and configuration."""
    ref = oracle.ref_run(inst.xs, inst.ys, ants=cfg.ants, iterations=cfg.iterations, alpha=cfg.alpha, beta=cfg.beta,
                         seed=cfg.seed, mode={Mode.partial_aco: "partial", Mode.paco_full: "paco",
                                              Mode.classic_aco: "classic"}[mode], workers=1,
                         partial_prob=cfg.partial_prob, max_mod_frac=cfg.max_mod_frac, rho=cfg.rho,
                         two_opt_prob=cfg.two_opt_prob, two_opt_window=cfg.two_opt_window, synchronous=True)
    assert rep.best_length == ref["best_length"]
    assert np.array_equal(rep.best_tour.order, ref["best_tour"])
    assert rep.comparisons_total == ref["comparisons"]
    assert rep.iterations_done == ref["iterations"]


@pytest.mark.parametrize("rule", RULES)
def test_iterations_1_reports_the_seeding_pass_only(rule):
    """test_engine.cpp:25-38"""
    inst = random_instance(MT19937_64(3), 25)
    rep = run(inst, small_cfg(11, rule, iterations=1), Mode.partial_aco)
    assert rep.iterations_done == 1
    # seeding builds one full tour per ant
    assert rep.comparisons_total == 4 * full_build_comparisons(25, rule)
    assert rep.best_length == tour_length(inst, rep.best_tour.order)
    assert rep.wall_time_s >= 0.0
    assert rep.pct_error is None


@pytest.mark.parametrize("rule", RULES)
def test_pct_error_uses_the_configured_optimum(rule):
    """test_engine.cpp:40-51"""
    inst = grid_instance(6, 4)
    assert inst.optimum == 240
    rep = run(inst, small_cfg(5, rule, iterations=200, two_opt_prob=0.05), Mode.partial_aco)
    assert rep.pct_error == pytest.approx(100.0 * (rep.best_length - 240.0) / 240.0)
    assert rep.pct_error >= 0.0


@pytest.mark.parametrize("rule", RULES)
def test_single_worker_runs_are_bit_reproducible_from_the_seed(rule):
    """test_engine.cpp:53-73"""
    inst = random_instance(MT19937_64(17), 40)
    cfg = small_cfg(123, rule, iterations=120, two_opt_prob=0.02, max_mod_frac=0.5)
    a = run(inst, cfg, Mode.partial_aco)
    b = run(inst, cfg, Mode.partial_aco)
    assert a.best_length == b.best_length
    assert np.array_equal(a.best_tour.order, b.best_tour.order)
    assert a.comparisons_total == b.comparisons_total
    assert a.iterations_done == b.iterations_done
    cfg.seed = 124
    c = run(inst, cfg, Mode.partial_aco)
    # different seed, almost surely a different trajectory
    assert a.comparisons_total != c.comparisons_total


@pytest.mark.parametrize("rule", RULES)
def test_synchronous_mode_is_independent_of_the_worker_count(rule):
    """test_engine.cpp:75-95. `workers` sizes the reference's thread pool; the GPU engine
    accepts it and runs one warp per ant whatever its value."""
    inst = random_instance(MT19937_64(19), 30)
    reps = [run(inst, small_cfg(77, rule, ants=6, iterations=60, two_opt_prob=0.05, workers=w), Mode.partial_aco)
            for w in (1, 2, 6)]
    for r in reps[1:]:
        assert np.array_equal(r.best_tour.order, reps[0].best_tour.order)
        assert r.comparisons_total == reps[0].comparisons_total


@pytest.mark.parametrize("rule", RULES)
def test_paco_full_comparisons_follow_the_closed_form(rule):
    """test_engine.cpp:97-105"""
    inst = random_instance(MT19937_64(23), 60)
    rep = run(inst, small_cfg(9, rule, iterations=50), Mode.paco_full)
    assert rep.comparisons_total == 50 * 4 * full_build_comparisons(60, rule)
    assert rep.iterations_done == 50


@pytest.mark.parametrize("rule", RULES)
def test_partial_prob_0_matches_paco_full_bit_for_bit(rule):
    """test_engine.cpp:107-118"""
    inst = random_instance(MT19937_64(29), 35)
    cfg = small_cfg(31, rule, iterations=80, partial_prob=0.0)
    full = run(inst, cfg, Mode.paco_full)
    degenerate = run(inst, cfg, Mode.partial_aco)
    assert np.array_equal(full.best_tour.order, degenerate.best_tour.order)
    assert full.comparisons_total == degenerate.comparisons_total


@pytest.mark.parametrize("rule", RULES)
def test_convergence_series_is_non_increasing_and_ends_with_the_result(rule):
    """test_engine.cpp:120-136"""
    inst = random_instance(MT19937_64(37), 50)
    rep = run(inst, small_cfg(41, rule, iterations=400, convergence_interval_s=0.005), Mode.partial_aco)
    cv = rep.convergence
    assert cv
    for prev, cur in zip(cv, cv[1:]):
        assert cur.g_best_length <= prev.g_best_length
        assert cur.elapsed_s >= prev.elapsed_s
    assert cv[-1].g_best_length == rep.best_length
    assert cv[-1].iterations_done == rep.iterations_done


def test_asynchronous_runs_produce_valid_tours_under_load():
    """test_engine.cpp:138-151 (asynchronous: the candidate rule's persistent kernel)"""
    inst = random_instance(MT19937_64(43), 40)
    cfg = RunConfig(ants=8, workers=4, iterations=300, seed=7, two_opt_prob=0.01, validate_tours=True,
                    synchronous=False)
    rep = run(inst, cfg, Mode.partial_aco)
    assert is_permutation_of_n(40, rep.best_tour.order)
    assert cycle_length(inst, rep.best_tour.order) == rep.best_length
    assert rep.iterations_done == 300


@pytest.mark.parametrize("rule", RULES)
def test_classic_mode_runs_improves_and_respects_the_size_limit(rule):
    """test_engine.cpp:153-178"""
    gen = MT19937_64(47)
    inst = random_instance(gen, 20)
    cfg = RunConfig(ants=8, workers=2, iterations=1, seed=13, rho=0.2, validate_tours=True, rule=rule)
    seed_only = run(inst, cfg, Mode.classic_aco)
    cfg.iterations = 150
    longer = run(inst, cfg, Mode.classic_aco)
    assert longer.best_length <= seed_only.best_length
    assert is_permutation_of_n(20, longer.best_tour.order)
    # classic mode needs the matrix, which is capped at 5000 cities
    big = random_instance(gen, 5001, box=100000.0, name="big")
    cfg.iterations = 1
    with pytest.raises(InvalidArgument):
        run(big, cfg, Mode.classic_aco)


@pytest.mark.parametrize("rule", RULES)
def test_a_tiny_time_budget_still_completes_the_in_flight_iteration(rule):
    """test_engine.cpp:180-192"""
    inst = random_instance(MT19937_64(53), 80)
    cfg = RunConfig(ants=4, workers=2, iterations=1000000, seed=3, rule=rule)
    rep = run_timed_baseline(inst, cfg, 1e-9)
    assert 1 <= rep.iterations_done < 1000000
    assert rep.comparisons_total >= 4 * full_build_comparisons(80, rule)


@pytest.mark.parametrize("rule", RULES)
def test_timed_baseline_runs_paco_full_until_the_budget_expires(rule):
    """test_engine.cpp:194-208"""
    inst = random_instance(MT19937_64(59), 60)
    cfg = RunConfig(ants=2, workers=1, iterations=1000000000, seed=21, rule=rule)
    rep = run_timed_baseline(inst, cfg, 0.25)
    assert 0.25 <= rep.wall_time_s < 5.0
    # full constructions only
    assert rep.comparisons_total % full_build_comparisons(60, rule) == 0
    assert rep.comparisons_total == rep.iterations_done * 2 * full_build_comparisons(60, rule)
    with pytest.raises(InvalidArgument):
        run_timed_baseline(inst, cfg, 0.0)


def brute_force_optimum(inst) -> int:
    """oracles.hpp brute_force_optimum: every tour through city 0."""
    return min(cycle_length(inst, (0,) + p) for p in itertools.permutations(range(1, inst.n)))


@pytest.mark.parametrize("rule", RULES)
def test_partial_mode_with_2opt_finds_the_optimum_of_a_tiny_instance(rule):
    """test_engine.cpp:210-224"""
    inst = random_instance(MT19937_64(61), 8)
    cfg = RunConfig(ants=16, workers=2, iterations=5000, seed=2, partial_prob=0.95, two_opt_prob=0.01, rule=rule)
    rep = run(inst, cfg, Mode.partial_aco)
    assert rep.best_length == brute_force_optimum(inst)


def test_config_validation_rejects_out_of_range_values():
    """test_engine.cpp:226-241"""
    inst = random_instance(MT19937_64(67), 10)
    for kw in (dict(partial_prob=1.5), dict(max_mod_frac=0.0), dict(ants=0), dict(iterations=0)):
        with pytest.raises(InvalidArgument):
            run(inst, RunConfig(**kw), Mode.partial_aco)


# ------------------------------------------------------------------ the same cases against paco::run


@needs_ref
@pytest.mark.parametrize("case", ["seeding", "pct_error", "reproducible", "closed_form", "pp0_partial", "pp0_paco",
                                  "convergence", "classic"])
def test_reference_rule_cases_match_paco_run(case):
    """The deterministic cases above with rule="independent", compared with the reference
    engine itself (synchronous, one worker) on the same instance."""
    inst, cfg, mode = {
        "seeding": (random_instance(MT19937_64(3), 25), small_cfg(11, "independent", iterations=1),
                    Mode.partial_aco),
        "pct_error": (grid_instance(6, 4), small_cfg(5, "independent", iterations=200, two_opt_prob=0.05),
                      Mode.partial_aco),
        "reproducible": (random_instance(MT19937_64(17), 40),
                         small_cfg(123, "independent", iterations=120, two_opt_prob=0.02, max_mod_frac=0.5),
                         Mode.partial_aco),
        "closed_form": (random_instance(MT19937_64(23), 60), small_cfg(9, "independent"), Mode.paco_full),
        "pp0_partial": (random_instance(MT19937_64(29), 35),
                        small_cfg(31, "independent", iterations=80, partial_prob=0.0), Mode.partial_aco),
        "pp0_paco": (random_instance(MT19937_64(29), 35),
                     small_cfg(31, "independent", iterations=80, partial_prob=0.0), Mode.paco_full),
        "convergence": (random_instance(MT19937_64(37), 50), small_cfg(41, "independent", iterations=400),
                        Mode.partial_aco),
        "classic": (random_instance(MT19937_64(47), 20),
                    RunConfig(ants=8, iterations=150, seed=13, rho=0.2, rule="independent"), Mode.classic_aco),
    }[case]
    check_against_reference(inst, cfg, mode, run(inst, cfg, mode))


# ------------------------------------------------------------------ device memory pool


def test_cached_memory_is_reused_and_released():
    """Destroyed engines return their buffers to the device's stream-ordered pool; a new
    engine reuses them with the same results, and paco_release_cached_memory trims it."""
    from paper_1709_03187_b200 import Colony, release_cached_memory

    inst = grid_instance(12, 9)
    cfg = RunConfig(ants=12, iterations=6, seed=3, candidates=8)
    lengths = []
    for _ in range(3):
        with Colony(inst, cfg, Mode.partial_aco) as col:
            col.iterate(6)
            lengths.append(col.g_best()[1])
        release_cached_memory() if len(lengths) == 2 else None
    assert lengths[0] == lengths[1] == lengths[2]
    release_cached_memory(0)


# ------------------------------------------------------------------ bench.py contract


def test_bench_line_contract():
    """bench.py on a small config prints one JSON line with the driver's keys."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--config", "C2", "--steps", "2",
                          "--warmup", "3", "--no-cpu"], capture_output=True, text=True, check=True, cwd=root).stdout
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks", "cpu_baseline"):
        assert key in d, key
    assert d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["gpu_launches"] == 6 * 2  # C2: k_weights, k_ant_order, k_construct, k_lengths, k_update, k_publish
    assert d["roofline"]["bound"] == "hbm" and 0 < d["roofline"]["frac"] < 1
    lat = d["roofline"]["latency"]  # null only when no SM clock was sampled
    assert lat is None or (lat["bound"] == "latency" and 0 < lat["frac"] <= 1.5 and lat["floor_terms"]["scan_levels"] == 5)
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert "workload" in d["config"] and "model" not in d["config"]
    # traffic is the committed ncu capture of THIS config, or null (never another config's)
    assert "C2" in d["roofline"]["traffic_source"]
    assert d["e2e"]["iterations"] == 200 and "host" in d
