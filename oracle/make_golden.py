#!/usr/bin/env python
"""Generate tests/golden/ref_golden.npz from the UNMODIFIED reference (O1).

Test infrastructure. Runs only in a container where /root/reference exists: it
builds oracle/_ref/libpaco_ref.so from the reference headers (oracle/Makefile)
and records the reference's own outputs for the pieces of the hot path that the
O2 restatement and the GPU engine must reproduce. The fixtures travel with the
repo, so the pinning tests run anywhere (including the GPU box, which has no
/root/reference).

    python oracle/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "ref_golden.npz")


def main() -> None:
    oracle.build(ref=True)
    rng = np.random.default_rng(20240917)
    L = oracle.reflib()
    g = {}

    # --- EUC_2D (instance.hpp:33-37): test_instance.cpp:136-145 points + random pairs
    kat = np.array([[0, 0, 3, 4], [0, 0, 1, 1], [0, 0, 0.5, 0], [0, 0, 10, 0], [0, 0, 0, 0]], dtype=np.float64)
    rnd_i = rng.integers(0, 10_000_000, size=(2000, 4)).astype(np.float64)
    rnd_f = rng.random((2000, 4)) * 1000.0
    pts = np.concatenate([kat, rnd_i, rnd_f])
    g["euc2d_pts"] = pts
    g["euc2d_ref"] = np.array([L.ref_euc2d(*p) for p in pts], dtype=np.int32)

    # --- Power (construction.hpp:19-44)
    es = np.array([0, 1, 2, 3, 5, 7, 64, 2.5, 0.5], dtype=np.float64)
    xs = np.array([1e-7, 0.5, 1.0, 2.0, 3.0, 123.4], dtype=np.float64)
    pe = np.array([(e, x) for e in es for x in xs], dtype=np.float64)
    g["power_args"] = pe
    g["power_ref"] = np.array([L.ref_power(e, x) for e, x in pe], dtype=np.float64)

    # --- tau^alpha through Colony + ColonyPheromone (colony.hpp:115-177, construction.hpp:104-158)
    cases = []
    for ci, (n, m, alpha) in enumerate([(10, 3, 1.0), (20, 5, 2.0), (37, 8, 5.0), (50, 16, 1.0), (12, 4, 0.0)]):
        x = rng.integers(0, 1000, n).astype(np.float64)
        y = rng.integers(0, 1000, n).astype(np.float64)
        tours = np.stack([rng.permutation(n) for _ in range(m)]).astype(np.uint32)
        if ci == 1:
            tours[3] = tours[1]  # equal lengths: the incumbent keeps g_best
        tau, direct, glen = oracle.ref_colony_tau(x, y, tours, 1.0, alpha, direct=True)
        g[f"tau{ci}_x"], g[f"tau{ci}_y"], g[f"tau{ci}_tours"] = x, y, tours
        g[f"tau{ci}_alpha"] = np.float64(alpha)
        g[f"tau{ci}_ref"] = tau
        g[f"tau{ci}_direct"] = direct
        g[f"tau{ci}_glen"] = np.int64(glen)
        cases.append(ci)
    g["tau_cases"] = np.array(cases)

    # --- eta^beta (Heuristic, construction.hpp:49-82), table path and on-the-fly path
    for tag, n in (("table", 200), ("fly", 5001)):
        x = rng.integers(0, 100_000, n).astype(np.float64)
        y = rng.integers(0, 100_000, n).astype(np.float64)
        x[5], y[5] = x[6], y[6]  # a duplicate point: d = 0 -> clamp to 1
        pairs = np.stack([rng.integers(0, n, 400), rng.integers(0, n, 400)], axis=1).astype(np.uint32)
        pairs[0] = (5, 6)
        pairs = pairs[pairs[:, 0] != pairs[:, 1]]
        for beta in (2.0, 5.0):
            g[f"eta_{tag}_b{int(beta)}_ref"] = oracle.ref_eta_beta(x, y, beta, pairs)
        g[f"eta_{tag}_x"], g[f"eta_{tag}_y"], g[f"eta_{tag}_pairs"] = x, y, pairs

    # --- completion-step update semantics (colony.hpp:115-139, engine.hpp:261-265)
    n, m = 9, 4
    x = rng.integers(0, 50, n).astype(np.float64)
    y = rng.integers(0, 50, n).astype(np.float64)
    count = 60
    tours = np.stack([rng.permutation(n) for _ in range(count)]).astype(np.uint32)
    tours[10] = tours[3]  # exact repeats -> ties
    tours[20] = np.roll(tours[7], 3)  # rotation -> equal length
    ants = rng.integers(0, m, count).astype(np.uint32)
    flags, gafter = oracle.ref_offer_sequence(x, y, m, tours, ants)
    g.update(offer_x=x, offer_y=y, offer_tours=tours, offer_ants=ants, offer_flags=flags, offer_g=gafter)

    # --- classic evaporate/deposit (construction.hpp:160-213)
    n = 12
    rounds, ntours = 3, 4
    ct = np.stack([[rng.permutation(n) for _ in range(ntours)] for _ in range(rounds)]).astype(np.uint32)
    cl = rng.integers(50, 200, size=(rounds, ntours)).astype(np.int64)
    g.update(classic_tours=ct, classic_lens=cl, classic_rho=np.float64(0.5), classic_tau=np.float64(1.0))
    g["classic_ref"] = oracle.ref_classic_update(n, 0.5, 1.0, ct, cl)

    # --- first-improvement 2-opt (two_opt.hpp:28-67): KAT square + random tours, windows
    sq_x = np.array([0.0, 10.0, 10.0, 0.0]); sq_y = np.array([0.0, 0.0, 10.0, 10.0])
    g["twoopt_sq"] = oracle.ref_two_opt(sq_x, sq_y, np.array([0, 2, 1, 3], np.uint32))[0]
    tcases = []
    for ti, (n, window) in enumerate([(9, 0), (25, 0), (60, 0), (60, 5), (120, 16), (200, 0)]):
        x = rng.integers(0, 1000, n).astype(np.float64)
        y = rng.integers(0, 1000, n).astype(np.float64)
        order = rng.permutation(n).astype(np.uint32)
        out, ln = oracle.ref_two_opt(x, y, order, window)
        g.update({f"twoopt{ti}_x": x, f"twoopt{ti}_y": y, f"twoopt{ti}_in": order, f"twoopt{ti}_out": out,
                  f"twoopt{ti}_len": np.int64(ln), f"twoopt{ti}_window": np.uint32(window)})
        tcases.append(ti)
    g["twoopt_cases"] = np.array(tcases)

    # --- Rng::for_stream (rng.hpp:33-50) raw outputs, for the IR-rule mode
    g["stream_ref"] = np.stack([oracle.ref_stream_u64(7, s, 64) for s in range(4)])

    # --- whole-run reference results (IR rule, sync mode) on small instances
    runs = []
    for ri, (n, m, iters, mode, p2, w2) in enumerate([(12, 4, 30, "partial", 0.0, 0), (30, 8, 20, "paco", 0.0, 0),
                                                      (25, 6, 10, "classic", 0.0, 0), (40, 6, 25, "partial", 0.3, 0),
                                                      (80, 8, 15, "partial", 0.05, 10)]):
        x = rng.integers(0, 1000, n).astype(np.float64)
        y = rng.integers(0, 1000, n).astype(np.float64)
        r = oracle.ref_run(x, y, ants=m, iterations=iters, alpha=1.0, beta=2.0, seed=11 + ri, mode=mode,
                           workers=2, rho=0.5, two_opt_prob=p2, two_opt_window=w2)
        g[f"run{ri}_x"], g[f"run{ri}_y"] = x, y
        g[f"run{ri}_cfg"] = np.array([n, m, iters, ["partial", "paco", "classic"].index(mode), 11 + ri])
        g[f"run{ri}_twoopt"] = np.array([p2, w2], dtype=np.float64)
        g[f"run{ri}_best"] = np.int64(r["best_length"])
        g[f"run{ri}_tour"] = r["best_tour"]
        g[f"run{ri}_comparisons"] = np.uint64(r["comparisons"])
        runs.append(ri)
    g["run_cases"] = np.array(runs)

    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes, {len(g)} arrays)")
    bench_fixtures()


BENCH_OUT = os.path.join(ROOT, "tests", "golden", "bench_golden.json")

# scripts for oracle/ref_bench_tool (rows mode): ROW label instance mode iterations max_mod pp
# two_opt_prob window pairing error|- ; REC instance row trial seed best pct_error wall_s
# iterations comparisons ; AGG ; SPEEDUP i j ; LABEL mode max_mod pp two_opt_prob
BENCH_SCRIPTS = [
    """ROW table4 pcb442 paco 100000 1 1 0 0 equal_iterations -
REC pcb442 baseline 0 1000 50903 0.21653543307086615 12.5 100000 160000000
REC pcb442 baseline 1 1001 50850 0.11220472440944881 12.25 100000 160000000
REC pcb442 baseline 2 1002 51002 0.41141732283464566 13.125 100000 160000000
ROW table4 pcb442 partial 100000 0.5 0.95 0 0 equal_iterations -
REC pcb442 partial_mm0.5_pp0.95_ls0 0 1000 50990 0.38779527559055116 3.1 100000 41000000
REC pcb442 partial_mm0.5_pp0.95_ls0 1 1001 50779 -0.027559055118110236 2.9 100000 40000000
REC pcb442 partial_mm0.5_pp0.95_ls0 2 1002 51204 0.80708661417322836 3.30000000001 100000 42000000
ROW table4 pcb442 partial 100000 0.1 0.95 0.001 500 equal_iterations boom
REC pcb442 partial_mm0.1_pp0.95_ls0.001 0 1000 50779 0 0.1 100000 7
AGG
SPEEDUP 1 0
SPEEDUP 2 0
LABEL partial 0.5 0.95 0
LABEL partial 0.1 1 0.001
LABEL paco 0.30000000000000004 0.95 1e-07
LABEL classic 1 1 0.33333333333333331
""",
    """ROW t8 earring200K partial 500 0.01 1 0.001 500 time_budget -
REC earring200K partial_mm0.01_pp1_ls0.001 0 1000 7990000 nan 3600.5 500 99999999999
REC earring200K partial_mm0.01_pp1_ls0.001 1 1001 7980000 nan 3599.75 500 88888888888
ROW t8 earring200K paco_timed 500 1 1 0 0 time_budget -
REC earring200K timed_baseline 0 8777 8100000 nan 3600.5 37 11111111111
REC earring200K timed_baseline 1 8778 8090000 nan 3599.75 41 22222222222
ROW t8 other partial 499 1 1 0 0 equal_iterations -
AGG
SPEEDUP 0 1
SPEEDUP 0 2
SPEEDUP 2 0
LABEL partial 0.01 1 0.001
""",
    """ROW solo x.tsp partial 7 1 1 0 3 equal_iterations -
REC x a 0 5 123 1e-20 1e-300 7 0
AGG
""",
]

BENCH_CONFIGS = [
    """# full experiment
label = "sweep one"   # quoted
instances = ["data/a.tsp", "data/b c.tsp"]
optima = data/optima.txt
mode = partial
trials = 5
ants = 32
iterations = 2000
alpha = 1.5
beta = 2
workers = 4
seed = 77
rho = 0.25
tau_max = 2.5
tau0 = 0.5
two_opt_window = 50
convergence_interval = 0.5
synchronous = true
validate_tours = false
baseline = false
timed_baseline = true
out_dir = out/run1
max_mod = [0.5, 0.25, 0.1]
partial_prob = [1.0, 0.95]
two_opt_prob = [0.0, 0.001]
""",
    "mode = paco\nmax_mod = []\n",
    "alpha = 1.5abc\ntrials = 12x\n",
    "trials = -1\n",
    "label = x\nnot a key value\n",
    "bogus = 3\n",
    "alpha = fast\n",
    "baseline = yes\n",
    "max_mod = [0.5, 0.2\n",
    "label = \"open\n",
    "alpha = [1, 2]\n",
    "alpha = 1, 2\n",
    "mode = turbo\n",
    "max_mod = [0.5, x]\n",
    "trials = \n",
    "   \n# only comments\n\n",
]

BENCH_PRESETS = ["table1", "table2", "table3", "table4", "table5", "table6", "table7", "table8", "table9"]


def bench_fixtures() -> None:
    import json
    import subprocess

    tool = os.path.join(HERE, "_ref", "ref_bench_tool")
    out = {"rows": [], "config": [], "preset": []}
    for sc in BENCH_SCRIPTS:
        r = subprocess.run([tool, "rows"], input=sc, capture_output=True, text=True, check=True)
        out["rows"].append({"input": sc, "output": r.stdout})
    for cf in BENCH_CONFIGS:
        r = subprocess.run([tool, "config"], input=cf, capture_output=True, text=True, check=True)
        out["config"].append({"input": cf, "output": r.stdout})
    for name in BENCH_PRESETS:
        r = subprocess.run([tool, "preset", name], capture_output=True, text=True, check=True)
        out["preset"].append({"input": name, "output": r.stdout})
    with open(BENCH_OUT, "w") as f:
        json.dump(out, f, indent=1)
    print(f"wrote {BENCH_OUT}")


if __name__ == "__main__":
    main()
