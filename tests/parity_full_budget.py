"""Full-budget parity run: the GPU engine against the O2 oracle (the checker, on the host
cores) over a config's whole iteration budget, several seeds; best lengths, g_best tours
and counters must be identical. Writes one JSON line per seed.

    python tests/parity_full_budget.py C2 1 2 3 4 5   (results: profiles/parity/*.jsonl)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402

import oracle  # noqa: E402  (test infrastructure: the checker)
from paper_1709_03187_b200 import Colony, Mode, RunConfig, make_config_instance  # noqa: E402

SPECS = {"C1": (64, 20, 100), "C2": (256, 20, 200), "C3": (256, 20, 200), "C4": (512, 16, 50),
         "C5": (1024, 16, 20)}

name = sys.argv[1]
m, k, iters = SPECS[name]
inst = make_config_instance(name)
for seed in [int(x) for x in sys.argv[2:]]:
    cfg = RunConfig(ants=m, iterations=iters, alpha=1.0, beta=2.0, rho=0.5, partial_prob=0.95, max_mod_frac=1.0,
                    candidates=k, seed=seed, synchronous=True)
    t0 = time.perf_counter()
    with Colony(inst, cfg, Mode.partial_aco) as col:
        col.iterate(iters)
        gt, gl = col.g_best()
        cg = col.counters()
    t_gpu = time.perf_counter() - t0
    t0 = time.perf_counter()
    ref = oracle.O2(inst.xs, inst.ys, m=m, k=k, seed=seed)
    for _ in range(iters):
        ref.iterate()
    rt, rl = ref.g_best()
    cr = ref.counters()
    t_cpu = time.perf_counter() - t0
    same = bool(gl == rl and np.array_equal(gt, rt) and all(cg[x] == cr[x] for x in ("decisions", "fallbacks", "ties")))
    print(json.dumps({"config": name, "seed": seed, "iterations": iters, "g_best_gpu": int(gl), "g_best_o2": int(rl),
                      "identical": same, "decisions": int(cg["decisions"]), "fallbacks": int(cg["fallbacks"]),
                      "ties": int(cg["ties"]), "gpu_s": round(t_gpu, 2), "o2_s": round(t_cpu, 2),
                      "o2_threads": os.cpu_count()}), flush=True)
