# 2-opt at the paper's large-instance setting (config.hpp:242-249: two_opt_prob = 0.001,
# two_opt_window = 500) on a BASELINE config: seeding + ITERS synchronous iterations, per
# iteration wall ms, searches and moves; the final g_best identifies the move sequence
# (dense and neighbour-list searches must agree). Run as
#   [PACO_B200_LIB=lib.so] python profiles/ubench/two_opt_bench.py C4 [seed] [iters]
import sys, time, json
sys.path.insert(0, "/root/repo")
from paper_1709_03187_b200 import Colony, Mode, RunConfig, make_config_instance
from paper_1709_03187_b200.instances import CONFIGS
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 4
spec = CONFIGS[name]
inst = make_config_instance(name)
cfg = RunConfig(ants=spec["m"], iterations=iters + 1, alpha=1.0, beta=2.0, rho=0.5, candidates=spec["k"], seed=seed,
                synchronous=True, two_opt_prob=0.001, two_opt_window=500)
rows = []
with Colony(inst, cfg, Mode.partial_aco) as col:
    prev = col.counters()
    for it in range(iters + 1):
        t0 = time.perf_counter()
        col.iterate(1)
        g = col.g_best()[1]
        ms = (time.perf_counter() - t0) * 1e3
        c = col.counters()
        rows.append({"iter": it, "ms": round(ms, 1), "searches": c["two_opts"] - prev["two_opts"],
                     "moves": c["two_opt_moves"] - prev["two_opt_moves"], "g_best": int(g)})
        prev = c
print(json.dumps({"config": name, "seed": seed, "rows": rows}))
