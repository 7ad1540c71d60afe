"""A/B of engine library variants on one config: same instance, seed and iterations.

    python profiles/ubench/ab.py [--config C5] [--iters 6] lib1.so lib2.so ...

Each library runs in its own process (PACO_B200_LIB), seeding + `iters` synchronous
iterations; prints the construction kernel's mean time over the iterations after the
first two, g_best and the counters (which must agree between variants).
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CHILD = r"""
import json, sys
sys.path.insert(0, %(root)r)
from paper_1709_03187_b200 import Colony, Mode, RunConfig, make_config_instance
import bench
cfgname, iters, sync = sys.argv[1], int(sys.argv[2]), sys.argv[3] == "1"
spec = bench.workload(cfgname)
inst = make_config_instance(cfgname)
cfg = RunConfig(ants=spec["m"], iterations=iters + 1, alpha=1.0, beta=2.0, rho=0.5, partial_prob=0.95,
                max_mod_frac=1.0, candidates=spec["k"], seed=1, synchronous=sync)
col = Colony(inst, cfg, Mode.partial_aco)
out = {"construct_ms": [], "update_ms": []}
if sync:
    for _ in range(iters + 1):
        col.iterate(1)
        c, u, _ = col.timing()
        out["construct_ms"].append(round(c, 3)); out["update_ms"].append(round(u, 3))
else:
    col.iterate(1)
    d0 = col.counters()["decisions"]
    col.iterate(iters)
    ms = col.timing()[0]
    out["async_dec_per_s"] = (col.counters()["decisions"] - d0) / (ms / 1e3)
out["g_best"] = int(col.g_best()[1])
out["counters"] = col.counters()
col.close()
print(json.dumps(out))
"""


def main() -> int:
    args = sys.argv[1:]
    cfg, iters, sync = "C5", 6, "1"
    libs = []
    while args:
        a = args.pop(0)
        if a == "--config":
            cfg = args.pop(0)
        elif a == "--iters":
            iters = int(args.pop(0))
        elif a == "--async":
            sync = "0"
        else:
            libs.append(a)
    for lib in libs:
        env = dict(os.environ, PACO_B200_LIB=os.path.abspath(lib))
        res = subprocess.run([sys.executable, "-c", CHILD % {"root": ROOT}, cfg, str(iters), sync], env=env,
                             capture_output=True, text=True, cwd=ROOT)
        if res.returncode != 0:
            print(f"{lib}: FAILED\n{res.stderr[-2000:]}")
            continue
        out = json.loads(res.stdout.strip().splitlines()[-1])
        if sync == "1":
            c = out["construct_ms"]
            tail = c[3:] if len(c) > 3 else c
            out["construct_ms_mean_after_2"] = round(sum(tail) / len(tail), 3)
        print(json.dumps({"lib": os.path.basename(lib), "config": cfg, **out}), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
