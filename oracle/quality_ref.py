"""Quality-gate reference means (TEST INFRASTRUCTURE ONLY; runs in the CPU container).

Runs O1 -- the unmodified reference `paco::run` (engine.hpp:156-333), synchronous,
Mode::partial_aco, the BASELINE.json parameters (alpha=1, beta=2, tau0=1,
partial_prob=0.95, max_mod_frac=1.0, 2-opt off) -- on the seeded config instances
and records the final best length per seed in tests/golden/quality_ref.json. The
-m gpu quality test compares the GPU's 5-seed mean against these committed means
(north_star: "within 1% of the reference's mean over 5 seeds").

Usage: python oracle/quality_ref.py C1 1 2 3 4 5 [--workers W] [--iterations I]
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

OUT = os.path.join(ROOT, "tests", "golden", "quality_ref.json")


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("seeds", type=int, nargs="+")
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--iterations", type=int, default=None)
    a = ap.parse_args()

    import oracle as O
    from paper_1709_03187_b200.instances import CONFIGS, make_config_instance

    spec = CONFIGS[a.config]
    iters = a.iterations or spec["iterations"]
    inst = make_config_instance(a.config)
    for seed in a.seeds:
        t0 = time.time()
        r = O.ref_run(inst.xs, inst.ys, spec["m"], iters, 1.0, 2.0, seed=seed, mode="partial",
                      workers=a.workers, partial_prob=0.95, max_mod_frac=1.0, synchronous=True)
        rec = dict(config=a.config, seed=seed, iterations=iters, ants=spec["m"], best_length=r["best_length"],
                   comparisons=r["comparisons"], wall_s=round(time.time() - t0, 2), workers=a.workers,
                   cpu=cpu_model(), rule="reference Independent Roulette, paco::run sync, partial_aco")
        db = {}
        if os.path.exists(OUT):
            with open(OUT) as f:
                db = json.load(f)
        key = a.config if iters == spec["iterations"] else f"{a.config}@{iters}"  # shortened budgets apart
        db.setdefault(key, {})[str(seed)] = rec
        with open(OUT, "w") as f:
            json.dump(db, f, indent=1, sort_keys=True)
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
