# Reference-rule mode (rule = independent) against the unmodified reference on the same
# host: C1-shaped instances, synchronous paco::run (O1, all host threads) and the GPU's
# bit-identical run, best length / comparisons / wall time each. With a library built with
# -DPACO_IRSEG the per-decision cycle split of the GPU construction is printed too.
#   [PACO_B200_LIB=lib.so] python profiles/ubench/ir_time.py [n] [ants] [iterations]
import ctypes, os, sys, time, json
import numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/oracle")
import oracle as O
from paper_1709_03187_b200 import Colony, Mode, RunConfig, make_config_instance, _native
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 64
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 100
inst = make_config_instance("C1", n=n)
out = {"n": n, "ants": m, "iterations": iters}
t0 = time.perf_counter()
r = O.ref_run(inst.xs, inst.ys, m, iters, 1.0, 2.0, seed=1, mode="partial", synchronous=True)
out["reference"] = {"wall_s": round(time.perf_counter() - t0, 3), "best": r["best_length"], "comparisons": r["comparisons"],
                    "threads": os.cpu_count()}
cfg = RunConfig(ants=m, iterations=iters, alpha=1.0, beta=2.0, rho=0.5, seed=1, rule="independent")
lib = _native.load()
for rep in range(2):
    t0 = time.perf_counter()
    with Colony(inst, cfg, Mode.partial_aco) as col:
        col.iterate(iters)
        g = col.g_best()[1]
        c = col.counters()
        cms = col.timing()[0]
    out[f"gpu_{rep}"] = {"wall_s": round(time.perf_counter() - t0, 3), "construct_ms": round(cms, 1), "best": int(g),
                         "comparisons": c["comparisons"]}
if hasattr(lib, "paco_debug_timing"):
    t = np.zeros(16, np.uint64)
    lib.paco_debug_timing(t.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), 1)
    t = t.astype(np.int64)
    d = max(1, t[4] // 2)
    out["cycles_per_decision"] = {"begin": int(t[0] // 2 // d), "scan": int(t[1] // 2 // d), "wait": int(t[2] // 2 // d),
                                  "end": int(t[3] // 2 // d), "loads": int(t[6] // 2 // d), "score_loop": int(t[7] // 2 // d),
                                  "draws_per_decision": int(t[5] // max(1, t[4]))}
out["identical"] = out["gpu_0"]["best"] == out["reference"]["best"] and out["gpu_0"]["comparisons"] == out["reference"]["comparisons"]
print(json.dumps(out))
