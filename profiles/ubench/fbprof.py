# Fallback anatomy of the longest (full) construction of synchronous C5 iterations: needs a
# library built with -DPACO_TIMING (nvcc ... -DPACO_TIMING -o lib.so paper_1709_03187_b200/csrc/paco_b200.cu),
# run as PACO_B200_LIB=lib.so python profiles/ubench/fbprof.py [config]
# g_prof is filled by CTA 0 (the first launched ant = a full construction, k_ant_order puts
# the longest constructions first): per 5% bucket of tour positions, cycles, fallbacks,
# F1 searches and F1 rings. g_timing holds the whole-launch totals.
import ctypes, sys, json
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_1709_03187_b200 import Colony, Mode, RunConfig, make_config_instance, _native
from paper_1709_03187_b200.instances import CONFIGS
name = sys.argv[1] if len(sys.argv) > 1 else "C5"
spec = CONFIGS[name]
inst = make_config_instance(name)
cfg = RunConfig(ants=spec["m"], iterations=8, alpha=1.0, beta=2.0, rho=0.5, partial_prob=0.95, max_mod_frac=1.0,
                candidates=spec["k"], seed=1, synchronous=True)
col = Colony(inst, cfg, Mode.partial_aco)
lib = _native.load()
P = ctypes.POINTER(ctypes.c_ulonglong)
prof = np.zeros(96, np.uint64)
tim = np.zeros(16, np.uint64)
col.iterate(1)
lib.paco_debug_timing(tim.ctypes.data_as(P), 1)
for it in range(3):
    col.iterate(1)
    lib.paco_debug_prof(prof.ctypes.data_as(P))
    lib.paco_debug_timing(tim.ctypes.data_as(P), 1)
    p = prof.astype(np.int64)
    cyc, fb, f1, rings = p[0:20], p[24:44], p[48:68], p[72:92]
    t = tim.astype(np.int64)
    out = {"iter": it + 1, "construct_ms": col.timing()[0],
           "loop_cycles": int(t[0]), "fallback_cycles": int(t[1]), "decisions": int(t[2]),
           "f1_searches": int(t[9]), "f1_rings": int(t[10]), "f1_sbs": int(t[11]), "f1_cities": int(t[12]),
           "f1_test": int(t[13]), "f1_scan": int(t[14]), "f1_argmin": int(t[15]), "f1_pre": int(t[3]),
           "f0": {"n": int(t[4]), "row_cycles": round(t[5] / max(1, t[4]), 1), "probe_cycles": round(t[6] / max(1, t[4]), 1),
                  "redux_cycles": round(t[7] / max(1, t[4]), 1), "fallback_cycles_each": round(t[1] / max(1, t[4]), 1)},
           "crit_total_mcycles": round(cyc.sum() / 1e6, 2), "crit_fallbacks": int(fb.sum()),
           "crit_f1": int(f1.sum()),
           "crit_buckets": [(round(c / 1e6, 2), int(f), int(s), int(r)) for c, f, s, r in zip(cyc, fb, f1, rings)]}
    print(json.dumps(out), flush=True)
col.close()
