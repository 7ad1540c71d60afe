# Construction phases of synchronous iterations (setup / decision loop / tail = 2-opt, tour
# length and permutation check), summed over full and partial constructions: needs a
# library built with -DPACO_PHASES; run as PACO_B200_LIB=lib.so python profiles/ubench/phases.py [config]
import ctypes, sys, json
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_1709_03187_b200 import Colony, Mode, RunConfig, make_config_instance, _native
from paper_1709_03187_b200.instances import CONFIGS
name = sys.argv[1] if len(sys.argv) > 1 else "C5"
spec = CONFIGS[name]
inst = make_config_instance(name)
cfg = RunConfig(ants=spec["m"], iterations=8, alpha=1.0, beta=2.0, rho=0.5, candidates=spec["k"], seed=1)
col = Colony(inst, cfg, Mode.partial_aco)
lib = _native.load()
P = ctypes.POINTER(ctypes.c_ulonglong)
t = np.zeros(16, np.uint64)
for it in range(4):
    col.iterate(1)
    lib.paco_debug_timing(t.ctypes.data_as(P), 1)
    v = t.astype(np.int64)
    out = {"iter": it}
    for o, kind in ((0, "full"), (5, "partial")):
        cnt = max(1, int(v[o + 4]))
        out[kind] = {"constructions": int(v[o + 4]), "setup_kcyc": round(v[o] / cnt / 1e3, 1),
                     "loop_kcyc": round(v[o + 1] / cnt / 1e3, 1), "tail_kcyc": round(v[o + 2] / cnt / 1e3, 1),
                     "decisions": int(v[o + 3] / cnt)}
    print(json.dumps(out), flush=True)
col.close()
