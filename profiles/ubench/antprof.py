# Per-ant construction profile of synchronous C5 iterations: needs a library built with
# -DPACO_ANTPROF (nvcc ... -DPACO_ANTPROF -o lib.so paper_1709_03187_b200/csrc/paco_b200.cu),
# run as PACO_B200_LIB=lib.so python profiles/ubench/antprof.py
import ctypes, os, sys, json
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_1709_03187_b200 import Colony, Mode, RunConfig, make_config_instance, _native
inst = make_config_instance("C5")
cfg = RunConfig(ants=1024, iterations=8, alpha=1.0, beta=2.0, rho=0.5, partial_prob=0.95, max_mod_frac=1.0,
                candidates=16, seed=1, synchronous=True)
col = Colony(inst, cfg, Mode.partial_aco)
lib = _native.load()
buf = np.zeros(4096 * 6, np.uint64)
for it in range(6):
    col.iterate(1)
    lib.paco_debug_ant(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)))
    a = buf.reshape(4096, 6)[:1024].astype(np.int64)
    t0 = a[:, 0].min()
    st, en, sm, dec, fb, part = (a[:, i] for i in range(6))
    dur = en - st
    crit = int(np.argmax(en))
    order = np.argsort(-dur)[:5]
    print(json.dumps({"iter": it, "construct_ms": col.timing()[0], "span_ms": (en.max() - t0) / 1e6,
                      "crit_ant": crit, "crit_start_us": (st[crit] - t0) / 1e3, "crit_ms": dur[crit] / 1e6,
                      "crit_dec": int(dec[crit]), "crit_fb": int(fb[crit]), "crit_partial": int(part[crit]),
                      "crit_ns_per_dec": dur[crit] / max(1, dec[crit]),
                      "crit_sm_coresidents": int((sm == sm[crit]).sum()),
                      "mean_ns_per_dec": float((dur / np.maximum(dec, 1)).mean()),
                      "full_ns_per_dec": float((dur[part == 0] / np.maximum(dec[part == 0], 1)).mean()),
                      "top5": [(int(i), round(dur[i] / 1e6, 2), int(dec[i]), int(fb[i]), int(part[i])) for i in order],
                      "max_start_us": (st.max() - t0) / 1e3}), flush=True)
    # fallback rate by decile of tour for full ants is not recorded here
    if it == 5:
        np.save("/root/repo/gpurun_out/antprof_it5.npy", a)
col.close()
