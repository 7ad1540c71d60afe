"""ctypes wrappers for the checkers (TEST INFRASTRUCTURE ONLY).

O2 = oracle/libo2.so, the CPU restatement of the north-star rule (o2.c).
O1 = oracle/_ref/libpaco_ref.so, the unmodified reference compiled in place.
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm
import this module.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, c_double, c_int, c_int32, c_int64, c_uint8, c_uint32, c_uint64

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
O2_PATH = os.path.join(HERE, "libo2.so")
REF_PATH = os.path.join(HERE, "_ref", "libpaco_ref.so")
REFERENCE_ROOT = "/root/reference"


def build(ref: bool = True) -> None:
    """Compile O2 and, when the reference tree is present, O1 (oracle/Makefile)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref and os.path.isdir(os.path.join(REFERENCE_ROOT, "proj", "include")):
        subprocess.run(["make", "-s", "-C", HERE, "ref", f"REF={REFERENCE_ROOT}"], check=True)


class O2Params(ctypes.Structure):
    _fields_ = [("n", c_uint32), ("m", c_uint32), ("k", c_uint32), ("threads", c_uint32),
                ("alpha", c_double), ("beta", c_double), ("tau0", c_double), ("partial_prob", c_double),
                ("max_mod_frac", c_double), ("rho", c_double), ("tau_max", c_double), ("two_opt_prob", c_double),
                ("two_opt_window", c_uint32), ("pad2_", c_uint32), ("seed", c_uint64),
                ("mode", c_int32), ("draw_source", c_int32), ("fallback_brute", c_int32), ("pad_", c_int32)]


class O2Counters(ctypes.Structure):
    _fields_ = [(f, c_uint64) for f in ("decisions", "fallbacks", "ties", "forced", "full_builds",
                                        "partial_builds", "iterations", "two_opts")]


def _p(a, t):
    return a.ctypes.data_as(POINTER(t))


_o2 = None


def o2lib():
    global _o2
    if _o2 is None:
        if not os.path.exists(O2_PATH):
            build(ref=False)
        L = ctypes.CDLL(O2_PATH)
        vp = ctypes.c_void_p
        L.o2_create.restype = vp
        L.o2_create.argtypes = [POINTER(c_double), POINTER(c_double), POINTER(O2Params)]
        L.o2_destroy.argtypes = [vp]
        L.o2_iterate.argtypes = [vp, POINTER(c_uint32), c_uint64]
        L.o2_get_knn.argtypes = [vp, POINTER(c_uint32)]
        L.o2_get_weights.argtypes = [vp, POINTER(ctypes.c_float)]
        L.o2_get_tours.argtypes = [vp, POINTER(c_uint32), POINTER(c_int64)]
        L.o2_get_lbest.argtypes = [vp, POINTER(c_uint32), POINTER(c_int64)]
        L.o2_get_gbest.restype = c_int64
        L.o2_get_gbest.argtypes = [vp, POINTER(c_uint32)]
        L.o2_get_counters.argtypes = [vp, POINTER(O2Counters)]
        L.o2_get_build_flags.argtypes = [vp, POINTER(c_uint8), POINTER(c_uint8)]
        L.o2_offer_tour.argtypes = [vp, c_uint32, POINTER(c_uint32)]
        L.o2_construct_at.argtypes = [vp, c_uint32, c_uint32, c_uint32, POINTER(c_uint32), c_uint64,
                                      POINTER(c_uint32), POINTER(c_int64)]
        L.o2_tau_row.argtypes = [vp, c_uint32, POINTER(c_double)]
        L.o2_get_T.argtypes = [vp, POINTER(c_double)]
        L.o2_classic_apply.argtypes = [vp, POINTER(c_uint32), POINTER(c_int64), c_uint32]
        L.o2_last_error.restype = ctypes.c_char_p
        L.o2_draw_word.restype = c_uint32
        L.o2_draw_word.argtypes = [c_uint64, c_uint32, c_uint64, c_uint32]
        L.o2_euc2d.restype = c_int32
        L.o2_euc2d.argtypes = [c_double] * 4
        L.o2_power.restype = c_double
        L.o2_power.argtypes = [c_double, c_double]
        L.o2_two_opt.restype = c_int64
        L.o2_two_opt.argtypes = [POINTER(c_double), POINTER(c_double), c_uint32, POINTER(c_uint32), c_uint32]
        L.o2_cycle_length.restype = c_int64
        L.o2_cycle_length.argtypes = [POINTER(c_double), POINTER(c_double), c_uint32, POINTER(c_uint32)]
        L.o2_knn_brute.argtypes = [POINTER(c_double), POINTER(c_double), c_uint32, c_uint32, POINTER(c_uint32)]
        L.o2_knn_rows.argtypes = [POINTER(c_double), POINTER(c_double), c_uint32, c_uint32, POINTER(c_uint32),
                                  c_uint32, POINTER(c_uint32)]
        L.o2_roulette.restype = c_int32
        L.o2_roulette.argtypes = [POINTER(ctypes.c_float), c_uint32, c_uint32, POINTER(c_int32)]
        L.o2_philox4x32_10.argtypes = [POINTER(c_uint32), POINTER(c_uint32), POINTER(c_uint32)]
        _o2 = L
    return _o2


MODES = {"partial": 0, "paco": 1, "classic": 2}


class O2:
    """The CPU restatement, driven like the GPU engine."""

    def __init__(self, xs, ys, m, k, alpha=1.0, beta=2.0, tau0=1.0, partial_prob=0.95, max_mod_frac=1.0,
                 rho=0.5, tau_max=1.0, seed=1, mode="partial", draws="philox", threads=None,
                 fallback_brute=False, two_opt_prob=0.0, two_opt_window=0):
        self.L = o2lib()
        self.xs = np.ascontiguousarray(xs, np.float64)
        self.ys = np.ascontiguousarray(ys, np.float64)
        self.n, self.m = self.xs.size, m
        self.k = min(k, self.n - 1, 32)
        p = O2Params(n=self.n, m=m, k=k, threads=threads or os.cpu_count() or 1, alpha=alpha, beta=beta,
                     tau0=tau0, partial_prob=partial_prob, max_mod_frac=max_mod_frac, rho=rho, tau_max=tau_max,
                     two_opt_prob=two_opt_prob, two_opt_window=two_opt_window, seed=seed, mode=MODES[mode], draw_source=1 if draws == "buffer" else 0,
                     fallback_brute=1 if fallback_brute else 0)
        self.h = self.L.o2_create(_p(self.xs, c_double), _p(self.ys, c_double), ctypes.byref(p))
        if not self.h:
            raise ValueError(self.L.o2_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.L.o2_destroy(self.h)
            self.h = None

    def iterate(self, words=None):
        if words is None:
            rc = self.L.o2_iterate(self.h, None, 0)
        else:
            w = np.ascontiguousarray(words, np.uint32)
            rc = self.L.o2_iterate(self.h, _p(w, c_uint32), w.shape[1])
        if rc:
            raise RuntimeError(self.L.o2_last_error().decode())

    def knn(self):
        out = np.empty((self.n, self.k), np.uint32)
        self.L.o2_get_knn(self.h, _p(out, c_uint32))
        return out

    def weights(self):
        out = np.empty((self.n, self.k), np.float32)
        self.L.o2_get_weights(self.h, _p(out, ctypes.c_float))
        return out

    def tau_row(self, i):
        out = np.empty(self.n, np.float64)
        self.L.o2_tau_row(self.h, i, _p(out, c_double))
        return out

    def T(self):
        out = np.empty((self.n, self.k), np.float64)
        self.L.o2_get_T(self.h, _p(out, c_double))
        return out

    def classic_apply(self, tours, lens):
        t = np.ascontiguousarray(tours, np.uint32)
        l = np.ascontiguousarray(lens, np.int64)
        if self.L.o2_classic_apply(self.h, _p(t, c_uint32), _p(l, c_int64), l.size):
            raise RuntimeError(self.L.o2_last_error().decode())

    def tours(self):
        t = np.empty((self.m, self.n), np.uint32)
        l = np.empty(self.m, np.int64)
        self.L.o2_get_tours(self.h, _p(t, c_uint32), _p(l, c_int64))
        return t, l

    def l_best(self):
        t = np.empty((self.m, self.n), np.uint32)
        l = np.empty(self.m, np.int64)
        self.L.o2_get_lbest(self.h, _p(t, c_uint32), _p(l, c_int64))
        return t, l

    def g_best(self):
        t = np.empty(self.n, np.uint32)
        ln = self.L.o2_get_gbest(self.h, _p(t, c_uint32))
        return t, int(ln)

    def counters(self):
        c = O2Counters()
        self.L.o2_get_counters(self.h, ctypes.byref(c))
        return {f: int(getattr(c, f)) for f, _ in c._fields_}

    def build_flags(self):
        p = np.empty(self.m, np.uint8)
        i = np.empty(self.m, np.uint8)
        self.L.o2_get_build_flags(self.h, _p(p, c_uint8), _p(i, c_uint8))
        return p, i

    def offer_tour(self, ant, order):
        o = np.ascontiguousarray(order, np.uint32)
        rc = self.L.o2_offer_tour(self.h, ant, _p(o, c_uint32))
        if rc < 0:
            raise ValueError(self.L.o2_last_error().decode())
        return bool(rc)

    def construct_at(self, ant, start_pos, m_mod, words):
        w = np.ascontiguousarray(words, np.uint32)
        out = np.empty(self.n, np.uint32)
        ln = c_int64()
        if self.L.o2_construct_at(self.h, ant, start_pos, m_mod, _p(w, c_uint32), w.size, _p(out, c_uint32),
                                  ctypes.byref(ln)):
            raise ValueError(self.L.o2_last_error().decode())
        return out, int(ln.value)


def draw_word(seed, ant, it, slot):
    return int(o2lib().o2_draw_word(seed, ant, it, slot))


def euc2d(x1, y1, x2, y2):
    return int(o2lib().o2_euc2d(x1, y1, x2, y2))


def power(e, x):
    return float(o2lib().o2_power(e, x))


def cycle_length(xs, ys, order):
    xs = np.ascontiguousarray(xs, np.float64)
    ys = np.ascontiguousarray(ys, np.float64)
    o = np.ascontiguousarray(order, np.uint32)
    return int(o2lib().o2_cycle_length(_p(xs, c_double), _p(ys, c_double), xs.size, _p(o, c_uint32)))


def knn_brute(xs, ys, k):
    xs = np.ascontiguousarray(xs, np.float64)
    ys = np.ascontiguousarray(ys, np.float64)
    out = np.empty((xs.size, k), np.uint32)
    o2lib().o2_knn_brute(_p(xs, c_double), _p(ys, c_double), xs.size, k, _p(out, c_uint32))
    return out


def knn_rows(xs, ys, k, rows):
    xs = np.ascontiguousarray(xs, np.float64)
    ys = np.ascontiguousarray(ys, np.float64)
    r = np.ascontiguousarray(rows, np.uint32)
    out = np.empty((r.size, k), np.uint32)
    o2lib().o2_knn_rows(_p(xs, c_double), _p(ys, c_double), xs.size, k, _p(r, c_uint32), r.size, _p(out, c_uint32))
    return out


def roulette(w, word):
    w = np.ascontiguousarray(w, np.float32)
    tie = c_int32()
    lane = o2lib().o2_roulette(_p(w, ctypes.c_float), w.size, word, ctypes.byref(tie))
    return int(lane), bool(tie.value)


def philox(ctr, key):
    c = (c_uint32 * 4)(*ctr)
    k = (c_uint32 * 2)(*key)
    o = (c_uint32 * 4)()
    o2lib().o2_philox4x32_10(c, k, o)
    return list(o)


# ------------------------------------------------------------------ O1 (reference)

class RefRunParams(ctypes.Structure):
    _fields_ = [("ants", c_uint32), ("workers", c_uint32), ("iterations", c_uint64), ("seed", c_uint64),
                ("alpha", c_double), ("beta", c_double), ("partial_prob", c_double), ("max_mod_frac", c_double),
                ("two_opt_prob", c_double), ("two_opt_window", c_uint32), ("synchronous", c_uint32),
                ("rho", c_double), ("tau_max", c_double), ("tau0", c_double), ("time_budget_s", c_double),
                ("mode", c_int32), ("pad_", c_int32)]


_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def reflib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_PATH):
            raise FileNotFoundError(f"{REF_PATH} not built (needs /root/reference at build time)")
        L = ctypes.CDLL(REF_PATH)
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_euc2d.restype = c_int32
        L.ref_euc2d.argtypes = [c_double] * 4
        L.ref_power.restype = c_double
        L.ref_power.argtypes = [c_double, c_double]
        L.ref_tour_length.argtypes = [POINTER(c_double), POINTER(c_double), c_uint32, POINTER(c_uint32), c_uint32,
                                      POINTER(c_int64)]
        L.ref_eta_beta.argtypes = [POINTER(c_double), POINTER(c_double), c_uint32, c_double, POINTER(c_uint32),
                                   c_uint32, POINTER(c_double)]
        L.ref_colony_tau.argtypes = [POINTER(c_double), POINTER(c_double), c_uint32, c_uint32, POINTER(c_uint32),
                                     c_double, c_double, POINTER(c_uint32), c_uint32, POINTER(c_double),
                                     POINTER(c_double), POINTER(c_int64)]
        L.ref_offer_sequence.argtypes = [POINTER(c_double), POINTER(c_double), c_uint32, c_uint32,
                                         POINTER(c_uint32), POINTER(c_uint32), c_uint32, POINTER(c_uint8),
                                         POINTER(c_int64)]
        L.ref_stream_u64.argtypes = [c_uint64, c_uint64, c_uint64, POINTER(c_uint64)]
        L.ref_two_opt.argtypes = [POINTER(c_double), POINTER(c_double), c_uint32, POINTER(c_uint32), c_uint32,
                                  POINTER(c_uint32), POINTER(c_int64)]
        L.ref_classic_update.argtypes = [c_uint32, c_double, c_double, POINTER(c_uint32), POINTER(c_int64),
                                         c_uint32, c_uint32, POINTER(c_double)]
        L.ref_run.argtypes = [POINTER(c_double), POINTER(c_double), c_uint32, POINTER(RefRunParams),
                              POINTER(c_int64), POINTER(c_uint32), POINTER(c_uint64), POINTER(c_uint64),
                              POINTER(c_double)]
        L.ref_sample_select.argtypes = [POINTER(c_double), POINTER(c_double), c_uint32, c_uint32, c_double,
                                        c_double, c_double, c_double, c_uint64, c_uint32, c_double,
                                        POINTER(c_uint64), POINTER(c_uint64), POINTER(c_double)]
        _ref = L
    return _ref


def two_opt(xs, ys, order, window=0):
    xs = np.ascontiguousarray(xs, np.float64)
    ys = np.ascontiguousarray(ys, np.float64)
    o = np.array(order, dtype=np.uint32)
    d = o2lib().o2_two_opt(_p(xs, c_double), _p(ys, c_double), xs.size, _p(o, c_uint32), window)
    return o, int(d)


def ref_run(xs, ys, ants, iterations, alpha, beta, seed=1, mode="partial", workers=None, partial_prob=0.95,
            max_mod_frac=1.0, rho=0.1, tau_max=1.0, tau0=1.0, synchronous=True, time_budget_s=0.0,
            two_opt_prob=0.0, two_opt_window=0):
    L = reflib()
    xs = np.ascontiguousarray(xs, np.float64)
    ys = np.ascontiguousarray(ys, np.float64)
    p = RefRunParams(ants=ants, workers=workers or os.cpu_count() or 1, iterations=iterations, seed=seed,
                     alpha=alpha, beta=beta, partial_prob=partial_prob, max_mod_frac=max_mod_frac,
                     two_opt_prob=two_opt_prob, two_opt_window=two_opt_window, synchronous=1 if synchronous else 0,
                     rho=rho,
                     tau_max=tau_max, tau0=tau0, time_budget_s=time_budget_s, mode=MODES[mode])
    best = c_int64()
    tour = np.empty(xs.size, np.uint32)
    it, cmp_, wall = c_uint64(), c_uint64(), c_double()
    rc = L.ref_run(_p(xs, c_double), _p(ys, c_double), xs.size, ctypes.byref(p), ctypes.byref(best),
                   _p(tour, c_uint32), ctypes.byref(it), ctypes.byref(cmp_), ctypes.byref(wall))
    if rc:
        raise RuntimeError(L.ref_last_error().decode())
    return dict(best_length=best.value, best_tour=tour, iterations=it.value, comparisons=cmp_.value,
                wall_s=wall.value)


def ref_sample_select(xs, ys, m, alpha, beta, partial_prob, max_mod_frac, seed, threads, seconds):
    L = reflib()
    xs = np.ascontiguousarray(xs, np.float64)
    ys = np.ascontiguousarray(ys, np.float64)
    d, c, b = c_uint64(), c_uint64(), c_double()
    rc = L.ref_sample_select(_p(xs, c_double), _p(ys, c_double), xs.size, m, alpha, beta, partial_prob,
                             max_mod_frac, seed, threads, seconds, ctypes.byref(d), ctypes.byref(c), ctypes.byref(b))
    if rc:
        raise RuntimeError(L.ref_last_error().decode())
    return dict(decisions=d.value, comparisons=c.value, busy_s=b.value)


def ref_colony_tau(xs, ys, tours, tau0, alpha, rows=None, direct=False):
    """tau^alpha rows through the reference ColonyPheromone after installing `tours` in ant order."""
    L = reflib()
    xs = np.ascontiguousarray(xs, np.float64)
    ys = np.ascontiguousarray(ys, np.float64)
    t = np.ascontiguousarray(tours, np.uint32)
    m, n = t.shape
    r = np.arange(n, dtype=np.uint32) if rows is None else np.ascontiguousarray(rows, np.uint32)
    out = np.empty((r.size, n), np.float64)
    outd = np.empty((r.size, n), np.float64) if direct else None
    g = c_int64()
    rc = L.ref_colony_tau(_p(xs, c_double), _p(ys, c_double), n, m, _p(t, c_uint32), tau0, alpha, _p(r, c_uint32),
                          r.size, _p(out, c_double), _p(outd, c_double) if direct else None, ctypes.byref(g))
    if rc:
        raise RuntimeError(L.ref_last_error().decode())
    return (out, outd, g.value) if direct else (out, g.value)


def ref_offer_sequence(xs, ys, m, tours, ants):
    L = reflib()
    xs = np.ascontiguousarray(xs, np.float64)
    ys = np.ascontiguousarray(ys, np.float64)
    t = np.ascontiguousarray(tours, np.uint32)
    a = np.ascontiguousarray(ants, np.uint32)
    flags = np.empty(a.size, np.uint8)
    g = np.empty(a.size, np.int64)
    rc = L.ref_offer_sequence(_p(xs, c_double), _p(ys, c_double), xs.size, m, _p(t, c_uint32), _p(a, c_uint32),
                              a.size, _p(flags, c_uint8), _p(g, c_int64))
    if rc:
        raise ValueError(L.ref_last_error().decode())
    return flags, g


def ref_classic_update(n, rho, tau_init, tours, lens):
    """tours: (rounds, ntours, n); lens: (rounds, ntours)."""
    L = reflib()
    t = np.ascontiguousarray(tours, np.uint32)
    l = np.ascontiguousarray(lens, np.int64)
    rounds, ntours = l.shape
    out = np.empty((n, n), np.float64)
    rc = L.ref_classic_update(n, rho, tau_init, _p(t, c_uint32), _p(l, c_int64), ntours, rounds, _p(out, c_double))
    if rc:
        raise RuntimeError(L.ref_last_error().decode())
    return out


def ref_tour_length(xs, ys, order):
    L = reflib()
    xs = np.ascontiguousarray(xs, np.float64)
    ys = np.ascontiguousarray(ys, np.float64)
    o = np.ascontiguousarray(order, np.uint32)
    out = c_int64()
    rc = L.ref_tour_length(_p(xs, c_double), _p(ys, c_double), xs.size, _p(o, c_uint32), o.size, ctypes.byref(out))
    if rc == -2:
        raise ValueError(L.ref_last_error().decode())
    if rc:
        raise RuntimeError(L.ref_last_error().decode())
    return out.value


def ref_eta_beta(xs, ys, beta, pairs):
    L = reflib()
    xs = np.ascontiguousarray(xs, np.float64)
    ys = np.ascontiguousarray(ys, np.float64)
    p = np.ascontiguousarray(pairs, np.uint32).reshape(-1, 2)
    out = np.empty(p.shape[0], np.float64)
    rc = L.ref_eta_beta(_p(xs, c_double), _p(ys, c_double), xs.size, beta, _p(p, c_uint32), p.shape[0],
                        _p(out, c_double))
    if rc:
        raise RuntimeError(L.ref_last_error().decode())
    return out


def ref_stream_u64(seed, stream, count):
    out = np.empty(count, np.uint64)
    reflib().ref_stream_u64(seed, stream, count, _p(out, c_uint64))
    return out


def ref_two_opt(xs, ys, order, window=0):
    L = reflib()
    xs = np.ascontiguousarray(xs, np.float64)
    ys = np.ascontiguousarray(ys, np.float64)
    o = np.ascontiguousarray(order, np.uint32)
    out = np.empty(o.size, np.uint32)
    ln = c_int64()
    rc = L.ref_two_opt(_p(xs, c_double), _p(ys, c_double), xs.size, _p(o, c_uint32), window, _p(out, c_uint32),
                       ctypes.byref(ln))
    if rc:
        raise RuntimeError(L.ref_last_error().decode())
    return out, ln.value
