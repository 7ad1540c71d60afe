"""Python mirror of the reference solver interface over the B200 C ABI.

Reference: /root/reference/proj/include/paco/engine.hpp -- Mode :24, mode_name /
mode_from_name :26-40, RunConfig :42-76, RunReport :84-92, run :156-333,
run_timed_baseline :339-344. Same names, same argument meaning, same errors
(ValueError for std::invalid_argument). Every call goes through
paper_1709_03187_b200/_lib/libpaco_b200.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes
import enum
import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _native as N
from .instances import Instance


class Mode(enum.IntEnum):
    partial_aco = N.MODE_PARTIAL
    paco_full = N.MODE_PACO
    classic_aco = N.MODE_CLASSIC


def mode_name(m: Mode) -> str:
    return {Mode.partial_aco: "partial", Mode.paco_full: "paco", Mode.classic_aco: "classic"}[Mode(m)]


def mode_from_name(s: str) -> Optional[Mode]:
    return {"partial": Mode.partial_aco, "paco": Mode.paco_full, "classic": Mode.classic_aco}.get(s)


@dataclass
class RunConfig:
    """engine.hpp:42-76, plus the north-star knobs `candidates` and `draws`."""

    ants: int = 16
    iterations: int = 100000
    alpha: float = 5.0
    beta: float = 5.0
    partial_prob: float = 0.95
    max_mod_frac: float = 1.0
    two_opt_prob: float = 0.0
    two_opt_window: int = 0
    workers: int = 8
    seed: int = 1
    rho: float = 0.1
    tau_max: float = 1.0
    tau0: float = 1.0
    time_budget_s: float = 0.0
    convergence_interval_s: float = 1.0
    synchronous: bool = True
    validate_tours: bool = False
    candidates: int = 16
    draws: str = "philox"  # or "buffer" (validation mode)
    device: int = -1
    rule: str = "roulette"  # north-star candidate-list roulette; "independent" = the reference's IR rule

    def to_c(self) -> N.Config:
        c = N.Config()
        for name, _ in N.Config._fields_:
            if name == "draws":
                c.draws = N.DRAWS_BUFFER if self.draws == "buffer" else N.DRAWS_PHILOX
            elif name == "rule":
                if self.rule not in ("roulette", "independent"):
                    raise ValueError(f"unknown rule {self.rule!r}")
                c.rule = N.RULE_INDEPENDENT_ROULETTE if self.rule == "independent" else N.RULE_CANDIDATE_ROULETTE
            else:
                setattr(c, name, getattr(self, name))
        return c

    def validate(self, n: int = 3, mode: Mode = Mode.partial_aco) -> None:
        """RunConfig::validate (engine.hpp:61-75) via the C ABI."""
        N.check(N.load().paco_config_validate(ctypes.byref(self.to_c()), n, int(mode)))


@dataclass
class ConvergenceSample:
    elapsed_s: float
    g_best_length: int
    iterations_done: int


@dataclass
class Tour:
    order: np.ndarray
    length: int


@dataclass
class RunReport:
    """engine.hpp:84-92 plus counters and device timings."""

    best_length: int = 0
    best_tour: Optional[Tour] = None
    pct_error: Optional[float] = None
    wall_time_s: float = 0.0
    iterations_done: int = 0
    comparisons_total: int = 0
    convergence: List[ConvergenceSample] = field(default_factory=list)
    counters: dict = field(default_factory=dict)
    construct_ms: float = 0.0
    update_ms: float = 0.0
    setup_ms: float = 0.0


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _u32(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


def _i64(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


class Colony:
    """A device-resident instance + colony (one paco_handle). Exposes the pieces
    run() composes, for tests and for callers that drive iterations themselves."""

    def __init__(self, inst: Instance, cfg: RunConfig, mode: Mode = Mode.partial_aco):
        self.lib = N.load()
        self.inst, self.cfg, self.mode = inst, cfg, Mode(mode)
        self._h = ctypes.c_void_p()
        c = cfg.to_c()
        N.check(self.lib.paco_create(_dptr(inst.xs), _dptr(inst.ys), inst.n, ctypes.byref(c), int(mode),
                                     ctypes.byref(self._h)))
        self.n, self.m = inst.n, cfg.ants
        self.k = min(cfg.candidates, inst.n - 1)

    def close(self):
        if self._h:
            self.lib.paco_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def iterate(self, count: int = 1) -> None:
        N.check(self.lib.paco_iterate(self._h, count))

    def set_draws(self, words: np.ndarray) -> None:
        w = np.ascontiguousarray(words, dtype=np.uint32)
        if w.ndim != 2 or w.shape[0] != self.m:
            raise ValueError("draw words must be an (ants, stride) array")
        N.check(self.lib.paco_set_draws(self._h, _u32(w), w.shape[1]))

    def tours(self):
        t = np.empty((self.m, self.n), np.uint32)
        l = np.empty(self.m, np.int64)
        N.check(self.lib.paco_get_tours(self._h, _u32(t), _i64(l)))
        return t, l

    def l_best(self):
        t = np.empty((self.m, self.n), np.uint32)
        l = np.empty(self.m, np.int64)
        N.check(self.lib.paco_get_l_best(self._h, _u32(t), _i64(l)))
        return t, l

    def g_best(self):
        t = np.empty(self.n, np.uint32)
        l = ctypes.c_int64()
        N.check(self.lib.paco_get_g_best(self._h, _u32(t), ctypes.byref(l)))
        return t, int(l.value)

    def counters(self) -> dict:
        c = N.Counters()
        N.check(self.lib.paco_get_counters(self._h, ctypes.byref(c)))
        return c.as_dict()

    def build_flags(self):
        p = np.empty(self.m, np.uint8)
        i = np.empty(self.m, np.uint8)
        N.check(self.lib.paco_get_build_flags(self._h, p.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)),
                                              i.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))))
        return p, i

    def candidates(self):
        knn = np.empty((self.n, self.k), np.uint32)
        w = np.empty((self.n, self.k), np.float32)
        k = ctypes.c_uint32()
        N.check(self.lib.paco_get_candidates(self._h, _u32(knn), w.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
                                             ctypes.byref(k)))
        return knn, w

    def timing(self):
        c, u, s = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        N.check(self.lib.paco_get_timing(self._h, ctypes.byref(c), ctypes.byref(u), ctypes.byref(s)))
        return c.value, u.value, s.value

    def offer_tour(self, ant: int, order) -> bool:
        o = np.ascontiguousarray(order, dtype=np.uint32)
        imp = ctypes.c_int()
        N.check(self.lib.paco_offer_tour(self._h, ant, _u32(o), ctypes.byref(imp)))
        return bool(imp.value)

    def construct_at(self, ant: int, start_pos: int, m_mod: int, words: np.ndarray):
        w = np.ascontiguousarray(words, dtype=np.uint32)
        out = np.empty(self.n, np.uint32)
        ln = ctypes.c_int64()
        N.check(self.lib.paco_construct_at(self._h, ant, start_pos, m_mod, _u32(w), w.size, _u32(out),
                                           ctypes.byref(ln)))
        return out, int(ln.value)


def release_cached_memory(device: int = -1) -> None:
    """Return the device memory of destroyed engines, kept in the device's stream-ordered
    pool for the next engine, to the driver (paco_release_cached_memory)."""
    N.check(N.load().paco_release_cached_memory(int(device)))


def run(inst: Instance, cfg: RunConfig, mode: Mode = Mode.partial_aco) -> RunReport:
    """paco::run (engine.hpp:156-333) on the B200 engine."""
    lib = N.load()
    rep = N.Report()
    best = np.empty(inst.n, np.uint32)
    opt = inst.optimum if inst.optimum else 0
    cap = 4096
    samples = (N.Sample * cap)()
    ns = ctypes.c_uint32()
    N.check(lib.paco_run_traced(_dptr(inst.xs), _dptr(inst.ys), inst.n, ctypes.byref(cfg.to_c()), int(mode), opt,
                                ctypes.byref(rep), _u32(best), samples, cap, ctypes.byref(ns)))
    out = RunReport(best_length=int(rep.best_length), best_tour=Tour(best, int(rep.best_length)),
                    pct_error=None if math.isnan(rep.pct_error) else float(rep.pct_error),
                    wall_time_s=float(rep.wall_time_s), iterations_done=int(rep.iterations_done),
                    comparisons_total=int(rep.comparisons_total), counters=rep.counters.as_dict(),
                    construct_ms=rep.construct_ms, update_ms=rep.update_ms, setup_ms=rep.setup_ms)
    out.convergence = [ConvergenceSample(float(x.elapsed_s), int(x.g_best_length), int(x.iterations_done))
                       for x in samples[:ns.value]]
    return out


def run_timed_baseline(inst: Instance, cfg: RunConfig, budget_s: float) -> RunReport:
    """engine.hpp:339-344"""
    if budget_s <= 0.0:
        raise N.InvalidArgument(N.PACO_E_INVALID, "budget must be positive")
    from dataclasses import replace
    return run(inst, replace(cfg, time_budget_s=budget_s), Mode.paco_full)
