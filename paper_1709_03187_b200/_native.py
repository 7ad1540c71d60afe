"""ctypes binding of the C ABI in include/paco_b200.h.

The shared library is built in-tree (paper_1709_03187_b200/_lib/libpaco_b200.so,
see build.py). There is no CPU fallback: if the library is missing, loading fails
loudly, and every compute entry point returns PACO_E_CUDA without an sm_100 GPU.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_uint8, c_uint32, c_uint64

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib")
LIB_PATH = os.environ.get("PACO_B200_LIB") or os.path.join(LIB_DIR, "libpaco_b200.so")

PACO_OK = 0
PACO_E_RUNTIME = -1
PACO_E_INVALID = -2
PACO_E_CUDA = -3
PACO_E_UNSUPPORTED = -4
PACO_E_LOGIC = -5

MODE_PARTIAL, MODE_PACO, MODE_CLASSIC = 0, 1, 2
DRAWS_PHILOX, DRAWS_BUFFER = 0, 1
RULE_CANDIDATE_ROULETTE, RULE_INDEPENDENT_ROULETTE = 0, 1

# every symbol include/paco_b200.h declares
EXPORTED = (
    "paco_last_error", "paco_version", "paco_config_default", "paco_config_validate", "paco_create",
    "paco_destroy", "paco_iterate", "paco_set_draws", "paco_get_tours", "paco_get_l_best",
    "paco_get_g_best", "paco_get_counters", "paco_get_build_flags", "paco_get_candidates",
    "paco_get_timing", "paco_offer_tour", "paco_construct_at", "paco_run", "paco_run_traced",
    "paco_release_cached_memory", "paco_rng_jump",
)


class Config(ctypes.Structure):
    _fields_ = [
        ("ants", c_uint32), ("workers", c_uint32), ("iterations", c_uint64),
        ("alpha", c_double), ("beta", c_double), ("partial_prob", c_double), ("max_mod_frac", c_double),
        ("two_opt_prob", c_double), ("two_opt_window", c_uint32), ("synchronous", c_uint32),
        ("seed", c_uint64), ("rho", c_double), ("tau_max", c_double), ("tau0", c_double),
        ("time_budget_s", c_double), ("convergence_interval_s", c_double), ("validate_tours", c_uint32),
        ("candidates", c_uint32), ("draws", c_uint32), ("device", c_int32), ("rule", c_uint32),
    ]


class Counters(ctypes.Structure):
    _fields_ = [(name, c_uint64) for name in (
        "decisions", "fallbacks", "ties", "forced", "full_builds", "partial_builds", "iterations",
        "improvements", "comparisons", "two_opts", "two_opt_moves")]

    def as_dict(self) -> dict:
        return {name: int(getattr(self, name)) for name, _ in self._fields_}


class Sample(ctypes.Structure):
    _fields_ = [("elapsed_s", c_double), ("g_best_length", c_int64), ("iterations_done", c_uint64)]


class Report(ctypes.Structure):
    _fields_ = [
        ("best_length", c_int64), ("pct_error", c_double), ("wall_time_s", c_double),
        ("iterations_done", c_uint64), ("comparisons_total", c_uint64), ("counters", Counters),
        ("construct_ms", c_double), ("update_ms", c_double), ("setup_ms", c_double),
    ]


class PacoError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"[{status}] {message}")
        self.status = status


class InvalidArgument(PacoError, ValueError):
    """std::invalid_argument analogue."""


class LogicError(PacoError):
    """std::logic_error analogue."""


_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`; "
                          "the engine has no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    vp = ctypes.c_void_p
    P = POINTER
    sig = {
        "paco_last_error": (c_char_p, []),
        "paco_version": (c_int, []),
        "paco_release_cached_memory": (c_int, [c_int]),
        "paco_rng_jump": (c_int, [P(ctypes.c_uint64), ctypes.c_uint64, P(ctypes.c_uint64)]),
        "paco_config_default": (c_int, [P(Config)]),
        "paco_config_validate": (c_int, [P(Config), c_uint32, c_int]),
        "paco_create": (c_int, [P(c_double), P(c_double), c_uint32, P(Config), c_int, P(vp)]),
        "paco_destroy": (None, [vp]),
        "paco_iterate": (c_int, [vp, c_uint64]),
        "paco_set_draws": (c_int, [vp, P(c_uint32), c_uint64]),
        "paco_get_tours": (c_int, [vp, P(c_uint32), P(c_int64)]),
        "paco_get_l_best": (c_int, [vp, P(c_uint32), P(c_int64)]),
        "paco_get_g_best": (c_int, [vp, P(c_uint32), P(c_int64)]),
        "paco_get_counters": (c_int, [vp, P(Counters)]),
        "paco_get_build_flags": (c_int, [vp, P(c_uint8), P(c_uint8)]),
        "paco_get_candidates": (c_int, [vp, P(c_uint32), P(ctypes.c_float), P(c_uint32)]),
        "paco_get_timing": (c_int, [vp, P(c_double), P(c_double), P(c_double)]),
        "paco_offer_tour": (c_int, [vp, c_uint32, P(c_uint32), P(c_int)]),
        "paco_construct_at": (c_int, [vp, c_uint32, c_uint32, c_uint32, P(c_uint32), c_uint64, P(c_uint32),
                                      P(c_int64)]),
        "paco_run": (c_int, [P(c_double), P(c_double), c_uint32, P(Config), c_int, c_int64, P(Report),
                             P(c_uint32)]),
        "paco_run_traced": (c_int, [P(c_double), P(c_double), c_uint32, P(Config), c_int, c_int64, P(Report),
                                    P(c_uint32), P(Sample), c_uint32, P(c_uint32)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int) -> None:
    if status == PACO_OK:
        return
    msg = load().paco_last_error().decode(errors="replace")
    if status == PACO_E_INVALID:
        raise InvalidArgument(status, msg)
    if status == PACO_E_LOGIC:
        raise LogicError(status, msg)
    raise PacoError(status, msg)
