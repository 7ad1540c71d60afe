"""B200-native tour construction for PartialACO (arXiv 1709.03187).

Python mirror of the reference's solver interface (paco::run and friends) over the
C ABI in include/paco_b200.h; the compute is hand-written sm_100a CUDA in csrc/.
"""
from .engine import (Colony, ConvergenceSample, Mode, RunConfig, RunReport, Tour, mode_from_name, mode_name,
                     release_cached_memory, run, run_timed_baseline)
from .instances import (CONFIGS, Instance, ParseError, cycle_length, emit_tsplib, euc2d, grid_instance,
                        is_permutation_of_n, load_optima, make_config_instance, parse_tsplib, tour_length)
from ._native import InvalidArgument, LogicError, PacoError

__all__ = [
    "Colony", "ConvergenceSample", "Mode", "RunConfig", "RunReport", "Tour", "mode_from_name", "mode_name",
    "release_cached_memory", "run",
    "run_timed_baseline", "CONFIGS", "Instance", "ParseError", "cycle_length", "emit_tsplib", "euc2d",
    "grid_instance", "is_permutation_of_n", "load_optima", "make_config_instance", "parse_tsplib", "tour_length",
    "InvalidArgument", "LogicError", "PacoError",
]
