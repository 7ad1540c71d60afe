"""Instances: coordinates, EUC_2D, tour validation, TSPLIB I/O and the synthetic
workloads of BASELINE.json.

Host-side mirror of /root/reference/proj/include/paco/instance.hpp (Instance
:41-101, euc2d :33-37, is_permutation_of_n :109-117, cycle_length :120-127,
tour_length :130-135, parse_tsplib :164-238, emit_tsplib :251-261,
load_optima :264-281). These run once per instance on the host; the per-iteration
work is on the GPU.
"""
from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field
from typing import Iterable, Optional, Sequence

import numpy as np

DIST_MATRIX_MAX_CITIES = 5000  # instance.hpp:23 (classic-mode cap)


class ParseError(RuntimeError):
    """instance.hpp:25-30: carries the 1-based line number."""

    def __init__(self, line: int, what: str):
        super().__init__(f"line {line}: {what}")
        self.line = line


def euc2d(x1: float, y1: float, x2: float, y2: float) -> int:
    """TSPLIB EUC_2D, nearest integer with .5 rounding up (instance.hpp:33-37)."""
    dx, dy = x1 - x2, y1 - y2
    return int(math.sqrt(dx * dx + dy * dy) + 0.5)


def euc2d_array(xs: np.ndarray, ys: np.ndarray, a: np.ndarray, b: np.ndarray) -> np.ndarray:
    dx = xs[a] - xs[b]
    dy = ys[a] - ys[b]
    return (np.sqrt(dx * dx + dy * dy) + 0.5).astype(np.int64)


@dataclass
class Instance:
    """Immutable city set (instance.hpp:41-101)."""

    name: str
    xs: np.ndarray
    ys: np.ndarray
    optimum: Optional[int] = None

    def __post_init__(self):
        self.xs = np.ascontiguousarray(self.xs, dtype=np.float64)
        self.ys = np.ascontiguousarray(self.ys, dtype=np.float64)
        if self.xs.shape != self.ys.shape or self.xs.ndim != 1:
            raise ValueError("xs and ys must be 1-D and of equal length")
        if self.xs.size < 3:
            raise ValueError(f"instance needs at least 3 cities, got {self.xs.size}")
        if self.optimum is not None and self.optimum <= 0:
            raise ValueError("known optimum must be positive")
        if not (np.isfinite(self.xs).all() and np.isfinite(self.ys).all()):
            raise ValueError("non-finite coordinate")

    @classmethod
    def from_coords(cls, name: str, coords: Sequence[tuple], optimum: Optional[int] = None) -> "Instance":
        arr = np.asarray(coords, dtype=np.float64).reshape(-1, 2)
        return cls(name, arr[:, 0].copy(), arr[:, 1].copy(), optimum)

    @property
    def n(self) -> int:
        return int(self.xs.size)

    def x(self, i: int) -> float:
        return float(self.xs[i])

    def y(self, i: int) -> float:
        return float(self.ys[i])

    def dist(self, i: int, j: int) -> int:
        return euc2d(self.xs[i], self.ys[i], self.xs[j], self.ys[j])

    def sha256(self) -> str:
        h = hashlib.sha256()
        h.update(self.xs.tobytes())
        h.update(self.ys.tobytes())
        return h.hexdigest()


def is_permutation_of_n(n: int, order) -> bool:
    """instance.hpp:109-117"""
    o = np.asarray(order)
    if o.size != n:
        return False
    if o.size and (o.min() < 0 or o.max() >= n):
        return False
    return np.unique(o).size == n


def cycle_length(inst: Instance, order) -> int:
    """instance.hpp:120-127 (int64 sum of rounded edges, closing edge included)."""
    o = np.asarray(order, dtype=np.int64)
    return int(euc2d_array(inst.xs, inst.ys, o, np.roll(o, -1)).sum())


def tour_length(inst: Instance, order) -> int:
    """instance.hpp:130-135: rejects non-permutations."""
    if not is_permutation_of_n(inst.n, order):
        raise ValueError(f"order is not a permutation of 0..{inst.n - 1}")
    return cycle_length(inst, order)


def parse_tsplib(text: str) -> Instance:
    """EUC_2D TSPLIB reader (instance.hpp:164-238), same error taxonomy."""
    name, dimension, ewt, in_coords = "unnamed", None, None, False
    coords: list = []
    line_no = 0
    for raw in text.splitlines():
        line_no += 1
        line = raw.strip()
        if not line:
            continue
        if line == "EOF":
            break
        if not in_coords:
            if line == "NODE_COORD_SECTION":
                if dimension is None:
                    raise ParseError(line_no, "NODE_COORD_SECTION before DIMENSION")
                if ewt is None:
                    raise ParseError(line_no, "missing EDGE_WEIGHT_TYPE header")
                in_coords = True
                continue
            if ":" not in line or not line.split(":", 1)[0].strip():
                raise ParseError(line_no, f"malformed header line: '{line}'")
            key, value = (s.strip() for s in line.split(":", 1))
            if key == "NAME":
                name = value
            elif key == "DIMENSION":
                try:
                    d = int(value)
                except ValueError:
                    raise ParseError(line_no, f"non-numeric DIMENSION: '{value}'") from None
                if d < 3:
                    raise ParseError(line_no, "DIMENSION must be at least 3")
                dimension = d
            elif key == "EDGE_WEIGHT_TYPE":
                if value != "EUC_2D":
                    raise ParseError(line_no, f"unsupported EDGE_WEIGHT_TYPE: '{value}' (only EUC_2D)")
                ewt = value
            continue
        if len(coords) == dimension:
            raise ParseError(line_no, f"more coordinate lines than DIMENSION {dimension}")
        fields = line.split()
        if len(fields) < 3:
            raise ParseError(line_no, f"expected 'id x y', got '{line}'")
        try:
            x, y = float(fields[1]), float(fields[2])
        except ValueError:
            raise ParseError(line_no, f"expected 'id x y', got '{line}'") from None
        if len(fields) > 3:
            raise ParseError(line_no, f"trailing content after coordinates: '{fields[3]}'")
        if not (math.isfinite(x) and math.isfinite(y)):
            raise ParseError(line_no, "non-finite coordinate")
        coords.append((x, y))
    if not in_coords:
        raise ParseError(line_no, "missing NODE_COORD_SECTION")
    if len(coords) != dimension:
        raise ParseError(line_no, f"DIMENSION is {dimension} but {len(coords)} coordinate lines were read")
    return Instance.from_coords(name, coords)


def emit_tsplib(inst: Instance) -> str:
    """instance.hpp:251-261 (17 significant digits)."""
    out = [f"NAME : {inst.name}", "TYPE : TSP", f"DIMENSION : {inst.n}", "EDGE_WEIGHT_TYPE : EUC_2D",
           "NODE_COORD_SECTION"]
    for i in range(inst.n):
        out.append(f"{i + 1} {inst.xs[i]:.17g} {inst.ys[i]:.17g}")
    out.append("EOF")
    return "\n".join(out) + "\n"


def load_optima(text: str) -> dict:
    """instance.hpp:264-281"""
    out = {}
    for line_no, raw in enumerate(text.splitlines(), 1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        f = line.split()
        try:
            v = int(f[1])
        except (IndexError, ValueError):
            v = 0
        if v <= 0:
            raise ParseError(line_no, f"expected 'instance-name optimum-length', got '{line}'")
        out[f[0]] = v
    return out


# ------------------------------------------------------------------ generators

def grid_instance(w: int, h: int, spacing: float = 10.0, name: str = "grid") -> Instance:
    """w x h lattice, row-major ids; for even w*h the optimum is w*h*spacing
    (the construction behind data/grid442.tsp, data/README.md:7-10)."""
    xs = np.tile(np.arange(w, dtype=np.float64) * spacing, h)
    ys = np.repeat(np.arange(h, dtype=np.float64) * spacing, w)
    opt = int(w * h * spacing) if (w * h) % 2 == 0 else None
    return Instance(name, xs, ys, opt)


def _uniform_int(rng: np.random.Generator, n: int, hi: int) -> np.ndarray:
    return rng.integers(0, hi + 1, size=n).astype(np.float64)


def _box_muller(rng: np.random.Generator, n: int) -> tuple:
    u1 = 1.0 - rng.random(n)  # (0, 1]
    u2 = rng.random(n)
    r = np.sqrt(-2.0 * np.log(u1))
    return r * np.cos(2 * np.pi * u2), r * np.sin(2 * np.pi * u2)


def _clusters(rng, n, nclusters, box, smin, smax):
    cx = rng.random(nclusters) * box
    cy = rng.random(nclusters) * box
    sig = smin + rng.random(nclusters) * (smax - smin)
    member = rng.integers(0, nclusters, size=n)  # uniform membership (BASELINE.json leaves it open)
    gx, gy = _box_muller(rng, n)
    x = np.clip(np.rint(cx[member] + sig[member] * gx), 0, box)
    y = np.clip(np.rint(cy[member] + sig[member] * gy), 0, box)
    return x, y


# BASELINE.json configs; instance seed = 1000 + config index
CONFIGS = {
    "C1": dict(n=1000, m=64, k=20, iterations=100, kind="uniform", box=100_000),
    "C2": dict(n=10_000, m=256, k=20, iterations=200, kind="uniform", box=1_000_000),
    "C3": dict(n=20_000, m=256, k=20, iterations=200, kind="clustered", box=1_000_000),
    "C4": dict(n=100_000, m=512, k=16, iterations=50, kind="uniform", box=10_000_000),
    "C5": dict(n=200_000, m=1024, k=16, iterations=20, kind="mixed", box=10_000_000),
}


def make_config_instance(cfg: str, n: Optional[int] = None) -> Instance:
    """Seeded synthetic stand-in for the paper's TSPLIB/art instances with the
    BASELINE.json shape. `n` overrides the size (same distribution) for tests."""
    spec = CONFIGS[cfg]
    idx = int(cfg[1])
    n = spec["n"] if n is None else n
    rng = np.random.Generator(np.random.PCG64(1000 + idx))
    box = spec["box"]
    if spec["kind"] == "uniform":
        x, y = _uniform_int(rng, n, box), _uniform_int(rng, n, box)
    elif spec["kind"] == "clustered":
        x, y = _clusters(rng, n, 50, box, 5_000, 40_000)
    else:
        nc = int(round(0.7 * n))
        x1, y1 = _clusters(rng, nc, 200, box, 20_000, 200_000)
        x2, y2 = _uniform_int(rng, n - nc, box), _uniform_int(rng, n - nc, box)
        x, y = np.concatenate([x1, x2]), np.concatenate([y1, y2])
    return Instance(f"{cfg.lower()}-{n}", x.astype(np.float64), y.astype(np.float64))
