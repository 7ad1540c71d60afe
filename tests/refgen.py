"""Test infrastructure: the reference test suite's instance generators, reproduced exactly.

The reference's tests draw their instances with std::mt19937_64 and
std::uniform_real_distribution<double> (tests/oracles.hpp:123-131, random_instance). The
generator below is the standard's mt19937_64 (seeded per [rand.eng.mt]) and libstdc++'s
generate_canonical<double, 53> (one 64-bit draw, converted to double, divided by 2^64,
clamped below 1), so tests/test_gpu_engine_behaviour.py runs on the very coordinates the
reference's test_engine.cpp uses. Pinned in tests/test_host.py against values printed by a
g++ build of the same calls.
"""
import math

import numpy as np

from paper_1709_03187_b200 import Instance

_M64 = (1 << 64) - 1


class MT19937_64:
    N, M = 312, 156
    A = 0xB5026F5AA96619E9
    UPPER, LOWER = 0xFFFFFFFF80000000, 0x7FFFFFFF

    def __init__(self, seed: int = 5489):
        self.x = [seed & _M64]
        for i in range(1, self.N):
            p = self.x[-1]
            self.x.append((6364136223846793005 * (p ^ (p >> 62)) + i) & _M64)
        self.i = self.N

    def _twist(self):
        x = self.x
        for k in range(self.N):
            y = (x[k] & self.UPPER) | (x[(k + 1) % self.N] & self.LOWER)
            x[k] = x[(k + self.M) % self.N] ^ (y >> 1) ^ (self.A if y & 1 else 0)
        self.i = 0

    def __call__(self) -> int:
        if self.i >= self.N:
            self._twist()
        y = self.x[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y


def uniform_real(gen: MT19937_64, a: float, b: float) -> float:
    r = float(gen()) / 18446744073709551616.0
    if r >= 1.0:
        r = math.nextafter(1.0, 0.0)
    return r * (b - a) + a


def random_instance(gen: MT19937_64, n: int, box: float = 1000.0, name: str = "random") -> Instance:
    """oracles.hpp:123-131. g++ evaluates the two emplace_back arguments right to left, so each
    point draws y first, then x."""
    xs = np.empty(n)
    ys = np.empty(n)
    for i in range(n):
        ys[i] = uniform_real(gen, 0.0, box)
        xs[i] = uniform_real(gen, 0.0, box)
    return Instance(name, xs, ys)


def held_karp(inst: Instance) -> int:
    """Exact optimum by the Held–Karp subset DP (the reference tests' oracle::held_karp), over
    TSPLIB EUC_2D distances; masks are processed layer by layer with numpy."""
    n = inst.n
    d = np.array([[inst.dist(i, j) for j in range(n)] for i in range(n)], np.int64)
    m = n - 1  # city 0 is the fixed start; bit k stands for city k + 1
    full = 1 << m
    inf = np.iinfo(np.int64).max // 4
    dp = np.full((full, m), inf, np.int64)
    for k in range(m):
        dp[1 << k, k] = d[0, k + 1]
    masks = np.arange(full)
    pop = np.array([bin(x).count("1") for x in range(full)])
    for size in range(1, m):
        layer = masks[pop == size]
        for j in range(m):
            src = layer[(layer >> j) & 1 == 1]
            for k in range(m):
                tgt = src[(src >> k) & 1 == 0]
                nxt = tgt | (1 << k)  # distinct for a fixed (j, k), so plain fancy indexing is safe
                dp[nxt, k] = np.minimum(dp[nxt, k], dp[tgt, j] + d[j + 1, k + 1])
    return int(min(dp[full - 1, j] + d[j + 1, 0] for j in range(m)))
