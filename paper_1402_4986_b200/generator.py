"""Synthetic point clouds: the splitmix64 generator of the reference's bench
harness (reference bench.py:32-77), bit-for-bit.

Stream for seed s: word k (k = 1, 2, ...) is mix(s + k * 0x9E3779B97F4A7C15)
with the 30/27/31 xor-multiply finaliser; uniform doubles take the top 53
bits; clouds consume words record-major (x0, y0, z0, x1, ...).  Pinned by
the published splitmix64 vectors and the reference's golden 10K sums
(tests/golden/).
"""

from __future__ import annotations

import numpy as np

from .core import PointRecord

K = 1024  # bench.py:30

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, count: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + np.arange(1, count + 1, dtype=np.uint64) * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def uniform01(seed: int, count: int) -> np.ndarray:
    return (splitmix64(seed, count) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def generate_cloud_arrays(n: int, seed: int, bounds=(0.0, 1.0, 0.0, 1.0), value_range=(0.0, 100.0)):
    if n < 1:
        raise ValueError("no data points")
    u = uniform01(seed, 3 * n).reshape(n, 3)
    xlo, xhi, ylo, yhi = bounds
    zlo, zhi = value_range
    return (xlo + u[:, 0] * (xhi - xlo), ylo + u[:, 1] * (yhi - ylo), zlo + u[:, 2] * (zhi - zlo))


def generate_cloud(n: int, seed: int, bounds=(0.0, 1.0, 0.0, 1.0), value_range=(0.0, 100.0)) -> list:
    x, y, z = generate_cloud_arrays(n, seed, bounds, value_range)
    return [PointRecord(float(a), float(b), float(c)) for a, b, c in zip(x, y, z)]


def query_seed(seed: int) -> int:
    return (seed + 1) & 0xFFFFFFFFFFFFFFFF
