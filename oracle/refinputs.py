"""Benchmark inputs for the CPU legs of bench.py, built without the product.

TEST INFRASTRUCTURE ONLY (see oracle.py).  The reference arm of bench.py
(`--impl reference`) must not import the product package or map its
library, so the inputs it times are generated and laid out here:

    cloud(n, seed)          the reference's splitmix64 cloud
                            (bench.py:37-63: word k = mix(seed + k*gamma),
                            top 53 bits -> [0,1), record-major x, y, z)
    query_seed(seed)        bench.py:75-77
    OracleStore(...)        the layout bytes of layouts.LayoutStore.from_arrays
                            (layouts.py:85-104,172-186) with strided
                            component views, the only thing the oracle reads

Pinned against the product generator and packers by tests/test_host.py.
"""

from __future__ import annotations

import numpy as np

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _words(seed: int, count: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + np.arange(1, count + 1, dtype=np.uint64) * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def cloud(n: int, seed: int):
    """(x, y, z) float64 arrays: x, y in [0, 1), z in [0, 100)."""
    u = (_words(seed, 3 * n) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    u = u.reshape(n, 3)
    return u[:, 0].copy(), u[:, 1].copy(), u[:, 2] * 100.0


def query_seed(seed: int) -> int:
    return (seed + 1) & 0xFFFFFFFFFFFFFFFF


class _Prec:
    def __init__(self, value: str):
        self.value = value


# record strides in elements and component offsets (layouts.py:3-21)
_GEOM = {
    "soa": None,
    "aos": (3, (0, 1, 2)),
    "aoas": (4, (0, 1, 2)),
}


class OracleStore:
    """Minimal store for oracle.* : precision, count, component_views()."""

    def __init__(self, x, y, z, layout: str, precision: str):
        dt = np.float32 if precision == "single" else np.float64
        self.precision = _Prec(precision)
        self.count = int(len(x))
        cols = [np.asarray(c, np.float64).astype(dt) for c in (x, y, z)]
        if layout == "soa":
            self.buffers = cols
            self._views = cols
        elif layout in _GEOM:
            stride, offs = _GEOM[layout]
            rec = np.zeros((self.count, stride), dt)
            for c, o in zip(cols, offs):
                rec[:, o] = c
            self.buffers = [rec]
            self._views = [rec[:, o] for o in offs]
        else:  # soaos / hybrid: fp64 xy pairs + z column (values are what matter here)
            xy = np.zeros((self.count, 2), dt)
            xy[:, 0], xy[:, 1] = cols[0], cols[1]
            zc = cols[2]
            self.buffers = [xy, zc]
            self._views = [xy[:, 0], xy[:, 1], zc]

    def component_views(self):
        return tuple(self._views)


def bench_inputs(n: int, m: int, layout: str, precision: str):
    """(store, (m, 2) float64 queries) of a bench config: data seed 0, query seed 1."""
    x, y, z = cloud(n, 0)
    qx, qy, _ = cloud(m, query_seed(0))
    return OracleStore(x, y, z, layout, precision), np.column_stack([qx, qy])
