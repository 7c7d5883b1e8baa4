"""ctypes wrapper of the C oracle (oracle/idw_oracle.c).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs, never by the product package.  Functions take
a store (ours or the reference's ``LayoutStore``: anything with
``component_views()``, ``precision`` and ``count``) and reproduce the
reference strategies' results:

    predict(store, ...)          kernels.predict_block / run_naive / idw_predict_seq
    tiled(store, ...)            run_tiled (load_tile + tile_accumulate)
    nested_improved(store, ...)  run_nested_improved (strided lanes + tree)
    nested_original(store, ...)  run_nested_original (group trees + serial merge)
    truth(store, ...)            fp64 double-double "fsum" truth on the
                                 run-precision inputs (tests/oracle_idw.py)
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle_idw.so"

_lib = None


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def load() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        _lib = ctypes.CDLL(str(LIB))
        P, I64, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        for sfx, T in (("f32", ctypes.c_float), ("f64", ctypes.c_double)):
            getattr(_lib, f"oracle_predict_{sfx}").argtypes = [P, P, I64, I64, P, I64, P, I64, P, I64, I64, I, T, T, P]
            getattr(_lib, f"oracle_tiled_{sfx}").argtypes = [P, P, I64, I64, P, I64, P, I64, P, I64, I64, I64, I, T, T, P]
            getattr(_lib, f"oracle_nested_improved_{sfx}").argtypes = [P, P, I64, I64, P, I64, P, I64, P, I64, I64, I64, I, T, T, P]
            fn = getattr(_lib, f"oracle_nested_original_{sfx}")
            fn.argtypes = [P, P, I64, I64, P, I64, P, I64, P, I64, I64, I64, I, T, T, P]
            fn.restype = I64
            getattr(_lib, f"oracle_tree_{sfx}").argtypes = [P, P, P, P, I64]
        D = ctypes.c_double
        _lib.oracle_truth_f64.argtypes = [P, P, I64, I64, P, P, P, I64, D, D, P]
        _lib.oracle_truth_mt_f64.argtypes = [P, P, I64, P, P, P, I64, D, D, P, I]
        _lib.oracle_predict_mt.argtypes = [I, P, P, I64, P, I64, P, I64, P, I64, I64, I, D, D, P, I]
        _lib.oracle_nested_improved_mt.argtypes = [I, P, P, I64, P, I64, P, I64, P, I64, I64, I64, I, D, D, P, I]
        _lib.oracle_max_threads.restype = I
    return _lib


def max_threads() -> int:
    return int(load().oracle_max_threads())


def _dtype(store) -> np.dtype:
    return np.dtype(np.float64 if store.precision.value == "double" else np.float32)


def _views(store):
    dt = _dtype(store)
    out = []
    for v in store.component_views():
        assert v.dtype == dt
        out.append((v.ctypes.data, v.strides[0] // dt.itemsize))
    return out


def _queries(queries, dt):
    qs = np.asarray(queries, dtype=np.float64).reshape(-1, 2)
    return (np.ascontiguousarray(qs[:, 0].astype(dt)), np.ascontiguousarray(qs[:, 1].astype(dt)))


def _scalars(p, zero_eps, dt):
    """kernels.scalar_args (kernels.py:20-24): fast, wexp, eps in the run dtype."""
    return int(p == 2.0), float(dt.type(-p / 2.0)), float(dt.type(zero_eps))


def _sfx(dt) -> str:
    return "f64" if dt == np.float64 else "f32"


def predict(store, queries, p=2.0, zero_eps=0.0) -> np.ndarray:
    dt = _dtype(store)
    qx, qy = _queries(queries, dt)
    out = np.empty(qx.shape[0], dt)
    (x, sx), (y, sy), (z, sz) = _views(store)
    fast, wexp, eps = _scalars(p, zero_eps, dt)
    getattr(load(), f"oracle_predict_{_sfx(dt)}")(qx.ctypes.data, qy.ctypes.data, 0, qx.shape[0], x, sx, y, sy,
                                                  z, sz, store.count, fast, wexp, eps, out.ctypes.data)
    return out


def tiled(store, queries, p=2.0, zero_eps=0.0, tile=1024) -> np.ndarray:
    dt = _dtype(store)
    qx, qy = _queries(queries, dt)
    out = np.empty(qx.shape[0], dt)
    (x, sx), (y, sy), (z, sz) = _views(store)
    fast, wexp, eps = _scalars(p, zero_eps, dt)
    getattr(load(), f"oracle_tiled_{_sfx(dt)}")(qx.ctypes.data, qy.ctypes.data, 0, qx.shape[0], x, sx, y, sy,
                                                z, sz, store.count, tile, fast, wexp, eps, out.ctypes.data)
    return out


def nested_improved(store, queries, p=2.0, zero_eps=0.0, group=1024) -> np.ndarray:
    dt = _dtype(store)
    qx, qy = _queries(queries, dt)
    out = np.empty(qx.shape[0], dt)
    (x, sx), (y, sy), (z, sz) = _views(store)
    fast, wexp, eps = _scalars(p, zero_eps, dt)
    getattr(load(), f"oracle_nested_improved_{_sfx(dt)}")(qx.ctypes.data, qy.ctypes.data, 0, qx.shape[0], x, sx,
                                                          y, sy, z, sz, store.count, group, fast, wexp, eps,
                                                          out.ctypes.data)
    return out


def nested_original(store, queries, p=2.0, zero_eps=0.0, group=1024):
    """Returns (predictions, merge count)."""
    dt = _dtype(store)
    qx, qy = _queries(queries, dt)
    out = np.empty(qx.shape[0], dt)
    (x, sx), (y, sy), (z, sz) = _views(store)
    fast, wexp, eps = _scalars(p, zero_eps, dt)
    merges = getattr(load(), f"oracle_nested_original_{_sfx(dt)}")(
        qx.ctypes.data, qy.ctypes.data, 0, qx.shape[0], x, sx, y, sy, z, sz, store.count, group, fast, wexp, eps,
        out.ctypes.data)
    return out, int(merges)


def run(strategy: str, store, queries, p=2.0, zero_eps=0.0, group=1024, tile=None) -> np.ndarray:
    """Oracle result of a reference strategy name (STRATEGIES keys)."""
    if strategy in ("naive", "seq"):
        return predict(store, queries, p, zero_eps)
    if strategy == "tiled":
        return tiled(store, queries, p, zero_eps, tile or group)
    if strategy == "nested_improved":
        return nested_improved(store, queries, p, zero_eps, group)
    if strategy == "nested_original":
        return nested_original(store, queries, p, zero_eps, group)[0]
    raise ValueError(strategy)


def tree(wp, wzp, hitp, hzp) -> None:
    dt = wp.dtype
    getattr(load(), f"oracle_tree_{_sfx(dt)}")(wp.ctypes.data, wzp.ctypes.data, hitp.ctypes.data, hzp.ctypes.data,
                                               wp.shape[0])


def truth(store, queries, p=2.0, zero_eps=0.0, threads: int | None = None) -> np.ndarray:
    """fp64 double-double truth on the store's run-precision values."""
    xs, ys, zs = (np.ascontiguousarray(v, dtype=np.float64) for v in store.component_views())
    dt = _dtype(store)
    qx, qy = (a.astype(np.float64) for a in _queries(queries, dt))
    out = np.empty(qx.shape[0], np.float64)
    eps = float(dt.type(zero_eps))
    load().oracle_truth_mt_f64(qx.ctypes.data, qy.ctypes.data, qx.shape[0], xs.ctypes.data, ys.ctypes.data,
                               zs.ctypes.data, store.count, float(p), eps, out.ctypes.data,
                               threads or max_threads())
    return out


def predict_mt(store, queries, p=2.0, zero_eps=0.0, threads: int | None = None) -> np.ndarray:
    """run_naive semantics on `threads` host threads (bench CPU baseline)."""
    dt = _dtype(store)
    qx, qy = _queries(queries, dt)
    out = np.empty(qx.shape[0], dt)
    (x, sx), (y, sy), (z, sz) = _views(store)
    fast, wexp, eps = _scalars(p, zero_eps, dt)
    load().oracle_predict_mt(int(dt == np.float64), qx.ctypes.data, qy.ctypes.data, qx.shape[0], x, sx, y, sy, z,
                             sz, store.count, fast, wexp, eps, out.ctypes.data, threads or max_threads())
    return out


def nested_improved_mt(store, queries, p=2.0, zero_eps=0.0, group=1024, threads: int | None = None):
    dt = _dtype(store)
    qx, qy = _queries(queries, dt)
    out = np.empty(qx.shape[0], dt)
    (x, sx), (y, sy), (z, sz) = _views(store)
    fast, wexp, eps = _scalars(p, zero_eps, dt)
    load().oracle_nested_improved_mt(int(dt == np.float64), qx.ctypes.data, qy.ctypes.data, qx.shape[0], x, sx, y,
                                     sy, z, sz, store.count, group, fast, wexp, eps, out.ctypes.data,
                                     threads or max_threads())
    return out


if os.environ.get("IDW_ORACLE_REBUILD"):
    build()
