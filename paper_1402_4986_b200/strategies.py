"""The four IDW strategies as a drop-in for ``idwlayout.strategies``.

Names, signatures, validation, error messages, read-counter formulas and
``RunStats`` semantics follow the reference (strategies.py:1-269).  What runs
underneath is one blocking call into libidw_b200 per strategy call:

    run_naive            K1  one query per thread             (kernels.py:34-67)
    run_tiled            K2  smem tiles via cp.async.bulk     (kernels.py:70-108)
    run_nested_improved  K3  G strided lanes + shuffle tree   (kernels.py:111-185)
    run_nested_original  K4  per-group tree + serial merge    (kernels.py:188-248)

``ExecConfig`` gains four GPU knobs with reference-neutral defaults:

    mode    "exact" (default; env IDW_MODE) -- IEEE RN ops in the reference's
            order: p = 2 results are bit-identical to the reference;
            "fast"  -- MUFU/FMA/f32x2 arithmetic, blocked compensated sums,
            exact fix-up of coincident queries; held to the tolerance table.
    device  CUDA ordinal (default env IDW_DEVICE or 0)
    devices device list (default env IDW_DEVICES="0,1,..." or none): one host
            thread drives them all from the one call -- the store goes to
            devices[0] once and on by a peer-copy broadcast tree, entry k
            evaluates the k-th 256-aligned query shard on its own stream and
            writes its slice of the result.  This is the reference's worker
            pool (``parallel_width`` threads over static query blocks,
            strategies.py:41-66,137-145) with GPUs as the workers; results
            are bit-identical for every list (repeats allowed).
    splits  FAST tiled summation chunks (0 = auto: a function of n alone).
            A nonzero value fixes the chunk count instead; it is part of the
            summation order, so it changes the FAST bits (still within the
            tolerance) -- nothing else the caller sets does.

``parallel_width`` is accepted and validated for compatibility; GPU results do
not depend on it.  ``tile_size`` is validated and kept for the read counters
(tiled: ceil(m/G)*n per component, as the reference counts them) but the GPU
tiles are fixed by the kernels (fp32 256 points, fp64 128): K2's arithmetic
does not change with it, so results never depend on it.
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np

from . import _capi
from .core import Params, Precision, as_query_array, ensure_finite

_MODES = ("exact", "fast")


@dataclass(frozen=True)
class ExecConfig:
    """Strategy parameters (reference strategies.py:41-66) plus GPU knobs."""

    group_size: int = 1024
    tile_size: int | None = None
    parallel_width: int | None = None
    deterministic_reduction: bool = True
    mode: str | None = None
    device: int | None = None
    splits: int = 0
    devices: tuple | None = None

    def __post_init__(self) -> None:
        if self.group_size < 1:
            raise ValueError("group_size must be >= 1")
        if self.tile_size is None:
            object.__setattr__(self, "tile_size", self.group_size)
        if self.tile_size < 1:
            raise ValueError("tile_size must be >= 1")
        if self.parallel_width is None:
            object.__setattr__(self, "parallel_width", os.cpu_count() or 1)
        if self.parallel_width < 1:
            raise ValueError("parallel_width must be >= 1")
        if self.mode is None:
            object.__setattr__(self, "mode", os.environ.get("IDW_MODE", "exact"))
        if self.mode not in _MODES:
            raise ValueError(f"mode must be one of {_MODES}")
        if self.device is None:
            object.__setattr__(self, "device", int(os.environ.get("IDW_DEVICE", "0")))
        if self.splits < 0:
            raise ValueError("splits must be >= 0")
        if self.devices is None and os.environ.get("IDW_DEVICES"):
            object.__setattr__(self, "devices",
                               tuple(int(d) for d in os.environ["IDW_DEVICES"].split(",") if d.strip()))
        if self.devices is not None:
            devs = tuple(int(d) for d in self.devices)
            if not devs or len(devs) > _capi.MAX_DEVICES or min(devs) < 0:
                raise ValueError(f"devices must list 1..{_capi.MAX_DEVICES} device ordinals >= 0")
            object.__setattr__(self, "devices", devs)


@dataclass
class Accumulator:
    """Partial state: weight sum, weighted-value sum, lowest coincident index."""

    sum_w: float = 0.0
    sum_wz: float = 0.0
    hit_index: int | None = None


def merge_accumulators(a: Accumulator, b: Accumulator) -> Accumulator:
    hits = [h for h in (a.hit_index, b.hit_index) if h is not None]
    return Accumulator(a.sum_w + b.sum_w, a.sum_wz + b.sum_wz, min(hits) if hits else None)


def reduce_tree(partials: Sequence[Accumulator]) -> Accumulator:
    """Adjacent-pair levels ((a+b)+(c+d)); an odd tail rides up unchanged.
    Same shape as the in-kernel pow2-padded tree (reference strategies.py:89-101)."""
    level = list(partials)
    if not level:
        raise ValueError("empty reduction")
    while len(level) > 1:
        nxt = [merge_accumulators(level[i], level[i + 1]) for i in range(0, len(level) - 1, 2)]
        if len(level) & 1:
            nxt.append(level[-1])
        level = nxt
    return level[0]


@dataclass
class RunStats:
    """Per-run instrumentation (reference strategies.py:104-115).

    merge_events: shared-accumulator merges (nested_original; 0 otherwise).
    worker_trips: strided-loop slots per worker of one group (nested_improved).
    The GPU-only fields report what the native call did.
    """

    merge_events: int = 0
    worker_trips: np.ndarray | None = None
    kernel_launches: int = 0
    kernel_ms: float = 0.0
    fixup_queries: int = 0


def strategy_tolerance(precision: Precision, n: int) -> float:
    """Max relative error vs the double sequential oracle (strategies.py:118-122)."""
    if precision is Precision.double:
        return 1e-9
    return 1e-4 if n <= 256 else 1e-3


# ---------------------------------------------------------------------------
def _store_codes(store) -> tuple:
    """(kind value, precision value) of our store or a reference LayoutStore."""
    return store.kind.value, store.precision.value


def _prepare(store, queries, params: Params):
    """Validation and casts of reference strategies._prepare (:125-134)."""
    qs = as_query_array(queries)
    ensure_finite(qs)
    if store.count == 0:
        raise ValueError("no data points")
    dt = np.dtype(np.float64 if store.precision.value == "double" else np.float32)
    qx = np.ascontiguousarray(qs[:, 0].astype(dt, copy=False))
    qy = np.ascontiguousarray(qs[:, 1].astype(dt, copy=False))
    return qx, qy, dt


def _native_store(store) -> _capi.IdwStore:
    kind, prec = _store_codes(store)
    ptrs, sizes = [], []
    for buf in store.buffers:
        arr = np.ascontiguousarray(buf)
        if arr is not buf:
            raise ValueError("store buffers must be contiguous")
        ptrs.append(arr.ctypes.data)
        sizes.append(arr.nbytes)
    return _capi.make_store(kind, prec, store.count, ptrs, sizes)


def _dispatch(variant: str, store, queries, params: Params, cfg: ExecConfig):
    """One blocking native call.  The query array goes to the device as the
    reference's (m, 2) float64 pairs (idw_run_xy): the finiteness test and the
    run-dtype cast of _prepare run there, with the same ValueError."""
    qs = as_query_array(queries)
    dt = np.dtype(np.float64 if store.precision.value == "double" else np.float32)
    if store.count == 0 or qs.shape[0] == 0:
        _prepare(store, qs, params)  # reference order: invalid coordinate, then no data points
        return np.empty(qs.shape[0], dtype=dt), None
    qs = np.ascontiguousarray(qs)
    out = np.empty(qs.shape[0], dtype=dt)
    prm = _capi.make_params(params.p, params.zero_eps, variant, cfg.mode, cfg.group_size,
                            cfg.tile_size, cfg.splits, cfg.device, cfg.devices)
    try:
        stats = _capi.run_host_xy(_native_store(store), qs, prm, out)
    except _capi.NativeError:
        # the input's own error outranks a device failure (e.g. no GPU):
        # report what the reference would raise, if anything
        _prepare(store, qs, params)
        raise
    return out, stats


def _copy_gpu_stats(instrumentation, st) -> None:
    if instrumentation is not None and st is not None:
        instrumentation.kernel_launches = int(st.kernel_launches)
        instrumentation.kernel_ms = float(st.kernel_ms)
        instrumentation.fixup_queries = int(st.fixup_queries)


def run_naive(store, queries, params: Params = Params(), cfg: ExecConfig | None = None,
              instrumentation: RunStats | None = None) -> np.ndarray:
    """Flat parallelism: one GPU thread per query scans all n points (K1)."""
    cfg = cfg or ExecConfig()
    out, st = _dispatch("naive", store, queries, params, cfg)
    m, n = out.shape[0], store.count
    if m:
        store.stats.add_reads(m * n, m * n, m * n)  # strategies.py:163
    _copy_gpu_stats(instrumentation, st)
    return out


def run_tiled(store, queries, params: Params = Params(), cfg: ExecConfig | None = None,
              instrumentation: RunStats | None = None) -> np.ndarray:
    """Query groups against shared-memory data tiles (K2).  Reads are counted
    as the reference's load_tile does: once per element per query group."""
    cfg = cfg or ExecConfig()
    out, st = _dispatch("tiled", store, queries, params, cfg)
    m, n = out.shape[0], store.count
    if m:
        groups = -(-m // cfg.group_size)
        store.stats.add_reads(groups * n, groups * n, groups * n)  # layouts.py:228 via :193
    _copy_gpu_stats(instrumentation, st)
    return out


def run_nested_original(store, queries, params: Params = Params(), cfg: ExecConfig | None = None,
                        instrumentation: RunStats | None = None) -> np.ndarray:
    """Per-group trees merged serially into one accumulator per query (K4)."""
    cfg = cfg or ExecConfig()
    out, st = _dispatch("nested_original", store, queries, params, cfg)
    m, n = out.shape[0], store.count
    if m:
        store.stats.add_reads(m * n, m * n, m * n)
    if instrumentation is not None:
        instrumentation.merge_events = m * (-(-n // cfg.group_size)) if m else 0
    _copy_gpu_stats(instrumentation, st)
    return out


def run_nested_improved(store, queries, params: Params = Params(), cfg: ExecConfig | None = None,
                        instrumentation: RunStats | None = None) -> np.ndarray:
    """G strided lanes per query, one adjacent-pair tree, no merges (K3)."""
    cfg = cfg or ExecConfig()
    G = cfg.group_size
    trips = np.zeros(G, dtype=np.int64)
    if instrumentation is not None:
        instrumentation.merge_events = 0
        instrumentation.worker_trips = trips
    out, st = _dispatch("nested_improved", store, queries, params, cfg)
    m, n = out.shape[0], store.count
    if m:
        trips[:] = -(-n // G)  # every worker runs ceil(n/G) strided slots
        store.stats.add_reads(m * n, m * n, m * n)
    _copy_gpu_stats(instrumentation, st)
    return out


STRATEGIES: dict[str, Callable] = {
    "naive": run_naive,
    "tiled": run_tiled,
    "nested_original": run_nested_original,
    "nested_improved": run_nested_improved,
}
