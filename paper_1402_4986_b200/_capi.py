"""ctypes binding of ``libidw_b200.so`` (declared in ``include/idw_b200.h``).

This is the only module that touches the native library.  It loads the
in-tree build (``paper_1402_4986_b200/libidw_b200.so``) and raises loudly when
it is missing or stale: the package has no CPU fallback, by design.  ctypes
releases the GIL for the duration of every call, like the reference's
``@njit(nogil=True)`` kernels (reference kernels.py:34).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

ABI_VERSION = 2

# enum codes -- include/idw_b200.h
KIND_CODES = {"soa": 0, "aos": 1, "aoas": 2, "soaos": 3, "hybrid": 4}  # layouts.py:65
PRECISION_CODES = {"single": 0, "double": 1}                            # layouts.py:66
VARIANT_CODES = {"naive": 0, "tiled": 1, "nested_original": 2, "nested_improved": 3}
MODE_CODES = {"exact": 0, "fast": 1}

_LIB_NAME = "libidw_b200.so"


class IdwStore(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("precision", ctypes.c_int32),
        ("count", ctypes.c_int64),
        ("nbuf", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("buf", ctypes.c_void_p * 3),
        ("nbytes", ctypes.c_int64 * 3),
    ]


class IdwParams(ctypes.Structure):
    _fields_ = [
        ("p", ctypes.c_double),
        ("zero_eps", ctypes.c_double),
        ("variant", ctypes.c_int32),
        ("mode", ctypes.c_int32),
        ("group_size", ctypes.c_int64),
        ("tile_size", ctypes.c_int64),
        ("splits", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("ndevices", ctypes.c_int32),
        ("devices", ctypes.c_int32 * 16),
    ]


class IdwStats(ctypes.Structure):
    _fields_ = [
        ("merge_events", ctypes.c_int64),
        ("kernel_launches", ctypes.c_int64),
        ("kernel_ms", ctypes.c_double),
        ("fixup_queries", ctypes.c_int64),
    ]


EXPORTS = ("idw_abi_version", "idw_device_count", "idw_last_error", "idw_run", "idw_run_xy",
           "idw_run_device", "idw_pack_device", "idw_convert_device", "idw_last_kernel_ms",
           "idw_mufu_peak", "idw_plan_create", "idw_plan_launch", "idw_plan_launches",
           "idw_plan_kernel_ms", "idw_plan_destroy")


class NativeError(RuntimeError):
    """A libidw_b200 call failed; the message is ``idw_last_error()``."""


def library_path() -> Path:
    override = os.environ.get("IDW_B200_LIB")
    if override:
        return Path(override)
    return Path(__file__).resolve().parent / _LIB_NAME


_lib = None


def load() -> ctypes.CDLL:
    """Load (once) and type the native library; raise if absent or stale."""
    global _lib
    if _lib is not None:
        return _lib
    path = library_path()
    if not path.exists():
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            f"or `make -C paper_1402_4986_b200/csrc` (there is no CPU fallback)")
    lib = ctypes.CDLL(str(path))
    lib.idw_abi_version.restype = ctypes.c_int
    lib.idw_abi_version.argtypes = []
    if lib.idw_abi_version() != ABI_VERSION:
        raise ImportError(f"{path}: ABI {lib.idw_abi_version()} != expected {ABI_VERSION}; rebuild")
    lib.idw_device_count.restype = ctypes.c_int
    lib.idw_device_count.argtypes = []
    lib.idw_last_error.restype = ctypes.c_char_p
    lib.idw_last_error.argtypes = []
    ptr = ctypes.c_void_p
    lib.idw_run.restype = ctypes.c_int
    lib.idw_run.argtypes = [ctypes.POINTER(IdwStore), ptr, ptr, ctypes.c_int64,
                            ctypes.POINTER(IdwParams), ptr, ctypes.POINTER(IdwStats)]
    lib.idw_run_xy.restype = ctypes.c_int
    lib.idw_run_xy.argtypes = [ctypes.POINTER(IdwStore), ptr, ctypes.c_int64,
                               ctypes.POINTER(IdwParams), ptr, ctypes.POINTER(IdwStats)]
    lib.idw_run_device.restype = ctypes.c_int
    lib.idw_run_device.argtypes = [ctypes.POINTER(IdwStore), ptr, ptr, ctypes.c_int64,
                                   ctypes.POINTER(IdwParams), ptr, ptr, ctypes.POINTER(IdwStats)]
    lib.idw_pack_device.restype = ctypes.c_int
    lib.idw_pack_device.argtypes = [ptr, ptr, ptr, ctypes.c_int64, ctypes.POINTER(IdwStore), ctypes.c_int, ptr]
    lib.idw_convert_device.restype = ctypes.c_int
    lib.idw_convert_device.argtypes = [ctypes.POINTER(IdwStore), ctypes.POINTER(IdwStore), ctypes.c_int, ptr]
    lib.idw_last_kernel_ms.restype = ctypes.c_int
    lib.idw_last_kernel_ms.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
    lib.idw_mufu_peak.restype = ctypes.c_int
    lib.idw_mufu_peak.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                  ctypes.POINTER(ctypes.c_double)]
    lib.idw_plan_create.restype = ctypes.c_int
    lib.idw_plan_create.argtypes = [ctypes.POINTER(IdwStore), ptr, ptr, ctypes.c_int64,
                                    ctypes.POINTER(IdwParams), ptr, ctypes.POINTER(ctypes.c_void_p)]
    lib.idw_plan_launch.restype = ctypes.c_int
    lib.idw_plan_launch.argtypes = [ptr, ptr]
    lib.idw_plan_launches.restype = ctypes.c_int64
    lib.idw_plan_launches.argtypes = [ptr]
    lib.idw_plan_kernel_ms.restype = ctypes.c_int
    lib.idw_plan_kernel_ms.argtypes = [ptr, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
    lib.idw_plan_destroy.restype = None
    lib.idw_plan_destroy.argtypes = [ptr]
    _lib = lib
    return lib


def device_count() -> int:
    return int(load().idw_device_count())


def _check(rc: int) -> None:
    if rc != 0:
        msg = load().idw_last_error().decode("utf-8", "replace")
        raise NativeError(f"libidw_b200 error {rc}: {msg}")


def make_store(kind: str, precision: str, count: int, pointers, nbytes) -> IdwStore:
    s = IdwStore()
    s.kind = KIND_CODES[kind]
    s.precision = PRECISION_CODES[precision]
    s.count = int(count)
    s.nbuf = len(pointers)
    for i, (p, nb) in enumerate(zip(pointers, nbytes)):
        s.buf[i] = int(p)
        s.nbytes[i] = int(nb)
    return s


MAX_DEVICES = 16  # IDW_MAX_DEVICES


def make_params(p: float, zero_eps: float, variant: str, mode: str, group_size: int,
                tile_size: int, splits: int = 0, device: int = 0,
                devices: tuple | None = None) -> IdwParams:
    prm = IdwParams()
    prm.p = float(p)
    prm.zero_eps = float(zero_eps)
    prm.variant = VARIANT_CODES[variant]
    prm.mode = MODE_CODES[mode]
    prm.group_size = int(group_size)
    prm.tile_size = int(tile_size)
    prm.splits = int(splits)
    prm.device = int(device)
    devs = tuple(devices or ())
    if len(devs) > MAX_DEVICES:
        raise ValueError(f"at most {MAX_DEVICES} devices per call")
    prm.ndevices = len(devs)
    for i, d in enumerate(devs):
        prm.devices[i] = int(d)
    return prm


def run_host(store: IdwStore, qx: np.ndarray, qy: np.ndarray, params: IdwParams,
             out: np.ndarray) -> IdwStats:
    """Blocking ``idw_run`` over host arrays (qx, qy, out contiguous, run dtype)."""
    lib = load()
    stats = IdwStats()
    m = out.shape[0]
    _check(lib.idw_run(ctypes.byref(store), qx.ctypes.data, qy.ctypes.data, m,
                       ctypes.byref(params), out.ctypes.data, ctypes.byref(stats)))
    return stats


E_NONFINITE = -5  # include/idw_b200.h


def run_host_xy(store: IdwStore, queries: np.ndarray, params: IdwParams, out: np.ndarray) -> IdwStats:
    """Blocking ``idw_run_xy``: the (m, 2) float64 C-contiguous query array of
    core.as_query_array goes to the device as is; the cast to the run dtype
    and core.ensure_finite's test run there.  A non-finite coordinate raises
    ValueError("invalid coordinate") like the reference (core.py:113-116)."""
    lib = load()
    stats = IdwStats()
    rc = lib.idw_run_xy(ctypes.byref(store), queries.ctypes.data, out.shape[0], ctypes.byref(params),
                        out.ctypes.data, ctypes.byref(stats))
    if rc == E_NONFINITE:
        raise ValueError("invalid coordinate")
    _check(rc)
    return stats


def run_device(store: IdwStore, qx_ptr: int, qy_ptr: int, m: int, params: IdwParams,
               out_ptr: int, stream: int = 0) -> IdwStats:
    """Asynchronous ``idw_run_device`` over device pointers on ``stream``."""
    lib = load()
    stats = IdwStats()
    _check(lib.idw_run_device(ctypes.byref(store), qx_ptr, qy_ptr, m, ctypes.byref(params),
                              out_ptr, stream, ctypes.byref(stats)))
    return stats


def pack_device(x_ptr: int, y_ptr: int, z_ptr: int, n: int, dst: IdwStore, device: int = 0,
                stream: int = 0) -> None:
    _check(load().idw_pack_device(x_ptr, y_ptr, z_ptr, n, ctypes.byref(dst), device, stream))


def convert_device(src: IdwStore, dst: IdwStore, device: int = 0, stream: int = 0) -> None:
    _check(load().idw_convert_device(ctypes.byref(src), ctypes.byref(dst), device, stream))


def last_kernel_ms() -> tuple[float, float]:
    """(variant kernels ms, fix-up ms) of this thread's last run_device call."""
    a = ctypes.c_double()
    b = ctypes.c_double()
    _check(load().idw_last_kernel_ms(ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


class Plan:
    """An ``idw_plan``: one run_device call captured into a CUDA graph over
    fixed device pointers, replayed by :meth:`launch`."""

    def __init__(self, store: IdwStore, qx_ptr: int, qy_ptr: int, m: int, params: IdwParams, out_ptr: int):
        self._lib = load()
        h = ctypes.c_void_p()
        _check(self._lib.idw_plan_create(ctypes.byref(store), qx_ptr, qy_ptr, m, ctypes.byref(params),
                                         out_ptr, ctypes.byref(h)))
        self._h = h
        self.launches = int(self._lib.idw_plan_launches(h))

    def launch(self, stream: int = 0) -> None:
        _check(self._lib.idw_plan_launch(self._h, stream))

    def kernel_ms(self) -> tuple[float, float]:
        a = ctypes.c_double()
        b = ctypes.c_double()
        _check(self._lib.idw_plan_kernel_ms(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def close(self) -> None:
        if self._h:
            self._lib.idw_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def mufu_peak(device: int = 0) -> tuple[float, float]:
    """(rcp results per second, implied SM clock in Hz) measured on ``device``."""
    lib = load()
    rate = ctypes.c_double()
    hz = ctypes.c_double()
    _check(lib.idw_mufu_peak(device, ctypes.byref(rate), ctypes.byref(hz)))
    return rate.value, hz.value
