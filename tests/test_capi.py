"""The C-ABI library: loads, exports every symbol include/idw_b200.h declares,
and refuses to compute without a GPU (no CPU fallback).  CPU-only."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_1402_4986_b200 import _capi
from paper_1402_4986_b200.layouts import LayoutKind, build
from paper_1402_4986_b200.core import Precision

HEADER = Path(__file__).resolve().parents[1] / "include" / "idw_b200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(idw_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_abi():
    fns = declared_functions()
    assert {"idw_run", "idw_run_device", "idw_last_error", "idw_abi_version"} <= set(fns)
    assert set(fns) == set(_capi.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_capi.library_path()))
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_abi_version_and_struct_layouts(tmp_path):
    """ctypes mirrors of the header structs match the C compiler's layout
    field by field (gcc on include/idw_b200.h)."""
    lib = _capi.load()
    assert lib.idw_abi_version() == _capi.ABI_VERSION == 2
    structs = {"idw_store": _capi.IdwStore, "idw_params": _capi.IdwParams, "idw_stats": _capi.IdwStats}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    lines.append('printf("IDW_MAX_DEVICES %d\\n", IDW_MAX_DEVICES); return 0; }')
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    import subprocess
    subprocess.run(["gcc", "-std=c11", "-o", str(exe), str(src)], check=True)
    got = dict(l.rsplit(" ", 1) for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                         check=True).stdout.splitlines())
    for cname, py in structs.items():
        assert int(got[f"{cname} size"]) == ctypes.sizeof(py), cname
        for f, _ in py._fields_:
            assert int(got[f"{cname}.{f}"]) == getattr(py, f).offset, (cname, f)
    assert int(got["IDW_MAX_DEVICES"]) == _capi.MAX_DEVICES == len(_capi.IdwParams().devices)


def test_device_list_validation():
    from paper_1402_4986_b200 import ExecConfig

    assert ExecConfig(devices=[0, 0, 1]).devices == (0, 0, 1)
    for bad in ((), (-1,), tuple(range(17))):
        with pytest.raises(ValueError):
            ExecConfig(devices=bad)
    prm = _capi.make_params(2.0, 0.0, "tiled", "fast", 1024, 1024, 0, 0, (3, 1))
    assert prm.ndevices == 2 and list(prm.devices[:2]) == [3, 1]
    lib = _capi.load()
    st = _store()
    ns = _capi.make_store("soa", "double", st.count, [b.ctypes.data for b in st.buffers],
                          [b.nbytes for b in st.buffers])
    q = np.zeros(4)
    # a captured plan runs on one device
    plan = ctypes.c_void_p()
    rc = lib.idw_plan_create(ctypes.byref(ns), q.ctypes.data, q.ctypes.data, 4, ctypes.byref(prm),
                             q.ctypes.data, ctypes.byref(plan))
    assert rc == -1 and b"one device" in lib.idw_last_error()
    prm.ndevices = 17
    rc = lib.idw_run(ctypes.byref(ns), q.ctypes.data, q.ctypes.data, 4, ctypes.byref(prm), q.ctypes.data, None)
    assert rc == -1 and b"ndevices" in lib.idw_last_error()


def test_device_list_env(monkeypatch):
    from paper_1402_4986_b200 import ExecConfig

    monkeypatch.setenv("IDW_DEVICES", "0,2, 1")
    assert ExecConfig().devices == (0, 2, 1)
    monkeypatch.delenv("IDW_DEVICES")
    assert ExecConfig().devices is None


def _store(kind=LayoutKind.SoA, precision=Precision.double):
    rng = np.random.default_rng(0)
    return build(rng.random((16, 3)), kind, precision)


def test_structural_validation_without_gpu():
    lib = _capi.load()
    st = _store()
    ns = _capi.make_store("soa", "double", st.count, [b.ctypes.data for b in st.buffers],
                          [b.nbytes for b in st.buffers])
    q = np.zeros(4)
    out = np.zeros(4)
    prm = _capi.make_params(2.0, 0.0, "tiled", "exact", 1024, 1024)
    # illegal layout/precision pair is refused before any device work
    bad = _capi.make_store("soaos", "single", st.count, [b.ctypes.data for b in st.buffers[:2]],
                           [b.nbytes for b in st.buffers[:2]])
    rc = lib.idw_run(ctypes.byref(bad), q.ctypes.data, q.ctypes.data, 4, ctypes.byref(prm), out.ctypes.data, None)
    assert rc == -2 and b"double precision" in lib.idw_last_error()
    # p <= 0
    prm_bad = _capi.make_params(0.0, 0.0, "tiled", "exact", 1024, 1024)
    rc = lib.idw_run(ctypes.byref(ns), q.ctypes.data, q.ctypes.data, 4, ctypes.byref(prm_bad), out.ctypes.data, None)
    assert rc == -1 and b"power p" in lib.idw_last_error()
    # buffer shorter than its shape
    short = _capi.make_store("soa", "double", st.count, [b.ctypes.data for b in st.buffers], [8, 8, 8])
    rc = lib.idw_run(ctypes.byref(short), q.ctypes.data, q.ctypes.data, 4, ctypes.byref(prm), out.ctypes.data, None)
    assert rc == -1 and b"shorter" in lib.idw_last_error()


@pytest.mark.skipif(_capi.device_count() > 0, reason="checks the no-GPU failure path")
def test_no_cpu_fallback():
    """Without a CUDA device every compute entry point fails loudly."""
    st = _store()
    ns = _capi.make_store("soa", "double", st.count, [b.ctypes.data for b in st.buffers],
                          [b.nbytes for b in st.buffers])
    q = np.full(4, 0.5)
    out = np.zeros(4)
    prm = _capi.make_params(2.0, 0.0, "naive", "exact", 1024, 1024)
    with pytest.raises(_capi.NativeError, match="no CUDA device"):
        _capi.run_host(ns, q, q, prm, out)
    import paper_1402_4986_b200 as il

    with pytest.raises(_capi.NativeError):
        il.run_tiled(st, [(0.5, 0.5)])


def test_header_codes_match_python_tables():
    """enum values of include/idw_b200.h == the codes the ctypes layer sends."""
    text = HEADER.read_text()
    enums = dict((k, int(v)) for k, v in re.findall(r"\b(IDW_[A-Z_0-9]+)\s*=\s*(-?\d+)", text))
    assert {k: enums[f"IDW_{k.upper()}"] for k in _capi.KIND_CODES} == _capi.KIND_CODES
    assert enums["IDW_SINGLE"] == _capi.PRECISION_CODES["single"]
    assert enums["IDW_DOUBLE"] == _capi.PRECISION_CODES["double"]
    for name, code in _capi.VARIANT_CODES.items():
        assert enums[f"IDW_{name.upper()}"] == code
    assert enums["IDW_EXACT"] == _capi.MODE_CODES["exact"] and enums["IDW_FAST"] == _capi.MODE_CODES["fast"]
    assert enums["IDW_E_NONFINITE"] == _capi.E_NONFINITE
