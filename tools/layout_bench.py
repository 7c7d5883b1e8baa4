"""§8f4 measurement: the device-side layout packers/converters
(idw_pack_device / idw_convert_device, byte-identical to the reference's
LayoutStore.from_arrays / convert, layouts.py:172-186, 251-255) at n = 64M
points, against the measured HBM copy bandwidth (MEASURED_PEAKS.json).
Algorithmic bytes = bytes read + bytes written (pads included: the layout
writes them).  The host packer (numpy, the reference's algorithm) is timed
on the same machine at n = 4M for the CPU column."""
import json, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np, torch
import paper_1402_4986_b200 as il
from paper_1402_4986_b200 import _capi
from paper_1402_4986_b200.device import DeviceStore
from paper_1402_4986_b200.layouts import buffer_shapes

peak = json.load(open(ROOT / "MEASURED_PEAKS.json")).get("hbm_gbs") if (ROOT / "MEASURED_PEAKS.json").exists() else None
n = 1 << 26
rng = np.random.default_rng(0)
xyz = [torch.tensor(rng.random(n), dtype=torch.float64, device="cuda") for _ in range(3)]
st = torch.cuda.current_stream()


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        best = t if best is None else min(best, t)
    return best


def nbytes(kind, prec):
    return sum(sh.nbytes for sh in buffer_shapes(kind, prec, n))


nh = 1 << 22
hx = [rng.random(nh) for _ in range(3)]
for kind, prec in il.legal_pairs():
    dst = DeviceStore._alloc(kind, prec, n, 0)
    nat = dst.native()
    t = timed(lambda: _capi.pack_device(xyz[0].data_ptr(), xyz[1].data_ptr(), xyz[2].data_ptr(), n, nat, 0,
                                        st.cuda_stream))
    b = 24 * n + nbytes(kind, prec)
    t0 = time.perf_counter(); il.LayoutStore.from_arrays(hx[0], hx[1], hx[2], kind, prec); tc = time.perf_counter() - t0
    print(json.dumps(dict(op="pack", kind=kind.value, precision=prec.value, n=n, s=t, gbs=b / t / 1e9,
                          frac_hbm=(b / t / 1e9 / peak) if peak else None,
                          cpu_numpy_gbs=(24 * nh + nbytes(kind, prec) * nh / n) / tc / 1e9)), flush=True)
    for k2 in il.LayoutKind:
        if not k2.legal_for(prec) or k2 == kind:
            continue
        out = DeviceStore._alloc(k2, prec, n, 0)
        onat = out.native()
        t = timed(lambda: _capi.convert_device(nat, onat, 0, st.cuda_stream))
        b = nbytes(kind, prec) + nbytes(k2, prec)
        print(json.dumps(dict(op="convert", src=kind.value, dst=k2.value, precision=prec.value, n=n, s=t,
                              gbs=b / t / 1e9, frac_hbm=(b / t / 1e9 / peak) if peak else None)), flush=True)
        del out
    del dst
    torch.cuda.empty_cache()
