"""K4 (nested_original) threads-per-query A/B: one JSON line per setting."""
import json, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1])); sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
import numpy as np, torch
import paper_1402_4986_b200 as il, oracle
from paper_1402_4986_b200.device import DeviceStore, predict_device
n, m = 102400, 8192
x, y, z = il.generate_cloud_arrays(n, 0); qx, qy, _ = il.generate_cloud_arrays(m, 1)
for prec in (il.Precision.single, il.Precision.double):
    st = il.LayoutStore.from_arrays(x, y, z, il.LayoutKind.SoA, prec)
    ds = DeviceStore(st, 0)
    tq = [torch.tensor(a.astype(prec.dtype), device="cuda") for a in (qx, qy)]
    out = torch.empty(m, dtype=ds.dtype, device="cuda")
    for mode in ("exact", "fast"):
        cfg = il.ExecConfig(mode=mode)
        predict_device(ds, tq[0], tq[1], out, il.Params(), cfg, "nested_original"); torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); predict_device(ds, tq[0], tq[1], out, il.Params(), cfg, "nested_original"); e1.record(); torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        res = out.cpu().numpy()
        ok = None
        if mode == "exact":
            ref = oracle.nested_original(st, np.column_stack([qx[:256], qy[:256]]))[0]
            ok = bool(np.array_equal(res[:256], ref))
        print(json.dumps(dict(threads=os.environ.get("IDW_K4_THREADS", "1024"), prec=prec.value, mode=mode,
                              gpairs=n * m / t / 1e9, bitwise_vs_oracle=ok)), flush=True)
