"""Quick device-resident timing of the variants (development aid)."""
import sys, time, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1402_4986_b200 as il
from paper_1402_4986_b200.device import DeviceStore, predict_device

def run(n, m, kind, prec, variant, mode, p=2.0, reps=3, G=1024, splits=0):
    x, y, z = il.generate_cloud_arrays(n, 0)
    qx, qy, _ = il.generate_cloud_arrays(m, 1)
    st = il.LayoutStore.from_arrays(x, y, z, il.LayoutKind(kind), il.Precision(prec))
    ds = DeviceStore(st, 0)
    dt = ds.dtype
    tqx = torch.tensor(qx, dtype=dt, device="cuda"); tqy = torch.tensor(qy, dtype=dt, device="cuda")
    out = torch.empty(m, dtype=dt, device="cuda")
    cfg = il.ExecConfig(mode=mode, group_size=G, splits=splits)
    predict_device(ds, tqx, tqy, out, il.Params(p), cfg, variant)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record(); predict_device(ds, tqx, tqy, out, il.Params(p), cfg, variant); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    t = min(ts)
    r = dict(n=n, m=m, kind=kind, prec=prec, variant=variant, mode=mode, p=p, s=t, gpairs=n * m / t / 1e9)
    print(json.dumps(r), flush=True)
    return out

import subprocess as _sp
print(json.dumps({"clocks": _sp.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
                                     "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()}), flush=True)
if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "nested":  # noqa
    K = 1024
    run(1024 * K, 64 * K, "soa", "double", "nested_improved", "fast", p=3.5, reps=2)
    run(102400, 102400, "soa", "double", "nested_improved", "fast", p=2.0, reps=2)
    run(10240 * K, 100 * K, "aoas", "single", "nested_improved", "fast", reps=2)
    sys.exit(0)
if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "exact":  # noqa
    K = 1024
    for v in ("naive", "tiled", "nested_improved", "nested_original"):
        for prec, kind in (("single", "aoas"), ("double", "soa")):
            run(100 * K, 100 * K if v != "nested_original" else 8 * K, kind, prec, v, "exact", reps=5)
    sys.exit(0)
if __name__ == "__main__":
    rate, hz = il._capi.mufu_peak(0)
    print(json.dumps(dict(mufu_rcp_per_s=rate, pairs_roofline_gpairs=rate / 1e9, sm_hz=hz)), flush=True)
    K = 1024
    for args in [
        (100 * K, 100 * K, "aoas", "single", "tiled", "fast"),
        (100 * K, 100 * K, "soa", "single", "tiled", "fast"),
        (100 * K, 100 * K, "aoas", "single", "naive", "fast"),
        (100 * K, 100 * K, "aoas", "single", "nested_improved", "fast"),
        (100 * K, 100 * K, "aoas", "single", "tiled", "exact"),
        (100 * K, 100 * K, "aoas", "single", "naive", "exact"),
        (100 * K, 100 * K, "aoas", "double", "tiled", "fast"),
        (100 * K, 100 * K, "soa", "double", "tiled", "exact"),
        (1024 * K, 1024 * K, "aoas", "single", "tiled", "fast"),
    ]:
        run(*args)
    run(1024 * K, 64 * K, "soa", "double", "nested_improved", "fast", p=3.5, reps=1)
    run(10240 * K, 100 * K, "aoas", "single", "tiled", "fast", reps=1)
    run(10240 * K, 100 * K, "aoas", "single", "nested_improved", "fast", reps=1)
