"""K3 EXACT fp32 at C2 size through IDW_B200_LIB (A/B helper)."""
import json, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1402_4986_b200 as il
from paper_1402_4986_b200.device import DeviceStore, predict_device
n = m = 102400
x, y, z = il.generate_cloud_arrays(n, 0); qx, qy, _ = il.generate_cloud_arrays(m, 1)
for kind in ("soa", "aos", "aoas"):
    ds = DeviceStore(il.LayoutStore.from_arrays(x, y, z, il.LayoutKind(kind), il.Precision.single), 0)
    tq = [torch.tensor(a, dtype=torch.float32, device="cuda") for a in (qx, qy)]
    out = torch.empty(m, dtype=torch.float32, device="cuda")
    for mode in ("exact", "fast"):
        cfg = il.ExecConfig(mode=mode)
        predict_device(ds, tq[0], tq[1], out, il.Params(), cfg, "nested_improved"); torch.cuda.synchronize()
        best = None
        for _ in range(3):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); predict_device(ds, tq[0], tq[1], out, il.Params(), cfg, "nested_improved"); e1.record()
            torch.cuda.synchronize(); t = e0.elapsed_time(e1) / 1e3; best = t if best is None else min(best, t)
        print(json.dumps(dict(lib=Path(os.environ.get("IDW_B200_LIB", "default")).name, kind=kind, mode=mode,
                              gpairs=n * m / best / 1e9)), flush=True)
