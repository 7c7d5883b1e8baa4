"""C2 (100K x 100K fp32 AoaS FAST tiled): forced data-split counts vs auto."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1402_4986_b200 as il
from paper_1402_4986_b200.device import DeviceStore, predict_device
for n, m in ((102400, 102400), (1 << 20, 1 << 20), (1 << 20, 1 << 17)):
    x, y, z = il.generate_cloud_arrays(n, 0); qx, qy, _ = il.generate_cloud_arrays(m, 1)
    ds = DeviceStore(il.LayoutStore.from_arrays(x, y, z, il.LayoutKind.AoaS, il.Precision.single), 0)
    tq = [torch.tensor(a, dtype=torch.float32, device="cuda") for a in (qx, qy)]
    out = torch.empty(m, dtype=torch.float32, device="cuda")
    for splits in (0, 12, 25, 50, 100):
        cfg = il.ExecConfig(mode="fast", splits=splits)
        predict_device(ds, tq[0], tq[1], out, il.Params(), cfg, "tiled"); torch.cuda.synchronize()
        best = None
        for _ in range(3):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); predict_device(ds, tq[0], tq[1], out, il.Params(), cfg, "tiled"); e1.record()
            torch.cuda.synchronize(); t = e0.elapsed_time(e1) / 1e3; best = t if best is None else min(best, t)
        print(json.dumps(dict(n=n, m=m, splits=splits, gpairs=n * m / best / 1e9)), flush=True)
