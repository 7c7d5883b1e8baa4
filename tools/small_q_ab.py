"""FAST fp32 tiled at small m through graph plans: C1 (10K x 10K SoA) and 100K x 10K, 100K x 100K AoaS."""
import json, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1402_4986_b200 as il
from paper_1402_4986_b200.device import DevicePlan, DeviceStore
for n, m, kind in ((10240, 10240, "soa"), (102400, 10240, "aoas"), (102400, 102400, "aoas"), (1 << 20, 1 << 17, "aoas")):
    x, y, z = il.generate_cloud_arrays(n, 0); qx, qy, _ = il.generate_cloud_arrays(m, 1)
    ds = DeviceStore(il.LayoutStore.from_arrays(x, y, z, il.LayoutKind(kind), il.Precision.single), 0)
    tq = [torch.tensor(a, dtype=torch.float32, device="cuda") for a in (qx, qy)]
    out = torch.empty(m, dtype=torch.float32, device="cuda")
    plan = DevicePlan(ds, tq[0], tq[1], out, il.Params(), il.ExecConfig(mode="fast"), "tiled")
    for _ in range(3): plan.launch()
    torch.cuda.synchronize()
    reps = 20
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): plan.launch()
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / reps
    print(json.dumps(dict(q4=os.environ.get("IDW_FAST_Q4", "0"), n=n, m=m, kind=kind, us=t * 1e6, gpairs=n * m / t / 1e9,
                          kernel_ms=plan.kernel_ms()[0])), flush=True)
