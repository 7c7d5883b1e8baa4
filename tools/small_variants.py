"""C1-size (10K x 10K fp32 SoA, p = 2, FAST) through DevicePlan replays for
every variant and a few group sizes: which one serves a small batch best."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1402_4986_b200 as il
from paper_1402_4986_b200.device import DevicePlan, DeviceStore
n = m = 10240
x, y, z = il.generate_cloud_arrays(n, 0); qx, qy, _ = il.generate_cloud_arrays(m, 1)
ds = DeviceStore(il.LayoutStore.from_arrays(x, y, z, il.LayoutKind.SoA, il.Precision.single), 0)
tq = [torch.tensor(a, dtype=torch.float32, device="cuda") for a in (qx, qy)]
out = torch.empty(m, dtype=torch.float32, device="cuda")
for variant, G in (("tiled", 1024), ("naive", 1024), ("nested_improved", 1024), ("nested_improved", 256),
                   ("nested_improved", 64), ("nested_improved", 32)):
    plan = DevicePlan(ds, tq[0], tq[1], out, il.Params(), il.ExecConfig(mode="fast", group_size=G), variant)
    for _ in range(3):
        plan.launch()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        plan.launch()
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / 20
    k, f = plan.kernel_ms()
    print(json.dumps(dict(variant=variant, G=G, step_us=t * 1e6, gpairs=n * m / t / 1e9, kernel_ms=k, fixup_ms=f,
                          launches=plan.launches)), flush=True)
