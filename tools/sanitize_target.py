"""Small runs of every variant / mode / precision for compute-sanitizer
(memcheck, racecheck, synccheck): the smem rings of K2, the cp.async ring,
cluster/DSMEM tree and persistent loop of K3, K4's trees, the fix-up and
combine passes, the device packers/converters and a graph plan."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1402_4986_b200 as il
from paper_1402_4986_b200.device import DevicePlan, DeviceStore
rng = np.random.default_rng(5)
data = rng.random((3000, 3)); data[:, 2] *= 100
queries = rng.random((700, 2)); queries[3] = data[9, :2]  # one coincidence -> fix-up
for precision in il.Precision:
    for kind in (il.LayoutKind.SoA, il.LayoutKind.AoaS):
        store = il.build(data, kind, precision)
        for variant in ("naive", "tiled", "nested_improved", "nested_original"):
            for mode in ("exact", "fast"):
                for G in (1024, 64):
                    il.STRATEGIES[variant](store, queries, cfg=il.ExecConfig(mode=mode, group_size=G))
        il.run_tiled(store, queries, il.Params(3.5), cfg=il.ExecConfig(mode="fast", splits=7))
        ds = DeviceStore(store, 0)
        ds.convert(il.LayoutKind.SoA if kind is not il.LayoutKind.SoA else il.LayoutKind.AoS)
        q = [torch.tensor(queries[:, k].astype(precision.dtype), device="cuda") for k in (0, 1)]
        out = torch.empty(len(queries), dtype=ds.dtype, device="cuda")
        plan = DevicePlan(ds, q[0], q[1], out, il.Params(), il.ExecConfig(mode="fast"), "tiled")
        plan.launch(); torch.cuda.synchronize(); plan.close()
print("sanitize target done")
