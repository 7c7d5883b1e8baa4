"""Small runs of every variant / mode / precision for compute-sanitizer
(memcheck, racecheck, synccheck): the smem rings of K2, the cp.async ring,
cluster/DSMEM tree and persistent loop of K3, K4's trees, the fix-up and
fix-up passes, the device packers/converters and a graph plan; round 2: the
chunked K2 FAST scheduler (ring-slot reuse), K3's warp split, the
device-list host path and the batched exact fix-up."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1402_4986_b200 as il
from paper_1402_4986_b200.device import DevicePlan, DeviceStore
if len(sys.argv) > 1 and sys.argv[1] == "band":  # run with IDW_BAND=3: K2 FAST banded order, ring reuse
    for prec in il.Precision:
        x, y, z = il.generate_cloud_arrays(60_000, 0)
        qx, qy, _ = il.generate_cloud_arrays(40_000, 1)
        st = il.LayoutStore.from_arrays(x, y, z, il.LayoutKind.AoaS, prec)
        il.run_tiled(st, np.column_stack([qx, qy]), cfg=il.ExecConfig(mode="fast"))
    torch.cuda.synchronize()
    sys.exit(0)
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
# round 2: K2 FAST chunk ring with slot reuse (groups > ring slots), the
# device-list host path, the batched exact fix-up (subnormal d2, EXACT naive/tiled)
x, y, z = il.generate_cloud_arrays(60_000, 0)
qx, qy, _ = il.generate_cloud_arrays(60_000, 1)
big = il.LayoutStore.from_arrays(x, y, z, il.LayoutKind.AoaS, il.Precision.single)
il.run_tiled(big, np.column_stack([qx, qy]), cfg=il.ExecConfig(mode="fast"))
il.run_tiled(big, np.column_stack([qx, qy])[:5000], cfg=il.ExecConfig(mode="fast", devices=(0, 0, 0)))
sub = data.copy(); sub[:, :2] = 0.1 + 0.9 * sub[:, :2]; sub[7] = (0.0, 0.0, 0.37)
qs = np.vstack([[[2.0 ** -63.5, 0.0], [0.0, 2.0 ** -63.2]], queries[:100]])
st = il.build(sub, il.LayoutKind.SoA, il.Precision.single)
for variant in ("naive", "tiled", "nested_improved"):
    il.STRATEGIES[variant](st, qs, cfg=il.ExecConfig(mode="exact"))
# device-resident device list (peer-copy broadcast, shards, gather)
from paper_1402_4986_b200.device import predict_device
dsb = DeviceStore(big, 0)
qb = [torch.tensor(a[:4000].astype(np.float32), device="cuda") for a in (qx, qy)]
ob = torch.empty(4000, dtype=torch.float32, device="cuda")
predict_device(dsb, qb[0], qb[1], ob, il.Params(), il.ExecConfig(mode="fast", devices=(0, 0, 0)), "tiled")
torch.cuda.synchronize()
print("sanitize target done")
