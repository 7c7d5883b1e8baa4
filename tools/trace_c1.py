"""Per-warp timeline of the C1 K2 FAST launch (build with -DIDW_TRACE); development aid."""
import sys
sys.path.insert(0, ".")
import torch
import paper_1402_4986_b200 as il
from paper_1402_4986_b200.device import DeviceStore, predict_device

n = m = 10 << 10
x, y, z = il.generate_cloud_arrays(n, 0)
qx, qy, _ = il.generate_cloud_arrays(m, 1)
ds = DeviceStore(il.LayoutStore.from_arrays(x, y, z, il.LayoutKind.SoA, il.Precision.single), 0)
tqx = torch.tensor(qx, dtype=torch.float32, device="cuda")
tqy = torch.tensor(qy, dtype=torch.float32, device="cuda")
out = torch.empty(m, dtype=torch.float32, device="cuda")
cfg = il.ExecConfig(mode="fast")
for k in range(4):
    print(f"CALL {k}", flush=True)
    predict_device(ds, tqx, tqy, out, il.Params(2.0), cfg, "tiled")
    torch.cuda.synchronize()
import ctypes
import numpy as np

lib = il._capi.load()
buf = np.zeros(4096 * 8, dtype=np.uint64)
rc = lib.idw_trace_dump(buf.ctypes.data_as(ctypes.c_void_p))
a = buf.reshape(4096, 8).astype(np.int64)
a = a[a[:, 1] > 0]
t0 = a[:, 1].min()
t = (a[:, 1:] - t0) / 1000.0
names = ["start", "issued", "qbox", "tiles", "partial", "foldend", "exit"]
print("rc", rc, "warps", len(a), "SMs", len(set(a[:, 0])))
for i, nm in enumerate(names):
    v = t[:, i] if nm != "foldend" else t[a[:, 6] > 0, i]
    print(f"{nm:8s} min {v.min():7.2f} med {np.median(v):7.2f} p90 {np.percentile(v, 90):7.2f} max {v.max():7.2f}")
fold = a[:, 6] > 0
print("fold duration med/max", np.median(t[fold, 5] - t[fold, 4]), (t[fold, 5] - t[fold, 4]).max())
print("store+fence+atomic med/max", np.median(t[:, 4] - t[:, 3]), (t[:, 4] - t[:, 3]).max())
