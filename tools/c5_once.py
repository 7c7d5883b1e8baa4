"""One warm C5-shaped FAST tiled call (10M x 100K fp32 AoaS) for ncu DRAM
counters; development aid.  usage: c5_once.py [n m]"""
import sys
sys.path.insert(0, ".")
import torch
import paper_1402_4986_b200 as il
from paper_1402_4986_b200.device import DeviceStore, predict_device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10 << 20
m = int(sys.argv[2]) if len(sys.argv) > 2 else 100 << 10
x, y, z = il.generate_cloud_arrays(n, 0)
qx, qy, _ = il.generate_cloud_arrays(m, 1)
ds = DeviceStore(il.LayoutStore.from_arrays(x, y, z, il.LayoutKind.AoaS, il.Precision.single), 0)
tqx = torch.tensor(qx, dtype=torch.float32, device="cuda")
tqy = torch.tensor(qy, dtype=torch.float32, device="cuda")
out = torch.empty(m, dtype=torch.float32, device="cuda")
cfg = il.ExecConfig(mode="fast")
for _ in range(2):
    predict_device(ds, tqx, tqy, out, il.Params(2.0), cfg, "tiled")
torch.cuda.synchronize()
print("ok", float(out[:4].sum()))
