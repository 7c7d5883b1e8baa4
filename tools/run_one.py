"""One device-resident call of a variant (for ncu captures); development aid.
usage: run_one.py n m kind prec variant mode p [reps]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1402_4986_b200 as il
from paper_1402_4986_b200.device import DeviceStore, predict_device

n, m, kind, prec, variant, mode, p = sys.argv[1:8]
reps = int(sys.argv[8]) if len(sys.argv) > 8 else 2
n, m, p = int(n), int(m), float(p)
x, y, z = il.generate_cloud_arrays(n, 0)
qx, qy, _ = il.generate_cloud_arrays(m, 1)
ds = DeviceStore(il.LayoutStore.from_arrays(x, y, z, il.LayoutKind(kind), il.Precision(prec)), 0)
tq = [torch.tensor(a, dtype=ds.dtype, device="cuda") for a in (qx, qy)]
out = torch.empty(m, dtype=ds.dtype, device="cuda")
for _ in range(reps):
    predict_device(ds, tq[0], tq[1], out, il.Params(p), il.ExecConfig(mode=mode), variant)
torch.cuda.synchronize()
