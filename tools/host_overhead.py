"""Where does a small predict_device call spend host time? (C1-sized)"""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1402_4986_b200 as il
from paper_1402_4986_b200 import _capi
from paper_1402_4986_b200.device import DeviceStore, predict_device
n = m = 10240
x, y, z = il.generate_cloud_arrays(n, 0); qx, qy, _ = il.generate_cloud_arrays(m, 1)
ds = DeviceStore(il.LayoutStore.from_arrays(x, y, z, il.LayoutKind.SoA, il.Precision.single), 0)
tq = [torch.tensor(a, dtype=torch.float32, device="cuda") for a in (qx, qy)]
out = torch.empty(m, dtype=torch.float32, device="cuda")
cfg = il.ExecConfig(mode="fast")
for _ in range(3):
    predict_device(ds, tq[0], tq[1], out, il.Params(), cfg, "tiled")
torch.cuda.synchronize()
res = {}
for name, fn in [("predict_device", lambda: predict_device(ds, tq[0], tq[1], out, il.Params(), cfg, "tiled")),
                 ("native_struct", lambda: ds.native()),
                 ("make_params", lambda: _capi.make_params(2.0, 0.0, "tiled", "fast", 1024, 1024, 0, 0)),
                 ("current_stream", lambda: torch.cuda.current_stream(0)),
                 ("last_kernel_ms", lambda: _capi.last_kernel_ms())]:
    t0 = time.perf_counter()
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    res[name + "_us"] = (time.perf_counter() - t0) / 50 * 1e6
st = torch.cuda.current_stream(0)
prm = _capi.make_params(2.0, 0.0, "tiled", "fast", 1024, 1024, 0, 0)
nat = ds.native()
t0 = time.perf_counter()
for _ in range(50):
    _capi.run_device(nat, tq[0].data_ptr(), tq[1].data_ptr(), m, prm, out.data_ptr(), st.cuda_stream)
torch.cuda.synchronize()
res["raw_run_device_us"] = (time.perf_counter() - t0) / 50 * 1e6
print(json.dumps(res))
