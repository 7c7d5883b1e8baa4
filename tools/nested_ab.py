"""A/B one libidw_b200 variant (IDW_B200_LIB) on the fp64 K3 configs:
device-resident timing (CUDA events) + max rel err vs the fp64 truth on a
query sample.  Prints one JSON line per case."""
import json, os, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "oracle"))
import numpy as np, torch
import paper_1402_4986_b200 as il
import oracle
from paper_1402_4986_b200.device import DeviceStore, predict_device
K = 1024
lib = os.environ.get("IDW_B200_LIB", "default")
cases = [(1024 * K, 64 * K, "soa", "double", "nested_improved", 3.5),
         (102400, 102400, "soa", "double", "nested_improved", 2.0),
         (102400, 102400, "soa", "double", "nested_improved", 3.0),
         (102400, 102400, "aoas", "double", "tiled", 3.5)]
if len(sys.argv) > 1 and sys.argv[1] == "full":
    cases = [(1024 * K, 1024 * K, "soa", "double", "nested_improved", 3.5)]
if len(sys.argv) > 1 and sys.argv[1] == "fp32":
    cases = [(102400, 102400, "aoas", "single", "nested_improved", 2.0),
             (102400, 102400, "soa", "single", "nested_improved", 2.0),
             (102400, 102400, "aos", "single", "nested_improved", 2.0),
             (10240 * K, 25 * K, "aoas", "single", "nested_improved", 2.0),
             (102400, 102400, "aoas", "single", "nested_improved", 3.5)]
for n, m, kind, prec, variant, p in cases:
    x, y, z = il.generate_cloud_arrays(n, 0)
    qx, qy, _ = il.generate_cloud_arrays(m, 1)
    st = il.LayoutStore.from_arrays(x, y, z, il.LayoutKind(kind), il.Precision(prec))
    ds = DeviceStore(st, 0)
    tqx = torch.tensor(qx, dtype=ds.dtype, device="cuda"); tqy = torch.tensor(qy, dtype=ds.dtype, device="cuda")
    out = torch.empty(m, dtype=ds.dtype, device="cuda")
    cfg = il.ExecConfig(mode="fast")
    predict_device(ds, tqx, tqy, out, il.Params(p), cfg, variant)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(3):
        e0.record(); predict_device(ds, tqx, tqy, out, il.Params(p), cfg, variant); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) / 1e3)
    res = out.cpu().numpy()
    idx = np.linspace(0, m - 1, 512).astype(np.int64)
    q = np.column_stack([qx[idx], qy[idx]])
    tr = oracle.truth(st, q, p)
    err = float(np.max(np.abs(res[idx] - tr) / np.abs(tr)))
    t = min(ts)
    print(json.dumps(dict(lib=Path(lib).name, n=n, m=m, kind=kind, variant=variant, p=p, s=t,
                          gpairs=n * m / t / 1e9, max_rel_err=err)), flush=True)
