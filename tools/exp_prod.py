"""Experiment: shared-reciprocal pairs per point (IDW_PROD) on C3; time + accuracy."""
import json, os, subprocess, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "oracle"))
    import numpy as np, torch, oracle
    import paper_1402_4986_b200 as il
    from paper_1402_4986_b200 import _capi
    from paper_1402_4986_b200.device import DeviceStore, predict_device
    n = m = 1 << 20
    x, y, z = il.generate_cloud_arrays(n, 0); qx, qy, _ = il.generate_cloud_arrays(m, 1)
    st = il.LayoutStore.from_arrays(x, y, z, il.LayoutKind.AoaS, il.Precision.single)
    ds = DeviceStore(st, 0)
    tqx = torch.tensor(qx, dtype=torch.float32, device="cuda"); tqy = torch.tensor(qy, dtype=torch.float32, device="cuda")
    out = torch.empty(m, dtype=torch.float32, device="cuda")
    cfg = il.ExecConfig(mode="fast")
    ts = []
    for i in range(4):
        predict_device(ds, tqx, tqy, out, il.Params(), cfg, "tiled"); ts.append(_capi.last_kernel_ms()[0])
    sub = np.arange(0, m, m // 1024)
    truth = oracle.truth(st, np.column_stack([qx[sub], qy[sub]]))
    got = out.cpu().numpy()[sub].astype(np.float64)
    err = float(np.max(np.abs(got - truth) / np.abs(truth)))
    full = out.cpu().numpy()
    np.save(f"/tmp/out_prod{os.environ.get('IDW_PROD','0')}.npy", full)
    base = f"/tmp/out_prod0.npy"
    ndiff = int(np.sum(np.load(base) != full)) if os.path.exists(base) else -1
    print(json.dumps({"prod": int(os.environ.get("IDW_PROD", "0")), "ndiff_vs_prod0": ndiff, "kernel_ms": min(ts[1:]),
                      "gpairs": n * m / (min(ts[1:]) * 1e-3) / 1e9, "max_rel_err_1024q": err}), flush=True)
else:
    for prod in (0, 1, 2):
        env = dict(os.environ, IDW_PROD=str(prod))
        subprocess.run([sys.executable, __file__, "child"], env=env)
