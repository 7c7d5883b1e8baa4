"""Break down e2e run_tiled calls (host buffers) at C1 and C3: Python prep,
native call, kernel time.  Run twice: IDW_POOL_KEEP=0 and =1."""
import json, os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1402_4986_b200 as il
from paper_1402_4986_b200 import strategies as S
res = {"pool_keep": os.environ.get("IDW_POOL_KEEP", "1")}
for name, n, kind in (("c1", 10240, il.LayoutKind.SoA), ("c3", 1 << 20, il.LayoutKind.AoaS)):
    x, y, z = il.generate_cloud_arrays(n, 0); qx, qy, _ = il.generate_cloud_arrays(n, 1)
    st = il.LayoutStore.from_arrays(x, y, z, kind, il.Precision.single)
    pinned = []
    for b in st.buffers:
        t = torch.empty(b.nbytes, dtype=torch.uint8, pin_memory=True); t.numpy()[:] = b; pinned.append(t.numpy())
    hst = il.LayoutStore(st.kind, st.precision, n, pinned, st.shapes)
    q = np.column_stack([qx, qy]); cfg = il.ExecConfig(mode="fast")
    rows = []
    for i in range(6):
        rs = il.RunStats()
        t0 = time.perf_counter(); qx32, qy32, dt = S._prepare(hst, q, il.Params()); t1 = time.perf_counter()
        out = np.empty(n, np.float32)
        prm = S._capi.make_params(2.0, 0.0, "tiled", "fast", 1024, 1024, 0, 0)
        ns = S._native_store(hst); t2 = time.perf_counter()
        stt = S._capi.run_host(ns, qx32, qy32, prm, out); t3 = time.perf_counter()
        o2 = il.run_tiled(hst, q, il.Params(), cfg, rs); t4 = time.perf_counter()
        rows.append({"prep_ms": 1e3 * (t1 - t0), "native_ms": 1e3 * (t3 - t2), "kernel_ms": stt.kernel_ms,
                     "run_tiled_ms": 1e3 * (t4 - t3)})
    res[name] = rows[2:]
print(json.dumps(res))
