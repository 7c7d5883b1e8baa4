"""Break down one e2e run_tiled call (host buffers) on C3."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1402_4986_b200 as il
from paper_1402_4986_b200 import strategies as S
n = m = 1 << 20
x, y, z = il.generate_cloud_arrays(n, 0); qx, qy, _ = il.generate_cloud_arrays(m, 1)
st = il.LayoutStore.from_arrays(x, y, z, il.LayoutKind.AoaS, il.Precision.single)
pinned = []
for b in st.buffers:
    t = torch.empty(b.nbytes, dtype=torch.uint8, pin_memory=True); t.numpy()[:] = b; pinned.append(t.numpy())
hst = il.LayoutStore(st.kind, st.precision, n, pinned, st.shapes)
q = np.column_stack([qx, qy]); cfg = il.ExecConfig(mode="fast")
for i in range(5):
    rs = il.RunStats()
    t0 = time.perf_counter(); qx32, qy32, dt = S._prepare(hst, q, il.Params()); t1 = time.perf_counter()
    out = il.run_tiled(hst, q, il.Params(), cfg, rs); t2 = time.perf_counter()
    print(json.dumps({"prep_s": t1 - t0, "call_s": t2 - t1, "kernel_ms": rs.kernel_ms, "launches": rs.kernel_launches}), flush=True)
