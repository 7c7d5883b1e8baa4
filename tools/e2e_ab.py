"""A/B of the host-buffer (e2e) call path between library builds; development aid.
usage: e2e_ab.py lib1.so lib2.so ...  (C1 and C2 shapes, pinned inputs, median of 5 x 100 calls)"""
import os, subprocess, sys

CHILD = r'''
import sys, time, statistics
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1402_4986_b200 as il
for name, n, kind in (("c1", 10 << 10, "soa"), ("c2", 100 << 10, "aoas")):
    x, y, z = il.generate_cloud_arrays(n, 0)
    qx, qy, _ = il.generate_cloud_arrays(n, 1)
    st = il.LayoutStore.from_arrays(x, y, z, il.LayoutKind(kind), il.Precision.single)
    pinned = []
    for b in st.buffers:
        t = torch.empty(b.nbytes, dtype=torch.uint8, pin_memory=True); t.numpy()[:] = b; pinned.append(t.numpy())
    hs = il.LayoutStore(st.kind, st.precision, n, pinned, st.shapes)
    tq = torch.empty((n, 2), dtype=torch.float64, pin_memory=True); tq.numpy()[:] = np.column_stack([qx, qy])
    q = tq.numpy(); cfg = il.ExecConfig(mode="fast")
    reps = 100 if name == "c1" else 20
    for _ in range(5): il.run_tiled(hs, q, il.Params(), cfg)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        for _ in range(reps): il.run_tiled(hs, q, il.Params(), cfg)
        ts.append((time.perf_counter() - t0) / reps)
    t = statistics.median(ts)
    print(f"{sys.argv[1]} {name} {t * 1e6:8.1f} us/call {n * n / t / 1e9:8.1f} GPairs/s", flush=True)
'''
libs = sys.argv[1:]
for rep in range(2):
    for lib in libs:
        subprocess.run([sys.executable, "-c", CHILD, os.path.basename(lib)],
                       env=dict(os.environ, IDW_B200_LIB=os.path.abspath(lib)))
