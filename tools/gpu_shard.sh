mkdir -p gpurun_out/shard
python tools/shard_perf.py > gpurun_out/shard/shard_perf.jsonl 2> gpurun_out/shard/err.log
python - > gpurun_out/shard/devlist_e2e.jsonl 2>> gpurun_out/shard/err.log <<'PY'
import json, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1402_4986_b200 as il
n = m = 1 << 20
x, y, z = il.generate_cloud_arrays(n, 0); qx, qy, _ = il.generate_cloud_arrays(m, 1)
st = il.LayoutStore.from_arrays(x, y, z, il.LayoutKind.AoaS, il.Precision.single)
pinned = []
for b in st.buffers:
    t = torch.empty(b.nbytes, dtype=torch.uint8, pin_memory=True); t.numpy()[:] = b; pinned.append(t.numpy())
hs = il.LayoutStore(st.kind, st.precision, n, pinned, st.shapes)
tq = torch.empty((m, 2), dtype=torch.float64, pin_memory=True); tq.numpy()[:] = np.column_stack([qx, qy]); hq = tq.numpy()
for devs in (None, (0,), (0, 0), (0,) * 4, (0,) * 8):
    cfg = il.ExecConfig(mode="fast", devices=devs)
    il.run_tiled(hs, hq, il.Params(), cfg)
    t0 = time.perf_counter()
    for _ in range(3):
        il.run_tiled(hs, hq, il.Params(), cfg)
    dt = (time.perf_counter() - t0) / 3
    print(json.dumps(dict(devices=devs, s=dt, gpairs=n * m / dt / 1e9)), flush=True)
PY
