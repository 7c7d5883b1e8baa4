"""Per-rank workload of the query-sharded C3 job at N = 1, 2, 4, 8 on one
GPU: n = 1M data x m/N queries (the shard bounds of partition.shard_bounds),
device-resident, CUDA events, best of 3.  Shows whether the kernel keeps its
rate when the shard shrinks (the strong-scaling question)."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1402_4986_b200 as il
from paper_1402_4986_b200 import _capi
from paper_1402_4986_b200.device import DeviceStore, predict_device
from paper_1402_4986_b200.partition import shard_bounds
n = m = 1 << 20
x, y, z = il.generate_cloud_arrays(n, 0)
qx, qy, _ = il.generate_cloud_arrays(m, 1)
ds = DeviceStore(il.LayoutStore.from_arrays(x, y, z, il.LayoutKind.AoaS, il.Precision.single), 0)
cfg = il.ExecConfig(mode="fast")
for N in (1, 2, 4, 8):
    lo, hi = shard_bounds(m, N, 0, 256)
    tq = [torch.tensor(a[lo:hi], dtype=torch.float32, device="cuda") for a in (qx, qy)]
    out = torch.empty(hi - lo, dtype=torch.float32, device="cuda")
    predict_device(ds, tq[0], tq[1], out, il.Params(), cfg, "tiled")
    torch.cuda.synchronize()
    best = None
    for _ in range(3):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); predict_device(ds, tq[0], tq[1], out, il.Params(), cfg, "tiled"); e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        best = t if best is None else min(best, t)
    k, f = _capi.last_kernel_ms()
    print(json.dumps(dict(N=N, m_shard=hi - lo, s=best, gpairs=n * (hi - lo) / best / 1e9,
                          kernel_ms=k, fixup_ms=f, projected_job_gpairs=N * n * (hi - lo) / best / 1e9)), flush=True)
