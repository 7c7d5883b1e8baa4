"""BASELINE configs[1]: 100K x 100K, p = 2, all eight legal (layout,
precision) pairs x naive / tiled / split-reduce (nested_improved), FAST and
EXACT, on one B200.  Device-resident inputs, CUDA events on the launching
stream, best of 3 after a warm-up; GPairs/s = n*m / time.  Writes JSON lines
to stdout (one per run) -- the paper's layout study on B200."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1402_4986_b200 as il
from paper_1402_4986_b200 import _capi
from paper_1402_4986_b200.device import DeviceStore, predict_device

n = m = 100 * 1024
x, y, z = il.generate_cloud_arrays(n, 0)
qx, qy, _ = il.generate_cloud_arrays(m, il.query_seed(0))
modes = [a for a in sys.argv[1:] if a in ("fast", "exact")] or ["fast", "exact"]
VARIANTS = ("naive", "tiled", "nested_improved", "nested_original") if "orig" in sys.argv else \
    ("naive", "tiled", "nested_improved")
for kind, prec in il.legal_pairs():
    st = il.LayoutStore.from_arrays(x, y, z, kind, prec)
    ds = DeviceStore(st, 0)
    tq = [torch.tensor(a.astype(prec.dtype), device="cuda") for a in (qx, qy)]
    out = torch.empty(m, dtype=ds.dtype, device="cuda")
    for variant in VARIANTS:
        for mode in modes:
            cfg = il.ExecConfig(mode=mode)
            predict_device(ds, tq[0], tq[1], out, il.Params(), cfg, variant)
            torch.cuda.synchronize()
            best = None
            for _ in range(3):
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                e0.record(); predict_device(ds, tq[0], tq[1], out, il.Params(), cfg, variant); e1.record()
                torch.cuda.synchronize()
                t = e0.elapsed_time(e1) / 1e3
                best = t if best is None else min(best, t)
            kms, fms = _capi.last_kernel_ms()
            print(json.dumps(dict(layout=kind.value, precision=prec.value, variant=variant, mode=mode,
                                  s=best, gpairs=n * m / best / 1e9, kernel_ms=kms, fixup_ms=fms)), flush=True)
