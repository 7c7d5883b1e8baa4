"""§8f3: analytic transaction model vs measured sectors.

`python tools/xcheck_txn.py run <layout>` runs k_nested (fp64 FAST, G = 1024:
each warp-trip reads 32 consecutive points with plain LDGs, the model's access
pattern) on n = 32768 points x m = 1024 queries; under
`ncu --metrics lts__t_sectors_srcunit_tex_op_read.sum,...` that gives measured
sectors.  `python tools/xcheck_txn.py report <dir>` joins the ncu CSVs with
the reference model's count_transactions(segment_bytes=32) x warp-trips
(pinned in tests/golden/transactions_ref.json).
"""
import csv, json, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
N, M, G, Q = 32768, 1024, 1024, 2
LAYOUTS = ["soa", "aos", "aoas", "soaos", "hybrid"]

if sys.argv[1] == "run":
    import numpy as np, torch
    import paper_1402_4986_b200 as il
    from paper_1402_4986_b200.device import DeviceStore, predict_device
    kind = il.LayoutKind(sys.argv[2])
    x, y, z = il.generate_cloud_arrays(N, 0); qx, qy, _ = il.generate_cloud_arrays(M, 1)
    ds = DeviceStore(il.LayoutStore.from_arrays(x, y, z, kind, il.Precision.double), 0)
    tq = [torch.tensor(a, dtype=torch.float64, device="cuda") for a in (qx, qy)]
    out = torch.empty(M, dtype=torch.float64, device="cuda")
    for _ in range(2):
        predict_device(ds, tq[0], tq[1], out, il.Params(), il.ExecConfig(mode="fast", group_size=G), "nested_improved")
    torch.cuda.synchronize()
else:
    # the reference model's answers, pinned from the reference itself
    # (tests/golden/make_txn_golden.py): the product carries no copy of it
    fx = json.loads((ROOT / "tests" / "golden" / "transactions_ref.json").read_text())["cases"]
    model = {c["layout"]: c for c in fx if (c["precision"], c["components"], c["warp"], c["segment"], c["base"])
             == ("double", "xyz", 32, 32, 0)}
    d = Path(sys.argv[2])
    trips = (N // 32) * (M // Q)
    rows = []
    for L in LAYOUTS:
        rep = model[L]
        meas = {}
        f = d / f"xcheck_{L}.csv"
        if f.exists():
            for r in csv.reader(open(f)):
                if len(r) > 3 and r[-3].startswith(("lts__", "l1tex__", "smsp__")):
                    meas[r[-3]] = float(r[-1].replace(",", ""))
        l2 = meas.get("lts__t_sectors_srcunit_tex_op_read.sum")
        l1 = meas.get("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum")
        ins = meas.get("smsp__inst_executed_op_global_ld.sum")
        rows.append({"layout": L, "model_segments_per_warp_trip": rep["segments"], "model_utilization": rep["utilization"],
                     "measured_l2_to_l1_sectors_per_trip": None if l2 is None else l2 / trips,
                     "measured_l1_sectors_per_trip": None if l1 is None else l1 / trips,
                     "ld_instr_per_trip": None if ins is None else ins / trips})
    print(json.dumps(rows, indent=1))
