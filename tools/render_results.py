"""Markdown tables of the committed round evidence (profiles/r1/bench/*.json,
c2_grid.jsonl) for DESIGN.md / profiles/r1/SUMMARY.md."""
import json
from collections import defaultdict
from pathlib import Path
B = Path(__file__).resolve().parents[1] / "profiles" / "r1" / "bench"
names = {"c1": "C1 10K² fp32 SoA tiled", "c2": "C2 100K² fp32 AoaS tiled", "c3": "**C3 1M² fp32 AoaS tiled**",
         "c4": "C4 1M² fp64 SoA p = 3.5 split-reduce", "c5": "C5 10M × 100K fp32 AoaS tiled + splits"}
print("| config | value GPairs/s | dominant kernels | roofline frac | e2e | CPU port, threads |")
print("|---|---|---|---|---|---|")
for c in ("c1", "c2", "c3", "c4", "c5"):
    d = json.load(open(B / f"bench_{c}.json"))
    r = d["roofline"]
    frac = f"{r['frac']:.2f}"
    if "kernel_mix_bound" in r:
        frac += f" of MUFU ({r['kernel_mix_bound']['frac']:.2f} of the mix ceiling)"
    elif r["bound"] == "fp64":
        frac += f" of FP64 ({r['baseline_definition']['frac']:.2f}× the BASELINE-defined roofline)"
    print(f"| {names[c]} | {d['value']:.0f} | {r['achieved']:.0f} | {frac} | {d['e2e']['value']:.0f} | "
          f"{d['cpu_baseline']['value']:.1f} ({d['cpu_baseline']['cores']}) |")
ref = json.load(open(B / "bench_reference_c3.json"))
print(f"\nreference arm (C3 sample, {ref['cpu_baseline']['cores']} threads): {ref['value']:.1f} GPairs/s")
rows = [json.loads(l) for l in open(B / "c2_grid.jsonl")]
t = defaultdict(dict)
for r in rows:
    t[(r["precision"], r["layout"])][(r["variant"], r["mode"])] = r["gpairs"]
vs = ("naive", "tiled", "nested_improved", "nested_original")
cols = [(v, m) for m in ("fast", "exact") for v in vs]
print()
print("| precision | layout | " + " | ".join(
    f"{v.replace('nested_improved', 'split-reduce').replace('nested_original', 'orig-nested')} {m.upper()}"
    for v, m in cols) + " |")
print("|---|---|" + "---|" * len(cols))
for k, v in t.items():
    print(f"| {k[0]} | {k[1]} | " + " | ".join(f"{v.get(c, 0):.0f}" for c in cols) + " |")
