"""Generate tests/golden/transactions_ref.json from the REFERENCE's analytic
coalescing model (idwlayout.transactions.count_transactions, reference
transactions.py:63-81; out of scope for the product).

Run here (the only place /root/reference exists):

    python tests/golden/make_txn_golden.py

The model's answers for a fixed set of access patterns (random layouts,
precisions, component subsets, warp widths, segment sizes, base indices --
plus the k_nested pattern tools/xcheck_txn.py measures with ncu) and its
scorecard CSVs are stored, so the ncu cross-check and its test need neither
the reference nor a restated model on the GPU box.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/idw_numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from idwlayout.core import Precision  # noqa: E402
from idwlayout.layouts import LayoutKind  # noqa: E402
from idwlayout.transactions import AccessPattern, count_transactions, scorecard_csv  # noqa: E402

OUT = Path(__file__).resolve().parent / "transactions_ref.json"


def main() -> None:
    rng = np.random.default_rng(4)
    subsets = ["x", "y", "z", "xy", "xz", "yz", "xyz"]
    cases = []
    pats = [(k.value, "double", "xyz", 32, 32, 0) for k in LayoutKind]  # tools/xcheck_txn.py's pattern
    pats += [("aos", "single", "x", 32, 128, 0), ("soa", "single", "x", 32, 128, 0)]  # criterion-4 anchors
    for _ in range(400):
        kind = list(LayoutKind)[rng.integers(5)]
        prec = "double" if kind.requires_double else ["single", "double"][rng.integers(2)]
        pats.append((kind.value, prec, subsets[rng.integers(len(subsets))], int(rng.integers(1, 65)),
                     int(2 ** rng.integers(5, 10)), int(rng.integers(0, 64))))
    for kind, prec, comps, warp, seg, base in pats:
        rep = count_transactions(AccessPattern(LayoutKind(kind), Precision(prec), tuple(comps), warp, seg, base))
        cases.append({"layout": kind, "precision": prec, "components": comps, "warp": warp, "segment": seg,
                      "base": base, "segments": rep.segments, "useful_bytes": rep.useful_bytes,
                      "fetched_bytes": rep.fetched_bytes, "utilization": rep.utilization})
    scorecards = {p: scorecard_csv(Precision(p), "xyz") for p in ("single", "double")}
    OUT.write_text(json.dumps({"source": "idwlayout.transactions (reference transactions.py:63-114)",
                               "cases": cases, "scorecard_xyz": scorecards}, indent=0))
    print(f"wrote {OUT} ({len(cases)} patterns)")


if __name__ == "__main__":
    main()
