"""§8f3 transaction model (CPU): the reference's analytic coalescing model is
an out-of-scope subsystem, so the product carries no copy of it.  Its
answers are pinned as a fixture generated from the reference itself
(tests/golden/make_txn_golden.py) and used by the ncu cross-check
(tools/xcheck_txn.py).  Here the fixture is checked against an independent
byte-enumeration oracle over this package's layout shape table
(layouts.buffer_shapes): every pattern's segment count and useful bytes."""

import json
from pathlib import Path

from paper_1402_4986_b200.core import Precision
from paper_1402_4986_b200.layouts import LayoutKind, buffer_shapes

FIXTURE = Path(__file__).resolve().parent / "golden" / "transactions_ref.json"


def brute(layout, precision, comps, warp, seg, base):
    """Every byte each lane touches -> distinct (buffer, segment) pairs."""
    e = precision.itemsize
    specs = buffer_shapes(layout, precision, base + warp)
    segs = set()
    for lane in range(warp):
        i = base + lane
        for c in comps:
            for b, sp in enumerate(specs):
                if c in sp.offsets:
                    for byte in range(i * sp.stride + sp.offsets[c], i * sp.stride + sp.offsets[c] + e):
                        segs.add((b, byte // seg))
    return len(segs), warp * e * len(comps)


def test_fixture_matches_byte_enumeration():
    data = json.loads(FIXTURE.read_text())
    assert len(data["cases"]) > 400
    for c in data["cases"]:
        kind, prec = LayoutKind(c["layout"]), Precision(c["precision"])
        got = brute(kind, prec, tuple(c["components"]), c["warp"], c["segment"], c["base"])
        assert (c["segments"], c["useful_bytes"]) == got, c
        assert c["utilization"] == c["useful_bytes"] / c["fetched_bytes"]


def test_reference_anchor_values():
    # reference test_acceptance.py:114-117 (criterion 4)
    cases = json.loads(FIXTURE.read_text())["cases"]
    pick = {(c["layout"], c["precision"], c["components"], c["warp"], c["segment"], c["base"]): c for c in cases}
    assert pick[("aos", "single", "x", 32, 128, 0)]["utilization"] == 1 / 3
    assert pick[("soa", "single", "x", 32, 128, 0)]["utilization"] == 1.0
    sc = json.loads(FIXTURE.read_text())["scorecard_xyz"]["single"]
    assert "soaos,single,xyz,32,128,n/a" in sc and sc.count("\n") == 6
