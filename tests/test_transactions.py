"""Analytic transaction model (CPU): the reference's criterion-4 anchors and
an independent byte-enumeration oracle over random patterns."""

import numpy as np
import pytest

from paper_1402_4986_b200.core import Precision
from paper_1402_4986_b200.layouts import LayoutKind, buffer_shapes
from paper_1402_4986_b200.transactions import AccessPattern, count_transactions, scorecard_csv


def brute(layout, precision, comps, warp, seg, base):
    """Enumerate every byte each lane touches (independent of the model)."""
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


def test_reference_anchor_values():
    # reference test_acceptance.py:114-117
    assert count_transactions(AccessPattern(LayoutKind.AoS, Precision.single, ("x",))).utilization == 1 / 3
    assert count_transactions(AccessPattern(LayoutKind.SoA, Precision.single, ("x",))).utilization == 1.0


def test_random_patterns_match_byte_oracle():
    rng = np.random.default_rng(4)
    subsets = ["x", "y", "z", "xy", "xz", "yz", "xyz"]
    for _ in range(1000):
        layout = list(LayoutKind)[rng.integers(5)]
        precision = Precision.double if layout.requires_double else list(Precision)[rng.integers(2)]
        comps = tuple(subsets[rng.integers(len(subsets))])
        warp, seg, base = int(rng.integers(1, 65)), int(2 ** rng.integers(5, 10)), int(rng.integers(0, 64))
        rep = count_transactions(AccessPattern(layout, precision, comps, warp, seg, base))
        assert (rep.segments, rep.useful_bytes) == brute(layout, precision, comps, warp, seg, base)


def test_validation_and_scorecard():
    with pytest.raises(ValueError):
        AccessPattern(LayoutKind.SoA, Precision.single, ())
    with pytest.raises(ValueError):
        AccessPattern(LayoutKind.SoA, Precision.single, ("x",), segment_bytes=48)
    text = scorecard_csv(Precision.single, "xyz")
    assert "soaos,single,xyz,32,128,n/a" in text and text.count("\n") == 6
