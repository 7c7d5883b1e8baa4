"""Host layer (CPU): byte-exact layout packers, generator, validation and the
reference-compatible Python API, checked against fixtures the reference made
(tests/golden/) and against the reference's own test expectations."""

import math

import numpy as np
import pytest

import paper_1402_4986_b200 as il
from paper_1402_4986_b200 import core, layouts, strategies
from paper_1402_4986_b200.layouts import LayoutKind, LayoutStore, buffer_shapes, build, legal_pairs
from paper_1402_4986_b200.core import Params, Precision


# ---- layouts ---------------------------------------------------------------
def test_dumps_byte_identical_to_reference(golden):
    recs = golden["dump/records"]
    for kind, precision in legal_pairs():
        ours = np.frombuffer(build(recs, kind, precision).to_bytes(), dtype=np.uint8)
        assert np.array_equal(ours, golden[f"dump/{precision.value}/{kind.value}"]), (kind, precision)


def test_dump_roundtrip_and_errors(tmp_path):
    st = build(np.random.default_rng(1).random((33, 3)), LayoutKind.Hybrid, Precision.double)
    p = tmp_path / "s.idwl"
    st.dump(p)
    back = LayoutStore.load(p)
    assert back.kind is LayoutKind.Hybrid and back.count == 33
    for a, b in zip(st.component_views(), back.component_views()):
        assert np.array_equal(a, b)
    blob = st.to_bytes()
    with pytest.raises(ValueError, match="truncated"):
        LayoutStore.from_bytes(blob[:5])
    with pytest.raises(ValueError, match="bad magic"):
        LayoutStore.from_bytes(b"XXXX" + blob[4:])
    with pytest.raises(ValueError, match="wrong size"):
        LayoutStore.from_bytes(blob + b"\0")


@pytest.mark.parametrize("kind,precision,strides", [
    (LayoutKind.SoA, Precision.single, (4, 4, 4)),
    (LayoutKind.AoS, Precision.single, (12,)),
    (LayoutKind.AoS, Precision.double, (24,)),
    (LayoutKind.AoaS, Precision.single, (16,)),
    (LayoutKind.AoaS, Precision.double, (32,)),
    (LayoutKind.SoAoS, Precision.double, (16, 16)),
    (LayoutKind.Hybrid, Precision.double, (16, 8)),
])
def test_strides(kind, precision, strides):
    assert tuple(s.stride for s in buffer_shapes(kind, precision, 1)) == strides


def test_alignment_pads_and_illegal_pairs():
    st = build(np.random.default_rng(2).random((10, 3)), LayoutKind.AoaS, Precision.single)
    assert all(b.ctypes.data % 64 == 0 for b in st.buffers)
    raw = st.buffers[0].view(np.float32).reshape(10, 4)
    assert np.all(raw[:, 3] == 0)
    with pytest.raises(ValueError, match="layout requires double precision"):
        build([(0, 0, 0)], LayoutKind.SoAoS, Precision.single)
    with pytest.raises(ValueError, match="no data points"):
        build([], LayoutKind.SoA, Precision.double)
    with pytest.raises(ValueError, match="invalid coordinate"):
        build([(0, math.nan, 0)], LayoutKind.SoA, Precision.double)


def test_conversion_value_exact_and_counters():
    recs = np.random.default_rng(3).random((500, 3)) * 100
    for precision in Precision:
        kinds = [k for k in LayoutKind if k.legal_for(precision)]
        for a in kinds:
            for b in kinds:
                st = build(recs, a, precision)
                back = st.convert(b).convert(a)
                for u, v in zip(st.component_views(), back.component_views()):
                    assert np.array_equal(u, v)
    st = build(recs, LayoutKind.AoS, Precision.double)
    st.read_point(3)
    st.read_components(4, "xz")
    st.load_tile(10, 20)
    assert st.stats.snapshot() == (12, 11, 12)
    with pytest.raises(IndexError):
        st.read_point(500)
    with pytest.raises(ValueError, match="empty component set"):
        st.read_components(0, "")


def test_reference_store_is_accepted_shape(golden):
    """The host layer duck-types stores: kind/precision values and buffers are
    all it needs (a reference LayoutStore has exactly these)."""
    st = build(golden["dump/records"], LayoutKind.AoaS, Precision.single)
    ns = strategies._native_store(st)
    assert ns.kind == 2 and ns.precision == 0 and ns.count == 7 and ns.nbuf == 1
    assert ns.nbytes[0] == 7 * 16


# ---- generator ---------------------------------------------------------------
def test_generator_matches_reference(golden):
    assert il.splitmix64(0, 3).tolist() == golden["gen/splitmix_seed0"].tolist()
    assert il.splitmix64(1234567, 2).tolist() == golden["gen/splitmix_seed1234567"].tolist()
    x, y, z = il.generate_cloud_arrays(10 * 1024, 7)
    assert float(np.sum(x) + np.sum(y) + np.sum(z)) == golden["gen/cloud10k_seed7_sum"][0]
    ends = golden["gen/cloud10k_seed7_ends"]
    assert (x[0], y[0], z[0], x[-1], y[-1], z[-1]) == tuple(ends)
    assert il.query_seed(2 ** 64 - 1) == 0
    with pytest.raises(ValueError, match="no data points"):
        il.generate_cloud_arrays(0, 1)


# ---- core / strategies API ---------------------------------------------------------
def test_params_and_weights():
    assert Params() == Params(2.0, 0.0)
    for bad in ({"p": 0.0}, {"p": -1.0}, {"zero_eps": -0.5}):
        with pytest.raises(ValueError):
            Params(**bad)
    assert il.weight(4.0, 2.0) == 0.25 and il.weight(4.0, 3.0) == 0.125
    with pytest.raises(ValueError):
        il.weight(0.0)
    assert il.squared_distance((1.5, -2), (-0.5, 1)) == 13
    assert core.prediction_ulps(1.0, 1.0 + 2 * math.ulp(1.0)) == 2.0
    assert Precision.parse("Single") is Precision.single
    with pytest.raises(ValueError):
        Precision.parse("half")


def test_exec_config():
    cfg = strategies.ExecConfig()
    assert cfg.group_size == 1024 and cfg.tile_size == 1024 and cfg.parallel_width >= 1
    assert cfg.mode == "exact" and cfg.splits == 0
    for bad in ({"group_size": 0}, {"tile_size": 0}, {"parallel_width": 0}, {"mode": "turbo"}, {"splits": -1}):
        with pytest.raises(ValueError):
            strategies.ExecConfig(**bad)


def test_reduce_tree_shape():
    A = strategies.Accumulator
    assert strategies.reduce_tree([A(0.1, 0.2), A(0.2, 0.4), A(0.3, 0.6), A(0.4, 0.8)]).sum_w == (0.1 + 0.2) + (0.3 + 0.4)
    assert strategies.reduce_tree([A(v, 0.0) for v in (0.1, 0.7, 1e-17)]).sum_w == (0.1 + 0.7) + 1e-17
    got = strategies.reduce_tree([A(1, 1, None), A(1, 1, 9), A(1, 1, 2), A(1, 1, None)])
    assert got.hit_index == 2
    with pytest.raises(ValueError, match="empty reduction"):
        strategies.reduce_tree([])


def test_strategy_validation_before_native_call():
    st = build(np.random.default_rng(4).random((4, 3)), LayoutKind.SoA, Precision.double)
    for fn in il.STRATEGIES.values():
        with pytest.raises(ValueError, match="invalid coordinate"):
            fn(st, [(np.nan, 0.0)])
        with pytest.raises(ValueError, match="queries must be"):
            fn(st, [(0.0, 0.0, 0.0)])
    assert strategies.strategy_tolerance(Precision.double, 10) == 1e-9
    assert strategies.strategy_tolerance(Precision.single, 256) == 1e-4
    assert strategies.strategy_tolerance(Precision.single, 257) == 1e-3
    assert set(il.STRATEGIES) == {"naive", "tiled", "nested_original", "nested_improved"}


def test_oracle_side_inputs_match_product(golden):
    """oracle/refinputs.py (used by bench's reference arm, which must not
    import the product) builds the same cloud and the same component values."""
    import refinputs

    x, y, z = refinputs.cloud(10 * 1024, 7)
    assert float(np.sum(x) + np.sum(y) + np.sum(z)) == golden["gen/cloud10k_seed7_sum"][0]
    assert refinputs.query_seed(0) == il.query_seed(0)
    px, py, pz = il.generate_cloud_arrays(5000, 3)
    for kind, precision in legal_pairs():
        ours = LayoutStore.from_arrays(px, py, pz, kind, precision)
        ref = refinputs.OracleStore(px, py, pz, kind.value, precision.value)
        for a, b in zip(ours.component_views(), ref.component_views()):
            assert a.dtype == b.dtype and np.array_equal(a, b), (kind, precision)
        if kind.value in ("soa", "aos", "aoas"):
            assert b"".join(bytes(np.ascontiguousarray(b)) for b in ref.buffers) == ours.to_bytes()[-sum(
                b.nbytes for b in ours.buffers):], (kind, precision)
