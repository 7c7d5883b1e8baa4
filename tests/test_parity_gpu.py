"""GPU parity: the CUDA path (through the C ABI) against the reference's bits.

EXACT mode must reproduce the reference bit-for-bit for p = 2 (every layout,
precision, strategy, G and T of the golden matrix).  General p goes through
CUDA pow instead of glibc pow, so it is held to the north-star tolerances
(1e-5 single, 1e-12 double).  FAST mode is held to those tolerances against
the fp64 double-double truth of the oracle, with coincident queries exact.
"""

import numpy as np
import pytest

import oracle
from conftest import golden_case, random_queries, random_records

pytestmark = pytest.mark.gpu

STRATS = ("naive", "tiled", "nested_original", "nested_improved")
TOL = {"single": 1e-5, "double": 1e-12}


@pytest.fixture(scope="module")
def il():
    import paper_1402_4986_b200 as pkg

    if pkg._capi.device_count() < 1:
        pytest.fail("no CUDA device visible: GPU tests must run on the B200 box")
    return pkg


def _names(g):
    return [str(s) for s in g["names"]]


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))) if a.size else 0.0


@pytest.mark.parametrize("strategy", STRATS)
def test_exact_mode_matches_reference_golden(il, golden, strategy):
    for name in _names(golden):
        data, queries, p, eps, G, T = golden_case(golden, name)
        cfg = il.ExecConfig(group_size=G, tile_size=T, mode="exact")
        for kind, precision in il.legal_pairs():
            store = il.build(data, kind, precision)
            got = il.STRATEGIES[strategy](store, queries, il.Params(p, eps), cfg)
            ref = golden[f"{name}/{precision.value}/{kind.value}/{strategy}"]
            assert got.dtype == ref.dtype
            if p == 2.0:
                assert np.array_equal(got.view(np.uint8), ref.view(np.uint8)), (name, kind, precision, strategy)
            else:
                assert rel(got, ref) <= TOL[precision.value], (name, kind, precision, strategy)


def test_runstats_match_reference(il, golden):
    """GPU-path RunStats (reference strategies.py:104-115, 202-261):
    nested_original's merge_events equal the reference's own count for every
    golden case (m * ceil(n/G), test_strategies.py:124-130), nested_improved
    reports zero merges and G workers of ceil(n/G) trips each
    (test_strategies.py:132-140, test_acceptance.py:97-109), in both modes."""
    for name in _names(golden):
        data, queries, p, eps, G, T = golden_case(golden, name)
        for mode in ("exact", "fast"):
            cfg = il.ExecConfig(group_size=G, tile_size=T, mode=mode)
            for kind, precision in il.legal_pairs():
                store = il.build(data, kind, precision)
                rs = il.RunStats()
                il.run_nested_original(store, queries, il.Params(p, eps), cfg, rs)
                assert rs.merge_events == golden[f"{name}/{precision.value}/{kind.value}/merges"][0], (name, mode)
                assert rs.kernel_launches >= 1
                rs = il.RunStats()
                il.run_nested_improved(store, queries, il.Params(p, eps), cfg, rs)
                assert rs.merge_events == 0
                assert rs.worker_trips is not None and len(rs.worker_trips) == G
                assert np.all(rs.worker_trips == -(-len(data) // G)), (name, mode)


def test_read_counters_match_reference(il, golden):
    for name in _names(golden):
        data, queries, p, eps, G, T = golden_case(golden, name)
        cfg = il.ExecConfig(group_size=G, tile_size=T, mode="exact")
        for kind, precision in il.legal_pairs():
            store = il.build(data, kind, precision)
            for s in STRATS:
                il.STRATEGIES[s](store, queries, il.Params(p, eps), cfg)
            assert store.stats.snapshot() == tuple(golden[f"{name}/{precision.value}/{kind.value}/reads"]), name


def test_idw_predict_seq_matches_reference(il, golden):
    for name in _names(golden):
        data, queries, p, eps, G, T = golden_case(golden, name)
        for precision in il.Precision:
            got = il.idw_predict_seq(data, queries, il.Params(p, eps), precision)
            ref = golden[f"{name}/{precision.value}/seq"]
            if p == 2.0:
                assert np.array_equal(got, ref), (name, precision)
            else:
                assert rel(got, ref) <= TOL[precision.value], (name, precision)


@pytest.mark.parametrize("strategy", ("naive", "tiled", "nested_improved"))
def test_fast_mode_within_tolerance_of_truth(il, golden, strategy):
    for name in _names(golden):
        data, queries, p, eps, G, T = golden_case(golden, name)
        cfg = il.ExecConfig(group_size=G, tile_size=T, mode="fast")
        for kind, precision in il.legal_pairs():
            store = il.build(data, kind, precision)
            got = il.STRATEGIES[strategy](store, queries, il.Params(p, eps), cfg)
            truth = oracle.truth(store, queries, p, eps)
            assert rel(got, truth) <= TOL[precision.value], (name, kind, precision, strategy)


def test_coincidence_exact_all_modes(il):
    rng = np.random.default_rng(3)
    data = random_records(rng, 90)
    data[20] = [data[57][0], data[57][1], 41.0]
    data[57, 2] = 17.0
    queries = np.vstack([random_queries(rng, 5), [data[20][:2]]])
    for mode in ("exact", "fast"):
        for kind, precision in il.legal_pairs():
            store = il.build(data, kind, precision)
            for s, fn in il.STRATEGIES.items():
                got = fn(store, queries, cfg=il.ExecConfig(group_size=16, tile_size=8, mode=mode))
                assert float(got[-1]) == float(np.asarray(41.0, precision.dtype)), (mode, kind, s)


def test_empty_queries_and_validation(il):
    store = il.build(random_records(np.random.default_rng(1), 10), il.LayoutKind.SoA, il.Precision.double)
    for fn in il.STRATEGIES.values():
        got = fn(store, [], cfg=il.ExecConfig(group_size=4))
        assert got.shape == (0,)
        with pytest.raises(ValueError, match="invalid coordinate"):
            fn(store, [(np.nan, 0.0)])
    assert store.stats.snapshot() == (0, 0, 0)


@pytest.mark.parametrize("precision", ["single", "double"])
def test_exact_bitwise_medium_random(il, precision):
    """n = m = 8192: exact naive/tiled bitwise vs oracle seq, nested vs oracle nested."""
    rng = np.random.default_rng(11)
    data = random_records(rng, 8192)
    queries = random_queries(rng, 8192)
    prec = il.Precision(precision)
    store = il.build(data, il.LayoutKind.AoS, prec)
    ref = oracle.predict(store, queries)
    for s in ("naive", "tiled"):
        got = il.STRATEGIES[s](store, queries, cfg=il.ExecConfig(mode="exact"))
        assert np.array_equal(got, ref), s
    sub = queries[:512]
    got = il.run_nested_improved(store, sub, cfg=il.ExecConfig(mode="exact"))
    assert np.array_equal(got, oracle.nested_improved(store, sub)), "nested_improved"


def test_determinism_repeated_runs(il):
    rng = np.random.default_rng(5)
    data = random_records(rng, 3000)
    queries = random_queries(rng, 5000)
    for mode in ("exact", "fast"):
        store = il.build(data, il.LayoutKind.AoaS, il.Precision.single)
        for s, fn in il.STRATEGIES.items():
            cfg = il.ExecConfig(group_size=64, mode=mode)
            assert np.array_equal(fn(store, queries, cfg=cfg), fn(store, queries, cfg=cfg)), (mode, s)


def test_fast_splits_tolerance(il):
    """FAST tiled with forced data splits (the skewed-workload path)."""
    rng = np.random.default_rng(9)
    data = random_records(rng, 200_000)
    queries = random_queries(rng, 3000)
    store = il.build(data, il.LayoutKind.AoaS, il.Precision.single)
    truth = oracle.truth(store, queries)
    for splits in (0, 1, 7, 64):
        got = il.run_tiled(store, queries, cfg=il.ExecConfig(mode="fast", splits=splits))
        assert rel(got, truth) <= 1e-5, splits


@pytest.mark.parametrize("scale", [1e-12, 1e-3, 1.0, 1e4, 1e10, 1e15])
def test_fast_coordinate_scales(il, scale):
    """FAST fp32 over clouds scaled to extreme ranges: the shared-reciprocal
    guard must fall back when a*b could overflow (large scales), and underflow
    (tiny scales: a*b < FLT_MIN for most pairs) must be screened and fixed up
    -- always within tolerance.  (Below ~1e-17 fp32 sums of 1/d2 overflow in
    the reference itself, which then returns NaN; that regime is not tested.)"""
    rng = np.random.default_rng(17)
    data = random_records(rng, 5000)
    data[:, :2] *= scale
    queries = random_queries(rng, 3000) * scale
    store = il.build(data, il.LayoutKind.AoaS, il.Precision.single)
    truth = oracle.truth(store, queries)
    for s in ("tiled", "naive", "nested_improved"):
        got = il.STRATEGIES[s](store, queries, cfg=il.ExecConfig(mode="fast"))
        assert np.all(np.isfinite(got)), (scale, s)
        assert rel(got, truth) <= 1e-5, (scale, s)


def test_fast_queries_on_data_points(il):
    """Every query coincides with a data point: all queries go through the
    exact fix-up and must return that point's z exactly."""
    rng = np.random.default_rng(23)
    data = random_records(rng, 4000)
    idx = rng.choice(4000, size=700, replace=False)
    queries = data[idx, :2]
    for precision in il.Precision:
        store = il.build(data, il.LayoutKind.SoA, precision)
        zs = store.to_arrays()[2]
        ref = oracle.predict(store, queries)
        for s in ("tiled", "naive", "nested_improved"):
            st = il.RunStats()
            got = il.STRATEGIES[s](store, queries, cfg=il.ExecConfig(mode="fast"), instrumentation=st)
            assert np.array_equal(got, ref), (precision, s)
            assert np.array_equal(got, zs[idx]), (precision, s)
            assert st.fixup_queries == len(idx), (precision, s)


def test_exact_zero_field_sign(il):
    """z == 0 everywhere: the reference returns +0.0 (its sums start at +0);
    the negated-sum EXACT path must not hand back -0.0."""
    rng = np.random.default_rng(29)
    data = random_records(rng, 1000)
    data[:, 2] = 0.0
    queries = random_queries(rng, 600)
    for kind, precision in il.legal_pairs():
        store = il.build(data, kind, precision)
        ref = oracle.predict(store, queries)
        for s in ("naive", "tiled"):
            got = il.STRATEGIES[s](store, queries, cfg=il.ExecConfig(mode="exact"))
            assert np.array_equal(got.view(np.uint8), ref.view(np.uint8)), (kind, precision, s)


@pytest.mark.parametrize("kind", ["soa", "aos", "aoas"])
def test_exact_tiled_bitwise_large(il, kind):
    """fp32 EXACT tiled (packed IEEE + inline __frcp_rn fast path) against the
    oracle's left-to-right loop, n = 65536 data x 4096 queries, bitwise."""
    rng = np.random.default_rng(31)
    data = random_records(rng, 65536)
    queries = random_queries(rng, 4096)
    store = il.build(data, il.LayoutKind(kind), il.Precision.single)
    ref = oracle.predict(store, queries)
    got = il.run_tiled(store, queries, cfg=il.ExecConfig(mode="exact"))
    assert np.array_equal(got.view(np.uint8), ref.view(np.uint8))


def test_device_packers_converters_and_dump_loader(il, tmp_path):
    """idw_pack_device / idw_convert_device / DeviceStore.from_dump produce the
    reference's bytes (host LayoutStore as the byte oracle, itself pinned to
    the reference's dumps in test_host.py)."""
    from paper_1402_4986_b200.device import DeviceStore

    rng = np.random.default_rng(37)
    recs = rng.random((1001, 3)) * np.array([1.0, 1.0, 100.0])
    for precision in il.Precision:
        kinds = [k for k in il.LayoutKind if k.legal_for(precision)]
        for a in kinds:
            host = il.build(recs, a, precision)
            dev = DeviceStore.from_arrays(recs[:, 0], recs[:, 1], recs[:, 2], a, precision)
            assert dev.to_host().to_bytes() == host.to_bytes(), (a, precision)
            for b in kinds:
                conv = dev.convert(b).to_host()
                assert conv.to_bytes() == host.convert(b).to_bytes(), (a, b, precision)
            path = tmp_path / f"{a.value}_{precision.value}.idwl"
            host.dump(path)
            assert DeviceStore.from_dump(path).to_host().to_bytes() == host.to_bytes()


def test_single_query_large_n_all_variants(il):
    """m = 1 against n = 300000 (FAST splits the data across the whole GPU;
    EXACT runs one block): exact bitwise vs oracle, fast within tolerance."""
    rng = np.random.default_rng(43)
    data = random_records(rng, 300_000, -50.0, 50.0)
    q = random_queries(rng, 1)
    for precision in il.Precision:
        store = il.build(data, il.LayoutKind.SoA, precision)
        ref = oracle.predict(store, q)
        truth = oracle.truth(store, q)
        for s in ("naive", "tiled"):
            assert np.array_equal(il.STRATEGIES[s](store, q, cfg=il.ExecConfig(mode="exact")), ref), (precision, s)
            assert rel(il.STRATEGIES[s](store, q, cfg=il.ExecConfig(mode="fast")), truth) <= TOL[precision.value]
        got = il.run_nested_improved(store, q, cfg=il.ExecConfig(mode="exact"))
        assert np.array_equal(got, oracle.nested_improved(store, q)), precision


def test_translation_invariance_exact(il):
    """Dyadic-grid coordinates shifted by integers give bit-identical results
    (reference test_core.py:137-163), through the GPU EXACT path."""
    rng = np.random.default_rng(47)
    data = random_records(rng, 2000)
    data[:, :2] = np.round(data[:, :2] * 2 ** 10) / 2 ** 10
    queries = np.round(random_queries(rng, 300) * 2 ** 10) / 2 ** 10
    for precision in il.Precision:
        base = il.run_tiled(il.build(data, il.LayoutKind.AoS, precision), queries, cfg=il.ExecConfig(mode="exact"))
        moved = data.copy()
        moved[:, 0] += 33.0
        moved[:, 1] -= 150.0
        got = il.run_tiled(il.build(moved, il.LayoutKind.AoS, precision), queries + np.array([33.0, -150.0]),
                           cfg=il.ExecConfig(mode="exact"))
        assert np.array_equal(got, base), precision


def test_negative_values_and_hull(il):
    """Negative z and coordinates; predictions stay inside the value hull
    (reference test_core.py:165-173)."""
    rng = np.random.default_rng(53)
    data = random_records(rng, 5000, -3.0, 7.0)
    data[:, :2] -= 0.5
    queries = random_queries(rng, 2000) - 0.5
    for mode in ("exact", "fast"):
        for kind, precision in il.legal_pairs():
            got = il.run_tiled(il.build(data, kind, precision), queries, cfg=il.ExecConfig(mode=mode))
            slack = 1e-4 if precision is il.Precision.single else 1e-12
            assert got.min() >= -3.0 - slack and got.max() <= 7.0 + slack, (mode, kind, precision)


def test_device_resident_path_matches_host_path(il):
    """predict_device (the bench/serving path: HBM-resident store, async on
    the torch stream) == the blocking host API, bitwise, every variant/mode;
    plus the kernel-time and MUFU-probe entry points."""
    import torch

    from paper_1402_4986_b200 import _capi
    from paper_1402_4986_b200.device import DeviceStore, predict_device

    rng = np.random.default_rng(59)
    data = random_records(rng, 20000)
    queries = random_queries(rng, 3000)
    for kind, precision in (("aoas", il.Precision.single), ("soa", il.Precision.double)):
        store = il.build(data, il.LayoutKind(kind), precision)
        ds = DeviceStore(store, 0)
        dt = ds.dtype
        q = [torch.tensor(queries[:, k].astype(precision.dtype), device="cuda") for k in (0, 1)]
        for variant in ("naive", "tiled", "nested_improved", "nested_original"):
            for mode in ("exact", "fast"):
                cfg = il.ExecConfig(mode=mode, group_size=256)
                host = il.STRATEGIES[variant](store, queries, cfg=cfg)
                out = torch.empty(len(queries), dtype=dt, device="cuda")
                predict_device(ds, q[0], q[1], out, il.Params(), cfg, variant)
                ms, fix_ms = _capi.last_kernel_ms()
                assert ms > 0 and fix_ms >= 0
                assert np.array_equal(out.cpu().numpy(), host), (kind, variant, mode)
    rate, _ = _capi.mufu_peak(0)
    assert 1e12 < rate < 2e13  # ~148 SMs x 16/clk x ~2 GHz


@pytest.mark.parametrize("precision", ["single", "double"])
def test_device_aos_store_alignment(il, precision):
    """A device AoS store 4 (fp32) / 8 (fp64) bytes off a 16-byte boundary:
    the kernels that stage tiles with cp.async.bulk (tiled, FAST split-reduce)
    refuse it with an error instead of a misaligned-address fault (which would
    poison the CUDA context); the scalar-load kernels run on it and match the
    host path bitwise; the context stays usable."""
    import torch

    from paper_1402_4986_b200 import _capi

    rng = np.random.default_rng(61)
    data = random_records(rng, 5000)
    queries = random_queries(rng, 700)
    prec = il.Precision(precision)
    store = il.build(data, il.LayoutKind.AoS, prec)
    raw = np.ascontiguousarray(store.buffers[0]).view(np.uint8)
    e = prec.dtype.itemsize
    dev = torch.zeros(raw.nbytes + 64, dtype=torch.uint8, device="cuda")
    dev[e:e + raw.nbytes] = torch.from_numpy(raw).cuda()
    ptr = dev.data_ptr() + e
    assert ptr % 16 != 0
    nstore = _capi.make_store("aos", precision, store.count, [ptr], [raw.nbytes])
    q = [torch.tensor(queries[:, k].astype(prec.dtype), device="cuda") for k in (0, 1)]
    out = torch.empty(len(queries), dtype=q[0].dtype, device="cuda")
    m = len(queries)
    for variant, mode, ok in (("tiled", "exact", False), ("tiled", "fast", False),
                              ("nested_improved", "fast", False), ("nested_improved", "exact", True),
                              ("naive", "fast", True), ("naive", "exact", True)):
        prm = _capi.make_params(2.0, 0.0, variant, mode, 1024, il.ExecConfig().tile_size)
        if not ok:
            with pytest.raises(_capi.NativeError, match="16-byte aligned"):
                _capi.run_device(nstore, q[0].data_ptr(), q[1].data_ptr(), m, prm, out.data_ptr())
            continue
        _capi.run_device(nstore, q[0].data_ptr(), q[1].data_ptr(), m, prm, out.data_ptr())
        torch.cuda.synchronize()
        host = il.STRATEGIES[variant](store, queries, cfg=il.ExecConfig(mode=mode))
        assert np.array_equal(out.cpu().numpy(), host), (variant, mode)
    torch.cuda.synchronize()  # no sticky error left behind
    assert np.array_equal(il.run_tiled(store, queries), oracle.predict(store, queries))


@pytest.mark.parametrize("scale", [1e-70, 1e-20, 1e-3, 1.0, 1e18, 1e40])
def test_fast_fp64_general_p_scales(il, scale):
    """FAST fp64 general p (quarter-root series for p in multiples of 1/2,
    exp2/log2 otherwise) across coordinate scales that put d2 below 2^-125 or
    above 2^125 -- outside the fp32 seed range every such weight is forced to
    NaN, so the query must come back through the exact fix-up -- and a few
    near-coincident queries.  Within 1e-12 of the fp64 truth, finite."""
    rng = np.random.default_rng(61)
    data = random_records(rng, 6000)
    data[:, :2] *= scale
    queries = random_queries(rng, 1500) * scale
    queries[:5] = data[:5, :2] * (1.0 + 1e-9)  # near-coincident (tiny d2 only)
    for kind in (il.LayoutKind.SoA, il.LayoutKind.AoaS):
        store = il.build(data, kind, il.Precision.double)
        for p in (3.5, 3.0, 1.5, 2.7):
            truth = oracle.truth(store, queries, p)
            for s in ("tiled", "naive", "nested_improved"):
                got = il.STRATEGIES[s](store, queries, il.Params(p), cfg=il.ExecConfig(mode="fast"))
                assert np.all(np.isfinite(got)), (scale, kind, p, s)
                assert rel(got, truth) <= 1e-12, (scale, kind, p, s)


@pytest.mark.parametrize("scale", [1e-160, 1e-140, 1e-3, 1e150])
def test_exact_fp64_scales_bitwise(il, scale):
    """fp64 EXACT p = 2 across exponent ranges: d2 ~ 1e-320 (denormal: the
    inline __drcp_rn path seeds inf, the query is screened and recomputed),
    d2 ~ 1e-280 (inline path, normal range), d2 ~ 1e300 (box guard off: the
    library __drcp_rn).  Bitwise against the reference loop (NaN where the
    reference itself overflows to inf/inf)."""
    rng = np.random.default_rng(67)
    data = random_records(rng, 3000)
    data[:, :2] *= scale
    queries = random_queries(rng, 700) * scale
    for kind in (il.LayoutKind.SoA, il.LayoutKind.AoaS, il.LayoutKind.Hybrid):
        store = il.build(data, kind, il.Precision.double)
        ref = oracle.predict(store, queries)
        for s in ("tiled", "naive"):
            got = il.STRATEGIES[s](store, queries, cfg=il.ExecConfig(mode="exact"))
            both_nan = np.isnan(got) & np.isnan(ref)
            assert np.array_equal(got[~both_nan].view(np.uint8), ref[~both_nan].view(np.uint8)), (scale, kind, s)
            assert np.array_equal(np.isnan(got), np.isnan(ref)), (scale, kind, s)


def test_device_side_prepare_matches_host_cast(il):
    """idw_run_xy (the (m, 2) float64 queries split, cast RN and checked on the
    device) == idw_run over the host-cast qx, qy (strategies._prepare), bitwise;
    a NaN or inf anywhere raises the reference's ValueError."""
    from paper_1402_4986_b200 import _capi, strategies

    rng = np.random.default_rng(71)
    data = random_records(rng, 5000)
    queries = random_queries(rng, 3001) * 3.0 - 1.0
    for kind, precision in (("aoas", il.Precision.single), ("soa", il.Precision.double)):
        store = il.build(data, il.LayoutKind(kind), precision)
        for variant in ("tiled", "naive", "nested_improved"):
            for mode in ("exact", "fast"):
                prm = _capi.make_params(2.0, 0.0, variant, mode, 1024, 1024)
                qx, qy, dt = strategies._prepare(store, queries, il.Params())
                a = np.empty(len(queries), dt)
                _capi.run_host(strategies._native_store(store), qx, qy, prm, a)
                b = np.empty(len(queries), dt)
                _capi.run_host_xy(strategies._native_store(store), np.ascontiguousarray(queries), prm, b)
                assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), (kind, variant, mode)
        for bad in (np.nan, np.inf, -np.inf):
            q = queries.copy()
            q[1234, 1] = bad
            with pytest.raises(ValueError, match="invalid coordinate"):
                il.run_tiled(store, q)


def test_plan_graph_replay_matches_run_device(il):
    """idw_plan (the call captured into a CUDA graph) == idw_run_device,
    bitwise, for every variant/mode; refilling the query tensors in place and
    relaunching gives the new batch's predictions; timing nodes work."""
    import torch

    from paper_1402_4986_b200.device import DevicePlan, DeviceStore, predict_device

    rng = np.random.default_rng(73)
    data = random_records(rng, 30000)
    qa, qb = random_queries(rng, 2500), random_queries(rng, 2500)
    qa[7] = data[11, :2]  # a coincidence: the fix-up node must run inside the graph
    for kind, precision in (("soa", il.Precision.single), ("aos", il.Precision.double)):
        store = il.build(data, il.LayoutKind(kind), precision)
        ds = DeviceStore(store, 0)
        for variant in ("tiled", "naive", "nested_improved", "nested_original"):
            for mode in ("exact", "fast"):
                cfg = il.ExecConfig(mode=mode, group_size=512)
                q = [torch.tensor(qa[:, k].astype(precision.dtype), device="cuda") for k in (0, 1)]
                out = torch.empty(len(qa), dtype=ds.dtype, device="cuda")
                plan = DevicePlan(ds, q[0], q[1], out, il.Params(), cfg, variant)
                assert plan.launches >= 1
                plan.launch()
                ms, _ = plan.kernel_ms()
                assert ms > 0
                ref = torch.empty_like(out)
                predict_device(ds, q[0], q[1], ref, il.Params(), cfg, variant)
                assert torch.equal(out.view(torch.uint8), ref.view(torch.uint8)), (kind, variant, mode)
                for k in (0, 1):
                    q[k].copy_(torch.tensor(qb[:, k].astype(precision.dtype)))
                plan.launch()
                predict_device(ds, q[0], q[1], ref, il.Params(), cfg, variant)
                assert torch.equal(out.view(torch.uint8), ref.view(torch.uint8)), (kind, variant, mode, "refill")
                plan.close()


def test_split_reduce_persistent_clusters(il):
    """K3 at a size where every persistent cluster walks many query groups
    (20K queries / 8 per team >> resident clusters) and the ring of the next
    group is primed during the tree: FAST within 1e-5 of the truth (fp32) /
    1e-12 (fp64), EXACT bitwise equal to the reference's nested_improved."""
    rng = np.random.default_rng(79)
    data = random_records(rng, 150_000)
    queries = random_queries(rng, 20_000)
    sub = np.arange(0, 20_000, 97)
    for precision in il.Precision:
        store = il.build(data, il.LayoutKind.AoaS, precision)
        truth = oracle.truth(store, queries[sub])
        fast = il.run_nested_improved(store, queries, cfg=il.ExecConfig(mode="fast"))
        assert np.all(np.isfinite(fast))
        assert rel(fast[sub], truth) <= TOL[precision.value], precision
        exact = il.run_nested_improved(store, queries[sub], cfg=il.ExecConfig(mode="exact"))
        assert np.array_equal(exact, oracle.nested_improved(store, queries[sub])), precision


@pytest.mark.parametrize("p", [1.0, 3.0, 4.0, 1.5])
def test_fast_fp32_integer_p(il, p):
    """FAST fp32 integer p compiles to one MUFU per pair (rsqrt^p for odd p,
    rcp^(p/2) for even p; p = 1.5 keeps lg2/ex2): within 1e-5 of the fp64
    truth for tiled, split-reduce and naive, with a coincident query fixed up
    exactly."""
    rng = np.random.default_rng(83)
    data = random_records(rng, 40_000)
    queries = random_queries(rng, 3000)
    queries[11] = data[5, :2]
    for kind in (il.LayoutKind.AoaS, il.LayoutKind.SoA):
        store = il.build(data, kind, il.Precision.single)
        truth = oracle.truth(store, queries, p)
        for s in ("tiled", "nested_improved", "naive"):
            got = il.STRATEGIES[s](store, queries, il.Params(p), cfg=il.ExecConfig(mode="fast"))
            assert got[11] == store.to_arrays()[2][5], (kind, s)
            assert rel(got, truth) <= 1e-5, (kind, p, s)


def test_exact_split_reduce_subnormal_d2_bitwise(il):
    """Screened EXACT split-reduce in fp32 runs packed query pairs with
    __frcp_rn's fast path inline; a subnormal d2 (which that path flushes)
    leaves the query flagged, and k_fixup recomputes it in K3's own order
    (G strided lanes + adjacent-pair tree).  Queries a subnormal distance
    (d2 ~ 2^-127.5, 1/d2 still finite) from a data point at the origin must
    come out bit-identical to the reference's nested_improved."""
    rng = np.random.default_rng(89)
    data = random_records(rng, 3000, 0.0, 1.0)
    data[:, :2] = 0.1 + 0.9 * data[:, :2]
    data[7] = (0.0, 0.0, 0.37)
    deltas = [2.0 ** -63.2, 2.0 ** -63.5, 2.0 ** -63.8, 2.0 ** -63.95]
    queries = np.vstack([np.array([[d, 0.0] for d in deltas] + [[0.0, d] for d in deltas]),
                         random_queries(rng, 200)])
    store = il.build(data, il.LayoutKind.SoA, il.Precision.single)
    for G in (1024, 256, 64):
        ref = oracle.nested_improved(store, queries, group=G)
        assert np.all(np.isfinite(ref[:8]))
        got = il.run_nested_improved(store, queries, cfg=il.ExecConfig(mode="exact", group_size=G))
        assert np.array_equal(got.view(np.uint8), ref.view(np.uint8)), G
    # the strict-order strategies take the same inline path (sequential recompute)
    ref = oracle.predict(store, queries)
    for s in ("naive", "tiled"):
        got = il.STRATEGIES[s](store, queries, cfg=il.ExecConfig(mode="exact"))
        assert np.array_equal(got.view(np.uint8), ref.view(np.uint8)), s


def test_exact_split_reduce_subnormal_d2_bitwise_fp64(il):
    """fp64 counterpart: the inline __drcp_rn path seeds inf for a subnormal
    d2 (~2^-1023.5, 1/d2 still finite); the query is recomputed in K3's order
    by k_fixup and must match the reference's nested_improved bitwise."""
    rng = np.random.default_rng(97)
    data = random_records(rng, 3000, 0.0, 1.0)
    data[:, :2] = 0.1 + 0.9 * data[:, :2]
    data[7] = (0.0, 0.0, 0.37)
    deltas = [2.0 ** -511.2, 2.0 ** -511.6, 2.0 ** -511.9]
    queries = np.vstack([np.array([[d, 0.0] for d in deltas] + [[0.0, d] for d in deltas]),
                         random_queries(rng, 200)])
    for kind in (il.LayoutKind.SoA, il.LayoutKind.Hybrid):
        store = il.build(data, kind, il.Precision.double)
        for G in (1024, 128):
            ref = oracle.nested_improved(store, queries, group=G)
            assert np.all(np.isfinite(ref[:6]))
            got = il.run_nested_improved(store, queries, cfg=il.ExecConfig(mode="exact", group_size=G))
            assert np.array_equal(got.view(np.uint8), ref.view(np.uint8)), (kind, G)


def test_exact_fixup_many_subnormal_queries_1m(il):
    """The strict-order recompute of flagged no-hit queries (EXACT naive and
    tiled; reference predict_block, kernels.py:49-63) is batched: 32 queries
    per block advance together through one pass over the data, their exact
    weights computed block-wide and summed left to right by one lane each.
    2048 queries a subnormal distance from a data point at n = 1M must come
    back bitwise equal to the reference's sums, in well under a second."""
    import time

    n = 1 << 20
    rng = np.random.default_rng(123)
    data = random_records(rng, n, 0.0, 1.0)
    data[:, :2] = 0.1 + 0.9 * data[:, :2]
    data[12345] = (0.0, 0.0, 0.37)
    k = 2048
    deltas = 2.0 ** -rng.uniform(63.05, 63.99, k)
    sub = np.where(rng.random(k)[:, None] < 0.5, np.column_stack([deltas, 0 * deltas]),
                   np.column_stack([0 * deltas, deltas]))
    queries = np.vstack([sub, random_queries(rng, 2048)])
    store = il.build(data, il.LayoutKind.AoaS, il.Precision.single)
    ref = oracle.predict_mt(store, queries)
    assert np.all(np.isfinite(ref[:k]))
    for s in ("tiled", "naive"):
        fn = il.STRATEGIES[s]
        cfg = il.ExecConfig(mode="exact")
        fn(store, queries[:300], cfg=cfg)  # warm-up (pool pages, first launch)
        st = il.RunStats()
        t0 = time.perf_counter()
        got = fn(store, queries, il.Params(), cfg, st)
        dt = time.perf_counter() - t0
        assert np.array_equal(got.view(np.uint8), ref.view(np.uint8)), s
        assert st.fixup_queries >= k, (s, st.fixup_queries)
        assert dt < 1.0, (s, dt)
