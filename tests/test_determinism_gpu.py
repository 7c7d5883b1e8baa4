"""Results independent of how the queries are cut up (GPU).

The reference pins its outputs bit-identical across worker counts
(test_acceptance.py:181-203, test_strategies.py:211-223): its query blocks
depend only on the workload (strategies.py:15-21,137-138) and every query is
summed in one fixed order.  The B200 analogue: a query's bits must not depend
on m, on the other queries of the call, or on how many devices share the job.

  EXACT   strict reference order -> trivially invariant (checked anyway).
  FAST    tiled: the summation chunks are a function of n alone and queries
          sit in fixed 32*Q-query groups, so any split of the query array at
          group-aligned boundaries (partition.shard_bounds with align=256)
          reproduces the single-call bits; split-reduce and naive have no
          m-dependent state at all.
"""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

ALIGN = 256  # partition.py's shard alignment (a multiple of every K2/K3 query group)


@pytest.fixture(scope="module")
def il():
    import paper_1402_4986_b200 as pkg

    if pkg._capi.device_count() < 1:
        pytest.fail("no CUDA device visible: GPU tests must run on the B200 box")
    return pkg


def cloud(il, n, m, kind="aoas", prec="single"):
    x, y, z = il.generate_cloud_arrays(n, 0)
    qx, qy, _ = il.generate_cloud_arrays(m, il.query_seed(0))
    store = il.LayoutStore.from_arrays(x, y, z, il.LayoutKind(kind), il.Precision(prec))
    return store, np.column_stack([qx, qy])


def sharded(il, fn, store, queries, world, params, cfg):
    from paper_1402_4986_b200.partition import shard_bounds

    parts = []
    for r in range(world):
        lo, hi = shard_bounds(len(queries), world, r, ALIGN)
        parts.append(fn(store, queries[lo:hi], params, cfg))
    return np.concatenate(parts)


def test_fast_tiled_c3_full_equals_eight_shards(il):
    """C3 (1M x 1M, fp32 AoaS, FAST tiled): one call == 8 shard calls, bitwise;
    also == 2 and 4 shards, and a group-aligned prefix of the queries."""
    n = m = 1 << 20
    store, queries = cloud(il, n, m)
    cfg = il.ExecConfig(mode="fast")
    full = il.run_tiled(store, queries, il.Params(), cfg)
    for world in (8, 2, 4):
        got = sharded(il, il.run_tiled, store, queries, world, il.Params(), cfg)
        assert np.array_equal(got, full), world
    pre = il.run_tiled(store, queries[: 3 * ALIGN], il.Params(), cfg)
    assert np.array_equal(pre, full[: 3 * ALIGN])
    idx = np.arange(0, m, m // 512)
    truth = oracle.truth(store, queries[idx])
    assert np.max(np.abs(full[idx] - truth) / np.abs(truth)) <= 1e-5


@pytest.mark.parametrize("prec", ["single", "double"])
def test_fast_tiled_banded_order_bits(il, prec):
    """A store larger than a quarter of L2 (10M points, 160 / 320 MB) is swept
    in bands of query groups, chunk-major inside a band (idw_tiled.cu): the
    item order must not change the bits.  One call (band order,
    several chunks per group in flight) == one call per 256-query shard (a
    group or two each) == a shard split in 3, and a sample is within the FAST
    tolerance of the fp64 truth.  fp32: 160 groups in bands of 100, fp64: 320
    groups in bands of 51 (a short last band in both)."""
    n, m = 10 * (1 << 20), 160 * 256
    store, queries = cloud(il, n, m, "aoas", prec)
    cfg = il.ExecConfig(mode="fast")
    full = il.run_tiled(store, queries, il.Params(), cfg)
    one = np.concatenate([il.run_tiled(store, queries[i:i + ALIGN], il.Params(), cfg) for i in range(0, m, ALIGN)])
    assert np.array_equal(one, full)
    assert np.array_equal(sharded(il, il.run_tiled, store, queries, 3, il.Params(), cfg), full)
    idx = np.arange(0, m, m // 16)
    truth = oracle.truth(store, queries[idx])
    assert np.max(np.abs(full[idx] - truth) / np.abs(truth)) <= {"single": 1e-5, "double": 1e-12}[prec]


BAND_CHILD = """
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_1402_4986_b200 as il
x, y, z = il.generate_cloud_arrays({n}, 0)
qx, qy, _ = il.generate_cloud_arrays({m}, il.query_seed(0))
st = il.LayoutStore.from_arrays(x, y, z, il.LayoutKind({kind!r}), il.Precision({prec!r}))
np.save({out!r}, il.run_tiled(st, np.column_stack([qx, qy]), il.Params({p}), il.ExecConfig(mode="fast")))
"""


@pytest.mark.parametrize("kind,prec,p", [("aoas", "single", 2.0), ("soa", "double", 3.5), ("aos", "single", 1.0)])
def test_fast_tiled_forced_bands_bits(il, tmp_path, kind, prec, p):
    """Band order forced small (IDW_BAND=3, a child process: the knob is read
    once per process) at a size where the default is group-major: dozens of
    bands, a short last band, ring slots reused across bands (groups > R) --
    bitwise equal to the default order."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    n, m = 300_000, 60_000
    store, queries = cloud(il, n, m, kind, prec)
    ref = il.run_tiled(store, queries, il.Params(p), il.ExecConfig(mode="fast"))
    out = tmp_path / "band.npy"
    code = BAND_CHILD.format(root=str(Path(__file__).resolve().parents[1]), n=n, m=m, kind=kind, prec=prec, p=p,
                             out=str(out))
    subprocess.run([sys.executable, "-c", code], check=True, env=dict(os.environ, IDW_BAND="3"))
    assert np.array_equal(np.load(out), ref)


@pytest.mark.parametrize("kind,prec,p", [("soa", "single", 2.0), ("aos", "single", 3.5),
                                         ("soa", "double", 2.0), ("hybrid", "double", 3.5),
                                         ("aoas", "single", 1.0)])
def test_fast_tiled_shards_all_arith(il, kind, prec, p):
    """Every FAST tiled arithmetic (fp32 shared reciprocal, fp32 general and
    integer p, fp64 p = 2 and quarter-root p) at a multi-chunk size."""
    n, m = 300_000, 20_000
    store, queries = cloud(il, n, m, kind, prec)
    cfg = il.ExecConfig(mode="fast")
    full = il.run_tiled(store, queries, il.Params(p), cfg)
    got = sharded(il, il.run_tiled, store, queries, 8, il.Params(p), cfg)
    assert np.array_equal(got, full)
    # a query's value does not depend on the rest of the call
    sub = il.run_tiled(store, queries[ALIGN : 5 * ALIGN], il.Params(p), cfg)
    assert np.array_equal(sub, full[ALIGN : 5 * ALIGN])


def test_fast_tiled_zero_eps_shards(il):
    """zero_eps > 0: the per-chunk hit flag rides the fold (NaN partial) and
    the fix-up returns the coincident z exactly, for any shard layout."""
    n, m = 100_000, 8_192
    store, queries = cloud(il, n, m)
    x, y, z = store.component_views()
    queries[::97] = np.column_stack([x[: len(queries[::97])], y[: len(queries[::97])]])
    prm = il.Params(2.0, 1e-12)
    cfg = il.ExecConfig(mode="fast")
    full = il.run_tiled(store, queries, prm, cfg)
    got = sharded(il, il.run_tiled, store, queries, 4, prm, cfg)
    assert np.array_equal(got, full)
    ref = oracle.predict(store, queries[::97], 2.0, 1e-12)
    assert np.array_equal(full[::97], ref)


@pytest.mark.parametrize("variant", ["run_naive", "run_nested_improved", "run_nested_original"])
@pytest.mark.parametrize("mode", ["fast", "exact"])
def test_other_variants_shards(il, variant, mode):
    n, m = 200_000, 4_096
    store, queries = cloud(il, n, m)
    cfg = il.ExecConfig(mode=mode)
    fn = getattr(il, variant)
    full = fn(store, queries, il.Params(), cfg)
    got = sharded(il, fn, store, queries, 8, il.Params(), cfg)
    assert np.array_equal(got, full)


def test_exact_tiled_shards(il):
    n, m = 200_000, 10_000
    store, queries = cloud(il, n, m, "soa", "single")
    cfg = il.ExecConfig(mode="exact")
    full = il.run_tiled(store, queries, il.Params(), cfg)
    got = sharded(il, il.run_tiled, store, queries, 8, il.Params(), cfg)
    assert np.array_equal(got, full)
    assert np.array_equal(full[::1000], oracle.predict(store, queries[::1000]))


# ---- one call, a device list (ExecConfig.devices; idw_params.devices, ABI 2).
# The 1-GPU box lists device 0 several times: every entry still gets its own
# stream, arena, broadcast copy (a same-device cudaMemcpyPeerAsync) and query
# shard, so the sharding, the broadcast tree and the gather into `out` run
# exactly as on 8 GPUs.

@pytest.mark.parametrize("variant,mode,kind,prec", [
    ("run_tiled", "fast", "aoas", "single"), ("run_tiled", "exact", "soa", "single"),
    ("run_naive", "fast", "aos", "double"), ("run_nested_improved", "fast", "soa", "single"),
    ("run_nested_original", "exact", "hybrid", "double")])
def test_device_list_bitwise(il, variant, mode, kind, prec):
    n, m = 150_000, 5_000
    store, queries = cloud(il, n, m, kind, prec)
    fn = getattr(il, variant)
    one = fn(store, queries, il.Params(), il.ExecConfig(mode=mode, devices=(0,)))
    assert np.array_equal(one, fn(store, queries, il.Params(), il.ExecConfig(mode=mode)))
    for devs in ((0, 0), (0, 0, 0), (0,) * 8):
        stats = il.RunStats()
        got = fn(store, queries, il.Params(), il.ExecConfig(mode=mode, devices=devs), stats)
        assert np.array_equal(got, one), devs
        if variant == "run_nested_original":
            assert stats.merge_events == m * -(-n // 1024)


def test_device_list_c3_fast(il):
    """C3 through one run_tiled call over an 8-entry device list == one device."""
    n = m = 1 << 20
    store, queries = cloud(il, n, m)
    one = il.run_tiled(store, queries, il.Params(), il.ExecConfig(mode="fast"))
    got = il.run_tiled(store, queries, il.Params(), il.ExecConfig(mode="fast", devices=(0,) * 8))
    assert np.array_equal(got, one)


def test_device_list_edges(il):
    """More entries than 256-query units (empty shards), the cast-query entry
    point (idw_run), and the reference's ValueError for a non-finite query."""
    store, queries = cloud(il, 50_000, 300)
    cfg1 = il.ExecConfig(mode="fast")
    one = il.run_tiled(store, queries, il.Params(), cfg1)
    got = il.run_tiled(store, queries, il.Params(), il.ExecConfig(mode="fast", devices=(0,) * 5))
    assert np.array_equal(got, one)
    from paper_1402_4986_b200 import _capi
    from paper_1402_4986_b200.strategies import _native_store

    qx = queries[:, 0].astype(np.float32)
    qy = queries[:, 1].astype(np.float32)
    out = np.empty(len(qx), np.float32)
    prm = _capi.make_params(2.0, 0.0, "tiled", "fast", 1024, 1024, 0, 0, (0, 0, 0))
    _capi.run_host(_native_store(store), qx, qy, prm, out)
    assert np.array_equal(out, one)
    bad = queries.copy()
    bad[299, 1] = np.inf
    with pytest.raises(ValueError, match="invalid coordinate"):
        il.run_tiled(store, bad, il.Params(), il.ExecConfig(mode="fast", devices=(0, 0)))


@pytest.mark.parametrize("variant,mode,kind,prec", [
    ("tiled", "fast", "aoas", "single"), ("tiled", "exact", "soa", "double"),
    ("nested_improved", "fast", "soa", "single"), ("naive", "fast", "aos", "single")])
def test_device_resident_device_list(il, variant, mode, kind, prec):
    """predict_device over a device list (idw_run_device, ABI 2): inputs and
    output on devices[0], the other entries fed by peer copies and their
    predictions gathered back by peer copies, asynchronous on the caller's
    stream -- bitwise equal to one device."""
    import torch

    from paper_1402_4986_b200.device import DeviceStore, predict_device

    store, queries = cloud(il, 120_000, 3_000, kind, prec)
    ds = DeviceStore(store, 0)
    tq = [torch.tensor(queries[:, k].astype(store.precision.dtype), device="cuda") for k in (0, 1)]
    outs = []
    for devs in (None, (0, 0), (0, 0, 0, 0, 0)):
        out = torch.full((len(queries),), float("nan"), dtype=ds.dtype, device="cuda")
        predict_device(ds, tq[0], tq[1], out, il.Params(), il.ExecConfig(mode=mode, devices=devs), variant)
        outs.append(out.cpu().numpy())  # ordered after the call on the current stream
    assert np.array_equal(outs[1], outs[0]) and np.array_equal(outs[2], outs[0])
    assert not np.any(np.isnan(outs[0]))
