"""Seeded randomized parity sweep (GPU): random sizes (including odd n and m,
n below / above a tile, m below / above a query group), layouts, precisions,
strategies, modes, powers, zero_eps windows with planted coincidences, group
sizes (powers of two and not), coordinate offsets and scales -- against the
reference-pinned C oracle, with the contract of tests/test_parity_gpu.py:

    EXACT, p = 2   bitwise vs the order-matched restatement (naive/tiled:
                   predict_block; split-reduce: nested_improved with G;
                   original nested: nested_original_block with G)
    EXACT, p != 2  1e-5 / 1e-12 relative (CUDA pow vs glibc pow)
    FAST           1e-5 / 1e-12 relative vs the fp64 double-double truth;
                   coincident queries return the first coincident z exactly

The scheduler paths this exercises that fixed-size tests do not: chunk
boundaries at arbitrary n (K2 FAST), the last partial query group, K3's warp
split with G not a power of two, ring-slot reuse, the batched fix-up.
"""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

CASES = 160
TOL = {"single": 1e-5, "double": 1e-12}


@pytest.fixture(scope="module")
def il():
    import paper_1402_4986_b200 as pkg

    if pkg._capi.device_count() < 1:
        pytest.fail("no CUDA device visible: GPU tests must run on the B200 box")
    return pkg


def draw(rng, il):
    kind, prec = il.legal_pairs()[rng.integers(len(il.legal_pairs()))]
    variant = ["naive", "tiled", "nested_improved", "nested_original"][rng.integers(4)]
    mode = ["exact", "fast"][rng.integers(2)]
    n = int(rng.choice([1, 7, 255, 256, 257, 1000, 4099, 20011, 70001]))
    m = int(rng.choice([1, 3, 255, 257, 1031, 2500]))
    if variant == "nested_original":
        n, m = min(n, 20011), min(m, 300)
    p = float(rng.choice([2.0, 2.0, 2.0, 3.0, 3.5, 1.0]))
    G = int(rng.choice([1024, 1024, 64, 100, 33, 512, 2048]))
    eps = float(rng.choice([0.0, 0.0, 0.0, 1e-9]))
    off, scale = float(rng.choice([0.0, 0.0, 1e3, -50.0])), float(rng.choice([1.0, 1.0, 1e-3, 1e4]))
    return kind, prec, variant, mode, n, m, p, G, eps, off, scale


@pytest.mark.parametrize("case", range(CASES))
def test_random_case_against_oracle(il, case):
    rng = np.random.default_rng(1000 + case)
    kind, prec, variant, mode, n, m, p, G, eps, off, scale = draw(rng, il)
    data = rng.random((n, 3))
    data[:, :2] = off + scale * data[:, :2]
    data[:, 2] = 100.0 * data[:, 2]
    queries = off + scale * rng.random((m, 2))
    store = il.build(data, kind, prec)
    xv, yv, _ = store.component_views()
    plant = rng.choice(m, size=min(m, 3), replace=False)  # queries exactly on data points
    src = rng.integers(n, size=plant.size)
    queries[plant] = np.column_stack([xv[src], yv[src]])
    cfg = il.ExecConfig(mode=mode, group_size=G)
    got = il.STRATEGIES[variant](store, queries, il.Params(p, eps), cfg)
    label = (kind.value, prec.value, variant, mode, n, m, p, G, eps, off, scale)
    if mode == "exact":
        ref = oracle.run(variant, store, queries, p, eps, group=G)
        if p == 2.0:
            assert np.array_equal(got.view(np.uint8), ref.view(np.uint8)), label
        else:
            assert np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300)) <= TOL[prec.value], label
        return
    truth = oracle.truth(store, queries, p, eps)
    hit = ~np.isfinite(truth) | np.isin(np.arange(m), plant)
    # coincident queries: the first coincident point's z, exactly (order-matched oracle)
    ref_hits = oracle.predict(store, queries[plant], p, eps)
    assert np.array_equal(got[plant], ref_hits), label
    ok = ~hit & (np.abs(truth) > 1e-300)
    if ok.any():
        rel = np.abs(got[ok].astype(np.float64) - truth[ok]) / np.abs(truth[ok])
        assert np.max(rel) <= TOL[prec.value], label
