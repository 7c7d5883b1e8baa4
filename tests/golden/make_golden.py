"""Generate tests/golden/reference_cases.npz from the REFERENCE itself.

Run here (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports the read-only reference package ``idwlayout`` from
/root/reference/pkg/src (numba cache redirected to /tmp so nothing is
written into the reference tree), runs every reference strategy on a set of
small cases that cover the reference's own test matrix, and stores inputs and
outputs.  The committed .npz pins the C oracle (tests/test_oracle_golden.py,
CPU) and the GPU path (tests/test_parity_gpu.py) to the reference's bits
without the reference being present on the GPU box.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/idw_numba_cache")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True
REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

import numpy as np  # noqa: E402

import idwlayout as il  # noqa: E402
from idwlayout.bench import query_seed  # noqa: E402
from idwlayout.core import Params, Precision  # noqa: E402
from idwlayout.layouts import LayoutKind, legal_pairs  # noqa: E402
from idwlayout.strategies import STRATEGIES, ExecConfig, RunStats  # noqa: E402

OUT = Path(__file__).resolve().parent / "reference_cases.npz"


def rng_records(seed, n, lo=0.0, hi=100.0):
    r = np.random.default_rng(seed)
    d = r.random((n, 3))
    d[:, 2] = lo + d[:, 2] * (hi - lo)
    return d


def grid_inputs(n, seed):
    data = il.generate_cloud_arrays(n, seed)
    qx, qy, _ = il.generate_cloud_arrays(n, query_seed(seed))
    return np.column_stack(data), np.column_stack([qx, qy])


def cases():
    """(name, data, queries, p, zero_eps, G, T, strategies)"""
    allS = tuple(STRATEGIES)
    d, q = rng_records(1, 400), np.random.default_rng(2).random((150, 2))
    yield "rand400", d, q, 2.0, 0.0, 64, None, allS
    d, q = rng_records(3, 333), np.random.default_rng(4).random((97, 2))
    yield "aos333_g32_t17", d, q, 2.0, 0.0, 32, 17, allS
    d, q = rng_records(5, 200), np.random.default_rng(6).random((31, 2))
    yield "p3_n200", d, q, 3.0, 0.0, 64, None, allS
    d, q = rng_records(7, 256), np.random.default_rng(8).random((40, 2))
    yield "p35_n256", d, q, 3.5, 0.0, 128, None, allS
    # two coincident sites, lowest index (20) must win; query 5 hits it
    d = rng_records(9, 90)
    d[20] = [d[57][0], d[57][1], 41.0]
    d[57, 2] = 17.0
    q = np.vstack([np.random.default_rng(10).random((5, 2)), [d[20][:2]]])
    yield "coincide90", d, q, 2.0, 0.0, 16, 8, allS
    # zero_eps window: d2 = 1e-8 <= 1e-6
    d = rng_records(11, 40)
    d[7, :2] = (0.5, 0.5)
    q = np.array([(0.5 + 1e-4, 0.5), (0.1, 0.9)])
    yield "eps_window", d, q, 2.0, 1e-6, 8, None, allS
    # remainders everywhere + coincident last query (test_acceptance c8)
    r = np.random.default_rng(12)
    d = r.random((1000, 3)) * np.array([1, 1, 50.0])
    site = (d[431, 0], d[431, 1])
    d[77] = [site[0], site[1], -7.0]
    q = np.vstack([r.random((529, 2)), [site]])
    yield "remainders1000", d, q, 2.0, 0.0, 128, 96, allS
    d, q = grid_inputs(1024, 2024)
    yield "grid1024", d, q, 2.0, 0.0, 1024, None, allS
    d, q = grid_inputs(1024, 77)
    yield "grid1024_p35", d, q[:64], 3.5, 0.0, 1024, None, allS
    d, q = rng_records(13, 100), np.random.default_rng(14).random((13, 2))
    yield "g_gt_n", d, q, 2.0, 0.0, 256, None, allS
    d, q = rng_records(15, 37), np.random.default_rng(16).random((9, 2))
    yield "g1", d, q, 2.0, 0.0, 1, None, allS
    d, q = rng_records(17, 300), np.random.default_rng(18).random((21, 2))
    yield "g100_nonpow2", d, q, 2.0, 0.0, 100, 37, allS
    d, q = rng_records(19, 3000), np.random.default_rng(20).random((8, 2))
    yield "g2048_wide", d, q, 2.0, 0.0, 2048, None, allS
    d = np.array([[0.25, 0.75, 5.0]])
    q = np.array([(0.25, 0.75), (0.9, 0.1)])
    yield "single_point", d, q, 2.0, 0.0, 4, None, allS


def main():
    blobs = {}
    names = []
    for name, data, queries, p, eps, G, T, strategies in cases():
        names.append(name)
        blobs[f"{name}/data"] = data
        blobs[f"{name}/queries"] = queries
        blobs[f"{name}/meta"] = np.array([p, eps, G, -1 if T is None else T], dtype=np.float64)
        cfg = ExecConfig(group_size=G, tile_size=T, parallel_width=2)
        for precision in Precision:
            seq = il.idw_predict_seq(data, queries, Params(p, eps), precision)
            blobs[f"{name}/{precision.value}/seq"] = seq
        for kind, precision in legal_pairs():
            store = il.build(data, kind, precision)
            for sname in strategies:
                rs = RunStats()
                got = STRATEGIES[sname](store, queries, Params(p, eps), cfg, rs)
                blobs[f"{name}/{precision.value}/{kind.value}/{sname}"] = got
                if sname == "nested_original":
                    blobs[f"{name}/{precision.value}/{kind.value}/merges"] = np.array([rs.merge_events])
            blobs[f"{name}/{precision.value}/{kind.value}/reads"] = np.array(store.stats.snapshot())
    # byte-exact layout dumps of a small cloud
    recs = rng_records(21, 7) * np.array([1.0, 1.0, 1.0])
    blobs["dump/records"] = recs
    for kind, precision in legal_pairs():
        blobs[f"dump/{precision.value}/{kind.value}"] = np.frombuffer(
            il.build(recs, kind, precision).to_bytes(), dtype=np.uint8)
    # generator: splitmix64 words and the reference's frozen 10K cloud sums
    blobs["gen/splitmix_seed0"] = il.splitmix64(0, 3)
    blobs["gen/splitmix_seed1234567"] = il.splitmix64(1234567, 2)
    x, y, z = il.generate_cloud_arrays(10 * 1024, 7)
    blobs["gen/cloud10k_seed7_sum"] = np.array([float(np.sum(x) + np.sum(y) + np.sum(z))])
    blobs["gen/cloud10k_seed7_ends"] = np.array([x[0], y[0], z[0], x[-1], y[-1], z[-1]])
    blobs["names"] = np.array(names)
    np.savez_compressed(OUT, **blobs)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(names)} cases)")


if __name__ == "__main__":
    main()
