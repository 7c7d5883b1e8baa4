"""Shared fixtures.  GPU tests carry @pytest.mark.gpu; everything else runs on
CPU (the driver runs `pytest -m "not gpu"` without a GPU)."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

GOLDEN = ROOT / "tests" / "golden" / "reference_cases.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libidw_b200.so")
    config.addinivalue_line("markers", "slow: long-running GPU case")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN, allow_pickle=False)


@pytest.fixture
def rng():
    return np.random.default_rng(0xC0FFEE)


def random_records(rng, n, lo=0.0, hi=100.0):
    out = rng.random((n, 3))
    out[:, 2] = lo + out[:, 2] * (hi - lo)
    return out


def random_queries(rng, m):
    return rng.random((m, 2))


def golden_case(g, name):
    """(data, queries, p, eps, G, T) of one golden case."""
    p, eps, G, T = g[f"{name}/meta"]
    return (g[f"{name}/data"], g[f"{name}/queries"], float(p), float(eps), int(G),
            None if T < 0 else int(T))
