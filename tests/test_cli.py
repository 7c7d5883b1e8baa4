"""CLI (run/bench callers of the hot path): argument handling and file
formats on CPU; the GPU round trip is in test_parity_gpu-style marked tests."""

import numpy as np
import pytest

import oracle
from paper_1402_4986_b200 import cli
from paper_1402_4986_b200.layouts import LayoutKind, build
from paper_1402_4986_b200.core import Precision


def test_parse_size():
    assert cli.parse_size("10k") == 10240 and cli.parse_size("7") == 7


def test_point_io_roundtrip(tmp_path):
    recs = [(0.25, 0.5, 3.0), (1e-17, 0.1, -2.5)]
    cli.write_points_csv(tmp_path / "p.csv", recs)
    assert cli.read_points_csv(tmp_path / "p.csv") == [tuple(r) for r in recs]
    (tmp_path / "bad.csv").write_text("a,b\n1,2\n")
    with pytest.raises(ValueError, match="expected header"):
        cli.read_points_csv(tmp_path / "bad.csv")
    assert cli.read_queries_csv(tmp_path / "p.csv") == [(0.25, 0.5), (1e-17, 0.1)]


def test_usage_errors_exit_2(tmp_path, capsys):
    assert cli.main(["run", "--queries", "q.csv"]) == 2
    assert cli.main(["bench", "--sizes", "8", "--strategies", "bogus", "--out", str(tmp_path / "r.csv")]) == 2
    assert cli.main(["run", "--data", str(tmp_path / "missing.csv"), "--queries", str(tmp_path / "q.csv"),
                     "--out", str(tmp_path / "o.csv")]) == 1
    assert "config:" in capsys.readouterr().out


@pytest.mark.gpu
def test_cli_run_matches_oracle(tmp_path):
    rng = np.random.default_rng(41)
    recs = rng.random((500, 3)) * np.array([1, 1, 100.0])
    qs = rng.random((64, 2))
    cli.write_points_csv(tmp_path / "d.csv", recs)
    with open(tmp_path / "q.csv", "w") as fh:
        fh.write("x,y\n" + "".join(f"{float(a)!r},{float(b)!r}\n" for a, b in qs))
    for strategy in ("seq", "naive", "tiled", "nested-improved", "nested-original"):
        out = tmp_path / f"{strategy}.csv"
        assert cli.main(["run", "--data", str(tmp_path / "d.csv"), "--queries", str(tmp_path / "q.csv"),
                         "--out", str(out), "--layout", "aoas", "--precision", "double",
                         "--strategy", strategy, "--group-size", "64"]) == 0
        got = np.array([float(line.split(",")[2]) for line in out.read_text().splitlines()[1:]])
        st = build(recs, LayoutKind.AoaS, Precision.double)
        ref = oracle.run("seq" if strategy == "seq" else strategy.replace("-", "_"), st, qs, group=64)
        assert np.array_equal(got, ref), strategy
    rep = tmp_path / "rep.csv"
    assert cli.main(["bench", "--sizes", "256", "--repeats", "1", "--warmup", "0", "--out", str(rep)]) == 0
    lines = rep.read_text().splitlines()
    assert lines[0] == cli.REPORT_HEADER and len(lines) == 1 + 1 + 5 * 4 * 2
