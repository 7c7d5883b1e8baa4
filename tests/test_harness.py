"""Benchmark harness API (CPU): reports byte-identical to the reference's on
the same records (fixture from the reference itself,
tests/golden/make_harness_golden.py), speedups, checksum cross-check and
validation; CLI flags of the reference (--config, --threads / IDW_THREADS,
--report, gen, convert) without a GPU."""

import json
import statistics
from pathlib import Path

import numpy as np
import pytest

from paper_1402_4986_b200 import cli, harness
from paper_1402_4986_b200.core import Precision
from paper_1402_4986_b200.layouts import LayoutKind, LayoutStore

FIXTURE = Path(__file__).resolve().parent / "golden" / "harness_ref.json"


def records():
    fx = json.loads(FIXTURE.read_text())
    out = []
    for layout, strategy, prec, n, p, times, cs, status in fx["records"]:
        r = harness.BenchRecord(layout, strategy, prec, n, p, list(times))
        r.status = status
        if status == "ok":
            r.median_s, r.min_s, r.checksum = statistics.median(times), min(times), cs
        out.append(r)
    return out, fx


def test_reports_identical_to_reference():
    recs, fx = records()
    table = harness.speedup_table(recs, harness.BaselineKey())
    assert [r.speedup for r in table] == fx["speedups"]
    assert harness.report_csv(table) == fx["csv"]
    # markdown: the reference's text plus one line naming the seq baseline
    md = harness.report_markdown(table)
    assert md.replace(f"_{harness.SEQ_NOTE}._\n\n", "") == fx["markdown"]


def test_speedup_and_checksum_rules(tmp_path):
    recs, _ = records()
    with pytest.raises(ValueError, match="baseline not found"):
        harness.speedup_table(recs, harness.BaselineKey(strategy="naive"))
    table = harness.speedup_table(recs, harness.BaselineKey())
    assert table[0].speedup == 1.0 and table[2].speedup is None
    assert table[1].times is not recs[1].times  # records are copied
    harness.verify_checksums(table[:4])  # 123.25 vs 123.2499 within single tol 1e-3
    bad = harness.replace_record(table[3], checksum=124.0)
    with pytest.raises(AssertionError, match="checksum mismatch"):
        harness.verify_checksums([table[1], harness.replace_record(bad, precision="single")])
    harness.emit_report(table, tmp_path / "r.csv", "csv")
    assert (tmp_path / "r.csv").read_text() == harness.report_csv(table)
    with pytest.raises(ValueError, match="unknown report format"):
        harness.emit_report(table, tmp_path / "r.x", "xml")


def test_bench_spec_validation():
    with pytest.raises(ValueError, match="repeats"):
        harness.BenchSpec(repeats=0)
    with pytest.raises(ValueError, match="no data points"):
        harness.BenchSpec(sizes=(0,))
    with pytest.raises(ValueError, match="unknown strategies"):
        harness.BenchSpec(strategies=("bogus",))
    spec = harness.BenchSpec()
    assert spec.sizes == (10240, 51200, 102400) and spec.repeats == 5 and spec.baseline.strategy == "seq"
    rec = harness.time_run(LayoutKind.SoAoS, "tiled", Precision.single, None, (np.zeros(4), np.zeros(4)))
    assert rec.status == "n/a" and rec.n == 4


def test_cli_config_threads_and_required(tmp_path, monkeypatch, capsys):
    cfgf = tmp_path / "c.json"
    cfgf.write_text(json.dumps({"n": "2k", "seed": 5, "format": "csv"}))
    out = tmp_path / "g.csv"
    assert cli.main(["gen", "--config", str(cfgf), "--out", str(out), "--seed", "6"]) == 0
    line = [l for l in capsys.readouterr().out.splitlines() if l.startswith("config:")][0]
    resolved = json.loads(line[len("config: "):])
    assert resolved["n"] == "2k" and resolved["seed"] == 6  # command line wins over the file
    assert len(out.read_text().splitlines()) == 2049
    cfgf.write_text(json.dumps({"bogus": 1}))
    assert cli.main(["gen", "--config", str(cfgf), "--out", str(out)]) == 2
    assert cli.main(["gen", "--out", str(out)]) == 2  # missing --n
    assert cli.main(["convert", "--out", str(out)]) == 2  # missing --in
    monkeypatch.setenv("IDW_THREADS", "3")
    assert cli.resolve_threads(8) == 3
    monkeypatch.delenv("IDW_THREADS")
    assert cli.resolve_threads(8) == 8 and cli.resolve_threads(None) is None
    # the reference's flags parse (no argparse error), e.g. run --threads / bench --report
    ap = cli.build_parser()
    ap.parse_args(["run", "--threads", "8", "--data", "d", "--queries", "q", "--out", "o"])
    ap.parse_args(["bench", "--report", "r.md", "--out", "r.csv", "--threads", "2"])


def test_cli_gen_bin_and_convert_roundtrip(tmp_path):
    dump = tmp_path / "g.bin"
    assert cli.main(["gen", "--n", "100", "--seed", "3", "--format", "bin", "--out", str(dump)]) == 0
    st = LayoutStore.load(dump)
    assert st.kind is LayoutKind.SoA and st.precision is Precision.double and st.count == 100
    aoas = tmp_path / "a.bin"
    assert cli.main(["convert", "--in", str(dump), "--to", "aoas", "--out", str(aoas)]) == 0
    back = LayoutStore.load(aoas)
    assert back.kind is LayoutKind.AoaS and back.records() == st.records()
    csvp = tmp_path / "a.csv"
    assert cli.main(["convert", "--in", str(aoas), "--out", str(csvp)]) == 0
    assert cli.main(["convert", "--in", str(csvp), "--to", "hybrid", "--out", str(tmp_path / "h.bin")]) == 0
    assert LayoutStore.load(tmp_path / "h.bin").records() == st.records()
    assert cli.main(["convert", "--in", str(aoas), "--from", "soa", "--out", str(csvp)]) == 2
