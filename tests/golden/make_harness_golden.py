"""Generate tests/golden/harness_ref.json from the REFERENCE's benchmark
harness (idwlayout.bench: speedup_table, report_csv, report_markdown,
verify_checksums; reference bench.py:205-303) on fixed synthetic records.

    python tests/golden/make_harness_golden.py      (here, where /root/reference exists)

tests/test_harness.py feeds the same records to paper_1402_4986_b200.harness
and requires byte-identical reports.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/idw_numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from idwlayout.bench import BaselineKey, BenchRecord, report_csv, report_markdown, speedup_table  # noqa: E402

OUT = Path(__file__).resolve().parent / "harness_ref.json"

RECORDS = [  # (layout, strategy, precision, n, p, times, checksum, status)
    ("-", "seq", "double", 8, 2.0, [0.5, 0.25, 0.75], 123.25, "ok"),
    ("soa", "naive", "single", 8, 2.0, [0.125, 0.0625], 123.2499, "ok"),
    ("soaos", "tiled", "single", 8, 2.0, [], None, "n/a"),
    ("aoas", "tiled", "double", 8, 2.0, [0.03125, 0.1, 0.2], 123.25000000001, "ok"),
    ("-", "seq", "double", 16, 3.5, [1.0], 7.0, "ok"),
    ("hybrid", "nested_improved", "double", 16, 3.5, [0.3, 0.1], 7.000000000001, "ok"),
]


def make(cls):
    import statistics
    out = []
    for layout, strategy, prec, n, p, times, cs, status in RECORDS:
        r = cls(layout, strategy, prec, n, p, list(times))
        r.status = status
        if status == "ok":
            r.median_s = statistics.median(times)
            r.min_s = min(times)
            r.checksum = cs
        out.append(r)
    return out


def main() -> None:
    recs = speedup_table(make(BenchRecord), BaselineKey())
    OUT.write_text(json.dumps({"records": RECORDS, "csv": report_csv(recs), "markdown": report_markdown(recs),
                               "speedups": [r.speedup for r in recs]}, indent=1))
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
