"""bench.py contract on CPU: the reference arm (the oracle port of the
reference loop) prints one JSON line with the driver's keys, on the same
metric/config as our arm; under torchrun only rank 0 prints."""

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def _run(args, env_extra=None):
    env = dict(os.environ)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT, env=env,
                          capture_output=True, text=True, timeout=300)


def test_reference_arm_json_line():
    r = _run(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "1"])
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["unit"] == "GPairs/s" and d["value"] > 0
    assert d["higher_is_better"] is True and d["steps"] == 1 and d["warmup"] == 1
    assert d["config"]["workload"].startswith("C1")
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_reference_arm_nonzero_rank_is_silent():
    r = _run(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "1"],
             {"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == ""


def test_reference_arm_never_loads_the_product():
    """the CPU arm runs the reference algorithm only --
    neither the product package nor libidw_b200.so may be loaded."""
    r = _run(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "1"])
    assert r.returncode == 0, r.stderr
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["product_loaded"] is False
    # and in-process: the oracle-side input builder alone imports no product module
    code = ("import sys; sys.path.insert(0, 'oracle'); import refinputs, oracle; "
            "s, q = refinputs.bench_inputs(4096, 64, 'aoas', 'single'); oracle.predict(s, q); "
            "assert not [k for k in sys.modules if k.startswith('paper_1402_4986_b200')]; "
            "assert 'libidw_b200' not in open('/proc/self/maps').read()")
    r2 = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=120)
    assert r2.returncode == 0, r2.stderr
