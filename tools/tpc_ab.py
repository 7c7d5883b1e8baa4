"""A/B of the FAST K2 chunk size (IDW_TPC tiles per chunk; development aid).
Each setting runs in its own process (the knob is read once)."""
import os, subprocess, sys
cases = sys.argv[1:] or ["c3"]
shapes = {"c3": (1 << 20, 1 << 20, "aoas"), "c5": (10 << 20, 100 << 10, "aoas"), "c2": (100 << 10, 100 << 10, "aoas"),
          "c2soa": (100 << 10, 100 << 10, "soa"), "c1": (10 << 10, 10 << 10, "soa"), "c3s8": (1 << 20, 1 << 17, "aoas")}
for tpc in (0, 8, 16, 32, 64, 128):
    for c in cases:
        n, m, kind = shapes[c]
        env = dict(os.environ, IDW_TPC=str(tpc))
        code = (f"import sys; sys.argv=['x']; __file__='tools/quick_perf.py'; exec(open('tools/quick_perf.py').read().split('import subprocess as _sp')[0]);"
                f"print('tpc={tpc} {c}', end=' '); run({n}, {m}, '{kind}', 'single', 'tiled', 'fast', reps=5)")
        subprocess.run([sys.executable, "-c", code], env=env)
