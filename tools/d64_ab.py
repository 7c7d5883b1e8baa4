"""A/B of library builds on fp64 FAST shapes (K2 tiled and K3), development aid."""
import os, subprocess, sys
libs = sys.argv[1:]
K = 1024
cases = [("tiled", 1024 * K, 64 * K, "soa", 3.5), ("nested_improved", 1024 * K, 64 * K, "soa", 3.5),
         ("tiled", 100 * K, 100 * K, "soa", 2.0), ("nested_improved", 100 * K, 100 * K, "soa", 2.0),
         ("tiled", 100 * K, 100 * K, "hybrid", 3.5)]
for rep in range(2):
    for v, n, m, kind, p in cases:
        for lib in libs:
            env = dict(os.environ, IDW_B200_LIB=os.path.abspath(lib))
            code = (f"import sys; sys.argv=['x']; __file__='tools/quick_perf.py'; "
                    f"exec(open('tools/quick_perf.py').read().split('import subprocess as _sp')[0]);"
                    f"print('{os.path.basename(lib)} {v}-{kind}-{p}', end=' '); run({n}, {m}, '{kind}', 'double', '{v}', 'fast', p={p}, reps=2)")
            subprocess.run([sys.executable, "-c", code], env=env)
