"""A/B of library builds on the K3 (split-reduce) FAST shapes; development aid.
usage: nested_ab.py lib1.so lib2.so ..."""
import os, subprocess, sys
libs = sys.argv[1:]
K = 1024
cases = {"c4": (1024 * K, 1024 * K, "soa", "double", 3.5), "c4s": (1024 * K, 64 * K, "soa", "double", 3.5),
         "c2d": (100 * K, 100 * K, "soa", "double", 2.0), "c2dh": (100 * K, 100 * K, "hybrid", "double", 3.5),
         "c2d_aoas": (100 * K, 100 * K, "aoas", "double", 2.0)}
for rep in range(2):
    for c, (n, m, kind, prec, p) in cases.items():
        for lib in libs:
            env = dict(os.environ, IDW_B200_LIB=os.path.abspath(lib))
            reps = 1 if n * m > 1e11 else 3
            code = (f"import sys; sys.argv=['x']; __file__='tools/quick_perf.py'; "
                    f"exec(open('tools/quick_perf.py').read().split('import subprocess as _sp')[0]);"
                    f"print('{os.path.basename(lib)} {c}', end=' '); run({n}, {m}, '{kind}', '{prec}', 'nested_improved', 'fast', p={p}, reps={reps})")
            subprocess.run([sys.executable, "-c", code], env=env)
