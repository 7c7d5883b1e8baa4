"""A/B of library builds (IDW_B200_LIB) on FAST tiled shapes; development aid.
usage: lib_ab.py lib1.so lib2.so ... [-- case ...]; each run in its own process,
libraries interleaved per case and repeated twice to expose drift."""
import os, subprocess, sys
argv = sys.argv[1:]
libs = argv[: argv.index("--")] if "--" in argv else argv
cases = argv[argv.index("--") + 1:] if "--" in argv else ["c3", "c1", "c2", "c2soa", "c5"]
shapes = {"c3": (1 << 20, 1 << 20, "aoas", "single", 2.0), "c5": (10 << 20, 100 << 10, "aoas", "single", 2.0),
          "c2": (100 << 10, 100 << 10, "aoas", "single", 2.0), "c2soa": (100 << 10, 100 << 10, "soa", "single", 2.0),
          "c1": (10 << 10, 10 << 10, "soa", "single", 2.0), "c3s8": (1 << 20, 1 << 17, "aoas", "single", 2.0),
          "c2d": (100 << 10, 100 << 10, "soa", "double", 2.0), "c2p": (100 << 10, 100 << 10, "aoas", "single", 3.5)}
mode = os.environ.get("AB_MODE", "fast")
for rep in range(2):
    for c in cases:
        n, m, kind, prec, p = shapes[c]
        for lib in libs:
            env = dict(os.environ, IDW_B200_LIB=os.path.abspath(lib))
            reps = 3 if n * m > 1e11 else 7
            code = (f"import sys; sys.argv=['x']; __file__='tools/quick_perf.py'; "
                    f"exec(open('tools/quick_perf.py').read().split('import subprocess as _sp')[0]);"
                    f"print('{os.path.basename(lib)} {c}', end=' '); run({n}, {m}, '{kind}', '{prec}', 'tiled', '{mode}', p={p}, reps={reps})")
            subprocess.run([sys.executable, "-c", code], env=env)
