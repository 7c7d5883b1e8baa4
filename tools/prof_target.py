"""Run one configuration twice (warm + profiled) for ncu captures."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
from quick_perf import run
K = 1024
T = {
    "c3": (1024 * K, 1024 * K, "aoas", "single", "tiled", "fast"),
    "c2_exact": (100 * K, 100 * K, "aoas", "single", "tiled", "exact"),
    "c2_fp64": (100 * K, 100 * K, "soa", "double", "tiled", "fast"),
    "c4": (1024 * K, 16 * K, "soa", "double", "nested_improved", "fast"),
    "c5_nested": (10240 * K, 25 * K, "aoas", "single", "nested_improved", "fast"),
    "naive_aoas": (100 * K, 100 * K, "aoas", "single", "naive", "fast"),
    "naive_soa": (100 * K, 100 * K, "soa", "single", "naive", "fast"),
    "naive_aos": (100 * K, 100 * K, "aos", "single", "naive", "fast"),
    "tiled64_p35": (100 * K, 100 * K, "aoas", "double", "tiled", "fast"),
    "c1": (10 * K, 10 * K, "soa", "single", "tiled", "fast"),
    "c2_nested": (100 * K, 100 * K, "aoas", "single", "nested_improved", "fast"),
    "c2": (100 * K, 100 * K, "aoas", "single", "tiled", "fast"),
    "c5": (10240 * K, 100 * K, "aoas", "single", "tiled", "fast"),
}
name = sys.argv[1]
if name.startswith("c2tiled:"):  # c2tiled:<layout>:<precision>
    _, kind, prec = name.split(":")
    T[name] = (100 * K, 100 * K, kind, prec, "tiled", "fast")
args = T[name]
p = 3.5 if name in ("c4", "tiled64_p35") else 2.0
run(*args, p=p, reps=1)
