#!/bin/bash
# round-2 GPU check: full GPU test suite (incl. BASELINE-config parity) + a short C3 bench
set -x
mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -x -rA --durations=30 -p no:cacheprovider -s > gpurun_out/r2/pytest_gpu.log 2>&1
echo "pytest_rc=$?" >> gpurun_out/r2/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2/bench_c3.json 2> gpurun_out/r2/bench_c3.err
echo bench_rc=$?
tail -3 gpurun_out/r2/pytest_gpu.log
