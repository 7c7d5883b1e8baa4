#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/quick_perf.py exact > gpurun_out/quick_perf_exact.log 2>&1
timeout 600 python tools/quick_perf.py nested > gpurun_out/quick_perf_nested.log 2>&1
