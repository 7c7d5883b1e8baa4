#!/bin/bash
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/quick_perf.py > gpurun_out/quick_perf.log 2>&1
echo "perf rc=$?" >> gpurun_out/quick_perf.log
