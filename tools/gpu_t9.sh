#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu --timeout 900 -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/c2_grid.py exact > gpurun_out/c2_grid_exact.jsonl 2> gpurun_out/c2_grid.err
