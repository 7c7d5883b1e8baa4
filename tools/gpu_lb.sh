#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 900 -x -k "packers or dump or device" > gpurun_out/pytest_gpu_layout.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_layout.log
timeout 600 python tools/layout_bench.py > gpurun_out/layout_bench.jsonl 2> gpurun_out/layout_bench.err
