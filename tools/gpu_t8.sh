#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu --timeout 900 -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/nested_ab.py fp32 > gpurun_out/nested_fp32.jsonl 2>&1
timeout 300 python tools/nested_ab.py > gpurun_out/nested_fp64.jsonl 2>&1
