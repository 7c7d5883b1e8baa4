#!/bin/bash
mkdir -p gpurun_out
timeout 120 ./tools/microbench > gpurun_out/microbench.json 2>&1
timeout 900 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python tools/quick_perf.py > gpurun_out/quick_perf.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tiled -s 1 -c 1 \
    -o gpurun_out/prof_tiled2 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/prof_tiled.log 2>&1
