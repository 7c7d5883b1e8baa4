#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/host_overhead.py > gpurun_out/host_overhead.json 2>&1
timeout 600 python bench.py --config c1 --no-cpu > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 1200 python tools/c2_grid.py > gpurun_out/c2_grid.jsonl 2> gpurun_out/c2_grid.err
