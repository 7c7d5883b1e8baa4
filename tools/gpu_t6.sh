#!/bin/bash
mkdir -p gpurun_out
for c in c1 c2; do
  timeout 600 python bench.py --config $c --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 300 python tools/host_overhead.py > gpurun_out/host_overhead.json 2>&1
