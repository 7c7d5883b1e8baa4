#!/bin/bash
# One bench line per BASELINE config (c3 is the driver's default line).
mkdir -p gpurun_out
for c in c3 c1 c2 c4 c5; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2>&1
