#!/bin/bash
mkdir -p gpurun_out
for c in c2 c5; do
  timeout 600 python bench.py --config $c --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches_$c.csv \
    python bench.py --config $c --steps 2 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
done
