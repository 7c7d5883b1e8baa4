#!/bin/bash
# One bench line per BASELINE config (c3 is the driver's default line), the
# reference arm, the launch list of the default command, the C2 layout grid,
# the per-shard scaling probe.
mkdir -p gpurun_out/bench
for c in c3 c1 c2 c4 c5; do
  timeout 900 python bench.py --config $c > gpurun_out/bench/bench_$c.json 2> gpurun_out/bench/bench_$c.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench/bench_reference_c3.json 2>&1
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/bench/launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
timeout 1200 python tools/c2_grid.py > gpurun_out/bench/c2_grid.jsonl 2> gpurun_out/bench/c2_grid.err
timeout 600 python tools/shard_perf.py > gpurun_out/bench/shard_perf.jsonl 2>&1
