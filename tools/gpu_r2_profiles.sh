#!/bin/bash
# Round-2 ncu evidence for FAST K2 (k_tiled_chunks): one --set full capture per
# bench config (raw CSV kept under profiles/r2), plus the C3 launch list.
set -x
mkdir -p gpurun_out/r2p
for c in c3 c1 c2 c5; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tiled_chunks --launch-skip 2 -c 1 \
    -o gpurun_out/r2p/prof_$c python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2p/ncu_$c.log 2>&1
  ncu -i gpurun_out/r2p/prof_$c.ncu-rep --page raw --csv > gpurun_out/r2p/prof_$c.raw.csv 2>/dev/null
  # keep the report only for C3 (gpurun copies back <= 64 MiB)
  [ "$c" = c3 ] || rm -f gpurun_out/r2p/prof_$c.ncu-rep
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2p/launches_c3.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2p/launches_c3.log 2>&1
ls -la gpurun_out/r2p
