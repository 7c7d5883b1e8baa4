#!/bin/bash
# Round evidence: one bench line per BASELINE config + reference arm, the
# launch list of the default command, ncu --set full of the dominant kernels,
# the C2 layout grid and the per-shard scaling probe.
OUT=gpurun_out/final
mkdir -p $OUT
nvidia-smi > $OUT/smi.txt 2>&1
for c in c3 c1 c2 c4 c5; do
  timeout 900 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference_c3.json 2>&1
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file $OUT/launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
timeout 1500 python tools/c2_grid.py orig > $OUT/c2_grid.jsonl 2> $OUT/c2_grid.err
timeout 600 python tools/layout_bench.py > $OUT/layout_bench.jsonl 2> $OUT/layout_bench.err
timeout 1200 python -m pytest tests -q -m gpu --timeout 900 > $OUT/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 600 python tools/shard_perf.py > $OUT/shard_perf.jsonl 2>&1
cap() {  # name kernel-regex target
  timeout 900 ncu --clock-control none --set full --import-source on -k regex:$2 -s 1 -c 1 -o $OUT/$1 \
      python tools/prof_target.py $3 > $OUT/$1.log 2>&1
  ncu -i $OUT/$1.ncu-rep --page raw --csv > $OUT/$1.raw.csv 2>/dev/null
  ncu -i $OUT/$1.ncu-rep --page details --csv > $OUT/$1.details.csv 2>/dev/null
  rm -f $OUT/$1.ncu-rep
}
cap prof_c3_tiled k_tiled c3
cap prof_c4 k_nested c4
cap prof_c2 k_tiled c2
cap prof_c5 k_tiled c5
cap prof_c1 k_tiled c1
cap prof_c2_fp64 k_tiled c2_fp64
cap prof_c2_exact k_tiled c2_exact
du -sh $OUT
