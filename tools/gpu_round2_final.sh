#!/bin/bash
# Round-2 evidence: GPU tests (incl. the reference's own suite), smoke, one
# bench line per BASELINE config + EXACT C3 + the reference arm, the C3 launch
# list, ncu --set full of the dominant kernels (raw CSVs; reports deleted so
# the copy-back stays < 64 MiB), the C2 grid, a 2-rank gloo bench on one GPU.
OUT=gpurun_out/final2
mkdir -p $OUT
nvidia-smi > $OUT/smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -rA --durations=20 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1
echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
cap() {  # name kernel-regex target
  timeout 900 ncu --clock-control none --set full --import-source on -k regex:$2 -s 1 -c 1 -o $OUT/$1 \
      python tools/prof_target.py $3 > $OUT/$1.log 2>&1
  ncu -i $OUT/$1.ncu-rep --page raw --csv > $OUT/$1.raw.csv 2>/dev/null
  rm -f $OUT/$1.ncu-rep
}
cap prof_c3 k_tiled_chunks c3
cap prof_c1 k_tiled_chunks c1
cap prof_c2 k_tiled_chunks c2
cap prof_c5 k_tiled_chunks c5
cap prof_c4 k_nested c4
cap prof_c2_fp64 k_tiled_chunks c2_fp64
cap prof_c2_exact k_tiled c2_exact
# the bench lines read their DRAM traffic from these captures
cp $OUT/prof_*.raw.csv profiles/r2/
for c in c3 c1 c2 c4 c5; do
  timeout 900 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 900 python bench.py --mode exact > $OUT/bench_c3_exact.json 2> $OUT/bench_c3_exact.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference_c3.json 2>&1
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file $OUT/launches_c3.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
timeout 1500 python tools/c2_grid.py orig > $OUT/c2_grid.jsonl 2> $OUT/c2_grid.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --device-override 0 --no-cpu \
    > $OUT/bench_2rank_gloo_single_gpu.json 2> $OUT/bench_2rank_gloo.err
du -sh $OUT
