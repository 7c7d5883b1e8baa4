#!/bin/bash
mkdir -p gpurun_out
for v in q2_u1 q2_u4 q4_u2 q4_u4; do
  IDW_B200_LIB=$PWD/build/variants/lib_$v.so timeout 300 python tools/nested_ab.py >> gpurun_out/nested_ab.jsonl 2>> gpurun_out/nested_ab.err
done
IDW_POOL_KEEP=0 timeout 300 python tools/e2e_breakdown.py > gpurun_out/e2e_pool0.json 2>&1
IDW_POOL_KEEP=1 timeout 300 python tools/e2e_breakdown.py > gpurun_out/e2e_pool1.json 2>&1
timeout 600 python bench.py --config c1 --no-cpu > gpurun_out/bench_c1_new.json 2> gpurun_out/bench_c1_new.err
