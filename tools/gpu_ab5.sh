#!/bin/bash
mkdir -p gpurun_out
python tools/nested_ab.py fp32 > gpurun_out/nested_ab5.jsonl 2>&1
for v in "$@"; do
  IDW_B200_LIB=$PWD/build/variants/lib_$v.so timeout 300 python tools/nested_ab.py fp32 >> gpurun_out/nested_ab5.jsonl 2>&1
done
