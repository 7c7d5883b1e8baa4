#!/bin/bash
mkdir -p gpurun_out
for v in "$@"; do
  IDW_B200_LIB=$PWD/build/variants/lib_$v.so timeout 300 python tools/nested_ab.py fp32 >> gpurun_out/nested_ab3.jsonl 2>> gpurun_out/nested_ab3.err
done
