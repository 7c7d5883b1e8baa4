#!/bin/bash
# Build libidw_b200 variants that differ only in idw_tiled.cu's compile-time
# knobs, for A/B timing: name:-DKNOB=v,-DKNOB2=w ...  Output build/tv/lib_<name>.so
set -e
cd "$(dirname "$0")/../paper_1402_4986_b200/csrc"
NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
OUT=../../build/tv
mkdir -p $OUT
for v in "$@"; do
  name=${v%%:*}; defs=$(echo ${v#*:} | tr ',' ' ')
  nvcc $NVFLAGS $defs -c idw_tiled.cu -o $OUT/tiled_$name.o &
done
wait
for v in "$@"; do
  name=${v%%:*}
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/lib_$name.so \
    build/idw_capi.o build/idw_naive.o build/idw_nested.o build/idw_layout_dev.o $OUT/tiled_$name.o
done
