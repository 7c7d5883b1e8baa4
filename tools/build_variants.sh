#!/bin/bash
# Build libidw_b200 variants that differ only in idw_nested.cu's compile-time
# knobs (fp64 K3 queries per thread Q, trips per batch U) for A/B timing.
set -e
cd "$(dirname "$0")/../paper_1402_4986_b200/csrc"
NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
OUT=../../build/nv
mkdir -p $OUT
# v = name:extra nvcc defines (comma separated), e.g. r0u8:-DIDW_NEST_RING32=0,-DIDW_NEST_U32=8
for v in "$@"; do
  name=${v%%:*}; defs=$(echo ${v#*:} | tr ',' ' ')
  nvcc $NVFLAGS $defs -c idw_nested.cu -o $OUT/nested_$name.o &
done
wait
for v in "$@"; do
  name=${v%%:*}
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/lib_$name.so \
    build/idw_capi.o build/idw_naive.o build/idw_tiled.o build/idw_layout_dev.o $OUT/nested_$name.o
done
