#!/bin/bash
# Full-library variants (every translation unit rebuilt with the given -D
# knobs) for A/B timing: name:-DKNOB=v,...  Output build/av/lib_<name>.so
set -e
cd "$(dirname "$0")/../paper_1402_4986_b200/csrc"
NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
OUT=../../build/av
mkdir -p $OUT
for v in "$@"; do
  name=${v%%:*}; defs=$(echo ${v#*:} | tr ',' ' ')
  for f in idw_tiled idw_nested; do nvcc $NVFLAGS $defs -c $f.cu -o $OUT/${f}_$name.o & done
done
wait
for v in "$@"; do
  name=${v%%:*}
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/lib_$name.so \
    build/idw_capi.o build/idw_naive.o build/idw_layout_dev.o $OUT/idw_tiled_$name.o $OUT/idw_nested_$name.o
done
rm -f $OUT/*.o
