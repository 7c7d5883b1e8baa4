#!/bin/bash
# Build libidw_b200 variants that differ only in idw_nested.cu's compile-time
# knobs (fp64 K3 queries per thread Q, trips per batch U) for A/B timing.
set -e
cd "$(dirname "$0")/../paper_1402_4986_b200/csrc"
NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
OUT=../../build/variants
mkdir -p $OUT
for v in "$@"; do   # v = Q,U
  q=${v%,*}; u=${v#*,}
  nvcc $NVFLAGS -DIDW_NEST_Q64=$q -DIDW_NEST_U=$u -c idw_nested.cu -o $OUT/nested_q${q}_u${u}.o &
done
wait
for v in "$@"; do
  q=${v%,*}; u=${v#*,}
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/lib_q${q}_u${u}.so \
    build/idw_capi.o build/idw_naive.o build/idw_tiled.o build/idw_layout_dev.o $OUT/nested_q${q}_u${u}.o
done
