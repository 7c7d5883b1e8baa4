#!/bin/bash
OUT=gpurun_out/k3
mkdir -p $OUT
cap() {  # name lib target
  IDW_B200_LIB=$PWD/build/variants/lib_$2.so timeout 900 ncu --clock-control none --set full --import-source on -k regex:k_nested -s 1 -c 1 -o $OUT/$1 \
      python tools/prof_target.py $3 > $OUT/$1.log 2>&1
  ncu -i $OUT/$1.ncu-rep --page raw --csv > $OUT/$1.raw.csv 2>/dev/null
  ncu -i $OUT/$1.ncu-rep --page source --csv --print-source sass > $OUT/$1.source.csv 2>/dev/null
  rm -f $OUT/$1.ncu-rep
}
cap ring_c5 ring c5_nested
cap r0u8_c5 r0u8 c5_nested
cap ring_c2 ring c2_nested
cap r0u8_c2 r0u8 c2_nested
