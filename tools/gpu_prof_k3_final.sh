#!/bin/bash
OUT=gpurun_out/k3final
mkdir -p $OUT
for t in c5_nested c2_nested; do
  timeout 900 ncu --clock-control none --set full -k regex:k_nested -s 1 -c 1 -o $OUT/prof_$t python tools/prof_target.py $t > $OUT/prof_$t.log 2>&1
  ncu -i $OUT/prof_$t.ncu-rep --page raw --csv > $OUT/prof_$t.raw.csv 2>/dev/null
  rm -f $OUT/prof_$t.ncu-rep
done
