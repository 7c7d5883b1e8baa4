#!/bin/bash
OUT=gpurun_out/soa
mkdir -p $OUT
for lp in soa:single aos:single; do
  l=${lp%%:*}
  timeout 600 ncu --clock-control none --set full -k regex:k_tiled -s 1 -c 1 -o $OUT/$l python tools/prof_target.py c2tiled:$lp > $OUT/$l.log 2>&1
  ncu -i $OUT/$l.ncu-rep --page raw --csv > $OUT/$l.raw.csv 2>/dev/null
  rm -f $OUT/$l.ncu-rep
done
