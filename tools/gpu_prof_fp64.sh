#!/bin/bash
mkdir -p gpurun_out
NCU="ncu --clock-control none"
cap() {  # name kernel-regex target
  timeout 600 $NCU --set full --import-source on -k regex:$2 -s 1 -c 1 -o gpurun_out/$1 \
      python tools/prof_target.py $3 > gpurun_out/$1.log 2>&1
  ncu -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1.raw.csv 2>/dev/null
  ncu -i gpurun_out/$1.ncu-rep --page details --csv > gpurun_out/$1.details.csv 2>/dev/null
  ncu -i gpurun_out/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/$1.source.csv 2>/dev/null
  rm -f gpurun_out/$1.ncu-rep
}
cap prof_c4 k_nested c4
cap prof_tiled64_p35 k_tiled tiled64_p35
cap prof_c2 k_tiled c2
cap prof_c5 k_tiled c5
du -sh gpurun_out
