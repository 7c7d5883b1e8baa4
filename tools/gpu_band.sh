#!/bin/bash
# Band order A/B (IDW_BAND / IDW_TPC) on C5: timing + ncu DRAM bytes.
O=gpurun_out/band; mkdir -p $O; rm -f $O/*
NEW=$PWD/build/tv/lib_band.so
for setting in ":" "IDW_TPC=128" "IDW_TPC=128,IDW_BAND=200" "IDW_TPC=128,IDW_BAND=400" "IDW_TPC=64,IDW_BAND=200" "IDW_TPC=256,IDW_BAND=400"; do
  envs=$(echo ${setting#:} | tr ',' ' ')
  echo "== $setting" >> $O/ab.log
  env $envs python tools/lib_ab.py $NEW -- c5 >> $O/ab.log 2>&1
  env $envs IDW_B200_LIB=$NEW timeout 300 ncu --kernel-name regex:k_tiled_chunks --launch-skip 1 --launch-count 1 \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv python tools/c5_once.py \
    > $O/ncu_$(echo $setting | tr ':=,' '___').csv 2>&1
done
