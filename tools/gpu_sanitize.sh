#!/bin/bash
OUT=gpurun_out/sanitizer2
mkdir -p $OUT
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
      python tools/sanitize_target.py > $OUT/$tool.log 2>&1
  echo "rc=$?" >> $OUT/$tool.log
done
for tool in memcheck racecheck synccheck; do  # K2 FAST banded order (forced), ring-slot reuse
  IDW_BAND=3 timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
      python tools/sanitize_target.py band > $OUT/band_$tool.log 2>&1
  echo "rc=$?" >> $OUT/band_$tool.log
done
for f in $OUT/*.log; do tail -n 4 $f; done
