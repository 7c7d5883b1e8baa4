mkdir -p gpurun_out/r2k
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_nested --launch-skip 1 -c 1 -o gpurun_out/r2k/c4s_tiles python tools/run_one.py 1048576 65536 soa double nested_improved fast 3.5 2 > gpurun_out/r2k/ncu.log 2>&1
ncu -i gpurun_out/r2k/c4s_tiles.ncu-rep --page raw --csv > gpurun_out/r2k/c4s_tiles.raw.csv
ncu -i gpurun_out/r2k/c4s_tiles.ncu-rep --page source --csv --print-source sass > gpurun_out/r2k/c4s_tiles.src.csv
rm -f gpurun_out/r2k/*.ncu-rep
