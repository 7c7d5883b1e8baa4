mkdir -p gpurun_out/k2k3
timeout 600 ncu --set full --clock-control none -k regex:k_tiled_chunks --launch-skip 1 -c 1 -o gpurun_out/k2k3/k2 python tools/run_one.py 1048576 65536 soa double tiled fast 3.5 2 > gpurun_out/k2k3/ncu_k2.log 2>&1
ncu -i gpurun_out/k2k3/k2.ncu-rep --page raw --csv > gpurun_out/k2k3/k2.raw.csv
timeout 600 ncu --set full --clock-control none -k regex:k_nested --launch-skip 1 -c 1 -o gpurun_out/k2k3/k3 python tools/run_one.py 1048576 65536 soa double nested_improved fast 3.5 2 > gpurun_out/k2k3/ncu_k3.log 2>&1
ncu -i gpurun_out/k2k3/k3.ncu-rep --page raw --csv > gpurun_out/k2k3/k3.raw.csv
rm -f gpurun_out/k2k3/*.ncu-rep
