mkdir -p gpurun_out/k3s
python tools/nested_ab.py build/nv/lib_s2.so build/nv/lib_s3.so > gpurun_out/k3s/ab.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_nested --launch-skip 1 -c 1 -o gpurun_out/k3s/c4w python tools/run_one.py 1048576 65536 soa double nested_improved fast 3.5 2 > gpurun_out/k3s/ncu.log 2>&1
ncu -i gpurun_out/k3s/c4w.ncu-rep --page raw --csv > gpurun_out/k3s/c4w.raw.csv
ncu -i gpurun_out/k3s/c4w.ncu-rep --page source --csv --print-source sass > gpurun_out/k3s/c4w.src.csv
rm -f gpurun_out/k3s/*.ncu-rep
