set -x
mkdir -p gpurun_out/r2c
timeout 900 python tools/tpc_ab.py c3 c1 c2 c5 c3s8 > gpurun_out/r2c/tpc.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_tiled_chunks --launch-skip 3 -c 1 -o gpurun_out/r2c/c1_chunks python bench.py --config c1 --steps 2 --warmup 3 > gpurun_out/r2c/ncu_c1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tiled_chunks --launch-skip 1 -c 1 -o gpurun_out/r2c/c3_chunks python bench.py --steps 1 --warmup 3 > gpurun_out/r2c/ncu_c3.log 2>&1
ls gpurun_out/r2c
