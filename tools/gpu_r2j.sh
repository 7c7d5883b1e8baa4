mkdir -p gpurun_out/r2j
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "nested or c4 or split or determinism" > gpurun_out/r2j/gpu.log 2>&1
echo rc=$? >> gpurun_out/r2j/gpu.log
timeout 1200 python tools/nested_ab.py build/nv/lib_t8.so build/nv/lib_t4.so build/nv/lib_old.so > gpurun_out/r2j/ab.log 2>&1
