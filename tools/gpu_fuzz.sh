mkdir -p gpurun_out/fuzz
timeout 1200 python -m pytest tests/test_fuzz_gpu.py -q -m gpu -p no:cacheprovider -rf > gpurun_out/fuzz/fuzz.log 2>&1
echo rc=$? >> gpurun_out/fuzz/fuzz.log
