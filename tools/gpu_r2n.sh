mkdir -p gpurun_out/r2n
timeout 900 python -m pytest tests/test_determinism_gpu.py tests/test_parity_configs.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2n/gpu.log 2>&1
echo rc=$? >> gpurun_out/r2n/gpu.log
for c in c1 c3 c2; do timeout 300 python bench.py --config $c --steps 10 --warmup 5 --no-cpu > gpurun_out/r2n/bench_$c.json 2>/dev/null; done
