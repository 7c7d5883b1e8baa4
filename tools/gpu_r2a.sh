set -x
mkdir -p gpurun_out/r2a
timeout 900 python -m pytest tests/test_determinism_gpu.py -q -x -rA -p no:cacheprovider > gpurun_out/r2a/det.log 2>&1
echo det_rc=$? >> gpurun_out/r2a/det.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2a/gpu.log 2>&1
echo gpu_rc=$? >> gpurun_out/r2a/gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2a/bench_c3.json 2> gpurun_out/r2a/bench_c3.err
for c in c1 c2 c5; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/r2a/bench_$c.json 2>> gpurun_out/r2a/bench_c3.err; done
tail -3 gpurun_out/r2a/det.log gpurun_out/r2a/gpu.log
