mkdir -p gpurun_out/r2f
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2f/gpu.log 2>&1
echo gpu_rc=$? >> gpurun_out/r2f/gpu.log
for c in c3 c1 c2 c4 c5; do timeout 400 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/r2f/bench_$c.json 2>> gpurun_out/r2f/bench.err; done
bash tools/gpu_r2_profiles.sh > gpurun_out/r2f/prof.log 2>&1
