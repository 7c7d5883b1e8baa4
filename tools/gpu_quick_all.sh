mkdir -p gpurun_out/qa
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/qa/gpu.log 2>&1
echo rc=$? >> gpurun_out/qa/gpu.log
for c in c1 c3 c2; do timeout 300 python bench.py --config $c --steps 10 --warmup 5 --no-cpu > gpurun_out/qa/bench_$c.json 2>/dev/null; done
