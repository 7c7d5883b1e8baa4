mkdir -p gpurun_out/r2m
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2m/gpu.log 2>&1
echo rc=$? >> gpurun_out/r2m/gpu.log
for sp in 1 0; do
IDW_FAST_SPLIT=$sp python -c "
import sys; sys.argv=['x']; __file__='tools/quick_perf.py'
exec(open('tools/quick_perf.py').read().split('import subprocess as _sp')[0])
print('split=$sp')
run(10240, 10240, 'soa', 'single', 'tiled', 'fast', reps=20)
run(10240, 10240, 'aoas', 'single', 'tiled', 'fast', reps=20)
run(102400, 10240, 'aoas', 'single', 'tiled', 'fast', reps=10)
run(1048576, 2048, 'aoas', 'single', 'tiled', 'fast', reps=5)
run(102400, 102400, 'aoas', 'single', 'tiled', 'fast', reps=5)
" >> gpurun_out/r2m/split.log 2>&1
done
timeout 300 python bench.py --config c1 --steps 20 --warmup 5 > gpurun_out/r2m/bench_c1.json 2>/dev/null
