mkdir -p gpurun_out/k2d
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/k2d/gpu.log 2>&1
echo rc=$? >> gpurun_out/k2d/gpu.log
python -c "
import sys; sys.argv=['x']; __file__='tools/quick_perf.py'
exec(open('tools/quick_perf.py').read().split('import subprocess as _sp')[0])
K=1024
for kind in ('soa','aos','aoas','soaos','hybrid'):
    run(100*K, 100*K, kind, 'double', 'tiled', 'fast', p=2.0, reps=3)
run(100*K, 100*K, 'soa', 'double', 'tiled', 'fast', p=3.5, reps=3)
run(1024*K, 64*K, 'soa', 'double', 'tiled', 'fast', p=3.5, reps=2)
run(1024*K, 64*K, 'soa', 'double', 'nested_improved', 'fast', p=3.5, reps=2)
" > gpurun_out/k2d/perf.log 2>&1
