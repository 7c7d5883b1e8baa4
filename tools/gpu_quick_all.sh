mkdir -p gpurun_out/qa
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/qa/gpu.log 2>&1
echo rc=$? >> gpurun_out/qa/gpu.log
python -c "
import sys; sys.argv=['x']; __file__='tools/quick_perf.py'
exec(open('tools/quick_perf.py').read().split('import subprocess as _sp')[0])
K=1024
for kind in ('soa','aos','aoas'):
    run(100*K, 100*K, kind, 'single', 'nested_improved', 'fast', p=2.0, reps=3)
run(10240*K, 100*K, 'aoas', 'single', 'nested_improved', 'fast', p=2.0, reps=1)
run(1024*K, 64*K, 'soa', 'double', 'nested_improved', 'fast', p=3.5, reps=2)
run(100*K, 100*K, 'soa', 'double', 'nested_improved', 'fast', p=2.0, reps=3)
" > gpurun_out/qa/perf.log 2>&1
