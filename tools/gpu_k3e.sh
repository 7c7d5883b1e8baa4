mkdir -p gpurun_out/k3e
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/k3e/gpu.log 2>&1
echo rc=$? >> gpurun_out/k3e/gpu.log
python -c "
import sys; sys.argv=['x']; __file__='tools/quick_perf.py'
exec(open('tools/quick_perf.py').read().split('import subprocess as _sp')[0])
K=1024
for kind in ('soa','aos','aoas'):
    run(100*K, 100*K, kind, 'single', 'nested_improved', 'exact', p=2.0, reps=3)
" > gpurun_out/k3e/perf.log 2>&1
