mkdir -p gpurun_out/k3i
python tools/d64_ab.py paper_1402_4986_b200/libidw_b200.so > gpurun_out/k3i/ab.log 2>&1
python -c "
import sys; sys.argv=['x']; __file__='tools/quick_perf.py'
exec(open('tools/quick_perf.py').read().split('import subprocess as _sp')[0])
K=1024
for kind in ('soa','aos','aoas'):
    run(100*K, 100*K, kind, 'single', 'nested_improved', 'fast', p=2.0, reps=3)
run(10240*K, 100*K, 'aoas', 'single', 'nested_improved', 'fast', p=2.0, reps=1)
" > gpurun_out/k3i/f32.log 2>&1
