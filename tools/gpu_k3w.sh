mkdir -p gpurun_out/k3w
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "nested or c4 or c5 or c2_grid or split or determinism or reference_suite or golden or runstats" > gpurun_out/k3w/gpu.log 2>&1
echo rc=$? >> gpurun_out/k3w/gpu.log
for w in 1 0; do
IDW_NEST_WARPS=$w python -c "
import sys; sys.argv=['x']; __file__='tools/quick_perf.py'
exec(open('tools/quick_perf.py').read().split('import subprocess as _sp')[0])
print('warps=$w')
K=1024
run(1024*K, 64*K, 'soa', 'double', 'nested_improved', 'fast', p=3.5, reps=2)
run(100*K, 100*K, 'soa', 'single', 'nested_improved', 'fast', p=2.0, reps=3)
run(100*K, 100*K, 'aos', 'single', 'nested_improved', 'fast', p=2.0, reps=3)
run(100*K, 100*K, 'aoas', 'single', 'nested_improved', 'fast', p=2.0, reps=3)
run(100*K, 100*K, 'aoas', 'single', 'nested_improved', 'fast', p=3.5, reps=3)
run(10240*K, 100*K, 'aoas', 'single', 'nested_improved', 'fast', p=2.0, reps=1)
run(10*K, 10*K, 'soa', 'single', 'nested_improved', 'fast', p=2.0, reps=5)
" >> gpurun_out/k3w/ab.log 2>&1
done
