mkdir -p gpurun_out/prod
for pr in 1 2 0; do
IDW_PROD=$pr python -c "
import sys; sys.argv=['x']; __file__='tools/quick_perf.py'
exec(open('tools/quick_perf.py').read().split('import subprocess as _sp')[0])
print('prod=$pr', end=' ')
run(1<<20, 1<<20, 'aoas', 'single', 'tiled', 'fast', reps=3)
print('prod=$pr', end=' ')
run(100<<10, 100<<10, 'aoas', 'single', 'tiled', 'fast', reps=5)
" >> gpurun_out/prod/ab.log 2>&1
done
