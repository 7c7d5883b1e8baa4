mkdir -p gpurun_out/r2l
for v in tiled nested_improved; do for p in 3.5 2.0; do
python - "$v" "$p" <<'PY' >> gpurun_out/r2l/k2k3.log 2>&1
import sys
sys.argv=['x']; __file__='tools/quick_perf.py'
exec(open('tools/quick_perf.py').read().split('import subprocess as _sp')[0])
import sys as s2
PY
done; done
python -c "
import sys; sys.argv=['x']; __file__='tools/quick_perf.py'
exec(open('tools/quick_perf.py').read().split('import subprocess as _sp')[0])
for v in ('tiled','nested_improved'):
    for p in (3.5, 2.0):
        for kind in ('soa','aoas'):
            run(1048576, 65536, kind, 'double', v, 'fast', p=p, reps=2)
" > gpurun_out/r2l/k2k3.log 2>&1
