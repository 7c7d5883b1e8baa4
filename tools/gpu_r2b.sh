set -x
mkdir -p gpurun_out/r2b
timeout 600 python -m pytest tests/test_determinism_gpu.py tests/test_parity_configs.py -q -x -p no:cacheprovider > gpurun_out/r2b/det.log 2>&1
echo det_rc=$? >> gpurun_out/r2b/det.log
timeout 900 python tools/tpc_ab.py c3 c1 c2 c5 c3s8 > gpurun_out/r2b/tpc.log 2>&1
timeout 300 python bench.py --config c1 --steps 5 --warmup 3 > gpurun_out/r2b/bench_c1.json 2> gpurun_out/r2b/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b/launches_c1.csv python bench.py --config c1 --steps 2 --warmup 3 > /dev/null 2>&1
tail -3 gpurun_out/r2b/det.log
