mkdir -p gpurun_out/r2h
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=15 > gpurun_out/r2h/gpu.log 2>&1
echo gpu_rc=$? >> gpurun_out/r2h/gpu.log
