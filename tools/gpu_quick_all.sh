mkdir -p gpurun_out/qa
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/qa/gpu.log 2>&1
echo rc=$? >> gpurun_out/qa/gpu.log
