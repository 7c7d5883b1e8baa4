mkdir -p gpurun_out/r2g
timeout 900 python -m pytest tests/test_determinism_gpu.py tests/test_partition.py tests/test_capi.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2g/det.log 2>&1
echo det_rc=$? >> gpurun_out/r2g/det.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --device-override 0 --no-cpu > gpurun_out/r2g/bench_2rank_gloo.json 2> gpurun_out/r2g/bench_2rank_gloo.err
echo "rc=$?" >> gpurun_out/r2g/bench_2rank_gloo.err
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r2g/bench_c3.json 2> gpurun_out/r2g/bench_c3.err
