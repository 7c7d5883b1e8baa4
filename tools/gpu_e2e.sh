mkdir -p gpurun_out/e2e
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/e2e/c3.json 2> gpurun_out/e2e/c3.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --device-override 0 --no-cpu > gpurun_out/e2e/r2.json 2> gpurun_out/e2e/r2.err
