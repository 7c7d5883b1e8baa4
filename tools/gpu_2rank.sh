#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --device-override 0 --no-cpu > gpurun_out/bench_2rank_gloo.json 2> gpurun_out/bench_2rank_gloo.err
echo "rc=$?" >> gpurun_out/bench_2rank_gloo.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 2 --warmup 1 --config c1 > gpurun_out/bench_ref_c1.json 2>&1
