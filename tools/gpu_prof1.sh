#!/bin/bash
# Profiling round: launch list of the bench command, full ncu captures of the
# dominant kernels, naive-kernel memory counters per layout, 2-rank bench (gloo).
mkdir -p gpurun_out
NCU="ncu --clock-control none"
timeout 600 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/launches_bench.log 2>&1
timeout 600 $NCU --set full --import-source on -k regex:k_tiled -s 1 -c 1 -o gpurun_out/prof_c3_tiled \
    python tools/prof_target.py c3 > gpurun_out/prof_c3.log 2>&1
timeout 600 $NCU --set full --import-source on -k regex:k_tiled -s 1 -c 1 -o gpurun_out/prof_c2_exact \
    python tools/prof_target.py c2_exact > gpurun_out/prof_c2_exact.log 2>&1
timeout 600 $NCU --set full --import-source on -k regex:k_nested -s 1 -c 1 -o gpurun_out/prof_c4_nested \
    python tools/prof_target.py c4 > gpurun_out/prof_c4.log 2>&1
timeout 600 $NCU --set full --import-source on -k regex:k_nested -s 1 -c 1 -o gpurun_out/prof_c5_nested \
    python tools/prof_target.py c5_nested > gpurun_out/prof_c5.log 2>&1
for L in aoas soa aos; do
  timeout 300 $NCU --section MemoryWorkloadAnalysis_Tables --section SpeedOfLight --metrics l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,smsp__inst_executed_op_global_ld.sum,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active \
      -k regex:k_naive -s 1 -c 1 -o gpurun_out/prof_naive_$L python tools/prof_target.py naive_$L > gpurun_out/prof_naive_$L.log 2>&1
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 2 --steps 2 --warmup 1 --dist-backend gloo --device-override 0 --no-cpu > gpurun_out/bench_2rank_gloo.json 2> gpurun_out/bench_2rank_gloo.err
