#!/bin/bash
# Profiling round: launch list of the bench command, full ncu captures of the
# dominant kernels (exported to CSV on the box; only the C3 report is kept
# whole), naive-kernel memory counters per layout, 2-rank bench (gloo), fp64
# microbench.
mkdir -p gpurun_out
NCU="ncu --clock-control none"
timeout 120 ./tools/microbench2 > gpurun_out/microbench2.json 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/launches_bench.log 2>&1
cap() {  # name kernel-regex target
  timeout 600 $NCU --set full --import-source on -k regex:$2 -s 1 -c 1 -o gpurun_out/$1 \
      python tools/prof_target.py $3 > gpurun_out/$1.log 2>&1
  ncu -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1.raw.csv 2>/dev/null
  ncu -i gpurun_out/$1.ncu-rep --page details --csv > gpurun_out/$1.details.csv 2>/dev/null
}
cap prof_c3_tiled k_tiled c3
ncu -i gpurun_out/prof_c3_tiled.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_c3_tiled.source.csv 2>/dev/null
for t in c2_exact:k_tiled c2_fp64:k_tiled c4:k_nested c5_nested:k_nested; do
  n=${t%%:*}; k=${t##*:}
  cap prof_$n $k $n
  rm -f gpurun_out/prof_$n.ncu-rep
done
for L in aoas soa aos; do
  timeout 300 $NCU --metrics l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,smsp__inst_executed_op_global_ld.sum,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum \
      --csv -k regex:k_naive -s 1 -c 1 python tools/prof_target.py naive_$L > gpurun_out/prof_naive_$L.csv 2>&1
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 2 --steps 2 --warmup 1 --dist-backend gloo --device-override 0 --no-cpu > gpurun_out/bench_2rank_gloo.json 2> gpurun_out/bench_2rank_gloo.err
du -sh gpurun_out
