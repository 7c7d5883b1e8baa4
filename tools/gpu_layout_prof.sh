#!/bin/bash
# k_tiled at C2 (100K x 100K FAST) for every legal layout: pipe utilisation,
# shared-memory wavefronts/bank conflicts of the stage reads, L2->SM bytes of
# the bulk-copy staging, DRAM bytes.
OUT=gpurun_out/layout_prof
mkdir -p $OUT
M=gpu__time_duration.sum,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum.pct_of_peak_sustained_elapsed,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,smsp__sass_inst_executed_op_shared_ld.sum,lts__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__issue_active.avg.pct_of_peak_sustained_active
for lp in soa:single aos:single aoas:single soa:double aos:double aoas:double soaos:double hybrid:double; do
  l=${lp%%:*}; p=${lp##*:}
  timeout 300 ncu --clock-control none --metrics $M --csv -k regex:k_tiled -s 1 -c 1 \
      python tools/prof_target.py c2tiled:$l:$p > $OUT/$l\_$p.csv 2>&1
done
