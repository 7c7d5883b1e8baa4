#!/bin/bash
mkdir -p gpurun_out
for L in soa aos aoas soaos hybrid; do
  timeout 300 ncu --clock-control none --metrics lts__t_sectors_srcunit_tex_op_read.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,smsp__inst_executed_op_global_ld.sum \
     --csv -k regex:k_nested -s 1 -c 1 python tools/xcheck_txn.py run $L > gpurun_out/xcheck_$L.csv 2>&1
done
python tools/xcheck_txn.py report gpurun_out > gpurun_out/xcheck_report.json
