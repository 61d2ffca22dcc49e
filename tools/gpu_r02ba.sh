#!/bin/bash
# round-2 GPU call ba: FP64 instruction counts of the Monte Carlo kernel after the
# arch-quad changes (profiles/r02_fp64_counts.json, bench C2 roofline)
O=gpurun_out/r02ba
mkdir -p $O
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum
for mode in fast exact; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:monte_carlo -s 1 -c 1 --csv python tools/mc_probe.py $mode > $O/ncu_mc_${mode}.csv 2>&1
done
