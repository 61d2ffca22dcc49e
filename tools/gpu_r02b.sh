#!/bin/bash
# round-2 GPU call b: multi-lane + bench-scale parity suites, the whole gpu
# suite, FP64 instruction counts of the chain / MC kernels, a bench line.
O=gpurun_out/r02b
mkdir -p $O
{ free -g; nproc; lscpu | grep -E "Model name|Socket|Thread|Core"; nvidia-smi -L; } > $O/host.txt 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=30 -rf > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/host.txt
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum
for cfg in "chain 10000000 fast" "chain 10000000 exact" "traffic 1000000 fast" "traffic 1000000 exact"; do
  set -- $cfg
  timeout 600 ncu --metrics $M --clock-control none -k regex:chain -s 2 -c 2 --csv python tools/prof_target.py $1 $2 $3 8 > $O/ncu_${1}_${3}.csv 2>&1
done
for mode in fast exact; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:monte_carlo -s 1 -c 1 --csv python tools/mc_probe.py $mode > $O/ncu_mc_${mode}.csv 2>&1
done
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err
echo "bench rc=$?" >> $O/host.txt
