#!/bin/bash
# round-2 first GPU call: FP64 peak, sanitizers on every kernel, the gpu suite
mkdir -p gpurun_out/r02a
./tools/bin/fp64_peak > gpurun_out/r02a/fp64_peak.json 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a/smi.txt
free -g > gpurun_out/r02a/host_mem.txt; nproc >> gpurun_out/r02a/host_mem.txt; lscpu | head -20 >> gpurun_out/r02a/host_mem.txt
for tool in memcheck racecheck synccheck; do
  for c in heat_fast heat_exact chain_fast traffic_exact mc_fast mc_exact; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_probe.py $c > gpurun_out/r02a/san_${tool}_${c}.log 2>&1
    echo "$tool $c rc=$?" >> gpurun_out/r02a/san_summary.txt
    tail -3 gpurun_out/r02a/san_${tool}_${c}.log >> gpurun_out/r02a/san_summary.txt
  done
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02a/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02a/san_summary.txt
