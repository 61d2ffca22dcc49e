#!/bin/bash
O=gpurun_out/r02w
mkdir -p $O
for b in kind3 nokind2 onlyint kind3 nokind2 onlyint; do
  echo "== $b" >> $O/ab.txt
  PIRK_LIB=build/ab/$b.so PROBE=heat PROBE_MODES=fast timeout 300 python tools/perf_probe.py 1600 >> $O/ab.txt 2>&1
done
PIRK_LIB=build/ab/kind3.so timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,smsp__cycles_active.avg,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:heat_strip -s 2 -c 1 python tools/prof_target.py heat 1600 fast 4 > $O/ncu_kind3.txt 2>&1
PIRK_LIB=build/ab/skipedge.so timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,smsp__cycles_active.avg,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:heat_strip -s 2 -c 1 python tools/prof_target.py heat 1600 fast 4 > $O/ncu_skipedge.txt 2>&1
PIRK_LIB=build/ab/onlyint.so timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,smsp__cycles_active.avg,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:heat_strip -s 2 -c 1 python tools/prof_target.py heat 1600 fast 4 > $O/ncu_onlyint.txt 2>&1
