#!/bin/bash
# round-2 GPU call ax: arch-quadrotor uniform divisions on the host: C1 / C2 timing, small-system parity
O=gpurun_out/r02ax
mkdir -p $O
for mode in fast exact; do
  PIRK_LIB=build/ab/base.so timeout 300 python tools/c1_probe.py $mode > $O/c1_base_$mode.log 2>&1
  timeout 300 python tools/c1_probe.py $mode > $O/c1_new_$mode.log 2>&1
done
PIRK_LIB=build/ab/base.so timeout 300 python tools/mc_probe.py > $O/mc_base.log 2>&1
timeout 300 python tools/mc_probe.py > $O/mc_new.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "arch or laub or scalar or small or frozen or golden or vdp or mc or monte or coverage or config" -rf > $O/pytest_small.log 2>&1
echo "pytest rc=$?" >> $O/pytest_small.log
