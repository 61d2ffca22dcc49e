#!/bin/bash
# round-2 GPU call ar: source-level ncu of the C1 warp integrator (fast and exact)
O=gpurun_out/r02ar
mkdir -p $O
for mode in fast exact; do
  timeout 600 python tools/c1_probe.py $mode > $O/c1_$mode.log 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:small_warp -s 1 -c 1 \
    -o $O/c1_$mode python tools/c1_probe.py $mode > $O/ncu_c1_$mode.log 2>&1
done
