#!/bin/bash
# round-2 GPU call aw: K2 A/B, x(j) carried in registers (XCARRY) on the S form
O=gpurun_out/r02aw
mkdir -p $O
for n in 1 2; do
  for lib in build/ab/base.so build/ab/xcarry.so; do
    echo "== $lib" >> $O/ab.log
    PIRK_LIB=$lib PROBE=heat PROBE_MODES=fast timeout 300 python tools/perf_probe.py 1600 >> $O/ab.log 2>&1
  done
done
