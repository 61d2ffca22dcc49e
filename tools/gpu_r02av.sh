#!/bin/bash
# round-2 GPU call av: K2 A/B of TMEM operand forms (64-bit asm operands; x16 stores)
O=gpurun_out/r02av
mkdir -p $O
for n in 1 2; do
  for lib in build/ab/base.so build/ab/tmpairs.so build/ab/st16.so; do
    echo "== $lib" >> $O/ab.log
    PIRK_LIB=$lib PROBE=heat PROBE_MODES=fast timeout 300 python tools/perf_probe.py 1600 >> $O/ab.log 2>&1
  done
done
