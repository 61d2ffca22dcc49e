#!/bin/bash
O=gpurun_out/r02p
mkdir -p $O
for b in base exonlyint base exonlyint; do
  echo "== $b" >> $O/ab.txt
  PIRK_LIB=build/ab/$b.so PROBE=heat PROBE_MODES=exact timeout 300 python tools/perf_probe.py 1600 >> $O/ab.txt 2>&1
done
