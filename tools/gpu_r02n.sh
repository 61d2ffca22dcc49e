#!/bin/bash
O=gpurun_out/r02n
mkdir -p $O
for c in 0 1 2 3 4 0; do
  echo "== zchunks=$c" >> $O/ab.txt
  if [ $c = 0 ]; then unset PIRK_HEAT_ZCHUNKS; else export PIRK_HEAT_ZCHUNKS=$c; fi
  PROBE=heat PROBE_MODES=fast timeout 300 python tools/perf_probe.py 1600 >> $O/ab.txt 2>&1
done
unset PIRK_HEAT_ZCHUNKS
for c in 0 1 2 3 4; do
  echo "== exact zchunks=$c" >> $O/ab.txt
  if [ $c = 0 ]; then unset PIRK_HEAT_ZCHUNKS; else export PIRK_HEAT_ZCHUNKS=$c; fi
  PROBE=heat PROBE_MODES=exact timeout 300 python tools/perf_probe.py 1600 >> $O/ab.txt 2>&1
done
