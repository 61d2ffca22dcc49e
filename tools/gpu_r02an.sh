#!/bin/bash
# round-2 GPU call an: K2 A/B on top of the S form + F32 screen: early TMEM
# loads, per-load store waits off, mbarrier suspend hint; z-chunk counts.
O=gpurun_out/r02an
mkdir -p $O
for n in 1 2; do
  for lib in paper_2001_10635_b200/lib/libpirk_b200.so build/ab/earlyld.so build/ab/waitst0.so build/ab/hint100.so; do
    echo "== $lib" >> $O/ab.log
    PIRK_LIB=$lib PROBE=heat PROBE_MODES=fast timeout 300 python tools/perf_probe.py 1600 >> $O/ab.log 2>&1
  done
done
for c in 1 2 3; do
  echo "== zchunks $c" >> $O/ab.log
  PIRK_HEAT_ZCHUNKS=$c PROBE=heat PROBE_MODES=fast timeout 300 python tools/perf_probe.py 1600 >> $O/ab.log 2>&1
done
