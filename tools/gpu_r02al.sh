#!/bin/bash
# round-2 GPU call al: K2 S form (polynomial in the neighbour-sum operator) A/B and heat parity.
O=gpurun_out/r02al
mkdir -p $O
for n in 1 2; do
  for lib in build/ab/sform0.so paper_2001_10635_b200/lib/libpirk_b200.so; do
    echo "== $lib" >> $O/ab.log
    PIRK_LIB=$lib PROBE=heat PROBE_MODES=fast timeout 300 python tools/perf_probe.py 1600 >> $O/ab.log 2>&1
    PIRK_LIB=$lib PROBE=heat PROBE_MODES=fast timeout 300 python tools/perf_probe.py 800 >> $O/ab.log 2>&1
  done
done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "heat" -rf > $O/pytest_heat.log 2>&1
echo "pytest rc=$?" >> $O/pytest_heat.log
