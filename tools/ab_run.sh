#!/bin/bash
# tools/ab_run.sh G NAME... : fast-mode timings at grid G for each A/B build (dev only);
# PROBE=heat|chain|all selects the workloads (default heat)
g=$1; shift
for n in "$@"; do
  echo "== $n"; PIRK_LIB=build/ab/$n.so PROBE=${PROBE:-heat} PROBE_MODES=${PROBE_MODES:-fast} timeout 300 python tools/perf_probe.py $g 2>&1 | grep "ms/step"
done
