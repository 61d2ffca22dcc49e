#!/bin/bash
# tools/ab_run.sh G NAME... : heat fast-mode timing at grid G for each A/B build (dev only)
g=$1; shift
for n in "$@"; do
  echo -n "$n: "; PIRK_LIB=build/ab/$n.so timeout 200 python tools/perf_probe.py $g 2>&1 | grep "heat.*fast"
done
