#!/bin/bash
O=gpurun_out/r02ab
mkdir -p $O
for b in kind3 k3re k3ni k7ni kind3 k3re k3ni k7ni; do
  echo "== $b" >> $O/ab.txt
  PIRK_LIB=build/ab/$b.so PROBE=heat PROBE_MODES=fast timeout 300 python tools/perf_probe.py 1600 >> $O/ab.txt 2>&1
done
