#!/bin/bash
# round-2 GPU call h: A/B of the edge-tile pair-sum path (PIRK_STRIP_EDGECSE)
O=gpurun_out/r02h
mkdir -p $O
for g in 1600 800; do
  for b in edgecse0 edgecse1 edgecse0 edgecse1; do
    echo "== $b g=$g" >> $O/ab.txt
    PIRK_LIB=build/ab/$b.so PROBE=heat PROBE_MODES=fast timeout 300 python tools/perf_probe.py $g >> $O/ab.txt 2>&1
  done
done
PIRK_LIB=build/ab/edgecse1.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -p no:cacheprovider -rf -k "heat or c5" > $O/pytest_heat.log 2>&1
echo "rc=$?" >> $O/pytest_heat.log
