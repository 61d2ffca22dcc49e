#!/bin/bash
O=gpurun_out/r02j
mkdir -p $O
for b in kind3 onlyint kind3 onlyint; do
  echo "== $b" >> $O/ab.txt
  PIRK_LIB=build/ab/$b.so PROBE=heat PROBE_MODES=fast timeout 300 python tools/perf_probe.py 1600 >> $O/ab.txt 2>&1
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_multilane.py -m gpu -q -p no:cacheprovider -rf -k "heat or c5 or lanes" > $O/pytest_heat.log 2>&1
echo "rc=$?" >> $O/pytest_heat.log
