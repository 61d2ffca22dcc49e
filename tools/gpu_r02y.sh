#!/bin/bash
O=gpurun_out/r02y
mkdir -p $O
for b in kind3 kind7 kind3 kind7; do
  echo "== $b" >> $O/ab.txt
  PIRK_LIB=build/ab/$b.so PROBE=heat PROBE_MODES=fast timeout 300 python tools/perf_probe.py 1600 >> $O/ab.txt 2>&1
done
PIRK_LIB=build/ab/kind7.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_multilane.py -m gpu -q -p no:cacheprovider -rf -k "heat or c5 or lanes" > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
