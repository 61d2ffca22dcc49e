#!/bin/bash
O=gpurun_out/r02k
mkdir -p $O
for b in kind3 nows kind3 nows; do
  echo "== $b" >> $O/ab.txt
  PIRK_LIB=build/ab/$b.so PROBE=heat PROBE_MODES=fast timeout 300 python tools/perf_probe.py 1600 >> $O/ab.txt 2>&1
done
PIRK_LIB=build/ab/nows.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -p no:cacheprovider -rf -k "heat_fast or interior_tiles_fast or pipelined or c5_full or fast-" > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
