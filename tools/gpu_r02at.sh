#!/bin/bash
# round-2 GPU call at: y-pair clusters v2 (parity-split barriers, st.async seam
# rows completing on the peer's barrier, relaxed remote arrivals): A/B + parity.
O=gpurun_out/r02at
mkdir -p $O
for n in 1 2; do
  for pr in 0 1; do
    echo "== PIRK_STRIP_PAIR=$pr" >> $O/ab.log
    PIRK_STRIP_PAIR=$pr PROBE=heat PROBE_MODES=fast timeout 300 python tools/perf_probe.py 1600 >> $O/ab.log 2>&1
    PIRK_STRIP_PAIR=$pr PROBE=heat PROBE_MODES=fast timeout 300 python tools/perf_probe.py 800 >> $O/ab.log 2>&1
  done
done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "pair or zslab or heat_fast or interior_tiles_fast or pipelined or tiny or sform" -rf > $O/pytest_pair.log 2>&1
echo "pytest rc=$?" >> $O/pytest_pair.log
