#!/bin/bash
# round-2 GPU call ap: K2 y-pair clusters (PIRK_STRIP_PAIR) A/B, heat parity
# with pairs on, sanitizers on the pair kernel.
O=gpurun_out/r02ap
mkdir -p $O
for n in 1 2; do
  for pr in 0 1; do
    echo "== PIRK_STRIP_PAIR=$pr" >> $O/ab.log
    PIRK_STRIP_PAIR=$pr PROBE=heat PROBE_MODES=fast timeout 300 python tools/perf_probe.py 1600 >> $O/ab.log 2>&1
    PIRK_STRIP_PAIR=$pr PROBE=heat PROBE_MODES=fast timeout 300 python tools/perf_probe.py 800 >> $O/ab.log 2>&1
  done
done
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -k "heat or smoke or peer or multilane or scale" -x -rf > $O/pytest_heat.log 2>&1
echo "pytest rc=$?" >> $O/pytest_heat.log
for tool in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 10 python tools/sanitize_probe.py heat_fast > $O/san_${tool}_pair.log 2>&1
  echo "rc=$?" >> $O/san_${tool}_pair.log
done
