#!/bin/bash
# round-2 GPU call e: K2 source-level ncu capture at C5 size; racecheck of the
# strip kernel built with __syncthreads instead of the split mbarrier.
O=gpurun_out/r02e
mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:heat_strip -s 2 -c 1 \
  -o $O/strip_g1600 python tools/prof_target.py heat 1600 fast 4 > $O/ncu_strip.log 2>&1
echo "ncu rc=$?" >> $O/ncu_strip.log
PIRK_LIB=build/ab/nosplit.so timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python tools/sanitize_probe.py heat_fast > $O/racecheck_nosplit.log 2>&1
echo "rc=$?" >> $O/racecheck_nosplit.log
PIRK_LIB=build/ab/nosplit.so PROBE=heat PROBE_MODES=fast timeout 600 python tools/perf_probe.py 1600 > $O/perf_nosplit.txt 2>&1
PROBE=heat PROBE_MODES=fast timeout 600 python tools/perf_probe.py 1600 > $O/perf_default.txt 2>&1
