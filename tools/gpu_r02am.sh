#!/bin/bash
# round-2 GPU call am: F32 finite screen A/B on top of the S form, new S-form
# tests, full gpu suite, smoke, bench line, ncu capture of K2.
O=gpurun_out/r02am
mkdir -p $O
for n in 1 2; do
  for lib in build/ab/sform1.so paper_2001_10635_b200/lib/libpirk_b200.so; do
    echo "== $lib" >> $O/ab.log
    PIRK_LIB=$lib PROBE=heat PROBE_MODES=fast timeout 300 python tools/perf_probe.py 1600 >> $O/ab.log 2>&1
  done
done
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 -rf > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err
echo "bench rc=$?" >> $O/bench.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:heat_strip -s 2 -c 1 \
  -o $O/strip_g1600 python tools/prof_target.py heat 1600 fast 4 > $O/ncu_strip.log 2>&1
echo "ncu rc=$?" >> $O/ncu_strip.log
