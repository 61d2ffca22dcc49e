#!/bin/bash
# round-2 GPU call ao: verification of v18b (S form, F32 screen, per-plane TMEM
# store wait): full gpu suite, smoke, bench line, reference arm, bench launch
# list, memcheck / synccheck of the strip kernel.
O=gpurun_out/r02ao
mkdir -p $O
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 -rf > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err
echo "bench rc=$?" >> $O/bench.err
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2>> $O/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/bench_launches.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu --no-secondary --no-exact > $O/bench_under_ncu.log 2>&1
for tool in memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 10 python tools/sanitize_probe.py heat_fast > $O/san_${tool}_heat_fast.log 2>&1
  echo "rc=$?" >> $O/san_${tool}_heat_fast.log
done
