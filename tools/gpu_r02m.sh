#!/bin/bash
# round-2 GPU call m: evidence for the current K2 (edge-tile instantiation):
# memcheck, DRAM traffic per launch, a full ncu capture, the bench launch list,
# and the bench line.
O=gpurun_out/r02m
mkdir -p $O
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python tools/sanitize_probe.py heat_fast lanes_fast > $O/memcheck_heat.log 2>&1
echo "rc=$?" >> $O/memcheck_heat.log
timeout 900 python tools/heat_traffic.py 1600 > $O/heat_traffic.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:heat_strip -s 2 -c 1 \
  -o $O/strip_g1600_kind3 python tools/prof_target.py heat 1600 fast 4 > $O/ncu_strip.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/bench_launches.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu --no-secondary --no-exact > $O/bench_under_ncu.log 2>&1
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err
echo "bench rc=$?" >> $O/bench.err
