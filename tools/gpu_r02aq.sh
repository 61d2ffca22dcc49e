#!/bin/bash
# round-2 GPU call aq: ncu --set full capture of the v18b strip kernel (S form,
# F32 screen, one TMEM store wait per plane) for profiles/; C1 probe.
O=gpurun_out/r02aq
mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:heat_strip -s 2 -c 1 \
  -o $O/strip_g1600_v18b python tools/prof_target.py heat 1600 fast 4 > $O/ncu_strip.log 2>&1
echo "ncu rc=$?" >> $O/ncu_strip.log
timeout 300 python tools/c1_probe.py > $O/c1_probe.log 2>&1
echo "rc=$?" >> $O/c1_probe.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "arch or laub or scalar or small or frozen or golden or vdp or user or config" -rf > $O/pytest_small.log 2>&1
echo "pytest rc=$?" >> $O/pytest_small.log
