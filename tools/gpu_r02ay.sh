#!/bin/bash
# round-2 GPU call ay: fast-mode arch-quad 1/cos(theta) by reciprocal + Newton: C1 / C2 timing, parity
O=gpurun_out/r02ay
mkdir -p $O
for lib in build/ab/base.so paper_2001_10635_b200/lib/libpirk_b200.so; do
  echo "== $lib" >> $O/ab.log
  PIRK_LIB=$lib timeout 300 python tools/c1_probe.py fast >> $O/ab.log 2>&1
  PIRK_LIB=$lib timeout 300 python tools/mc_probe.py >> $O/ab.log 2>&1
  PIRK_LIB=$lib timeout 300 python tools/mc_probe.py >> $O/ab.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "arch or laub or scalar or small or frozen or golden or vdp or mc or monte or coverage or config" -rf > $O/pytest_small.log 2>&1
echo "pytest rc=$?" >> $O/pytest_small.log
