#!/bin/bash
# round-2 GPU call af: skewed field-pipelined driver, revised fronts.
O=gpurun_out/r02af
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -rf -x \
   -k "pipelined" > $O/pytest_skew.log 2>&1
echo "pytest rc=$?" >> $O/pytest_skew.log
for v in "PIRK_SKEW=0" "PIRK_SKEW_S=200" "PIRK_SKEW_S0=100" "PIRK_SKEW_S0=64" "PIRK_SKEW_S=160" "PIRK_SKEW_S=260" "PIRK_SKEW_J=2"; do
  env $v timeout 300 python tools/e2e_probe.py 1600 2 >> $O/e2e.jsonl 2>> $O/e2e.err
done
