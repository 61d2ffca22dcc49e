#!/bin/bash
# round-2 GPU call ae: skewed field-pipelined driver -- parity of every strip
# width, the pipelined / record / scale tests, and the C5 e2e call A/B.
O=gpurun_out/r02ae
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -rf -x \
   -k "pipelined" > $O/pytest_skew.log 2>&1
echo "pytest rc=$?" >> $O/pytest_skew.log
timeout 900 python -m pytest tests/test_gpu_record.py tests/test_gpu_scale.py -q -p no:cacheprovider -rf > $O/pytest_rs.log 2>&1
echo "pytest rc=$?" >> $O/pytest_rs.log
for v in "PIRK_SKEW=0" "PIRK_SKEW_S=200" "PIRK_SKEW_S=100" "PIRK_SKEW_S=300"; do
  env $v PIRK_TRACE=1 timeout 300 python tools/e2e_probe.py 1600 2 >> $O/e2e.jsonl 2>> $O/e2e.err
done
