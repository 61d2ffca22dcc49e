#!/bin/bash
# round-2 GPU call g: record-callback tests, smoke, racecheck of the sanitize +
# __syncthreads build (expected clean).
O=gpurun_out/r02g
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_record.py tests/test_gpu_multilane.py -m gpu -q -p no:cacheprovider -rf > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "rc=$?" >> $O/smoke.log
PIRK_LIB=build/ab/sanitize_nosplit.so timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python tools/sanitize_probe.py heat_fast > $O/racecheck_sanitize_nosplit.log 2>&1
echo "rc=$?" >> $O/racecheck_sanitize_nosplit.log
