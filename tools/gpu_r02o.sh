#!/bin/bash
O=gpurun_out/r02o
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_multilane.py tests/test_gpu_record.py tests/test_cpp_shim.py tests/test_gpu_scale.py -m gpu -q -p no:cacheprovider -rf -k "not c2_ and not bench_ratio" > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
PROBE=all PROBE_MODES=fast timeout 600 python tools/perf_probe.py 1600 > $O/perf.txt 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python tools/sanitize_probe.py lanes_fast lanes_exact > $O/memcheck_lanes.log 2>&1
echo "rc=$?" >> $O/memcheck_lanes.log
