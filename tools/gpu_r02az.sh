#!/bin/bash
# round-2 GPU call az (same script as as): final verification of the round's tree (full gpu suite,
# smoke, bench line, reference arm).
O=gpurun_out/r02az
mkdir -p $O
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 -rf > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err
echo "bench rc=$?" >> $O/bench.err
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2>> $O/bench.err
