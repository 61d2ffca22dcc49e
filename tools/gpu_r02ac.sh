#!/bin/bash
# round-2 GPU call ac: final verification of the tree -- the whole gpu suite,
# smoke, bench line, reference arm.
O=gpurun_out/r02ac
mkdir -p $O
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 -rf > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err
echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2>> $O/bench.err
