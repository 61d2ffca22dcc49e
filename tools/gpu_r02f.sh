#!/bin/bash
# round-2 GPU call f: racecheck of the sanitize build (halo warps' wrapped
# reads redirected), the whole gpu suite, a bench line.
O=gpurun_out/r02f
mkdir -p $O
for c in heat_fast lanes_fast; do
  PIRK_LIB=build/ab/sanitize.so timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python tools/sanitize_probe.py $c > $O/racecheck_sanitize_$c.log 2>&1
  echo "rc=$?" >> $O/racecheck_sanitize_$c.log
done
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 -rf > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err
echo "bench rc=$?" >> $O/bench.err
