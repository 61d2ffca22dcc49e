#!/bin/bash
# round-2 GPU call d: sanitizers on the new kernels (lanes, NVRTC user models),
# variant-flag rebuild check, MC timing after the constant-bank change, bench.
O=gpurun_out/r02d
mkdir -p $O
for tool in memcheck racecheck synccheck; do
  for c in lanes_exact lanes_fast user_exact user_fast mc_fast; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 10 python tools/sanitize_probe.py $c > $O/san_${tool}_${c}.log 2>&1
    echo "$tool $c rc=$?" >> $O/san_summary.txt
    tail -2 $O/san_${tool}_${c}.log >> $O/san_summary.txt
  done
done
python tools/mc_probe.py fast > $O/mc_probe.txt 2>&1
python tools/mc_probe.py exact >> $O/mc_probe.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -rf -k "mc or variant or arch or laub" > $O/pytest_mc.log 2>&1
echo "rc=$?" >> $O/pytest_mc.log
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err
echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2>> $O/bench.err
