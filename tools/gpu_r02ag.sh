#!/bin/bash
# round-2 GPU call ag: skew tail length A/B for the C5 e2e call.
O=gpurun_out/r02ag
mkdir -p $O
for v in "PIRK_SKEW_J=3" "PIRK_SKEW_J=4" "PIRK_SKEW_J=5" "PIRK_SKEW_J=6" "PIRK_SKEW_J=8" "PIRK_SKEW_S=160 PIRK_SKEW_J=6" "PIRK_SKEW_S=120 PIRK_SKEW_J=8"; do
  env $v timeout 300 python tools/e2e_probe.py 1600 2 >> $O/e2e.jsonl 2>> $O/e2e.err
done
