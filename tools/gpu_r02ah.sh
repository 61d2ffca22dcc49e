#!/bin/bash
# round-2 GPU call ah: z-strip launch overhead of the heat strip kernel.
O=gpurun_out/r02ah
mkdir -p $O
timeout 300 python tools/strip_probe.py 1600 1600,800,400,200,100,50 >> $O/strips.jsonl 2>> $O/strips.err
PIRK_HEAT_ZCHUNKS=1 timeout 300 python tools/strip_probe.py 1600 1600,400,200,100 >> $O/strips.jsonl 2>> $O/strips.err
PIRK_HEAT_ZCHUNKS=2 timeout 300 python tools/strip_probe.py 1600 400,200,100 >> $O/strips.jsonl 2>> $O/strips.err
