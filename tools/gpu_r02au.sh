#!/bin/bash
# round-2 GPU call au: per-rank slab cost of the peer-store schedules with the
# v18b kernel (DESIGN (e) cost model), and C4 / C2 at one GPU for reference.
O=gpurun_out/r02au
mkdir -p $O
timeout 600 python tools/peer_probe.py 8,4,2 > $O/peer_probe.jsonl 2> $O/peer_probe.err
