#!/bin/bash
# round-2 GPU call ai: two-sided mirror stores; fused one-launch-per-step
# peer-store schedule; per-step cost of fused vs split vs plain slab launches.
O=gpurun_out/r02ai
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_peer.py tests/test_gpu_multilane.py tests/test_gpu_bench_ranks.py \
   -q -p no:cacheprovider -rf > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python tools/peer_probe.py 8,4,2 > $O/peer_probe.jsonl 2> $O/peer_probe.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
