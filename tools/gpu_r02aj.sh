#!/bin/bash
# round-2 GPU call aj: in-process lanes with one fused launch per lane and step.
O=gpurun_out/r02aj
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_multilane.py tests/test_gpu_peer.py tests/test_cpp_shim.py \
   -q -p no:cacheprovider -rf > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
