#!/bin/bash
# round-2 GPU call ad: peer-store halos for one process per GPU (CUDA IPC +
# stream flags) -- multi-process tests on cuda:0, the N=2 bench path with
# --halo peer and --halo nccl-equivalent (gloo staging) at a reduced grid.
O=gpurun_out/r02ad
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_peer.py -q -p no:cacheprovider -rf -x > $O/pytest_peer.log 2>&1
echo "pytest rc=$?" >> $O/pytest_peer.log
timeout 900 python -m pytest tests/test_gpu_bench_ranks.py -q -p no:cacheprovider -rf > $O/pytest_ranks.log 2>&1
echo "pytest rc=$?" >> $O/pytest_ranks.log
for halo in peer nccl; do
  timeout 600 python bench.py --gpus 2 --backend gloo --same-device --grid 800 --steps 10 --warmup 3 \
     --no-exact --no-secondary --no-cpu --halo $halo > $O/bench_n2_$halo.json 2> $O/bench_n2_$halo.err
  echo "rc=$?" >> $O/bench_n2_$halo.err
done
