#!/bin/bash
O=gpurun_out/r02c
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_user.py tests/test_gpu_multilane.py tests/test_cpp_shim.py -m gpu -q -p no:cacheprovider -rf --durations=15 > $O/pytest_user.log 2>&1
echo "rc=$?" >> $O/pytest_user.log
