#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_multirank.py tests/test_gpu_nccl.py -q > gpurun_out/p22_mp.log 2>&1
echo "mp rc=$?" >> gpurun_out/p22_mp.log
tail -n 3 gpurun_out/p22_mp.log
