#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_multirank.py -q > gpurun_out/p25_mp.log 2>&1
echo "mp rc=$?" >> gpurun_out/p25_mp.log
tail -n 3 gpurun_out/p25_mp.log
