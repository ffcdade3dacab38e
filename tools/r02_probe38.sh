#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_multirank.py -x -q > gpurun_out/p38_mp.log 2>&1; echo "rc=$?" >> gpurun_out/p38_mp.log
tail -30 gpurun_out/p38_mp.log
