#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_multirank.py -x -q > gpurun_out/p18_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/p18_tests.log
echo done
