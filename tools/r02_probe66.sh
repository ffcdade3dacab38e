#!/bin/bash
# the two boundary strips of a non-reducing slab pass as one masked launch: tests + slab overhead
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_multiproc.py tests/test_gpu_nccl.py tests/test_gpu_checked.py -x -q > gpurun_out/p66_tests.log 2>&1; echo "rc=$?" >> gpurun_out/p66_tests.log; tail -2 gpurun_out/p66_tests.log
for cfg in "512 512 512 40 12" "320 320 320 20 15" "640 640 80 40 12" "512 512 64 40 12"; do
  PYTHONPATH=. python tools/slab_overhead.py $cfg 2>&1 | tail -1 | cut -c1-230
done | tee gpurun_out/p66_slab.log
