#!/bin/bash
# boundary launches of non-reducing slab passes on a second stream: multi-rank tests, slab overhead with / without
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_multiproc.py tests/test_gpu_nccl.py -x -q > gpurun_out/p65_tests.log 2>&1; echo "rc=$?" >> gpurun_out/p65_tests.log; tail -2 gpurun_out/p65_tests.log
for cfg in "512 512 512 40 12" "320 320 320 20 15" "640 640 80 40 12" "512 512 64 40 12"; do
  for b in 0 1; do echo "bstream=$b"; PCGX_SLAB_BSTREAM=$b PYTHONPATH=. python tools/slab_overhead.py $cfg 2>&1 | tail -1 | cut -c1-230; done
done | tee gpurun_out/p65_slab.log
