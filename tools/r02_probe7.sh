#!/bin/bash
# full GPU suite (incl. the slow full-size tests) + adapter + bench + the CPU time-to-1e-8
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu -rs --durations=15 -s -k "not fullsize" > gpurun_out/p7_gputests.log 2>&1
echo "gpu tests rc=$?" >> gpurun_out/p7_gputests.log
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -q -s -rs > gpurun_out/p7_fullsize.log 2>&1
echo "fullsize rc=$?" >> gpurun_out/p7_fullsize.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/p7_bench.json 2> gpurun_out/p7_bench.log
timeout 900 python tools/cpu_full_solve.py 20 320 > gpurun_out/p7_cpu_full_k20.json 2> gpurun_out/p7_cpu_full.log
echo done
