#!/bin/bash
# HEAD validation after container re-creation: GPU suite, smoke, bench, launch list of k=20 / k=5
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/p30_gputests.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/p30_gputests.log
tail -3 gpurun_out/p30_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/p30_smoke.log 2>&1; tail -1 gpurun_out/p30_smoke.log
timeout 900 python bench.py > gpurun_out/p30_bench.json 2> gpurun_out/p30_bench.err; tail -c 600 gpurun_out/p30_bench.json
