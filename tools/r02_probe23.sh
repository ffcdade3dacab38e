#!/bin/bash
# full GPU suite + smoke + default bench (N=1) at HEAD
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/p23_gputests.log 2>&1
echo "gpu tests rc=$?" >> gpurun_out/p23_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/p23_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/p23_smoke.log
timeout 900 python bench.py > gpurun_out/p23_bench.json 2> gpurun_out/p23_bench.err
echo "bench rc=$?" >> gpurun_out/p23_bench.err
tail -n 2 gpurun_out/p23_gputests.log gpurun_out/p23_smoke.log gpurun_out/p23_bench.err
