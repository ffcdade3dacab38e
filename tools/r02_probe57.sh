#!/bin/bash
# flakiness check: the GPU suite twice more, with xdist-free sequential runs
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for i in 1 2; do timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/p57_gputests_$i.log 2>&1; echo "run $i rc=$?"; tail -1 gpurun_out/p57_gputests_$i.log; done
