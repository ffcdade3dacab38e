#!/bin/bash
# pruned kernel variants: parity suite + solves A/B against the previous build
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/p53_gputests.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/p53_gputests.log
tail -3 gpurun_out/p53_gputests.log
NEW=paper_2008_01440_b200/libpcgx.so; OLD=tools/bin/libpcgx_prev.so
for m in 0 5 20; do timeout 600 python tools/solve_ab.py 320 $m 3 $OLD $NEW > gpurun_out/p53_ab_k$m.log 2>&1; echo "k=$m"; cat gpurun_out/p53_ab_k$m.log; done
