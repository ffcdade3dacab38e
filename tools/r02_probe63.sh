#!/bin/bash
# direction step with the long-chunk plan in Chebyshev solves (explicit plan = two-step plan, so only the direction step changes)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
L=paper_2008_01440_b200/libpcgx.so
for m in 10 20 40; do timeout 600 python tools/solve_ab.py 320 $m 5 $L "$L+PCGX_C2PLAN=176,88,28,28" > gpurun_out/p63_ab_k$m.log 2>&1; echo "k=$m"; cat gpurun_out/p63_ab_k$m.log; done
