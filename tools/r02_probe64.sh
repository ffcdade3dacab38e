#!/bin/bash
# direction step with a 4-slot operand ring (room for a second p tile): k = 0 and k = 20 solves
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
L=paper_2008_01440_b200/libpcgx.so
for m in 0 20; do timeout 600 python tools/solve_ab.py 320 $m 4 $L tools/bin/libpcgx_ns4.so > gpurun_out/p64_ab_k$m.log 2>&1; echo "k=$m"; cat gpurun_out/p64_ab_k$m.log; done
