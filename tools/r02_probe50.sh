#!/bin/bash
# three-step schedule vs two-step schedule with the long-chunk planner (320^3, sustained), and whole solves
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
L=paper_2008_01440_b200/libpcgx.so
timeout 900 python tools/kbench_cheb2.py --rounds 3 --reps 50 PCGX_CHEB3=2 PCGX_CHEB3=1 "PCGX_CHEB3=1+PCGX_C2PLAN=320" "PCGX_CHEB3=1+PCGX_C2PLAN=160,160" > gpurun_out/p50_c3.log 2>&1
cat gpurun_out/p50_c3.log
for m in 20 40; do timeout 600 python tools/solve_ab.py 320 $m 3 $L $L+PCGX_CHEB3=1 > gpurun_out/p50_ab_k$m.log 2>&1; echo "k=$m"; cat gpurun_out/p50_ab_k$m.log; done
