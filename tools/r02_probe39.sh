#!/bin/bash
# ncu --set full of the three-step pass (PCGX_CHEB3=1) and of the two-step pass, for the stall breakdown
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
PCGX_CHEB3=1 PCGX_NO_GRAPH=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:stencil7_cheb3_kernel -s 4 -c 1 -o gpurun_out/p39_cheb3 -f python tools/solve_once.py 320 40 2 > gpurun_out/p39_a.log 2>&1
PCGX_CHEB3=0 PCGX_NO_GRAPH=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:stencil7_cheb2f_kernel -s 6 -c 1 -o gpurun_out/p39_cheb2 -f python tools/solve_once.py 320 40 2 > gpurun_out/p39_b.log 2>&1
ls -la gpurun_out/p39*
