#!/bin/bash
# ncu --set full of the fused first pass (update inside P r's first two-step pass) for the stall / source breakdown
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
PCGX_NO_GRAPH=1 timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:cheb2f_kernel<\\(bool\\)1, \\(bool\\)0, \\(bool\\)1>" -s 4 -c 1 -o gpurun_out/p55_upd -f python tools/solve_once.py 320 20 8 > gpurun_out/p55.log 2>&1
ls -la gpurun_out/p55_upd.ncu-rep
