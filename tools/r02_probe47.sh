#!/bin/bash
# direction-step chunk plans at 320^3 (k = 0 solve: direction step + update only)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
L=paper_2008_01440_b200/libpcgx.so
timeout 900 python tools/solve_ab.py 320 0 3 $L "$L+PCGX_C2PLAN=u+PCGX_KZ2=32" "$L+PCGX_C2PLAN=u+PCGX_KZ2=64" "$L+PCGX_C2PLAN=64,64,64,64,40,24" "$L+PCGX_C2PLAN=40,80,80,80,24,16" "$L+PCGX_C2PLAN=16,48,48,48,48,48,32,20,12" "$L+PCGX_C2PLAN=176,88,28,28" > gpurun_out/p47_dirplans.log 2>&1
cat gpurun_out/p47_dirplans.log
