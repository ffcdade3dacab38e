#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python tools/prof_cheb.py 40 2 > gpurun_out/p3_plain.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cheb3 -s 2 -c 1 -o gpurun_out/p3_cheb3 python tools/prof_cheb.py 40 2 > gpurun_out/p3_ncu3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil7_cheb2f -s 4 -c 1 -o gpurun_out/p3_cheb2f env PCGX_CHEB3=0 python tools/prof_cheb.py 40 2 > gpurun_out/p3_ncu2.log 2>&1
echo done
