#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
L=paper_2008_01440_b200/libpcgx.so
for k in 5 10 20 80; do
  timeout 900 python tools/solve_ab.py 320 $k 4 "$L+PCGX_COND_GRAPH=0" "$L+PCGX_COND_GRAPH=1" > gpurun_out/p12_cond_k$k.log 2>&1
done
timeout 600 python tools/solve_ab.py 320 0 4 "$L+PCGX_COND_GRAPH=0" "$L+PCGX_COND_GRAPH=1" > gpurun_out/p12_cond_k0.log 2>&1
PCGX_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:cheb2f_kernel<\\(bool\\)1, \\(bool\\)0, \\(bool\\)1>" -s 3 -c 1 -o gpurun_out/p12_first python tools/solve_ab.py --child 320 20 > gpurun_out/p12_ncu_first.log 2>&1
echo done
