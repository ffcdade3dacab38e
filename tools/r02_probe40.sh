#!/bin/bash
# three-step pass: plane-loop unroll 4 (default) / 2 / 1 (instruction-fetch stalls), sustained
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
L=paper_2008_01440_b200/libpcgx.so
PCGX_CHEB3=1 timeout 900 python tools/kbench_cheb2.py --rounds 3 --reps 50 lib=$L lib=tools/bin/libpcgx_c3u2.so lib=tools/bin/libpcgx_c3u1.so > gpurun_out/p40_c3unroll.log 2>&1
cat gpurun_out/p40_c3unroll.log
