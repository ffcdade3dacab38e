#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python tools/kbench_cheb2.py --rounds 3 --reps 20 --m 40 "PCGX_CHEB3=0" "PCGX_CHEB3=1" "lib=tools/bin/libpcgx_c3u2.so" "lib=tools/bin/libpcgx_c3ty14.so" "lib=tools/bin/libpcgx_c3ty14u2.so" > gpurun_out/p6_kbench.log 2>&1
echo done
