#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cheb3" > gpurun_out/p13_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/p13_tests.log
timeout 900 python tools/kbench_cheb2.py --rounds 3 --reps 20 --m 40 "PCGX_CHEB3=0" "PCGX_CHEB3=1" "lib=tools/bin/libpcgx_c3v2ty18.so+PCGX_CHEB3=1" "lib=tools/bin/libpcgx_c3v2u2.so+PCGX_CHEB3=1" > gpurun_out/p13_kbench.log 2>&1
PCGX_CHEB3=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:cheb3 -s 2 -c 1 -o gpurun_out/p13_cheb3 python tools/prof_cheb.py 40 2 > gpurun_out/p13_ncu3.log 2>&1
echo done
