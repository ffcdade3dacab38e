#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python tools/power_probe.py cheb2 5 > gpurun_out/p16_power_cheb2.log 2>&1
PCGX_LIB=tools/bin/libpcgx_nomath.so timeout 600 python tools/power_probe.py cheb2 5 > gpurun_out/p16_power_nomath.log 2>&1
timeout 600 python tools/power_probe.py copy 5 > gpurun_out/p16_power_copy.log 2>&1
timeout 600 python tools/kbench_cheb2.py --rounds 3 --reps 30 --m 40 "PCGX_CHEB3=0" "lib=tools/bin/libpcgx_nomath.so" > gpurun_out/p16_kbench.log 2>&1
timeout 900 python -m pytest tests/test_gpu_checked.py -q > gpurun_out/p16_checked.log 2>&1
echo done
