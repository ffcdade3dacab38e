#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for i in 1 2; do
timeout 600 python tools/power_probe.py cheb2 6 >> gpurun_out/p17_power_base.log 2>&1
PCGX_LIB=tools/bin/libpcgx_nbr0.so timeout 600 python tools/power_probe.py cheb2 6 >> gpurun_out/p17_power_nbr0.log 2>&1
done
timeout 600 python tools/kbench_cheb2.py --rounds 3 --reps 40 --m 40 "PCGX_CHEB3=0" "lib=tools/bin/libpcgx_nbr0.so" > gpurun_out/p17_kbench.log 2>&1
echo done
