#!/bin/bash
# round-2 probe 1: baseline bench on this box + power sensitivity of the two-step
# pass to its fp64 instruction count (the FMA-contracted build as an A/B only).
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi > gpurun_out/p1_smi.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/p1_bench.json 2> gpurun_out/p1_bench.log
timeout 600 python tools/kbench_cheb2.py --rounds 3 --reps 50 --m 40 "PCGX_CHEB2V=3" "lib=tools/bin/libpcgx_fma.so+PCGX_CHEB2V=3" > gpurun_out/p1_kbench.log 2>&1
timeout 300 python tools/power_probe.py cheb2 4 > gpurun_out/p1_power_cheb2.log 2>&1
timeout 300 python tools/power_probe.py copy 4 > gpurun_out/p1_power_copy.log 2>&1
PCGX_LIB=tools/bin/libpcgx_fma.so timeout 300 python tools/power_probe.py cheb2 4 > gpurun_out/p1_power_cheb2_fma.log 2>&1
echo done
