#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
./tools/bin/cond_probe > gpurun_out/p5_cond_probe.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cheb3 or cheb2_bitwise or per_degree or schedules or fused or on_iterate or pcg" > gpurun_out/p5_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/p5_tests.log
timeout 900 python tools/kbench_cheb2.py --same --rounds 5 --reps 20 --m 40 "PCGX_CHEB3=0" "PCGX_CHEB3=1" > gpurun_out/p5_kbench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cheb3 -s 2 -c 1 -o gpurun_out/p5_cheb3 python tools/prof_cheb.py 40 2 > gpurun_out/p5_ncu3.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/p5_bench.json 2> gpurun_out/p5_bench.log
echo done
