#!/bin/bash
# round-2 probe 2: three-step pass parity + A/B against the two-step schedule
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cheb3 or cheb2 or per_degree or large_degree or schedules or fused_update" > gpurun_out/p2_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/p2_tests.log
timeout 600 python tools/kbench_cheb2.py --same --rounds 5 --reps 20 --m 40 "PCGX_CHEB3=0" "PCGX_CHEB3=1" > gpurun_out/p2_kbench40.log 2>&1
timeout 600 python tools/kbench_cheb2.py --same --rounds 5 --reps 20 --m 20 "PCGX_CHEB3=0" "PCGX_CHEB3=1" > gpurun_out/p2_kbench20.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/p2_bench.json 2> gpurun_out/p2_bench.log
echo done
