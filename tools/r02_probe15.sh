#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or schedules or fullsize or per_degree or device_convergence" > gpurun_out/p15_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/p15_tests.log
timeout 900 python tools/solve_ab.py 320 5 5 tools/bin/libpcgx_upd_noahead.so tools/bin/libpcgx_upd_ahead.so > gpurun_out/p15_ab_k5.log 2>&1
timeout 900 python tools/solve_ab.py 320 20 5 tools/bin/libpcgx_upd_noahead.so tools/bin/libpcgx_upd_ahead.so > gpurun_out/p15_ab_k20.log 2>&1
PCGX_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:cheb2f_kernel<\\(bool\\)1, \\(bool\\)0, \\(bool\\)1>" -s 3 -c 1 -o gpurun_out/p15_first python tools/solve_ab.py --child 320 20 > gpurun_out/p15_ncu_first.log 2>&1
echo done
