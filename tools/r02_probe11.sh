#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python tools/solve_ab.py 320 5 5 tools/bin/libpcgx_div1.so tools/bin/libpcgx_div2.so > gpurun_out/p11_ab_k5.log 2>&1
timeout 900 python tools/solve_ab.py 320 20 5 tools/bin/libpcgx_div1.so tools/bin/libpcgx_div2.so > gpurun_out/p11_ab_k20.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:cheb2f_kernel<\\(bool\\)1, \\(bool\\)0, \\(bool\\)1>" -s 3 -c 1 -o gpurun_out/p11_first python tools/solve_ab.py --child 320 20 > gpurun_out/p11_ncu_first.log 2>&1
PCGX_LIB=tools/bin/libpcgx_checked.so timeout 900 python tools/sanitize_run.py > gpurun_out/p11_checked.log 2>&1
echo "checked rc=$?" >> gpurun_out/p11_checked.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "table1" > gpurun_out/p11_table1.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -q -s -k "cfg3 or cfg5s" > gpurun_out/p11_fullsize.log 2>&1
echo done
