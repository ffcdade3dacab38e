#!/bin/bash
# Where the capped two-step pass spends its power: variants without the j / i shared loads,
# the halo columns and the stencil arithmetic (experiment builds, not bitwise), sustained load
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
V="lib=paper_2008_01440_b200/libpcgx.so"
for e in 1 2 3 4; do V="$V lib=tools/bin/libpcgx_exp$e.so"; done
timeout 1200 python tools/kbench_cheb2.py --rounds 3 --reps 100 $V > gpurun_out/p31_kbench_exp.log 2>&1
cat gpurun_out/p31_kbench_exp.log
