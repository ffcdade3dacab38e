#!/bin/bash
# ablation of the two-step pass from the movement side (experiment builds): levels 4..7
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
V="lib=paper_2008_01440_b200/libpcgx.so"
for e in 4 5 6 7; do V="$V lib=tools/bin/libpcgx_exp$e.so"; done
timeout 1200 python tools/kbench_cheb2.py --rounds 3 --reps 100 $V > gpurun_out/p44_kbench_exp.log 2>&1
cat gpurun_out/p44_kbench_exp.log
