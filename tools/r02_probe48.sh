#!/bin/bash
# chunk lengths at 512^3 and 640^3 (more tiles than SMs): uniform chunks of various heights vs the planner
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 python tools/kbench_cheb2.py --same --nx 512 --m 20 --rounds 3 --reps 10 "PCGX_KZ2=32" "PCGX_C2PLAN=u+PCGX_KZ2=48" "PCGX_C2PLAN=u+PCGX_KZ2=64" "PCGX_C2PLAN=u+PCGX_KZ2=128" "PCGX_C2PLAN=u+PCGX_KZ2=256" "PCGX_C2PLAN=360,72,72,8" "PCGX_C2PLAN=216,256,40" > gpurun_out/p48_512.log 2>&1
cat gpurun_out/p48_512.log
timeout 1200 python tools/kbench_cheb2.py --same --nx 640 --m 20 --rounds 3 --reps 6 "PCGX_KZ2=32" "PCGX_C2PLAN=u+PCGX_KZ2=48" "PCGX_C2PLAN=u+PCGX_KZ2=64" "PCGX_C2PLAN=u+PCGX_KZ2=128" "PCGX_C2PLAN=216,320,104" "PCGX_C2PLAN=432,104,104" > gpurun_out/p48_640.log 2>&1
cat gpurun_out/p48_640.log
