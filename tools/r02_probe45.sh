#!/bin/bash
# chunk plans with long chunks at 320^3 (wider planner search) against the current plan: sustained A/B on one context
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 python tools/kbench_cheb2.py --same --rounds 5 --reps 50 "PCGX_KZ2=32" "PCGX_C2PLAN=176,88,28,28" "PCGX_C2PLAN=180,56,56,28" "PCGX_C2PLAN=180,84,28,28" "PCGX_C2PLAN=88,88,88,28,28" "PCGX_C2PLAN=184,80,32,24" > gpurun_out/p45_plans.log 2>&1
cat gpurun_out/p45_plans.log
