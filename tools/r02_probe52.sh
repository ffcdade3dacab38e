#!/bin/bash
# HEAD ncu --set full capture of the regular two-step pass inside bench.py (long-chunk plan) + per-k launch lists
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:cheb2f_kernel<\\(bool\\)0, \\(bool\\)0, \\(bool\\)0>" -s 100 -c 1 \
    -o gpurun_out/ncu_cfg2 -f python bench.py --config cfg2 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/p52_ncu.log 2>&1
echo "ncu rc=$?"
python tools/ncu_to_traffic.py gpurun_out/ncu_cfg2.ncu-rep cfg2 32768000 1310720000 > gpurun_out/p52_traffic.log 2>&1; cat gpurun_out/p52_traffic.log | tail -20
for k in 20 5; do
PCGX_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/p52_launches_k$k.csv python tools/solve_timeline.py 320 $k > gpurun_out/p52_tl_k$k.log 2>&1
python tools/launch_summary.py gpurun_out/p52_launches_k$k.csv | tee gpurun_out/p52_launches_k${k}_summary.txt
done
