#!/bin/bash
# full launch list of the bench command (graphs off so ncu sees every kernel)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
PCGX_NO_GRAPH=1 timeout 3300 ncu --metrics gpu__time_duration.sum --clock-control none -c 100000 --csv --log-file gpurun_out/p43_launches_bench.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/p43_ncu_bench.log 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/p43_launches_bench.csv > gpurun_out/p43_launches_bench_summary.txt 2>&1
cat gpurun_out/p43_launches_bench_summary.txt | head -30
rm -f gpurun_out/p43_launches_bench.csv.tmp
