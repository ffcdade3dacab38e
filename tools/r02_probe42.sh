#!/bin/bash
# launch list of the bench command with the solver's CUDA graphs off (ncu lists no kernels inside
# graph launches / conditional nodes), and the power draw of the three-step pass
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
PCGX_NO_GRAPH=1 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file gpurun_out/p42_launches_bench.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/p42_ncu_bench.log 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/p42_launches_bench.csv > gpurun_out/p42_launches_bench_summary.txt 2>&1
cat gpurun_out/p42_launches_bench_summary.txt | head -30
for w in cheb3 cheb2 copy; do PYTHONPATH=. timeout 300 python tools/power_probe.py $w 5 > gpurun_out/p42_power_$w.json 2>&1; tail -c 700 gpurun_out/p42_power_$w.json; echo; done
