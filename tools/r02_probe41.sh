#!/bin/bash
# HEAD bench lines for every config + the reference arm + the launch list of the bench command
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/p41_bench_cfg2.json 2> gpurun_out/p41_bench_cfg2.err; echo "cfg2 rc=$?"
for cfg in cfg1 cfg3 cfg4 cfg5s cfg5w; do
  timeout 1500 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/p41_bench_$cfg.json 2> gpurun_out/p41_bench_$cfg.err; echo "$cfg rc=$?"
done
timeout 900 python bench.py --impl reference > gpurun_out/p41_bench_ref.json 2> gpurun_out/p41_bench_ref.err; echo "ref rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/p41_launches_bench.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/p41_ncu_bench.log 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/p41_launches_bench.csv > gpurun_out/p41_launches_bench_summary.txt 2>&1
cat gpurun_out/p41_launches_bench_summary.txt | head -30
