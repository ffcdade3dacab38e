#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/p10_smi.csv
timeout 900 python bench.py > gpurun_out/p10_bench.json 2> gpurun_out/p10_bench.log
echo "bench rc=$?" >> gpurun_out/p10_bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/p10_ref.json 2> gpurun_out/p10_ref.log
echo "ref rc=$?" >> gpurun_out/p10_ref.log
python bench.py --degrees 20 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/p10_k20_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/p10_launches_k20.csv python bench.py --degrees 20 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/p10_ncu_k20.log 2>&1
python bench.py --degrees 5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/p10_k5_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/p10_launches_k5.csv python bench.py --degrees 5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/p10_ncu_k5.log 2>&1
bash tools/profile_configs.sh cfg2 > gpurun_out/p10_profile.log 2>&1
echo done
