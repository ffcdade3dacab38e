#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -q -m gpu -rs --durations=20 -s > gpurun_out/p14_gputests.log 2>&1
echo "gpu tests rc=$?" >> gpurun_out/p14_gputests.log
./oracle/_ref/adapter_test > gpurun_out/p14_adapter.log 2>&1; echo "adapter rc=$?" >> gpurun_out/p14_adapter.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/p14_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/p14_smoke.log
for cfg in cfg1 cfg3 cfg4 cfg5s cfg5w; do
  timeout 1200 python bench.py --config $cfg --no-cpu-baseline > gpurun_out/p14_bench_$cfg.json 2> gpurun_out/p14_bench_$cfg.log
done
echo done
