#!/bin/bash
# three-step tail as the default: GPU suite and the cfg2 bench
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/p34_gputests.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/p34_gputests.log
tail -3 gpurun_out/p34_gputests.log
timeout 900 python bench.py > gpurun_out/p34_bench.json 2> gpurun_out/p34_bench.err; python - <<'PY'
import json
d=json.loads(open('gpurun_out/p34_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['time_to_1e8_s'], d['clocks'])
PY
