#!/bin/bash
# conditional-graph threshold A/B at low degrees (k = 0, 5, 10)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for th in 10 1; do
  for rep in 1 2; do
    PCGX_COND_GRAPH=$th timeout 600 python bench.py --degrees 0,5,10 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/p24_th${th}_${rep}.json 2> gpurun_out/p24_th${th}_${rep}.err
  done
done
python - <<'PY'
import json
for th in (10, 1):
    for rep in (1, 2):
        d = json.load(open(f"gpurun_out/p24_th{th}_{rep}.json"))
        print(th, rep, [(p["k"], p["iters"], p["median_s"], p["ms_per_iter"]) for p in d["per_k"]], d["clocks"]["sm_mhz"])
PY
