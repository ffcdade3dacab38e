#!/bin/bash
# L2-capped chunk plans: regular pass / direction kernel under ncu at 640/512/320, live cfg5s / cfg5w bench
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
M="dram__bytes_read.sum,gpu__time_duration.sum"
for nx in 640 512 320; do
  timeout 600 ncu --metrics $M --clock-control none --kernel-name-base demangled \
    -k "regex:cheb2f_kernel<\\(bool\\)0, \\(bool\\)0, \\(bool\\)0>" -s 4 -c 3 --csv \
    python tools/prof_cheb.py 40 1 $nx > gpurun_out/p28_pass_$nx.csv 2> gpurun_out/p28_pass_$nx.err
  timeout 600 ncu --metrics $M --clock-control none -k regex:stencil7_dir_kernel -s 3 -c 3 --csv \
    python tools/solve_once.py $nx 20 6 > gpurun_out/p28_dir_$nx.csv 2> gpurun_out/p28_dir_$nx.err
done
python - <<'PY'
import csv, glob
for f in sorted(glob.glob("gpurun_out/p28_*.csv")):
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    if not rows: print(f, "no rows"); continue
    hdr = rows[0]; vals = {}
    for r in rows[1:]:
        d = dict(zip(hdr, r)); vals.setdefault(d["Metric Name"], []).append(float(d["Metric Value"]))
    rd = sum(vals["dram__bytes_read.sum"]) / len(vals["dram__bytes_read.sum"]) / 1e9
    t = sorted(vals["gpu__time_duration.sum"])[len(vals["gpu__time_duration.sum"]) // 2] / 1e3
    print(f"{f:32s} read {rd:6.3f} GB  t {t:8.1f} us")
PY
for cfg in cfg5s cfg5w; do
  timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/p28_bench_$cfg.json 2> gpurun_out/p28_bench_$cfg.err
  python -c "import json;d=json.load(open('gpurun_out/p28_bench_$cfg.json'));print('$cfg',d['value'],d['ms_per_step'],d['roofline']['frac'],d['roofline']['avg_launch_ms'],d['clocks']['sm_mhz'])"
done
