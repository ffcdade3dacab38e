#!/bin/bash
# chunk-plan sweep of the regular two-step pass at 640^3 / 512^3 (DRAM bytes, duration under ncu)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
M="dram__bytes_read.sum,gpu__time_duration.sum"
run() {  # tag nx env...
  tag=$1; nx=$2; shift 2
  env "$@" timeout 600 ncu --metrics $M --clock-control none --kernel-name-base demangled \
    -k "regex:cheb2f_kernel<\\(bool\\)0, \\(bool\\)0, \\(bool\\)0>" -s 4 -c 3 --csv \
    python tools/prof_cheb.py 40 1 $nx > gpurun_out/p27_$tag.csv 2> gpurun_out/p27_$tag.err
}
for nx in 640 512; do
  run ${nx}_auto $nx X=1
  for h in 24 40 48 80 96 128; do run ${nx}_u$h $nx PCGX_C2PLAN=u PCGX_KZ2=$h; done
done
python - <<'PY'
import csv, glob
for f in sorted(glob.glob("gpurun_out/p27_*.csv")):
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    if not rows: print(f, "no rows"); continue
    hdr = rows[0]; vals = {}
    for r in rows[1:]:
        d = dict(zip(hdr, r)); vals.setdefault(d["Metric Name"], []).append(float(d["Metric Value"]))
    rd = sum(vals["dram__bytes_read.sum"]) / len(vals["dram__bytes_read.sum"]) / 1e9
    t = sorted(vals["gpu__time_duration.sum"])[1] / 1e3
    print(f"{f:32s} read {rd:6.3f} GB  t {t:8.1f} us")
PY
