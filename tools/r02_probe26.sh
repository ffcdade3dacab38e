#!/bin/bash
# cfg5s (640^3) regular two-step pass: DRAM bytes and duration per chunk plan
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum"
run() {  # tag env...
  tag=$1; shift
  env "$@" timeout 600 ncu --metrics $M --clock-control none --kernel-name-base demangled \
    -k "regex:cheb2f_kernel<\\(bool\\)0, \\(bool\\)0, \\(bool\\)0>" -s 4 -c 2 --csv \
    python tools/prof_cheb.py 40 1 ${NX:-640} > gpurun_out/p26_$tag.csv 2> gpurun_out/p26_$tag.err
}
run auto X=1
run u32 PCGX_C2PLAN=u PCGX_KZ2=32
run u64 PCGX_C2PLAN=u PCGX_KZ2=64
run u160 PCGX_C2PLAN=u PCGX_KZ2=160
run one PCGX_C2PLAN=640
NX=512 run w_auto X=1
NX=512 run w_u64 PCGX_C2PLAN=u PCGX_KZ2=64
NX=320 run c2_auto X=1
python - <<'PY'
import csv, glob
for f in sorted(glob.glob("gpurun_out/p26_*.csv")):
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    if not rows: print(f, "no rows"); continue
    hdr = rows[0]; vals = {}
    for r in rows[1:]:
        d = dict(zip(hdr, r)); vals.setdefault(d["Metric Name"], []).append((d["Metric Unit"], d["Metric Value"]))
    print(f, {k: v for k, v in vals.items()})
PY
