#!/bin/bash
# A/B (same box, interleaved) of the L2-capped chunk plans against the previous plans
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
NEW=paper_2008_01440_b200/libpcgx.so; OLD=tools/bin/libpcgx_old.so
for cfg in "640 40" "512 40" "320 20"; do
  set -- $cfg
  timeout 900 python tools/solve_ab.py $1 $2 5 $OLD $NEW > gpurun_out/p29_ab_$1.log 2>&1
  echo "nx=$1 k=$2"; cat gpurun_out/p29_ab_$1.log
done
M="dram__bytes_read.sum,gpu__time_duration.sum"
for nx in 640 512; do for L in $OLD $NEW; do
  PCGX_LIB=$L PCGX_NO_GRAPH=1 timeout 600 ncu --metrics $M --clock-control none -k regex:stencil7_dir_kernel -s 3 -c 3 --csv \
    python tools/solve_once.py $nx 20 6 2>/dev/null | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]; hdr=rows[0]; v={}
for r in rows[1:]:
    d=dict(zip(hdr,r)); v.setdefault(d['Metric Name'],[]).append(float(d['Metric Value']))
print('dir nx=$nx $L', round(sum(v['dram__bytes_read.sum'])/3e9,3), sorted(v['gpu__time_duration.sum'])[1]/1e3)"
done; done
