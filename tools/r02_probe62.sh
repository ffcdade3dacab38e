#!/bin/bash
# single-domain constants in the two-step kernels (experiment build): solves A/B
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
L=paper_2008_01440_b200/libpcgx.so; S=tools/bin/libpcgx_single.so
for m in 5 20 80; do timeout 600 python tools/solve_ab.py 320 $m 3 $L $S > gpurun_out/p62_ab_k$m.log 2>&1; echo "k=$m"; cat gpurun_out/p62_ab_k$m.log; done
for lib in $L $S; do
PCGX_LIB=$lib PCGX_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:stencil7_cheb2f_kernel -c 40 --csv python tools/solve_once.py 320 20 3 2>/dev/null | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]; hdr=rows[0]; v={}
for r in rows[1:]:
    d=dict(zip(hdr,r)); v.setdefault((d['Kernel Name'][:38],d['Metric Name']),[]).append(float(d['Metric Value'].replace(',','')))
for k in sorted(v): print('$lib', k, len(v[k]), sorted(v[k])[len(v[k])//2])"
done
