#!/bin/bash
# L2 eviction hints on the streaming operands of the two-step pass (experiment builds): 320 / 512 / 640, DRAM traffic at 640
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
L=paper_2008_01440_b200/libpcgx.so
for nx in 320 512 640; do
  reps=50; [ $nx -gt 320 ] && reps=10
  timeout 900 python tools/kbench_cheb2.py --nx $nx --m 20 --rounds 3 --reps $reps lib=$L lib=tools/bin/libpcgx_l2h1.so lib=tools/bin/libpcgx_l2h2.so > gpurun_out/p59_l2h_$nx.log 2>&1
  echo "nx=$nx"; cat gpurun_out/p59_l2h_$nx.log
done
for lib in $L tools/bin/libpcgx_l2h1.so tools/bin/libpcgx_l2h2.so; do
PCGX_LIB=$lib PCGX_NO_GRAPH=1 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:stencil7_cheb2f_kernel -s 6 -c 4 --csv python tools/solve_once.py 640 20 2 2>/dev/null | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]; hdr=rows[0]; v={}
for r in rows[1:]:
    d=dict(zip(hdr,r)); v.setdefault((d['Kernel Name'][:38],d['Metric Name']),[]).append(float(d['Metric Value'].replace(',','')))
for k in sorted(v): print('$lib', k, len(v[k]), sorted(v[k])[len(v[k])//2])"
done
