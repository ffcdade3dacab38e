#!/bin/bash
# fused first pass: incremental r pointer + one-compare plane range; parity + A/B + ncu time of the pass
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_checked.py tests/test_gpu_multirank.py -x -q > gpurun_out/p56_tests.log 2>&1; echo "rc=$?" >> gpurun_out/p56_tests.log; tail -2 gpurun_out/p56_tests.log
NEW=paper_2008_01440_b200/libpcgx.so; OLD=tools/bin/libpcgx_prev.so
for m in 5 10; do timeout 600 python tools/solve_ab.py 320 $m 3 $OLD $NEW > gpurun_out/p56_ab_k$m.log 2>&1; echo "k=$m"; cat gpurun_out/p56_ab_k$m.log; done
for L in $OLD $NEW; do
PCGX_LIB=$L PCGX_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:stencil7_cheb2f_kernel -c 40 --csv python tools/solve_once.py 320 20 3 2>/dev/null | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]; hdr=rows[0]; v={}
for r in rows[1:]:
    d=dict(zip(hdr,r)); v.setdefault((d['Kernel Name'][:40],d['Metric Name']),[]).append(float(d['Metric Value'].replace(',','')))
for k in v:
    if '1, 0, 1' in k[0]: print('$L', k, len(v[k]), sorted(v[k])[len(v[k])//2])"
done
