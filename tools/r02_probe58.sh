#!/bin/bash
# persisting-L2 window over r in the regular two-step passes: apply A/B, DRAM traffic under ncu
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "
import torch
p=torch.cuda.get_device_properties(0)
print('L2', p.L2_cache_size/2**20, 'MB')
import ctypes
rt=ctypes.CDLL('libcudart.so.12')
for name,idx in (('MaxPersistingL2CacheSize',108),('MaxAccessPolicyWindowSize',109)):
    v=ctypes.c_int(); rt.cudaDeviceGetAttribute(ctypes.byref(v), idx, 0); print(name, v.value/2**20,'MB')
" 2>&1 | tail -3
timeout 900 python tools/kbench_cheb2.py --rounds 3 --reps 50 PCGX_L2_PERSIST_MB=0 PCGX_L2_PERSIST_MB=48 PCGX_L2_PERSIST_MB=72 PCGX_L2_PERSIST_MB=96 > gpurun_out/p58_l2.log 2>&1
cat gpurun_out/p58_l2.log
for mb in 0 72; do
PCGX_L2_PERSIST_MB=$mb PCGX_NO_GRAPH=1 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:stencil7_cheb2f_kernel -s 12 -c 6 --csv python tools/solve_once.py 320 20 3 2>/dev/null | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]; hdr=rows[0]; v={}
for r in rows[1:]:
    d=dict(zip(hdr,r)); v.setdefault((d['Kernel Name'][:38],d['Metric Name']),[]).append(float(d['Metric Value'].replace(',','')))
for k in sorted(v): print('mb=$mb', k, len(v[k]), sorted(v[k])[len(v[k])//2], d['Metric Unit'] if False else '')"
done
