#!/bin/bash
# wider chunk-plan search (long chunks when all tiles of a level are resident): whole solves A/B, apply A/B, first-apply latency
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
NEW=paper_2008_01440_b200/libpcgx.so; OLD=tools/bin/libpcgx_oldplan.so
timeout 600 python tools/kbench_cheb2.py --rounds 3 --reps 50 lib=$OLD lib=$NEW > gpurun_out/p46_kbench.log 2>&1; cat gpurun_out/p46_kbench.log
for m in 0 5 20 80; do
  timeout 600 python tools/solve_ab.py 320 $m 3 $OLD $NEW > gpurun_out/p46_ab_k$m.log 2>&1
  echo "k=$m"; cat gpurun_out/p46_ab_k$m.log
done
for nx in 512; do
  timeout 600 python tools/solve_ab.py $nx 40 2 $OLD $NEW > gpurun_out/p46_ab_${nx}.log 2>&1
  echo "nx=$nx"; cat gpurun_out/p46_ab_${nx}.log
done
PYTHONPATH=. python - <<'PY'
import time, numpy as np
import paper_2008_01440_b200 as P
with P.Context(0) as ctx:
    for nx in (320, 100, 640):
        op,_=P.jacobi_scale(P.StencilOperator(nx),ctx)
        a,b=P.analytic_extremes(3,nx)
        r=P.random_uniform_vector(nx**3,1,ctx=ctx)
        prm=P.cheb_params(a,b,8,1.001)
        t=time.time(); z=P.apply_chebyshev(prm,op,r); ctx.synchronize(); t1=time.time()-t
        t=time.time(); z=P.apply_chebyshev(prm,op,r); ctx.synchronize(); t2=time.time()-t
        print('nx',nx,'first apply %.3f s, second %.3f s'%(t1,t2))
        op.close()
PY
