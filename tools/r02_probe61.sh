#!/bin/bash
# plan search with early exit: first-apply latency, same plans (bitwise reductions => same solve), quick parity
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
PYTHONPATH=. python - <<'PY'
import time
import paper_2008_01440_b200 as P
with P.Context(0) as ctx:
    for nx, m in ((320, 8), (320, 5), (640, 8)):
        op,_=P.jacobi_scale(P.StencilOperator(nx),ctx)
        a,b=P.analytic_extremes(3,nx)
        r=P.random_uniform_vector(nx**3,1,ctx=ctx)
        prm=P.cheb_params(a,b,m,1.001)
        t=time.time(); z=P.apply_chebyshev(prm,op,r); ctx.synchronize(); t1=time.time()-t
        t=time.time(); z=P.apply_chebyshev(prm,op,r); ctx.synchronize(); t2=time.time()-t
        print('nx',nx,'m',m,'first apply %.3f s, second %.3f s'%(t1,t2))
        op.close()
PY
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -k "cfg2" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
python bench.py --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['in_solve']['frac'])"
