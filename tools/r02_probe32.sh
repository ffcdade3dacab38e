#!/bin/bash
# Odd degrees ending with one three-step pass (PCGX_CHEB3=2) against two-step pass + single step:
# bitwise check of P_m(A) r, then whole solves A/B at 320^3 for k = 5, 7, 15
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
L=paper_2008_01440_b200/libpcgx.so
python - > gpurun_out/p32_bitwise.log 2>&1 <<'PY'
import os, numpy as np
import paper_2008_01440_b200 as P
res = {}
for mode in ("0", "2"):
    os.environ["PCGX_CHEB3"] = mode
    with P.Context(0) as ctx:
        for nx in (64, 96):
            op, _ = P.jacobi_scale(P.StencilOperator(nx), ctx)
            a, b = P.analytic_extremes(3, nx)
            r = P.random_uniform_vector(nx ** 3, 3)
            for m in (5, 7, 9, 13, 21):
                res[(mode, nx, m)] = P.apply_chebyshev(P.cheb_params(a, b, m, 1.001), op, r)
            rhs = op.apply(P.random_uniform_vector(nx ** 3, 5))
            x, rep = P.pcg_solve(op, rhs, None, P.ChebyshevPreconditioner(P.cheb_params(a, b, 5, 1.001)))
            res[(mode, nx, "x")] = x; res[(mode, nx, "it")] = rep.iters
ok = all(np.array_equal(res[("0",) + k[1:]], res[k]) for k in res if k[0] == "2")
print("tail3 bitwise vs two-step + single:", ok, [res[(md, 96, "it")] for md in ("0", "2")])
PY
cat gpurun_out/p32_bitwise.log
for m in 5 7 15; do
  timeout 600 python tools/solve_ab.py 320 $m 3 $L $L+PCGX_CHEB3=2 > gpurun_out/p32_ab_k$m.log 2>&1
  echo "k=$m"; cat gpurun_out/p32_ab_k$m.log
done
