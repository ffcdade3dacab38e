# bitwise check of the three-step tail (PCGX_CHEB3=2) against the default schedule, key by key
import os, numpy as np
import paper_2008_01440_b200 as P
res = {}
for mode in ("0", "2"):
    os.environ["PCGX_CHEB3"] = mode
    with P.Context(0) as ctx:
        for nx in (64, 96, 100):
            op, _ = P.jacobi_scale(P.StencilOperator(nx), ctx)
            a, b = P.analytic_extremes(3, nx)
            r = P.random_uniform_vector(nx ** 3, 3)
            for m in (5, 7, 9, 13, 21):
                res[(mode, nx, m)] = P.apply_chebyshev(P.cheb_params(a, b, m, 1.001), op, r)
            rhs = op.apply(P.random_uniform_vector(nx ** 3, 5))
            x, rep = P.pcg_solve(op, rhs, None, P.ChebyshevPreconditioner(P.cheb_params(a, b, 5, 1.001)))
            res[(mode, nx, "x")] = x; res[(mode, nx, "it")] = rep.iters
for k in res:
    if k[0] == "2":
        a, b = res[("0",) + k[1:]], res[k]
        if isinstance(a, np.ndarray):
            print(k[1:], "bitwise" if np.array_equal(a, b) else "max rel diff %.3e" % (np.abs(a - b).max() / np.abs(a).max()))
        else:
            print(k[1:], a, b)
