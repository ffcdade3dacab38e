# SPDX-License-Identifier: Apache-2.0
"""One Chebyshev-PCG solve on the nx^3 matrix-free Laplacian (profiling driver).

    python tools/solve_once.py NX M [MAXIT]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_01440_b200 as P  # noqa: E402

nx, m = int(sys.argv[1]), int(sys.argv[2])
maxit = int(sys.argv[3]) if len(sys.argv) > 3 else 10
with P.Context(0) as ctx:
    op, _ = P.jacobi_scale(P.StencilOperator(nx), ctx)
    a, b = P.analytic_extremes(3, nx)
    rhs = op.apply(P.random_uniform_vector(nx ** 3, 20240801, ctx=ctx))
    prec = P.ChebyshevPreconditioner(P.cheb_params(a, b, m, 1.001)) if m >= 0 else None
    x, rep = P.pcg_solve(op, rhs, P.SolveOptions(maxit=maxit), prec)
    print(rep.iters, rep.rel_res)
