# SPDX-License-Identifier: Apache-2.0
"""Config-3 solve (256^3 Q1 FE27, k = 40) for launch lists: python tools/solve_fe27.py [NX] [K] [MAXIT]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_01440_b200 as P  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 256
k = int(sys.argv[2]) if len(sys.argv) > 2 else 40
maxit = int(sys.argv[3]) if len(sys.argv) > 3 else 3
A = P.gen_fe27(nx, sigma=1.0, seed=20240801)
with P.Context(0) as ctx:
    op, _ = P.jacobi_scale(P.CsrMatrix(A.n, A.row_ptr, A.col_idx, A.values), ctx)
    lo, hi = P.lanczos_bounds(op, 20, 30, 20240801)
    rhs = op.apply(P.random_uniform_vector(A.n, 20240801, ctx=ctx))
    prec = P.ChebyshevPreconditioner(P.cheb_params(lo, hi, k, 1.001))
    for i in range(2):
        x, rep = P.pcg_solve(op, rhs, P.SolveOptions(maxit=maxit), prec)
        print(f"solve {i}: {rep.wall_time * 1e3:.3f} ms, iters {rep.iters}", flush=True)
