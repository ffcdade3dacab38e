# SPDX-License-Identifier: Apache-2.0
"""Small-grid workload for compute-sanitizer (memcheck / synccheck / racecheck):
every hand-written TMA / mbarrier kernel on ragged shapes -- the two-step pass
(first, fused-update, regular, reducing), the three-step pass, the direction
step, the offset-storage grid kernels (dia3 / dia3t), BSR-3 (bsr3 / bsr3t), the
update kernels, the conditional-graph solve -- plus the host-visible results
checked against the oracle (a sanitizer run must also compute the right thing).

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle, OracleOp  # noqa: E402
from paper_2008_01440_b200 import pcgx as P  # noqa: E402

SEED = 20240801


def main():
    O = Oracle()
    with P.Context(0) as ctx:
        for cheb3 in ("0", "1"):
            os.environ["PCGX_CHEB3"] = cheb3
            for dims in ((66, 26, 9), (64, 20, 5)):
                nx, ny, nz = dims
                op, _ = P.jacobi_scale(P.StencilOperator(nx, ny, nz), ctx)
                opo = OracleOp("lap3d", nx=nx, ny=ny, nz=nz)
                a, b = P.analytic_extremes_box(nx, ny, nz)
                r = O.random_uniform(nx * ny * nz, 3)
                for m in (2, 5, 8):
                    out = P.apply_chebyshev(P.cheb_params(a, b, m, 1.001), op, r)
                    assert np.array_equal(out, O.apply_chebyshev(opo, O.cheb_params(a, b, m, 1.001), r)), (dims, m)
                rhs = O.apply(opo, O.random_uniform(nx * ny * nz, SEED))
                for m in (0, 3, 6):
                    x, rep = P.pcg_solve(op, rhs, P.SolveOptions(maxit=4000),
                                         P.ChebyshevPreconditioner(P.cheb_params(a, b, m, 1.001)))
                    assert rep.converged, (dims, m)
                op.close()
        os.environ["PCGX_CHEB3"] = "0"
        for gen, nx in (("fe27", 36), ("elast27", 36)):
            A = P.gen_fe27(nx, 1.0, SEED) if gen == "fe27" else P.gen_elast27(nx, 1.0, 0.5, 0.1, SEED)
            op, _ = P.jacobi_scale(A, ctx)
            opo = OracleOp("csr", row_ptr=A.row_ptr, col_idx=A.col_idx, values=A.values)
            x = O.random_uniform(A.n, 5)
            assert np.array_equal(op.apply(x), O.apply(opo, x))
            prm = P.cheb_params(0.01, 2.6, 4, 1.001)
            assert np.array_equal(P.apply_chebyshev(prm, op, x),
                                  O.apply_chebyshev(opo, O.cheb_params(0.01, 2.6, 4, 1.001), x))
            _, rep = P.pcg_solve(op, op.apply(x), P.SolveOptions(maxit=200), P.ChebyshevPreconditioner(prm))
            print(gen, op.storage(), rep.iters, flush=True)
            op.close()
    print("sanitize workload ok", flush=True)


if __name__ == "__main__":
    main()
