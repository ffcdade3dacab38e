# SPDX-License-Identifier: Apache-2.0
"""CSR kernel micro-benchmark on the config-3/4 matrices.

    python tools/kbench_csr.py fe27|elast27|lap NX [VAR=VAL,...]...

Times the plain scaled SpMV (20 launches) and the fused Chebyshev middle step
(FLAG_TIME_KERNELS) with CUDA events; prints GB/s against the int32-CSR
algorithmic bytes (12 nnz + 4(n+1) + 16 n resp. + 40 n).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2008_01440_b200 as P  # noqa: E402
from paper_2008_01440_b200 import pcgx  # noqa: E402


def main():
    kind, nx = sys.argv[1], int(sys.argv[2])
    variants = sys.argv[3:] or [""]
    if kind == "fe27":
        A = P.gen_fe27(nx, 1.0, 20240801)
    elif kind == "elast27":
        A = P.gen_elast27(nx, 1.0, 0.5, 0.1, 20240801)
    else:
        sys.path.insert(0, ROOT)
        import bench
        rp, ci, va = bench.lap3d_csr_i32(nx)
        A = P.CsrMatrix(nx ** 3, rp, ci, va)
    n, nnz = A.n, A.nnz()
    with P.Context(0) as ctx:
        for v in variants:
            env = dict(kv.split("=") for kv in v.split(",") if kv)
            os.environ.update(env)
            op, _ = P.jacobi_scale(A, ctx)
            xt = P.random_uniform_vector(n, 1, ctx=ctx)
            y = op.apply(xt)
            ctx.synchronize()
            reps = 20
            ctx.timer_start()
            for _ in range(reps):
                pcgx._check(pcgx.lib().pcgx_operator_apply_device(ctx.h, op.h, xt.ptr, y.ptr), ctx.h)
            ms = ctx.timer_stop() / reps
            spmv_b = 12.0 * nnz + 4.0 * (n + 1) + 16.0 * n
            prec = P.ChebyshevPreconditioner(P.cheb_params(0.01, 2.0, 20, 1.001))
            _, rep = P.pcg_solve(op, y, P.SolveOptions(maxit=1, flags=pcgx.FLAG_TIME_KERNELS), prec)
            st = rep.step_ms / max(rep.step_launches, 1)
            print(json.dumps({"env": env, "n": n, "nnz": nnz, "spmv_ms": round(ms, 4),
                              "spmv_GBps": round(spmv_b / ms / 1e6, 1), "step_ms": round(st, 4),
                              "step_GBps": round(rep.step_bytes / st / 1e6, 1)}), flush=True)
            for k in env:
                del os.environ[k]
            op.close()


if __name__ == "__main__":
    main()
