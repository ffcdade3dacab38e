# SPDX-License-Identifier: Apache-2.0
"""Strong-scaling PROJECTION of cfg5s (640^3, k = 40) from one GPU: the global problem
is the same at every P (28 iterations, tests/golden/full/cfg5s_k40.json), so the
projected speed-up is the single domain's per-iteration time over a middle rank's on
its 640 x 640 x (640 / P) slab (loopback context: the whole slab code path, no link
time, no all-reduce latency).   python tools/strong_projection.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_01440_b200 as P  # noqa: E402

NX, K, ITERS = 640, 40, 10


def per_iter(ctx, nz_global):
    op, _ = P.jacobi_scale(P.StencilOperator(NX, NX, nz_global), ctx)
    nl = op.local_size()
    a, b = P.analytic_extremes_box(NX, NX, NX)
    rhs = op.apply(P.random_uniform_vector(nl, 20240801, ctx=ctx, offset=op.row0()))
    prec = P.ChebyshevPreconditioner(P.cheb_params(a, b, K, 1.001))
    x = P.DeviceVector(ctx, nl)
    ts = []
    for i in range(4):
        _, rep = P.pcg_solve(op, rhs, P.SolveOptions(tol=1e-30, maxit=ITERS), prec, x_out=x)
        if i:
            ts.append(rep.wall_time / rep.iters)
    op.close()
    return sorted(ts)[1] * 1e3


def main():
    with P.Context(0) as ctx:
        t1 = per_iter(ctx, NX)
    rows = [{"P": 1, "slab": [NX, NX, NX], "ms_per_iter": round(t1, 4), "speedup": 1.0, "efficiency": 1.0}]
    for p in (2, 4, 8):
        nzl = NX // p
        with P.Context(0, nranks=3, rank=1, loopback=True) as ctx:
            tp = per_iter(ctx, 3 * nzl)
        rows.append({"P": p, "slab": [NX, NX, nzl], "ms_per_iter": round(tp, 4), "speedup": round(t1 / tp, 3),
                     "efficiency": round(t1 / tp / p, 4)})
    print(json.dumps({"config": "cfg5s 640^3 k=40", "rows": rows,
                      "note": "projection: a middle rank (two neighbours) on the loopback context; link transfer "
                              "and all-reduce latency not included"}))


if __name__ == "__main__":
    main()
