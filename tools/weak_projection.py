# SPDX-License-Identifier: Apache-2.0
"""Weak-scaling PROJECTION from one GPU (no multi-GPU node was available): for P = 1,
2, 4, 8 the global cfg5w problem 512 x 512 x (512 P), k = 40, is solved to 1e-8 as a
SINGLE domain on one B200 (it fits: 1.07e9 unknowns x 11 vectors = 94 GB at P = 8),
which gives the iteration counts the P-rank job will take (iterations grow with the
condition number); a middle rank's per-iteration time on its 512^3 slab comes from
the loopback context (tools/slab_overhead.py: the whole slab code path, no link).
projected time(P) = iterations(P) x ms_per_iter(middle rank); the NVLink transfer
(overlapped with the interior launches) and two small all-reduces per iteration are
NOT in it.   python tools/weak_projection.py [PMAX]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_01440_b200 as P  # noqa: E402

NX = NY = NZL = 512
K = 40


def solve_single(nz):
    with P.Context(0) as ctx:
        op, _ = P.jacobi_scale(P.StencilOperator(NX, NY, nz), ctx)
        n = op.local_size()
        a, b = P.analytic_extremes_box(NX, NY, nz)
        xt = P.random_uniform_vector(n, 20240801, ctx=ctx)
        rhs = op.apply(xt)
        del xt
        prec = P.ChebyshevPreconditioner(P.cheb_params(a, b, K, 1.001))
        x = P.DeviceVector(ctx, n)
        best = None
        for _ in range(2):
            _, rep = P.pcg_solve(op, rhs, P.SolveOptions(tol=1e-8, maxit=100000), prec, x_out=x)
            best = rep.wall_time if best is None else min(best, rep.wall_time)
        op.close()
        return rep.iters, best, rep.rel_res, rep.true_rel_res


def middle_rank_ms(iters=12):
    with P.Context(0, nranks=3, rank=1, loopback=True) as ctx:
        op, _ = P.jacobi_scale(P.StencilOperator(NX, NY, 3 * NZL), ctx)
        nl = op.local_size()
        a, b = P.analytic_extremes_box(NX, NY, 3 * NZL)
        rhs = op.apply(P.random_uniform_vector(nl, 20240801, ctx=ctx, offset=op.row0()))
        prec = P.ChebyshevPreconditioner(P.cheb_params(a, b, K, 1.001))
        x = P.DeviceVector(ctx, nl)
        ts = []
        for i in range(4):
            _, rep = P.pcg_solve(op, rhs, P.SolveOptions(tol=1e-30, maxit=iters), prec, x_out=x)
            if i:
                ts.append(rep.wall_time / rep.iters)
        op.close()
        return sorted(ts)[1] * 1e3


def main():
    pmax = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    mid = middle_rank_ms()
    rows = []
    for p in (1, 2, 4, 8):
        if p > pmax:
            break
        it, t, rr, tr = solve_single(NZL * p)
        rows.append({"P": p, "grid": [NX, NY, NZL * p], "unknowns": NX * NY * NZL * p, "iterations": it,
                     "single_domain_one_gpu_s": round(t, 4), "rel_res": rr, "true_rel_res": tr})
        print(json.dumps(rows[-1]), flush=True)
    t1 = rows[0]["single_domain_one_gpu_s"]
    ms1 = t1 / rows[0]["iterations"] * 1e3
    for r in rows:
        if r["P"] == 1:
            r["projected_s"] = t1
        else:
            r["projected_s"] = round(r["iterations"] * mid / 1e3 * (t1 / (rows[0]["iterations"] * ms1 / 1e3)), 4)
        r["weak_efficiency_time_to_1e8"] = round(t1 / r["projected_s"], 4)
        r["weak_efficiency_per_iteration"] = 1.0 if r["P"] == 1 else round(ms1 / mid, 4)
    print(json.dumps({"k": K, "slab_per_rank": [NX, NY, NZL], "ms_per_iter_single_512": round(ms1, 4),
                      "ms_per_iter_middle_rank_loopback": round(mid, 4), "rows": rows,
                      "note": "projection: iterations from single-domain solves of the global problem on one GPU, "
                              "per-iteration time from a loopback middle rank; link transfer and all-reduce "
                              "latency not included"}))


if __name__ == "__main__":
    main()
