# SPDX-License-Identifier: Apache-2.0
"""The z-slab code path's own overhead on ONE GPU (no link): a rank with two
neighbours (pcgx_context_create_loopback: ghost planes = its own opposite boundary
planes, copied with the real exchange's sizes on the comm stream) against the same
slab as a single domain. Same grid per GPU, same degree, a fixed number of PCG
iterations; prints ms per iteration for both and their ratio -- what weak scaling
keeps of a rank's throughput before the NVLink transfer itself (which the interior
launches overlap) and the all-reduce latency.

    python tools/slab_overhead.py [NX NY NZ_LOCAL] [K] [ITERS]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_01440_b200 as P  # noqa: E402


def run(ctx, nx, ny, nz_global, k, iters, reps=3):
    op, _ = P.jacobi_scale(P.StencilOperator(nx, ny, nz_global), ctx)
    nl = op.local_size()
    a, b = P.analytic_extremes_box(nx, ny, nz_global)
    xt = P.random_uniform_vector(nl, 20240801, ctx=ctx, offset=op.row0())
    rhs = op.apply(xt)
    prec = P.ChebyshevPreconditioner(P.cheb_params(a, b, k, 1.001))
    x = P.DeviceVector(ctx, nl)
    ts = []
    for i in range(reps + 1):
        _, rep = P.pcg_solve(op, rhs, P.SolveOptions(tol=1e-30, maxit=iters), prec, x_out=x)
        if i:
            ts.append(rep.wall_time / rep.iters)
    op.close()
    return sorted(ts)[len(ts) // 2] * 1e3, rep.halo_bytes, rep.kernel_launches


def main():
    a = [int(v) for v in sys.argv[1:]]
    nx, ny, nzl = (a[0], a[1], a[2]) if len(a) >= 3 else (512, 512, 512)
    k = a[3] if len(a) >= 4 else 40
    iters = a[4] if len(a) >= 5 else 12
    with P.Context(0) as ctx:
        single, _, l1 = run(ctx, nx, ny, nzl, k, iters)
    with P.Context(0, nranks=3, rank=1, loopback=True) as ctx:
        slab, halo, l2 = run(ctx, nx, ny, 3 * nzl, k, iters)
    print(json.dumps({"grid_per_rank": [nx, ny, nzl], "k": k, "iters": iters,
                      "ms_per_iter_single_domain": round(single, 4),
                      "ms_per_iter_middle_rank_loopback": round(slab, 4),
                      "slab_path_efficiency": round(single / slab, 4),
                      "halo_bytes_per_solve": halo, "launches_per_solve": [l1, l2],
                      "note": "loopback: the rank's neighbours are its own opposite planes (device copies of "
                              "the real exchange's sizes), all-reduces keep the local value; no link time"}))


if __name__ == "__main__":
    main()
