"""One k-degree Chebyshev-PCG solve at NX^3 after a warm-up solve (profiling aid).

    python tools/solve_timeline.py [NX] [K]      (K < 0: Newton form, nlev = -K)
Prints the device-timed solve; run under
    ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none
to get the warm-cache per-launch times of the same solve (the last solve's launches).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_01440_b200 as P  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 320
k = int(sys.argv[2]) if len(sys.argv) > 2 else 20
with P.Context(0) as ctx:
    op, _ = P.jacobi_scale(P.StencilOperator(nx), ctx)
    a, b = P.analytic_extremes(3, nx)
    rhs = op.apply(P.random_uniform_vector(nx ** 3, 20240801, ctx=ctx))
    prec = (P.NewtonPreconditioner(P.newton_params(a, b, -k, 1.001)) if k < 0 else
            P.ChebyshevPreconditioner(P.cheb_params(a, b, k, 1.001)))
    x = P.DeviceVector(ctx, nx ** 3)
    for i in range(3):
        l0 = ctx.kernel_launches
        _, rep = P.pcg_solve(op, rhs, None, prec, x_out=x)
        print(f"solve {i}: {rep.wall_time * 1e3:.3f} ms, iters {rep.iters}, launches "
              f"{ctx.kernel_launches - l0}, alg {rep.alg_bytes / rep.wall_time / 1e9:.0f} GB/s", flush=True)
