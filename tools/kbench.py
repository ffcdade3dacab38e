# SPDX-License-Identifier: Apache-2.0
"""Kernel micro-benchmark: the fused Chebyshev step and the plain SpMV of the
7-point stencil at 320^3 under launch-shape variants (env knobs read at
operator creation). CUDA-event timed on the library's compute stream.

    python tools/kbench.py [nx] [variant ...]   variant = "kz=16,scalar=0"
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2008_01440_b200 as P  # noqa: E402
from paper_2008_01440_b200 import pcgx  # noqa: E402


def run(ctx, nx, env, reps=30):
    for k, v in env.items():
        os.environ[k] = str(v)
    op, _ = P.jacobi_scale(P.StencilOperator(nx), ctx)
    n = op.local_size()
    a, b = P.analytic_extremes(3, nx)
    xt = P.random_uniform_vector(n, 1, ctx=ctx)
    rhs = op.apply(xt)
    y = op.apply(rhs)
    ctx.synchronize()
    ctx.timer_start()
    for _ in range(reps):
        pcgx._check(pcgx.lib().pcgx_operator_apply_device(ctx.h, op.h, rhs.ptr, y.ptr), ctx.h)
    spmv_ms = ctx.timer_stop() / reps
    prec = P.ChebyshevPreconditioner(P.cheb_params(a, b, 20, 1.001))
    _, rep = P.pcg_solve(op, rhs, P.SolveOptions(maxit=1, flags=pcgx.FLAG_TIME_KERNELS), prec)
    step_ms = rep.step_ms / rep.step_launches
    _, rep2 = P.pcg_solve(op, rhs, P.SolveOptions(), prec)
    for k in env:
        del os.environ[k]
    out = {"env": env, "spmv_GBps": round(16 * n / spmv_ms / 1e6, 1),
           "step_GBps": round(32 * n / step_ms / 1e6, 1), "step_ms": round(step_ms, 4),
           "solve_k20_s": round(rep2.wall_time, 4), "iters": rep2.iters,
           "solve_alg_GBps": round(rep2.alg_bytes / rep2.wall_time / 1e9, 1)}
    op.close()
    return out


def main():
    nx = int(sys.argv[1]) if len(sys.argv) > 1 else 320
    variants = sys.argv[2:] or ["kz=16,scalar=1", "kz=16,scalar=0", "kz=8,scalar=0",
                                "kz=32,scalar=0", "kz=64,scalar=0", "kz=320,scalar=0"]
    with P.Context(0) as ctx:
        for v in variants:
            env = {}
            for kv in v.split(","):
                k, val = kv.split("=")
                env[{"kz": "PCGX_KZ", "pfd": "PCGX_PFD"}.get(k, k)] = val
            print(json.dumps(run(ctx, nx, env)), flush=True)


if __name__ == "__main__":
    main()
