# SPDX-License-Identifier: Apache-2.0
"""Minimal driver for ncu captures of the Chebyshev passes: apply_chebyshev of
degree m on the 320^3 scaled Laplacian, `reps` times (device buffers).

    ncu ... python tools/prof_cheb.py [m] [reps] [nx]
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_01440_b200 as P  # noqa: E402
from paper_2008_01440_b200 import pcgx  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 40
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
nx = int(sys.argv[3]) if len(sys.argv) > 3 else 320
with P.Context(0) as ctx:
    op, _ = P.jacobi_scale(P.StencilOperator(nx), ctx)
    n = op.local_size()
    a, b = P.analytic_extremes(3, nx)
    cp = P.cheb_params(a, b, m, 1.001)._c()
    r = P.random_uniform_vector(n, 1, ctx=ctx)
    out = P.DeviceVector(ctx, n)
    L = pcgx.lib()
    for _ in range(reps):
        pcgx._check(L.pcgx_cheb_apply_device(ctx.h, op.h, C.byref(cp), r.ptr, out.ptr), ctx.h)
    ctx.synchronize()
    print("ok", ctx.kernel_launches)
