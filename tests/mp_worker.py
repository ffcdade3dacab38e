# SPDX-License-Identifier: Apache-2.0
"""One rank of a multi-PROCESS job on one GPU (tests/test_gpu_multiproc.py):
pcgx_context_create_host -- halo planes, block-row segments and scalars through a
shared-memory segment -- or, with PCGX_MP_COMM=ipc, pcgx_context_create_ipc
(CUDA-IPC device mailboxes ordered by IPC events); no kernel waits on another rank. Writes its slab /
block of b = A x_true, P_m(A) r, the solution and the report to OUT/rank<r>.npz.

    python tests/mp_worker.py NAME NRANKS RANK OUT KIND NX NY NZ M
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SEED = 20240801


def main():
    name, nranks, rank, out, kind = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5]
    nx, ny, nz, m = (int(v) for v in sys.argv[6:10])
    from paper_2008_01440_b200 import pcgx as P
    mb = int(os.environ.get("PCGX_MP_MAILBOX", "0"))  # bytes per message (0: the library default)
    if os.environ.get("PCGX_MP_COMM", "host") == "ipc":  # CUDA-IPC device mailboxes
        ctx = P.Context(0, nranks=nranks, rank=rank, ipc_comm=name, mailbox_bytes=mb)
    else:  # host shared memory
        ctx = P.Context(0, nranks=nranks, rank=rank, host_comm=name, mailbox_bytes=mb)
    if kind == "stencil":
        op, _ = P.jacobi_scale(P.StencilOperator(nx, ny, nz), ctx)
        a, b = P.analytic_extremes_box(nx, ny, nz)
        n = nx * ny * nz
    elif kind in ("fe27", "elast27"):
        A = P.gen_fe27(nx, 1.0, SEED) if kind == "fe27" else P.gen_elast27(nx, 1.0, 0.5, 0.1, SEED)
        op, _ = P.jacobi_scale(A, ctx)
        a, b = (0.01, 2.5) if kind == "fe27" else (0.005, 3.2)
        n = A.n
    else:
        # this rank's block of rows only (pcgx_csr_create_local): "fe27_local[_asym]" the
        # balanced rows, "fe27_planes" whole node planes (keeps the offset storage),
        # "elast27_local" whole 3 x 3 block rows (keeps BSR-3)
        if kind == "elast27_local":
            A = P.gen_elast27(nx, 1.0, 0.5, 0.1, SEED)
            b0, nb = P.slab_partition(A.n // 3, nranks, rank)
            r0, nl = 3 * b0, 3 * nb
        else:
            A = P.gen_fe27(nx, 1.0, SEED)
            if kind == "fe27_planes":
                z0, nzl = P.slab_partition(nx, nranks, rank)
                r0, nl = z0 * nx * nx, nzl * nx * nx
            else:
                r0, nl = P.slab_partition(A.n, nranks, rank)
        n = A.n
        lo, hi = int(A.row_ptr[r0]), int(A.row_ptr[r0 + nl])
        rp, ci, va = A.row_ptr[r0:r0 + nl + 1].astype(np.int64), A.col_idx[lo:hi], A.values[lo:hi]
        if kind.endswith("_asym") and rank == 0:
            # drop every coupling of rank 0's rows to rank 1's first row: rank 0 no
            # longer needs that value, rank 1 (whose row still couples back) sends it
            c = r0 + nl
            keep = ci != c
            ck = np.concatenate([[0], np.cumsum(keep)])
            rp = ck[rp - rp[0]].astype(np.int64)
            ci, va = ci[keep], va[keep]
        try:
            op = P.csr_block_rows(ctx, n, rp, ci, va, row0=r0)
        except P.InvalidArgument as e:
            with open(os.path.join(out, f"rank{rank}.err"), "w") as f:
                f.write(str(e))
            ctx.close()
            return
        del A
        a, b = (0.005, 3.2) if kind == "elast27_local" else (0.01, 2.5)
    lo, nl = op.row0(), op.local_size()
    xt = P.random_uniform_vector(nl, SEED, offset=lo)
    bl = op.apply(xt)
    r_full = P.random_uniform_vector(n, 77)
    prm = P.cheb_params(a, b, m, 1.001)
    zl = P.apply_chebyshev(prm, op, r_full[lo:lo + nl])
    x, rep = P.pcg_solve(op, bl, P.SolveOptions(), P.ChebyshevPreconditioner(prm))
    np.savez(os.path.join(out, f"rank{rank}.npz"), lo=lo, b=bl, z=zl, x=x,
             rep=json.dumps({"iters": rep.iters, "ddot": rep.ddot, "matvec": rep.matvec,
                             "converged": bool(rep.converged), "allreduces": rep.allreduces,
                             "halo_bytes": rep.halo_bytes, "rel_res": rep.rel_res,
                             "true_rel_res": rep.true_rel_res}),
             storage=op.storage())
    op.close()
    ctx.close()


if __name__ == "__main__":
    main()
