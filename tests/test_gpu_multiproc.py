# SPDX-License-Identifier: Apache-2.0
"""The multi-rank algorithm across PROCESSES on one GPU: P Python processes, one
pcgx context each (pcgx_context_create_host: halo planes, block-row segments and
scalars through a POSIX shared-memory segment, host-staged; or
pcgx_context_create_ipc: CUDA-IPC device mailboxes, stream-ordered by IPC events
-- in neither does a kernel wait on another rank, so ranks sharing one GPU cannot
deadlock it). This is the
process layout of a torchrun job; only the transport differs from NCCL.

SpMV and every Chebyshev step are elementwise exact across slabs / row blocks,
so b and P_m(A) r must be BITWISE the single-domain oracle's; the solve matches
within the PCG parity bar (its reductions are per-rank trees summed in rank order)."""
import json
import os
import subprocess
import sys
import uuid

import numpy as np
import pytest

from oracle.oracle import OracleOp
from tests._util import rel_norm

pytestmark = pytest.mark.gpu
SEED = 20240801
HERE = os.path.dirname(os.path.abspath(__file__))


def run_job(nranks, kind, dims, m, tmp_path, comm="host"):
    name = f"pcgx_test_{uuid.uuid4().hex[:12]}"
    env = dict(os.environ, PCGX_MP_COMM=comm)
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "mp_worker.py"), name, str(nranks), str(r),
                               str(tmp_path), kind, *map(str, dims), str(m)],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True, env=env)
             for r in range(nranks)]
    outs = []
    for p in procs:
        try:
            o, _ = p.communicate(timeout=600)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        outs.append((p.returncode, o))
    for rc, o in outs:
        assert rc == 0, o
    res = [np.load(os.path.join(tmp_path, f"rank{r}.npz")) for r in range(nranks)]
    return res


@pytest.mark.parametrize("comm", ["host", "ipc"])
@pytest.mark.parametrize("nranks,dims,m", [(2, (24, 24, 24), 10), (3, (20, 16, 26), 5), (2, (64, 40, 33), 20)])
def test_multiprocess_slabs_match_single_domain(pcgx, oracle, nranks, dims, m, comm, tmp_path):
    P = pcgx
    nx, ny, nz = dims
    res = run_job(nranks, "stencil", dims, m, tmp_path, comm)
    a, b = P.analytic_extremes_box(nx, ny, nz)
    opo = OracleOp("lap3d", nx=nx, ny=ny, nz=nz)
    xt = oracle.random_uniform(nx * ny * nz, SEED)
    b_full = oracle.apply(opo, xt)
    prm = oracle.cheb_params(a, b, m, 1.001)
    z_full = oracle.apply_chebyshev(opo, prm, oracle.random_uniform(nx * ny * nz, 77))
    x_full, rep_o = oracle.pcg_solve(opo, prm, b_full)
    assert np.array_equal(np.concatenate([r["b"] for r in res]), b_full)
    assert np.array_equal(np.concatenate([r["z"] for r in res]), z_full)
    reps = [json.loads(str(r["rep"])) for r in res]
    assert all(r["iters"] == reps[0]["iters"] for r in reps)
    assert reps[0]["converged"] and abs(reps[0]["iters"] - rep_o["iters"]) <= 1
    assert reps[0]["ddot"] == rep_o["ddot"] and reps[0]["matvec"] == rep_o["matvec"]
    if reps[0]["iters"] == rep_o["iters"]:
        assert rel_norm(np.concatenate([r["x"] for r in res]), x_full) <= 1e-10
    assert all(r["halo_bytes"] > 0 for r in reps)


@pytest.mark.parametrize("comm", ["host", "ipc"])
def test_multiprocess_slabs_match_local_group(pcgx, comm, tmp_path):
    """Processes + shared memory (or CUDA-IPC device mailboxes) and threads +
    stream-ordered copies run the same algorithm with scalars summed in rank order:
    the solutions are bit-identical."""
    P = pcgx
    nx, ny, nz, m = 24, 20, 30, 8
    res = run_job(3, "stencil", (nx, ny, nz), m, tmp_path, comm)
    ctxs = P.Context.local_group(3)
    from concurrent.futures import ThreadPoolExecutor
    a, b = P.analytic_extremes_box(nx, ny, nz)

    def rank(r, ctx):
        op, _ = P.jacobi_scale(P.StencilOperator(nx, ny, nz), ctx)
        xt = P.random_uniform_vector(op.local_size(), SEED, offset=op.row0())
        x, rep = P.pcg_solve(op, op.apply(xt), P.SolveOptions(),
                             P.ChebyshevPreconditioner(P.cheb_params(a, b, m, 1.001)))
        return x, rep

    with ThreadPoolExecutor(3) as ex:
        outs = [f.result(timeout=600) for f in [ex.submit(rank, r, c) for r, c in enumerate(ctxs)]]
    assert np.array_equal(np.concatenate([o[0] for o in outs]), np.concatenate([r["x"] for r in res]))
    assert outs[0][1].iters == json.loads(str(res[0]["rep"]))["iters"]
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("kind,nranks,comm", [("fe27", 2, "host"), ("fe27_local", 2, "host"),
                                              ("fe27_local", 3, "host"), ("elast27", 2, "host"),
                                              ("elast27", 3, "host"), ("fe27", 3, "ipc"),
                                              ("fe27_local", 3, "ipc"), ("elast27", 2, "ipc"),
                                              ("fe27_planes", 3, "host"), ("fe27_planes", 2, "ipc"),
                                              ("elast27_local", 2, "host"), ("elast27_local", 3, "ipc")])
def test_multiprocess_block_rows_match_single_domain(pcgx, oracle, kind, nranks, comm, tmp_path):
    """CSR block rows (the paper's distributed SpMV) across
    processes: per-neighbour packed halos through the shared segment; every rank
    given the full matrix ("fe27") or only its own rows ("fe27_local",
    pcgx_csr_create_local: lists from the symmetric pattern, ghost Jacobi values
    exchanged once). Local rows cut at whole node planes ("fe27_planes") keep the
    offset storage, at whole 3 x 3 block rows ("elast27_local") BSR-3 -- partitions
    that differ from the balanced rows at these sizes."""
    P = pcgx
    nx, m = (14, 6) if kind.startswith("fe27") else ((7, 6) if kind == "elast27_local" else (8, 6))
    res = run_job(nranks, kind, (nx, nx, nx), m, tmp_path, comm)
    if kind.startswith("elast27"):
        assert all(str(r["storage"]) == "bsr3" for r in res)
    if kind in ("fe27", "fe27_planes"):
        assert all(str(r["storage"]) == "dia_grid" for r in res)
    if kind == "fe27_local":  # 14 planes: two ranks' balanced rows ARE whole planes, three ranks' are not
        assert all(str(r["storage"]) == ("dia_grid" if nranks == 2 else "sell32") for r in res)
    A = P.gen_fe27(nx, 1.0, SEED) if kind.startswith("fe27") else P.gen_elast27(nx, 1.0, 0.5, 0.1, SEED)
    opo = OracleOp("csr", row_ptr=A.row_ptr, col_idx=A.col_idx, values=A.values)
    xt = oracle.random_uniform(A.n, SEED)
    b_full = oracle.apply(opo, xt)
    prm = oracle.cheb_params(*((0.01, 2.5) if kind.startswith("fe27") else (0.005, 3.2)), m, 1.001)
    z_full = oracle.apply_chebyshev(opo, prm, oracle.random_uniform(A.n, 77))
    assert np.array_equal(np.concatenate([r["b"] for r in res]), b_full)
    assert np.array_equal(np.concatenate([r["z"] for r in res]), z_full)
    x_full, rep_o = oracle.pcg_solve(opo, prm, b_full)
    rep = json.loads(str(res[0]["rep"]))
    assert rep["converged"] and abs(rep["iters"] - rep_o["iters"]) <= 1


def test_multiprocess_local_rows_reject_asymmetric_pattern(pcgx, tmp_path):
    """pcgx_csr_create_local derives its halo lists from the symmetric pattern; a
    pattern that is not symmetric across ranks is caught on EVERY rank before any
    point-to-point exchange (InvalidArgument naming the ranks), instead of a hang.
    (13 planes: the balanced rows are not whole planes, so the rows go through the
    packed per-neighbour exchange; plane-aligned rows take the plane exchange, whose
    messages do not depend on the pattern.)"""
    name = f"pcgx_test_{uuid.uuid4().hex[:12]}"
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "mp_worker.py"), name, "2", str(r),
                               str(tmp_path), "fe27_local_asym", "13", "13", "13", "4"],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(2)]
    for p in procs:
        out, _ = p.communicate(timeout=600)
        assert p.returncode == 0, out
    for r in range(2):
        msg = open(os.path.join(tmp_path, f"rank{r}.err")).read()
        assert "block rows are not symmetric" in msg, msg


@pytest.mark.parametrize("comm", ["host", "ipc"])
def test_multiprocess_small_mailbox_fails_every_rank_fast(pcgx, comm, tmp_path):
    """A halo plane larger than the mailbox: the rank that finds out marks the job
    aborted, so EVERY rank fails promptly (no rank waits out the barrier timeout)."""
    import time
    name = f"pcgx_test_{uuid.uuid4().hex[:12]}"
    env = dict(os.environ, PCGX_MP_COMM=comm, PCGX_MP_MAILBOX="4096")
    t0 = time.time()
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "mp_worker.py"), name, "2", str(r),
                               str(tmp_path), "stencil", "40", "40", "12", "4"],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True, env=env)
             for r in range(2)]
    outs = [p.communicate(timeout=300)[0] for p in procs]
    assert time.time() - t0 < 240
    for p, o in zip(procs, outs):
        assert p.returncode != 0, o
        assert "mailbox" in o or "gave up" in o, o
