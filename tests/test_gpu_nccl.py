# SPDX-License-Identifier: Apache-2.0
"""The NCCL communicator path on one GPU: a 1-rank dist context with
PCGX_FORCE_NCCL=1 routes every all-reduce through NCCL (loaded at run time from
the process's libnccl.so.2), launched directly (the multi-rank default) or inside
the per-iteration CUDA graphs (PCGX_GRAPH_MULTI=1), with the
multi-GPU schedule (PCGX_MERGED=1: merged [r'r, r'z] all-reduce, scalar snapshot
taken by an external event node inside the graph)."""
import numpy as np
import pytest

from oracle.oracle import OracleOp
from tests._util import rel_norm

pytestmark = pytest.mark.gpu
SEED = 20240801


@pytest.mark.parametrize("graphs", ["0", "1"])
@pytest.mark.parametrize("m", [-1, 0, 4, 10])
def test_nccl_one_rank_solve(pcgx, oracle, m, graphs, monkeypatch):
    P = pcgx
    monkeypatch.setenv("PCGX_FORCE_NCCL", "1")
    monkeypatch.setenv("PCGX_MERGED", "1")
    monkeypatch.setenv("PCGX_GRAPH_MULTI", graphs)  # multi-rank default: direct launches
    nid = P.Context.nccl_unique_id()
    with P.Context(0, nranks=1, rank=0, nccl_id=nid, dist=True) as ctx:
        assert ctx.nranks == 1
        nx = 24
        op, _ = P.jacobi_scale(P.StencilOperator(nx), ctx)
        a, b = P.analytic_extremes(3, nx)
        rhs = op.apply(P.random_uniform_vector(nx ** 3, SEED))
        prec = None if m < 0 else P.ChebyshevPreconditioner(P.cheb_params(a, b, m, 1.001))
        x, rep = P.pcg_solve(op, P.DeviceVector.from_numpy(ctx, rhs), None, prec)
        x = x.numpy()
        po = None if m < 0 else oracle.cheb_params(a, b, m, 1.001)
        xo, ro = oracle.pcg_solve(OracleOp("lap3d", nx=nx), po, rhs)
        assert rep.allreduces >= 2 * rep.iters
        assert rep.converged and abs(rep.iters - ro["iters"]) <= 1
        if rep.iters == ro["iters"]:
            assert rel_norm(x, xo) <= 1e-10
