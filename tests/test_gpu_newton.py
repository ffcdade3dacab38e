# SPDX-License-Identifier: Apache-2.0
"""Newton-form preconditioner on the device:
apply_newton (polyprec.cpp:135-160) and pcg_solve with a NewtonPreconditioner
(pcg.hpp:27-40), against the reference's golden outputs and the C oracle.

The device plan fuses every SpMV of the recursion with the element-wise steps
that follow it, but performs the reference's IEEE operations in its order per
element, so every apply is BITWISE the reference's."""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from oracle.oracle import OracleOp
from tests._util import fh, fhs, rel_norm, sha

pytestmark = pytest.mark.gpu
SEED = 20240801


@pytest.fixture(scope="module")
def P(pcgx):
    return pcgx


def stencil(P, ctx, nx, ny=None, nz=None):
    op, _ = P.jacobi_scale(P.StencilOperator(nx, ny, nz), ctx)
    return op


def csr(P, ctx, rp, ci, va):
    op, _ = P.jacobi_scale(P.CsrMatrix(len(rp) - 1, np.asarray(rp), np.asarray(ci),
                                       np.asarray(va)), ctx)
    return op


def test_apply_newton_bitwise_vs_reference(P, ctx, golden):
    g = golden["apply_newton"]
    nx = g["nx"]
    a, b = P.analytic_extremes(3, nx)
    r = P.random_uniform_vector(nx ** 3, g["r_seed"])
    op = stencil(P, ctx, nx)
    for lv in g["levels"]:
        prm = P.newton_params(a, b, lv["nlev"], fh(g["scale"]))
        before = op.matvec_count()
        out = P.apply_newton(prm, op, r)
        assert sha(out) == lv["sha256"], lv["nlev"]
        assert op.matvec_count() - before == 2 ** lv["nlev"] - 1  # exactly 2^nlev - 1 matvecs


@pytest.mark.parametrize("nlev", [0, 1, 2, 3, 4, 5, 6, 7])
def test_apply_newton_all_levels_vs_oracle(P, ctx, oracle, nlev):
    """Every chain shape of the fused plan (SpMV epilogue chains of 1-3 combines,
    the element-wise remainder beyond 3)."""
    nx, ny, nz = 19, 12, 11
    a, b = P.analytic_extremes_box(nx, ny, nz)
    r = oracle.random_uniform(nx * ny * nz, 5)
    prm = P.newton_params(a, b, nlev, 1.001)
    out = P.apply_newton(prm, stencil(P, ctx, nx, ny, nz), r)
    ref = oracle.apply_newton(OracleOp("lap3d", nx=nx, ny=ny, nz=nz), prm.zeta, r)
    assert np.array_equal(out, ref)


def test_apply_newton_csr_and_device_entry(P, ctx, oracle, golden):
    g = golden["csr_apply"]
    rp, ci, va = np.array(g["row_ptr"]), np.array(g["col_idx"]), fhs(g["values"])
    op = csr(P, ctx, rp, ci, va)
    opo = OracleOp("csr", row_ptr=rp, col_idx=ci, values=va)
    r = oracle.random_uniform(len(rp) - 1, 9)
    for nlev in (1, 3, 5):
        prm = P.newton_params(0.05, 1.9, nlev, 1.01)
        ref = oracle.apply_newton(opo, prm.zeta, r)
        assert np.array_equal(P.apply_newton(prm, op, r), ref)
        rd = P.DeviceVector.from_numpy(ctx, r)
        assert np.array_equal(P.apply_newton(prm, op, rd).numpy(), ref)


def test_apply_newton_base_case_and_identity(P, ctx):
    # test_polyprec.cpp:65-86: nlev 0 is zeta0 r; on the identity (scaled diag) with
    # alpha = beta = 1 every level gives r
    op = csr(P, ctx, np.array([0, 1, 2]), np.array([0, 1]), np.array([5.0, 7.0]))
    r = np.array([2.0, -4.0])
    out = P.apply_newton(P.newton_params(2.0, 6.0, 0, 1.0), op, r)
    assert np.array_equal(out, 0.25 * r)
    for nlev in range(1, 5):
        assert np.allclose(P.apply_newton(P.newton_params(1.0, 1.0, nlev, 1.0), op, r), r,
                           rtol=0, atol=1e-14)


def test_newton_equals_chebyshev_on_device(P, ctx):
    # test_polyprec.cpp:112-144
    nx = 12
    a, b = P.analytic_extremes(3, nx)
    op = stencil(P, ctx, nx)
    r = P.random_uniform_vector(nx ** 3, 31)
    for nlev in (1, 3, 5):
        for s in (1.0, 1.01):
            zn = P.apply_newton(P.newton_params(a, b, nlev, s), op, r)
            zc = P.apply_chebyshev(P.cheb_params(a, b, 2 ** nlev - 1, s), op, r)
            assert rel_norm(zc, zn) <= 1e-10


def test_apply_newton_rejects_alias_and_bad_params(P, ctx):
    import ctypes as C
    op = stencil(P, ctx, 6)
    prm = P.newton_params(0.1, 1.9, 2, 1.0)
    rd = P.DeviceVector.from_numpy(ctx, np.ones(216))
    cp = prm._c()
    with pytest.raises(P.InvalidArgument, match="alias"):
        P._check(P.lib().pcgx_newton_apply_device(ctx.h, op.h, C.byref(cp), rd.ptr, rd.ptr), ctx.h)
    with pytest.raises(P.InvalidArgument):
        P.apply_newton(prm, op, np.ones(5))


@pytest.mark.parametrize("tag", ["lap24_n0", "lap24_n3", "lap24_n5"])
def test_pcg_solve_newton_vs_reference(P, ctx, oracle, golden, tag):
    c = next(s for s in golden["pcg_solve_newton"] if s["tag"] == tag)
    nx = c["nx"]
    op = stencil(P, ctx, nx)
    xt = P.random_uniform_vector(nx ** 3, SEED)
    b = op.apply(xt)
    assert sha(b) == c["b_sha256"]
    prm = P.newton_params(fh(c["alpha"]), fh(c["beta"]), c["nlev"], fh(c["scale"]))
    x, rep = P.pcg_solve(op, b, None, P.NewtonPreconditioner(prm))
    g = c["report"]
    assert abs(rep.iters - g["iters"]) <= 1 and rep.converged == bool(g["converged"])
    deg = 2 ** c["nlev"] - 1
    assert rep.ddot == 3 * rep.iters + 2
    assert rep.matvec == rep.iters * (deg + 1) + 1
    assert rep.prec_applies == rep.iters
    xo, ro = oracle.pcg_solve_newton(OracleOp("lap3d", nx=nx), prm.zeta, b)
    assert ro["iters"] == g["iters"] and sha(xo) == c["x_sha256"]  # oracle pinned to the reference
    if rep.iters == ro["iters"]:
        assert rel_norm(x, xo) <= 1e-10
        assert abs(rep.rel_res - ro["rel_res"]) <= 1e-10 * ro["rel_res"]
    # device entry, same answer
    bd = P.DeviceVector.from_numpy(ctx, b)
    xd, rep_d = P.pcg_solve(op, bd, None, P.NewtonPreconditioner(prm))
    assert rep_d.iters == rep.iters and rel_norm(xd.numpy(), x) <= 1e-12


def test_pcg_solve_newton_csr_vs_reference(P, ctx, oracle, golden):
    g = golden["csr_apply"]
    c = next(s for s in golden["pcg_solve_newton"] if s["tag"] == "csr300_n3")
    rp, ci, va = np.array(g["row_ptr"]), np.array(g["col_idx"]), fhs(g["values"])
    op = csr(P, ctx, rp, ci, va)
    b = op.apply(P.random_uniform_vector(len(rp) - 1, SEED))
    assert sha(b) == c["b_sha256"]
    prm = P.newton_params(fh(c["alpha"]), fh(c["beta"]), c["nlev"], fh(c["scale"]))
    x, rep = P.pcg_solve(op, b, None, P.NewtonPreconditioner(prm))
    assert abs(rep.iters - c["report"]["iters"]) <= 1
    xo, ro = oracle.pcg_solve_newton(OracleOp("csr", row_ptr=rp, col_idx=ci, values=va), prm.zeta, b)
    if rep.iters == ro["iters"]:
        assert rel_norm(x, xo) <= 1e-10


def test_newton_slab_ranks_bitwise(pcgx, oracle):
    """z-slab ranks (local group on one GPU): the Newton apply is bitwise the
    single-domain oracle's, the solve within the PCG parity bar."""
    P = pcgx
    nx, ny, nz, nranks, nlev = 20, 18, 23, 3, 3
    ctxs = P.Context.local_group(nranks)
    a, b = P.analytic_extremes_box(nx, ny, nz)
    opo = OracleOp("lap3d", nx=nx, ny=ny, nz=nz)
    prm = P.newton_params(a, b, nlev, 1.001)
    r_full = oracle.random_uniform(nx * ny * nz, 77)
    z_full = oracle.apply_newton(opo, prm.zeta, r_full)
    b_full = oracle.apply(opo, oracle.random_uniform(nx * ny * nz, SEED))
    x_full, rep_o = oracle.pcg_solve_newton(opo, prm.zeta, b_full)

    def rank(rk, ctx):
        op, _ = P.jacobi_scale(P.StencilOperator(nx, ny, nz), ctx)
        lo = op.z0() * nx * ny
        hi = lo + op.local_size()
        zl = P.apply_newton(prm, op, r_full[lo:hi])
        x, rep = P.pcg_solve(op, b_full[lo:hi], None, P.NewtonPreconditioner(prm))
        return zl, x, rep

    with ThreadPoolExecutor(max_workers=nranks) as ex:
        outs = [f.result(timeout=600) for f in [ex.submit(rank, r, c) for r, c in enumerate(ctxs)]]
    assert np.array_equal(np.concatenate([o[0] for o in outs]), z_full)
    x_g = np.concatenate([o[1] for o in outs])
    rep = outs[0][2]
    assert abs(rep.iters - rep_o["iters"]) <= 1
    if rep.iters == rep_o["iters"]:
        assert rel_norm(x_g, x_full) <= 1e-10
    for c in ctxs:
        c.close()
