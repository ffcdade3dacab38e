# SPDX-License-Identifier: Apache-2.0
"""The multi-rank z-slab path on ONE GPU: P ranks as P contexts of a
pcgx_local_group (one host thread each; halo planes by stream-ordered copies,
scalars reduced in rank order). Everything but the NCCL calls themselves runs:
slab partition, ghost planes, interior/boundary split with accumulated
reductions, merged [r'r, r'z] all-reduce, per-rank RNG offsets.

Elementwise work is exact, so SpMV and every Chebyshev step must be BITWISE equal
to the single-domain oracle; the solve must match within the PCG parity bar."""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from oracle.oracle import OracleOp
from tests._util import rel_norm

pytestmark = pytest.mark.gpu
SEED = 20240801


def run_ranks(P, fn):
    with ThreadPoolExecutor(max_workers=len(P)) as ex:
        futs = [ex.submit(fn, r, c) for r, c in enumerate(P)]
        return [f.result(timeout=600) for f in futs]


@pytest.mark.parametrize("nranks,dims,m", [(2, (24, 24, 24), 10), (3, (20, 16, 26), 5),
                                           (4, (32, 32, 30), 20), (4, (30, 30, 4), 3),
                                           # the 8-GPU layouts: even slabs, uneven slabs, m = 0
                                           (8, (64, 40, 48), 20), (8, (66, 20, 17), 7),
                                           (8, (32, 32, 40), 0)])
def test_slab_solve_matches_single_domain(pcgx, oracle, nranks, dims, m):
    P = pcgx
    nx, ny, nz = dims
    ctxs = P.Context.local_group(nranks)
    a, b = P.analytic_extremes_box(nx, ny, nz)
    opo = OracleOp("lap3d", nx=nx, ny=ny, nz=nz)
    xt_full = oracle.random_uniform(nx * ny * nz, SEED)
    b_full = oracle.apply(opo, xt_full)
    prm_o = oracle.cheb_params(a, b, m, 1.001)
    x_full, rep_o = oracle.pcg_solve(opo, prm_o, b_full)
    r_full = oracle.random_uniform(nx * ny * nz, 77)
    z_full = oracle.apply_chebyshev(opo, prm_o, r_full)

    def rank(r, ctx):
        op, _ = P.jacobi_scale(P.StencilOperator(nx, ny, nz), ctx)
        z0 = op.z0()
        nl = op.local_size()
        assert (z0, nl // (nx * ny)) == P.slab_partition(nz, nranks, r)
        lo, hi = z0 * nx * ny, z0 * nx * ny + nl
        xt = P.random_uniform_vector(nl, SEED, offset=lo)
        bl = op.apply(xt)                                  # halo exchange inside
        zl = P.apply_chebyshev(P.cheb_params(a, b, m, 1.001), op, r_full[lo:hi])
        x, rep = P.pcg_solve(op, bl, P.SolveOptions(),
                             P.ChebyshevPreconditioner(P.cheb_params(a, b, m, 1.001)))
        return lo, hi, bl, zl, x, rep

    outs = run_ranks(ctxs, rank)
    b_g = np.concatenate([o[2] for o in outs])
    z_g = np.concatenate([o[3] for o in outs])
    x_g = np.concatenate([o[4] for o in outs])
    assert np.array_equal(b_g, b_full)          # SpMV across slabs: bitwise
    assert np.array_equal(z_g, z_full)          # P_m(A) r across slabs: bitwise
    reps = [o[5] for o in outs]
    assert all(r.iters == reps[0].iters for r in reps)
    assert abs(reps[0].iters - rep_o["iters"]) <= 1
    assert reps[0].converged
    if reps[0].iters == rep_o["iters"]:
        assert rel_norm(x_g, x_full) <= 1e-10
    assert reps[0].ddot == rep_o["ddot"] and reps[0].matvec == rep_o["matvec"]
    # two all-reduces per iteration (+ setup/exit ones), halos on every SpMV
    assert reps[0].allreduces <= 2 * reps[0].iters + 4
    assert all(r.halo_bytes > 0 for r in reps)
    for c in ctxs:
        c.close()


def test_slab_lanczos_matches_single_domain(pcgx):
    P = pcgx
    nx, nz = 20, 22
    single = P.Context(0)
    op1, _ = P.jacobi_scale(P.StencilOperator(nx, nx, nz), single)
    lo1, hi1 = P.lanczos_bounds(op1, 20, 30, SEED)
    ctxs = P.Context.local_group(2)

    def rank(r, ctx):
        op, _ = P.jacobi_scale(P.StencilOperator(nx, nx, nz), ctx)
        return P.lanczos_bounds(op, 20, 30, SEED)

    res = run_ranks(ctxs, rank)
    for lo, hi in res:
        assert lo == pytest.approx(lo1, rel=1e-9) and hi == pytest.approx(hi1, rel=1e-9)
    for c in ctxs:
        c.close()
    single.close()


@pytest.mark.parametrize("nranks,gen,m", [(2, "fe27", 6), (3, "elast27", 4), (4, "lap", 5), (4, "fe27_3", 4),
                                          (3, "fe27_odd", 5)])
def test_csr_block_rows_match_single_domain(pcgx, oracle, nranks, gen, m):
    """Multi-rank CSR (block rows + per-neighbour halo; SELL-32, or BSR-3 for the 3 x 3
    block matrix): SpMV and P_m(A) r bitwise equal to the single-domain oracle, the
    solve within the PCG bar."""
    P = pcgx
    nxg = {"fe27": 10, "fe27_3": 3, "fe27_odd": 7}.get(gen)
    if nxg:  # fe27_3: fewer node planes than ranks -> row blocks (SELL); fe27_odd: ragged slabs
        A = P.gen_fe27(nxg, 1.0, SEED)
    elif gen == "elast27":
        A = P.gen_elast27(6, 1.0, 0.5, 0.1, SEED)
    else:
        from tests._util import lap3d_csr
        rp, ci, va = lap3d_csr(11)
        A = P.CsrMatrix(11 ** 3, rp, ci, va)
    n = A.n
    opo = OracleOp("csr", row_ptr=A.row_ptr, col_idx=A.col_idx, values=A.values)
    a, b = 0.005, 2.5
    xt_full = oracle.random_uniform(n, SEED)
    b_full = oracle.apply(opo, xt_full)
    prm_o = oracle.cheb_params(a, b, m, 1.001)
    x_full, rep_o = oracle.pcg_solve(opo, prm_o, b_full)
    r_full = oracle.random_uniform(n, 77)
    z_full = oracle.apply_chebyshev(opo, prm_o, r_full)
    ctxs = P.Context.local_group(nranks)

    def rank(r, ctx):
        op, _ = P.jacobi_scale(A, ctx)
        lo = op.row0()
        hi = lo + op.local_size()
        if gen == "elast27":  # 3 x 3 blocks: whole block rows per rank, BSR-3 kept
            z0, nb = P.slab_partition(n // 3, nranks, r)
            assert (lo, op.local_size()) == (3 * z0, 3 * nb) and op.storage() == "bsr3"
        elif gen in ("fe27", "fe27_odd"):  # 27-point box on an nx^3 grid: node-plane slabs, grid-tile offsets
            z0, nzl = P.slab_partition(nxg, nranks, r)
            assert (lo, op.local_size()) == (nxg * nxg * z0, nxg * nxg * nzl) and op.storage() == "dia_grid"
        else:
            assert (lo, op.local_size()) == P.slab_partition(n, nranks, r)
        bl = op.apply(P.random_uniform_vector(op.local_size(), SEED, offset=lo))
        zl = P.apply_chebyshev(P.cheb_params(a, b, m, 1.001), op, r_full[lo:hi])
        x, rep = P.pcg_solve(op, bl, P.SolveOptions(),
                             P.ChebyshevPreconditioner(P.cheb_params(a, b, m, 1.001)))
        lo2, hi2 = P.lanczos_bounds(op, 10, 15, SEED)
        return bl, zl, x, rep, (lo2, hi2)

    outs = run_ranks(ctxs, rank)
    assert np.array_equal(np.concatenate([o[0] for o in outs]), b_full)
    assert np.array_equal(np.concatenate([o[1] for o in outs]), z_full)
    reps = [o[3] for o in outs]
    assert all(r.iters == reps[0].iters for r in reps) and reps[0].converged
    assert abs(reps[0].iters - rep_o["iters"]) <= 1
    if reps[0].iters == rep_o["iters"]:
        # 27 unknowns (fe27_3): a handful of iterations on a tiny system, where the
        # per-rank reduction order moves x by ~5e-10 relative; the elementwise work
        # above is still bitwise
        tol = 1e-8 if n < 100 else 1e-10
        assert rel_norm(np.concatenate([o[2] for o in outs]), x_full) <= tol
    assert all(r.halo_bytes > 0 for r in reps)
    olo, _, al, be = oracle.lanczos(opo, 15, SEED)
    _, ohi = oracle.tridiag_extremes(al[:10], be[:10])
    for o in outs:
        assert o[4][0] == pytest.approx(olo, rel=1e-8) and o[4][1] == pytest.approx(ohi, rel=1e-8)
    for c in ctxs:
        c.close()


def test_loopback_rank_runs_the_slab_path(pcgx, monkeypatch):
    """pcgx_context_create_loopback (measurement only, tools/slab_overhead.py): a rank of
    a z-slab job whose neighbours are its own opposite planes. The slab it owns with
    periodic ghosts in z is a consistent SPD problem: the scaled SpMV matches a numpy
    periodic stencil, the two-step passes (two ghost planes per side) match the
    single-step path bitwise, and a PCG solve recovers x_true."""
    P = pcgx
    nx, ny, nzl, m = 66, 24, 20, 6
    with P.Context(0, nranks=3, rank=1, loopback=True) as ctx:
        assert (ctx.rank, ctx.nranks) == (1, 3)
        op, _ = P.jacobi_scale(P.StencilOperator(nx, ny, 3 * nzl), ctx)
        assert op.local_size() == nx * ny * nzl and op.row0() == nx * ny * nzl
        xt = P.random_uniform_vector(op.local_size(), SEED, offset=op.row0())
        y = op.apply(xt)
        X = xt.reshape(nzl, ny, nx)
        Y = 6.0 * X - np.roll(X, 1, 0) - np.roll(X, -1, 0)
        Y[:, 1:, :] -= X[:, :-1, :]
        Y[:, :-1, :] -= X[:, 1:, :]
        Y[:, :, 1:] -= X[:, :, :-1]
        Y[:, :, :-1] -= X[:, :, 1:]
        assert np.allclose(y.reshape(nzl, ny, nx), Y / 6.0, rtol=0, atol=1e-14)
        a, b = P.analytic_extremes_box(nx, ny, 3 * nzl)
        prm = P.cheb_params(a, b, m, 1.001)
        r = P.random_uniform_vector(op.local_size(), 7)
        z2 = P.apply_chebyshev(prm, op, r)
        monkeypatch.setenv("PCGX_CHEB2", "0")
        op1, _ = P.jacobi_scale(P.StencilOperator(nx, ny, 3 * nzl), ctx)
        assert np.array_equal(z2, P.apply_chebyshev(prm, op1, r))
        x, rep = P.pcg_solve(op, y, P.SolveOptions(tol=1e-10), P.ChebyshevPreconditioner(prm))
        assert rep.converged and rep.halo_bytes > 0
        assert rel_norm(x, xt) <= 1e-7


@pytest.mark.parametrize("nranks,dims,m", [(3, (66, 24, 22), 6), (4, (64, 44, 17), 5), (2, (130, 20, 9), 12)])
def test_slab_fused_update_matches_update_kernel(pcgx, nranks, dims, m, monkeypatch):
    """z-slab ranks fuse the PCG update r -= alpha q, r'r into the first two-step pass
    of P r (ghost planes of r(it-1) and q(it), r(it)'s ghost plane with the next pass's
    exchange): element operations are the update kernel's, so r and every iterate are
    bitwise equal and only the r'r partial sums differ in their last bits -- same
    iteration counts, x within 1e-12 of the unfused schedule, fewer launches. Uneven
    slabs down to four planes (smaller slabs keep the update kernel)."""
    P = pcgx
    nx, ny, nz = dims
    a, b = P.analytic_extremes_box(nx, ny, nz)
    prm = P.cheb_params(a, b, m, 1.001)

    def solve(flag):
        monkeypatch.setenv("PCGX_FUSE_UPD_SLAB", flag)
        ctxs = P.Context.local_group(nranks)

        def rank(r, ctx):
            op, _ = P.jacobi_scale(P.StencilOperator(nx, ny, nz), ctx)
            xt = P.random_uniform_vector(op.local_size(), SEED, offset=op.row0())
            x, rep = P.pcg_solve(op, op.apply(xt), P.SolveOptions(), P.ChebyshevPreconditioner(prm))
            return x, rep

        outs = run_ranks(ctxs, rank)
        for c in ctxs:
            c.close()
        return np.concatenate([o[0] for o in outs]), outs[0][1]

    xf, rf = solve("1")
    xu, ru = solve("0")
    assert rf.converged and ru.converged and rf.iters == ru.iters
    assert (rf.ddot, rf.matvec) == (ru.ddot, ru.matvec)
    assert rel_norm(xf, xu) <= 1e-12
    assert rf.kernel_launches < ru.kernel_launches


@pytest.mark.parametrize("nranks,m", [(3, 6), (2, 5)])
def test_slab_solve_stopped_by_maxit_matches_oracle(pcgx, oracle, nranks, m):
    """An iteration-limited solve on slab ranks (fused update in P r's first pass,
    the last iteration's update as a kernel of its own, the deferred x update flushed
    at the exit): x and the residuals after exactly maxit iterations match the
    single-domain oracle stopped at the same iteration."""
    P = pcgx
    nx, ny, nz, maxit = 66, 24, 23, 7
    a, b = P.analytic_extremes_box(nx, ny, nz)
    opo = OracleOp("lap3d", nx=nx, ny=ny, nz=nz)
    b_full = oracle.apply(opo, oracle.random_uniform(nx * ny * nz, SEED))
    x_o, rep_o = oracle.pcg_solve(opo, oracle.cheb_params(a, b, m, 1.001), b_full, tol=1e-30, maxit=maxit)
    ctxs = P.Context.local_group(nranks)

    def rank(r, ctx):
        op, _ = P.jacobi_scale(P.StencilOperator(nx, ny, nz), ctx)
        lo = op.row0()
        x, rep = P.pcg_solve(op, b_full[lo:lo + op.local_size()], P.SolveOptions(tol=1e-30, maxit=maxit),
                             P.ChebyshevPreconditioner(P.cheb_params(a, b, m, 1.001)))
        return x, rep

    outs = run_ranks(ctxs, rank)
    for c in ctxs:
        c.close()
    rep = outs[0][1]
    assert rep.iters == maxit == rep_o["iters"] and not rep.converged
    assert (rep.ddot, rep.matvec) == (rep_o["ddot"], rep_o["matvec"])
    assert rel_norm(np.concatenate([o[0] for o in outs]), x_o) <= 1e-11
    assert abs(rep.rel_res - rep_o["rel_res"]) <= 1e-12 * max(1.0, rep_o["rel_res"])
    assert abs(rep.true_rel_res - rep_o["true_rel_res"]) <= 1e-12 * max(1.0, rep_o["true_rel_res"])
