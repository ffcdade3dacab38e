# SPDX-License-Identifier: Apache-2.0
"""Pins the C oracle (oracle/polycg_oracle.c) against the REFERENCE's own outputs.

tests/golden/reference_golden.json was produced by the reference library itself
(oracle/_ref/libpolycg_ref.so, built from /root/reference/proj/src by
oracle/Makefile) via tests/golden/make_golden.py. Every check here is bitwise
(float.hex / SHA-256 of the float64 bytes) unless stated.
"""
import numpy as np
import pytest

from oracle.oracle import InvalidArgument, NumericalError, OracleOp
from tests._util import fh, fhs, rel_norm, sha

SEED = 20240801


def test_cheb_params_bitwise(oracle, golden):
    for c in golden["cheb_params"]:
        p = oracle.cheb_params(fh(c["alpha"]), fh(c["beta"]), c["m"], fh(c["scale"]))
        assert p["theta"] == fh(c["theta"])
        assert p["delta"] == fh(c["delta"])
        assert p["sigma"] == fh(c["sigma"])
        assert np.array_equal(p["rho"], fhs(c["rho"]))


def test_cheb_params_hand_values(oracle):
    # test_polyprec.cpp:38-46
    p = oracle.cheb_params(1.0, 3.0, 2, 1.0)
    assert (p["theta"], p["delta"], p["sigma"]) == (2.0, 1.0, 2.0)
    assert p["rho"] == pytest.approx([0.5, 2 / 7, 7 / 26], rel=1e-15)


def test_cheb_params_errors(oracle, golden):
    for e in golden["cheb_params_errors"]:
        a, b, m, s = e["args"]
        if e["error"] is None:
            oracle.cheb_params(a, b, m, s)
            continue
        exc = InvalidArgument if e["error"] == "invalid_argument" else NumericalError
        with pytest.raises(exc) as ei:
            oracle.cheb_params(a, b, m, s)
        assert str(ei.value) == e["msg"]


def test_eval_poly_bitwise(oracle, golden):
    g = golden["eval_poly"]
    lams = fhs(g["lams"])
    for key, vals in g["by_m"].items():
        m, s = key.split(":")
        p = oracle.cheb_params(fh(g["alpha"]), fh(g["beta"]), int(m), float(s))
        got = np.array([oracle.eval_poly(p, l) for l in lams])
        assert np.array_equal(got, fhs(vals)), key


def test_newton_params_bitwise(oracle, golden):
    for c in golden["newton_params"]:
        z = oracle.newton_params(fh(c["alpha"]), fh(c["beta"]), c["nlev"], fh(c["scale"]))
        assert np.array_equal(z, fhs(c["zeta"]))


def test_analytic_extremes_bitwise(oracle, golden):
    for c in golden["analytic_extremes"]:
        lo, hi = oracle.analytic_extremes(c["dim"], c["nx"])
        assert lo == fh(c["lo"]) and hi == fh(c["hi"]), c


def test_analytic_extremes_box_matches_cubic(oracle):
    for nx in (5, 100, 320, 512):
        lo, hi = oracle.analytic_extremes(3, nx)
        blo, bhi = oracle.analytic_extremes_box(nx, nx, nx)
        assert blo == pytest.approx(lo, rel=1e-14) and bhi == pytest.approx(hi, rel=1e-14)
    # 512x512x(512P) alpha0
    for P, a0 in ((1, 1.8751e-5), (2, 1.4067e-5), (4, 1.2893e-5), (8, 1.2599e-5)):
        lo, _ = oracle.analytic_extremes_box(512, 512, 512 * P)
        assert lo == pytest.approx(a0, rel=1e-4)


def test_random_uniform_bitwise(oracle, golden):
    g = golden["random_uniform"]
    v = oracle.random_uniform(g["n"], g["seed"])
    assert np.array_equal(v[:64], fhs(g["first"]))
    assert sha(v) == g["sha256"]
    assert sha(oracle.random_uniform(4096, 7)) == g["seed7_sha256_4096"]
    # counter-based: any slab offset reproduces the same elements
    assert np.array_equal(oracle.random_uniform(1000, g["seed"], offset=5000), v[5000:6000])


def test_stencil_apply_bitwise(oracle, golden):
    for c in golden["stencil_apply"]:
        nx = c["nx"]
        x = oracle.random_uniform(nx ** 3, c["x_seed"])
        y = oracle.apply(OracleOp("lap3d", nx=nx), x)
        assert sha(y) == c["sha256"], nx
        if "y" in c:
            assert np.array_equal(y, fhs(c["y"]))


def test_csr_apply_bitwise(oracle, golden):
    g = golden["csr_apply"]
    op = OracleOp("csr", row_ptr=g["row_ptr"], col_idx=g["col_idx"], values=fhs(g["values"]))
    x = oracle.random_uniform(len(g["row_ptr"]) - 1, g["x_seed"])
    y = oracle.apply(op, x)
    assert np.array_equal(y, fhs(g["y"]))


def test_apply_chebyshev_per_step_bitwise(oracle, golden):
    for c in golden["apply_chebyshev"]:
        nx = c["nx"]
        op = OracleOp("lap3d", nx=nx)
        a, b = oracle.analytic_extremes(3, nx)
        r = oracle.random_uniform(nx ** 3, c["r_seed"])
        if "steps" in c:
            for st in c["steps"]:
                p = oracle.cheb_params(a, b, st["m"], fh(c["scale"]))
                out = oracle.apply_chebyshev(op, p, r)
                assert sha(out) == st["sha256"], (nx, st["m"])
        else:
            p = oracle.cheb_params(a, b, 5, fh(c["scale"]))
            assert np.array_equal(oracle.apply_chebyshev(op, p, r), fhs(c["m5_out"]))


def test_apply_chebyshev_csr_bitwise(oracle, golden):
    g, c = golden["csr_apply"], golden["apply_chebyshev_csr"]
    op = OracleOp("csr", row_ptr=g["row_ptr"], col_idx=g["col_idx"], values=fhs(g["values"]))
    x = oracle.random_uniform(len(g["row_ptr"]) - 1, c["x_seed"])
    p = oracle.cheb_params(fh(c["alpha"]), fh(c["beta"]), c["m"], fh(c["scale"]))
    assert sha(oracle.apply_chebyshev(op, p, x)) == c["sha256"]


def test_apply_newton_bitwise(oracle, golden):
    g = golden["apply_newton"]
    nx = g["nx"]
    a, b = oracle.analytic_extremes(3, nx)
    r = oracle.random_uniform(nx ** 3, g["r_seed"])
    op = OracleOp("lap3d", nx=nx)
    for lv in g["levels"]:
        z = oracle.newton_params(a, b, lv["nlev"], fh(g["scale"]))
        assert sha(oracle.apply_newton(op, z, r)) == lv["sha256"]


def test_newton_equals_chebyshev(oracle):
    # test_polyprec.cpp:112-144 on the scaled 3D operator
    nx = 9
    a, b = oracle.analytic_extremes(3, nx)
    r = oracle.random_uniform(nx ** 3, 31)
    op = OracleOp("lap3d", nx=nx)
    for nlev in (1, 3, 5):
        for s in (1.0, 1.01):
            zn = oracle.apply_newton(op, oracle.newton_params(a, b, nlev, s), r)
            zc = oracle.apply_chebyshev(op, oracle.cheb_params(a, b, 2 ** nlev - 1, s), r)
            assert rel_norm(zc, zn) <= 1e-10


def _solve_case(oracle, c):
    kind = c["kind"]
    if kind.startswith("lap3d"):
        op = OracleOp("lap3d", nx=c["nx"])  # stencil and assembled forms are bitwise equal
        n = c["nx"] ** 3
    else:
        return None
    b = oracle.apply(op, oracle.random_uniform(n, SEED))
    params = None if c["m"] < 0 else oracle.cheb_params(fh(c["alpha"]), fh(c["beta"]), c["m"],
                                                        fh(c["scale"]))
    return op, b, params


@pytest.mark.parametrize("tag", ["cfg1", "cfg1_s1", "lap24_m0", "lap24_m1", "lap24_m5",
                                 "lap24_m10", "lap24_m20", "lap24_m40", "lap24_cg",
                                 "lap24_maxit", "lap32_m80"])
def test_pcg_solve_bitwise_vs_reference(oracle, golden, tag):
    c = next(s for s in golden["pcg_solve"] if s["tag"] == tag)
    op, b, params = _solve_case(oracle, c)
    assert sha(b) == c["b_sha256"]
    x, rep = oracle.pcg_solve(op, params, b, tol=c["tol"], maxit=c["maxit"])
    g = c["report"]
    for k in ("iters", "ddot", "matvec", "prec_applies", "converged"):
        assert rep[k] == g[k], k
    assert rep["rel_res"] == fh(g["rel_res"])
    assert rep["true_rel_res"] == fh(g["true_rel_res"])
    assert sha(x) == c["x_sha256"]


def test_pcg_solve_csr_vs_reference(oracle, golden):
    g = golden["csr_apply"]
    c = next(s for s in golden["pcg_solve"] if s["tag"] == "csr300_m7")
    op = OracleOp("csr", row_ptr=g["row_ptr"], col_idx=g["col_idx"], values=fhs(g["values"]))
    n = len(g["row_ptr"]) - 1
    b = oracle.apply(op, oracle.random_uniform(n, SEED))
    assert sha(b) == c["b_sha256"]
    p = oracle.cheb_params(fh(c["alpha"]), fh(c["beta"]), c["m"], fh(c["scale"]))
    x, rep = oracle.pcg_solve(op, p, b)
    assert rep["iters"] == c["report"]["iters"]
    assert sha(x) == c["x_sha256"]


def test_table1_iterations(oracle, golden):
    """spectrum_table(78, ...) iteration columns (PAPER.md:496-501 shape) via the 2D oracle."""
    nx = 78
    op = OracleOp("lap2d", nx=nx)
    a, b = oracle.analytic_extremes(2, nx)
    for key, rows in golden["table1"].items():
        sol, s = key.split(":")
        xt = np.ones(nx * nx) if sol == "ones" else oracle.random_uniform(nx * nx, SEED)
        rhs = oracle.apply(op, xt)
        for row in rows:
            m, iters = row[0], row[1]
            _, rep = oracle.pcg_solve(op, oracle.cheb_params(a, b, m, float(s)), rhs)
            assert rep["iters"] == iters, (key, m)


def test_cfg1_known_answer(golden):
    """SURVEY.md Appendix A known answer, as the reference itself produced it."""
    c = next(s for s in golden["pcg_solve"] if s["tag"] == "cfg1")["report"]
    assert (c["iters"], c["ddot"], c["matvec"], c["prec_applies"]) == (19, 59, 400, 19)
    assert fh(c["rel_res"]) == pytest.approx(6.703e-9, rel=1e-3)


def test_lanczos_bounds_bracket_analytic(oracle):
    nx = 20
    op = OracleOp("lap3d", nx=nx)
    lo_a, hi_a = oracle.analytic_extremes(3, nx)
    lo, hi, al, be = oracle.lanczos(op, 30, SEED)
    # Ritz values lie inside the spectrum
    assert lo_a <= lo <= hi <= hi_a
    assert hi == pytest.approx(hi_a, rel=2e-2)
    lo20, hi20 = oracle.tridiag_extremes(al[:20], be[:20])
    assert hi20 <= hi + 1e-15


def _eig_op(oracle, golden, c):
    if c["kind"] == "lap3d":
        return OracleOp("lap3d", nx=c["nx"])
    g = golden["csr_apply"]
    return OracleOp("csr", row_ptr=g["row_ptr"], col_idx=g["col_idx"], values=fhs(g["values"]))


def test_power_dacg_bitwise_vs_reference(oracle, golden):
    """power_method / dacg_smallest (eigenest.cpp:48-167) restated in C: same value
    bits, iterations and matvec counts as the reference itself."""
    for c in golden["eigen_estimators"]:
        op = _eig_op(oracle, golden, c)
        pm = oracle.power_method(op, tol=c["power"]["tol"], maxit=c["power"]["maxit"], seed=SEED)
        assert pm["value"] == fh(c["power"]["value"]), c["tag"]
        assert (pm["iters"], pm["matvecs"], pm["converged"]) == (
            c["power"]["iters"], c["power"]["matvecs"], c["power"]["converged"])
        dg = oracle.dacg_smallest(op, tol=c["dacg"]["tol"], maxit=c["dacg"]["maxit"], seed=SEED)
        assert dg["value"] == fh(c["dacg"]["value"]), c["tag"]
        assert (dg["iters"], dg["matvecs"], dg["converged"]) == (
            c["dacg"]["iters"], c["dacg"]["matvecs"], c["dacg"]["converged"])


@pytest.mark.parametrize("tag", ["lap24_n0", "lap24_n3", "lap24_n5", "csr300_n3"])
def test_pcg_solve_newton_bitwise_vs_reference(oracle, golden, tag):
    """pcg_solve with NewtonPreconditioner (pcg.hpp:27-40): counters, residuals, x."""
    c = next(s for s in golden["pcg_solve_newton"] if s["tag"] == tag)
    if c["kind"] == "csr":
        g = golden["csr_apply"]
        op = OracleOp("csr", row_ptr=g["row_ptr"], col_idx=g["col_idx"], values=fhs(g["values"]))
        n = len(g["row_ptr"]) - 1
    else:
        op = OracleOp("lap3d", nx=c["nx"])
        n = c["nx"] ** 3
    b = oracle.apply(op, oracle.random_uniform(n, SEED))
    assert sha(b) == c["b_sha256"]
    z = oracle.newton_params(fh(c["alpha"]), fh(c["beta"]), c["nlev"], fh(c["scale"]))
    x, rep = oracle.pcg_solve_newton(op, z, b)
    g = c["report"]
    for k in ("iters", "ddot", "matvec", "prec_applies", "converged"):
        assert rep[k] == g[k], k
    assert rep["rel_res"] == fh(g["rel_res"])
    assert rep["true_rel_res"] == fh(g["true_rel_res"])
    assert sha(x) == c["x_sha256"]
