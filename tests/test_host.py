# SPDX-License-Identifier: Apache-2.0
"""CPU-only checks of the native library: it builds, loads, exports every symbol
include/pcgx.h declares, and its host-side math and generators are right.
No kernel is launched here (no GPU in the build container)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from tests._util import fh, fhs, sha

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_symbols_exported(pcgx):
    hdr = open(os.path.join(ROOT, "include", "pcgx.h")).read()
    declared = set(re.findall(r"\b(pcgx_[a-z0-9_]+)\s*\(", hdr))
    declared -= {"pcgx_context_s", "pcgx_operator_s"}
    L = C.CDLL(pcgx.LIB_PATH)
    missing = [s for s in sorted(declared) if not hasattr(L, s)]
    assert not missing, missing
    assert declared == set(pcgx.SYMBOLS)


def test_library_is_sm100a(pcgx):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", pcgx.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_context_without_gpu_fails_loudly(pcgx):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(pcgx.CudaError):
        pcgx.Context(0)


def test_cheb_params_bitwise(pcgx, golden):
    for c in golden["cheb_params"]:
        p = pcgx.cheb_params(fh(c["alpha"]), fh(c["beta"]), c["m"], fh(c["scale"]))
        assert (p.theta, p.delta, p.sigma) == (fh(c["theta"]), fh(c["delta"]), fh(c["sigma"]))
        assert np.array_equal(p.rho, fhs(c["rho"]))


def test_cheb_params_errors_match_reference(pcgx, golden):
    for e in golden["cheb_params_errors"]:
        a, b, m, s = e["args"]
        if e["error"] is None:
            pcgx.cheb_params(a, b, m, s)
            continue
        exc = pcgx.InvalidArgument if e["error"] == "invalid_argument" else pcgx.NumericalError
        with pytest.raises(exc) as ei:
            pcgx.cheb_params(a, b, m, s)
        assert str(ei.value) == e["msg"]


def test_eval_poly_bitwise(pcgx, golden):
    g = golden["eval_poly"]
    for key, vals in g["by_m"].items():
        m, s = key.split(":")
        p = pcgx.cheb_params(fh(g["alpha"]), fh(g["beta"]), int(m), float(s))
        got = np.array([pcgx.eval_poly(p, l) for l in fhs(g["lams"])])
        assert np.array_equal(got, fhs(vals))


def test_positivity_grid(pcgx):
    # test_polyprec.cpp:296-306
    for s in (1.0, 1.01, 1.1):
        for m in (0, 1, 3, 7, 15, 31, 63):
            p = pcgx.cheb_params(7.9064e-4, 1.99921, m, s)
            lam = np.linspace(7.9064e-4, 1.99921, 2001)
            assert all(pcgx.eval_poly(p, l) > 0 for l in lam)


def test_optimality(pcgx):
    # test_polyprec.cpp:173-188: max |1 - lambda p(lambda)| = 1 / T_{m+1}(sigma)
    for a, b in ((7.9064e-4, 1.99921), (1e-3, 1.0), (0.02, 2.0)):
        for m in (1, 3, 7, 15, 31):
            p = pcgx.cheb_params(a, b, m, 1.0)
            lam = a + (b - a) * np.arange(20001) / 20000
            gm = max(abs(1 - l * pcgx.eval_poly(p, l)) for l in lam)
            exp = 1.0 / np.cosh((m + 1) * np.arccosh(p.sigma))
            assert gm == pytest.approx(exp, rel=1e-10)


def test_newton_params_bitwise(pcgx, golden):
    for c in golden["newton_params"]:
        p = pcgx.newton_params(fh(c["alpha"]), fh(c["beta"]), c["nlev"], fh(c["scale"]))
        assert np.array_equal(p.zeta, fhs(c["zeta"]))
        assert p.degree() == 2 ** c["nlev"] - 1


def test_newton_params_hand_values_and_errors(pcgx):
    # test_polyprec.cpp:19-36, 55-60
    p = pcgx.newton_params(1.0, 1.0, 4, 1.0)
    assert p.zeta == pytest.approx([1.0] * 5, rel=1e-15)
    p = pcgx.newton_params(1.0, 3.0, 2, 1.0)
    assert p.zeta == pytest.approx([0.5, 8.0 / 7.0, 98.0 / 97.0], rel=1e-15)
    p = pcgx.newton_params(7.9064e-4, 1.99921, 1, 1.0)
    assert p.zeta[1] == pytest.approx(1.99684, rel=1e-5)
    for args, msg in [((0.0, 1.0, 1, 1.0), "newton_params: need 0 < alpha0 <= beta0"),
                      ((-1.0, 1.0, 1, 1.0), "newton_params: need 0 < alpha0 <= beta0"),
                      ((1.0, 2.0, -1, 1.0), "newton_params: nlev must be >= 0"),
                      ((1.0, 2.0, 1, 0.5), "newton_params: scale must be >= 1")]:
        with pytest.raises(pcgx.InvalidArgument) as ei:
            pcgx.newton_params(*args)
        assert str(ei.value) == msg


def test_newton_eval_and_forms_agree(pcgx):
    # test_polyprec.cpp:38-43, 155-170: eval at the fixed point; the scalar forms agree
    for nlev in (0, 2, 5):
        assert pcgx.eval_poly(pcgx.newton_params(1.0, 1.0, nlev, 1.0), 1.0) == pytest.approx(1.0, rel=1e-15)
    for s in (1.0, 1.01):
        for nlev in (0, 1, 3, 6):
            pn = pcgx.newton_params(0.01, 1.99, nlev, s)
            pc = pcgx.cheb_params(0.01, 1.99, pn.degree(), s)
            for g in range(101):
                lam = 0.01 + (1.99 - 0.01) * g / 100.0
                assert pcgx.eval_poly(pn, lam) == pytest.approx(pcgx.eval_poly(pc, lam), rel=1e-12)
    # the scalar mirror of the recursion (polyprec.cpp:81-87), restated
    p = pcgx.newton_params(0.02, 1.95, 4, 1.001)
    for lam in (0.02, 0.5, 1.3, 1.95):
        r = p.zeta[0]
        for j in range(1, 5):
            r = p.zeta[j] * (2.0 * r - lam * r * r)
        assert pcgx.eval_poly(p, lam) == r


def test_chi_sequence(pcgx):
    # test_polyprec.cpp:308-321, and chi == zeta[1:] of newton_params at scale 1
    chi = pcgx.chi_sequence(1.0, 3.0, 2)
    assert chi == pytest.approx([8.0 / 7.0, 98.0 / 97.0], rel=1e-15)
    tight = pcgx.chi_sequence(1.0, 1.0 + 1e-9, 30)
    assert len(tight) == 30 and all(abs(c - 1.0) <= 1e-15 for c in tight[5:])
    z = pcgx.newton_params(0.01, 1.99, 6, 1.0).zeta
    assert pcgx.chi_sequence(0.01, 1.99, 6) == pytest.approx(z[1:], rel=1e-12)
    with pytest.raises(pcgx.InvalidArgument):
        pcgx.chi_sequence(1.0, 1.0, 1)
    with pytest.raises(pcgx.InvalidArgument):
        pcgx.chi_sequence(1.0, 2.0, 31)


def test_analytic_extremes_bitwise(pcgx, golden):
    for c in golden["analytic_extremes"]:
        lo, hi = pcgx.analytic_extremes(c["dim"], c["nx"])
        assert lo == fh(c["lo"]) and hi == fh(c["hi"])


def test_random_uniform_host_bitwise(pcgx, golden):
    g = golden["random_uniform"]
    v = pcgx.random_uniform_vector(g["n"], g["seed"])
    assert sha(v) == g["sha256"]
    assert np.array_equal(pcgx.random_uniform_vector(100, g["seed"], offset=777), v[777:877])


def _check_sym_spd(A, n, dense_ok=True):
    rp, ci, va = A.row_ptr, A.col_idx, A.values
    assert rp[0] == 0 and rp[-1] == len(ci)
    assert np.all(np.diff(rp) >= 0)
    for i in range(n):
        row = ci[rp[i]:rp[i + 1]]
        assert np.all(np.diff(row) > 0)
    # bitwise symmetry: CsrMatrix(..., sym_tol = 0) contract
    rows = np.repeat(np.arange(n), np.diff(rp))
    key = rows.astype(np.int64) * n + ci
    keyT = ci.astype(np.int64) * n + rows
    order = np.argsort(key)
    orderT = np.argsort(keyT)
    assert np.array_equal(key[order], keyT[orderT])
    assert np.array_equal(va[order].view(np.uint64), va[orderT].view(np.uint64))
    if dense_ok:
        D = np.zeros((n, n))
        D[rows, ci] = va
        assert np.linalg.eigvalsh(D).min() > 0


@pytest.mark.parametrize("nx", [1, 2, 4, 6])
def test_gen_fe27(pcgx, nx):
    A = pcgx.gen_fe27(nx, sigma=1.0, seed=5)
    assert A.n == nx ** 3 and A.nnz() == (3 * nx - 2) ** 3
    assert np.all(np.diff(A.row_ptr) <= 27)
    _check_sym_spd(A, A.n)
    # every one of the 27 couplings is nonzero (anisotropic Q1 element)
    assert np.count_nonzero(A.values) == A.nnz()
    # deterministic
    B = pcgx.gen_fe27(nx, sigma=1.0, seed=5)
    assert sha(A.values) == sha(B.values)


@pytest.mark.parametrize("nx", [1, 2, 4])
def test_gen_elast27(pcgx, nx):
    A = pcgx.gen_elast27(nx, 1.0, 0.5, 0.1, seed=9)
    assert A.n == 3 * nx ** 3 and A.nnz() == 9 * (3 * nx - 2) ** 3
    assert np.all(np.diff(A.row_ptr) <= 81)
    _check_sym_spd(A, A.n)


def test_gen_sizes_at_configs(pcgx):
    n, nnz = C.c_int64(), C.c_int64()
    pcgx.lib().pcgx_gen_fe27_size(256, C.byref(n), C.byref(nnz))
    assert (n.value, nnz.value) == (16_777_216, 449_455_096)
    pcgx.lib().pcgx_gen_elast27_size(160, C.byref(n), C.byref(nnz))
    assert (n.value, nnz.value) == (12_288_000, 982_938_168)


def test_device_quotient_model_matches_ieee_division(tmp_path):
    # host model of div_rn / div_rn_wide (csrc/kernels.cuh: Markstein's correction,
    # power-of-two scaling outside [2^-960, 2^961), the subnormal tie fix): bitwise
    # x / b over 2.4e6 operands of every class for six divisors
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc not available")
    src = os.path.join(os.path.dirname(__file__), "cpp", "div_rn_model.c")
    exe = str(tmp_path / "div_rn_model")
    subprocess.run([gcc, "-O2", "-ffp-contract=off", "-o", exe, src, "-lm"], check=True)
    out = subprocess.run([exe, "400000"], capture_output=True, text=True)
    assert out.returncode == 0 and out.stdout.strip().endswith("bad=0"), out.stdout


def test_chunk_plans(pcgx):
    """The z-chunk planner of the temporally blocked passes (host code): plans cover
    the span exactly, respect the chunk limit, and admit a long first chunk exactly
    when every tile of a z-level is resident (tiles <= resident CTAs)."""
    P = pcgx
    for span, tiles, slots in ((320, 80, 148), (512, 208, 148), (640, 320, 148), (1, 1, 148), (7, 3, 148),
                               (97, 10, 148), (200, 148, 148), (4096, 208, 148), (33, 1000, 296)):
        for lc in (True, False):
            h = P.chunk_plan(span, tiles, slots, lc)
            assert 1 <= len(h) <= 48 and sum(h) == span and min(h) >= 1, (span, tiles, h)
    # 320^3: 80 tiles of 64 x 20 on 148 SMs -- one long chunk, the other SMs share the rest
    assert P.chunk_plan(320, 80, 148, True) == [176, 88, 28, 28]
    assert max(P.chunk_plan(320, 80, 148, False)) <= 96      # the direction step keeps short chunks
    assert max(P.chunk_plan(512, 208, 148, True)) <= 96      # more tiles than resident CTAs: short chunks
    assert max(P.chunk_plan(640, 320, 148, True)) <= 96
