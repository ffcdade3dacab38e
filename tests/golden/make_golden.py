# SPDX-License-Identifier: Apache-2.0
"""Generate tests/golden/*.json from the REFERENCE ITSELF.

Runs in the build container only (needs oracle/_ref/libpolycg_ref.so, which
oracle/Makefile compiles from /root/reference/proj/src). The fixtures it writes
are committed, so the GPU box (which has no /root/reference) checks against
them. Bitwise fixtures are stored as float.hex() strings or SHA-256 digests of
the little-endian float64 bytes.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from oracle.oracle import RefLib, NumericalError, InvalidArgument, OracleError  # noqa: E402

SEED = 20240801


def h(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def hx(v):
    return float(v).hex()


def sparse_spd(n, seed):
    """Small exactly-symmetric, diagonally dominant SPD CSR (int64) for CSR fixtures."""
    rng = np.random.default_rng(seed)
    rows, cols, vals = [], [], []
    for i in range(n):
        for j in rng.choice(n, size=4, replace=False):
            if j < i:
                v = -float(rng.integers(1, 9)) / 8.0
                rows += [i, j]
                cols += [j, i]
                vals += [v, v]
    A = {}
    for r, c, v in zip(rows, cols, vals):
        A[(r, c)] = A.get((r, c), 0.0) + v
    offsum = np.zeros(n)
    for (r, c), v in A.items():
        offsum[r] += abs(v)
    for i in range(n):
        A[(i, i)] = offsum[i] + 1.0 + (i % 7) * 0.25
    keys = sorted(A)
    rp = np.zeros(n + 1, dtype=np.int64)
    for r, _ in keys:
        rp[r + 1] += 1
    rp = np.cumsum(rp)
    ci = np.array([c for _, c in keys], dtype=np.int64)
    va = np.array([A[k] for k in keys])
    return rp, ci, va


def main():
    R = RefLib()
    R.set_threads(8)
    out = {}

    # ---- coefficients (polyprec.cpp:56-79) -----------------------------------------
    cases = [(1.0, 3.0, 2, 1.0), (7.9064e-4, 1.99921, 31, 1.01), (7.9064e-4, 1.99921, 31, 1.0),
             (0.02, 1.95, 31, 1.01), (0.1, 1.9, 12, 1.0)]
    for nx in (100, 160, 320, 640):
        a, b = R.analytic_extremes(3, nx)
        for m in (0, 5, 10, 20, 30, 40, 80):
            cases.append((a, b, m, 1.001))
    coeffs = []
    for a, b, m, s in cases:
        p = R.cheb_params(a, b, m, s)
        coeffs.append({"alpha": hx(a), "beta": hx(b), "m": m, "scale": hx(s), "theta": hx(p["theta"]),
                       "delta": hx(p["delta"]), "sigma": hx(p["sigma"]),
                       "rho": [hx(v) for v in p["rho"]]})
    out["cheb_params"] = coeffs

    errs = []
    for a, b, m, s in [(1.0, 1.0, 1, 1.0), (0.0, 1.0, 1, 1.0), (1.0, 2.0, -1, 1.0), (1.0, 2.0, 1, 0.5),
                       (-1.0, 2.0, 1, 1.0)]:
        try:
            R.cheb_params(a, b, m, s)
            errs.append({"args": [a, b, m, s], "error": None})
        except InvalidArgument as e:
            errs.append({"args": [a, b, m, s], "error": "invalid_argument", "msg": str(e)})
        except NumericalError as e:
            errs.append({"args": [a, b, m, s], "error": "numerical", "msg": str(e)})
    out["cheb_params_errors"] = errs

    lams = np.linspace(7.9064e-4, 1.99921, 101)
    out["eval_poly"] = {"alpha": hx(7.9064e-4), "beta": hx(1.99921), "lams": [hx(v) for v in lams],
                        "by_m": {}}
    for m, s in [(0, 1.0), (7, 1.01), (31, 1.01), (40, 1.001)]:
        out["eval_poly"]["by_m"][f"{m}:{s}"] = [hx(v) for v in R.eval_poly(7.9064e-4, 1.99921, m, s, lams)]

    out["newton_params"] = []
    for a, b, nl, s in [(1.0, 3.0, 2, 1.0), (0.02, 1.95, 5, 1.01), (7.9064e-4, 1.99921, 5, 1.0)]:
        out["newton_params"].append({"alpha": hx(a), "beta": hx(b), "nlev": nl, "scale": hx(s),
                                     "zeta": [hx(v) for v in R.newton_params(a, b, nl, s)]})

    # ---- analytic extremes (linop.cpp:382-390) -----------------------------------------
    out["analytic_extremes"] = []
    for dim in (2, 3):
        for nx in (2, 5, 16, 78, 100, 160, 256, 320, 512, 640):
            lo, hi = R.analytic_extremes(dim, nx)
            out["analytic_extremes"].append({"dim": dim, "nx": nx, "lo": hx(lo), "hi": hx(hi)})

    # ---- RNG (eigenest.cpp:13-30) -------------------------------------------------------
    v = R.random_uniform(1_000_000, SEED)
    out["random_uniform"] = {"seed": SEED, "first": [hx(x) for x in v[:64]], "n": 1_000_000,
                             "sha256": h(v), "seed7_sha256_4096": h(R.random_uniform(4096, 7))}

    # ---- scaled stencil / CSR applies (linop.cpp:171-187, 236-258, 271-275) ----------------
    applies = []
    for nx in (2, 3, 5, 9, 16, 33):
        x = R.random_uniform(nx ** 3, 7000 + nx)
        y = R.apply("lap3d", x, nx=nx)
        ya = R.apply("lap3d_assembled", x, nx=nx)
        assert np.array_equal(y, ya)
        rec = {"nx": nx, "x_seed": 7000 + nx, "sha256": h(y)}
        if nx <= 5:
            rec["y"] = [hx(t) for t in y]
        applies.append(rec)
    out["stencil_apply"] = applies

    rp, ci, va = sparse_spd(300, 11)
    x = R.random_uniform(300, 77)
    y = R.apply("csr", x, csr=(rp, ci, va))
    out["csr_apply"] = {"row_ptr": rp.tolist(), "col_idx": ci.tolist(), "values": [hx(t) for t in va],
                        "x_seed": 77, "y": [hx(t) for t in y], "sha256": h(y)}

    # ---- Chebyshev apply per degree step (polyprec.cpp:169-198) ----------------------------
    cheb = []
    for nx, scale in ((17, 1.001), (8, 1.01)):
        a, b = R.analytic_extremes(3, nx)
        r = R.random_uniform(nx ** 3, 4242)
        steps = []
        for j in range(0, 13):
            o, mv = R.apply_chebyshev("lap3d", a, b, j, scale, r, nx=nx)
            assert mv == j
            steps.append({"m": j, "sha256": h(o), "norm": hx(float(np.sqrt(np.sum(o * o))))})
        cheb.append({"nx": nx, "scale": hx(scale), "r_seed": 4242, "steps": steps})
    a, b = R.analytic_extremes(3, 5)
    r = R.random_uniform(125, 4243)
    o, _ = R.apply_chebyshev("lap3d", a, b, 5, 1.001, r, nx=5)
    cheb.append({"nx": 5, "scale": hx(1.001), "r_seed": 4243, "m5_out": [hx(t) for t in o]})
    out["apply_chebyshev"] = cheb

    # CSR Chebyshev (sparse_spd; bounds from a generous interval)
    o, _ = R.apply_chebyshev("csr", 0.05, 1.9, 7, 1.01, x, csr=(rp, ci, va))
    out["apply_chebyshev_csr"] = {"alpha": hx(0.05), "beta": hx(1.9), "m": 7, "scale": hx(1.01),
                                  "x_seed": 77, "sha256": h(o)}

    # Newton vs Chebyshev (test_polyprec.cpp:112-144 shape on the 3D operator)
    a, b = R.analytic_extremes(3, 9)
    r = R.random_uniform(729, 31)
    newton = []
    for nlev in (0, 1, 3, 5):
        on = R.apply_newton("lap3d", a, b, nlev, 1.01, r, nx=9)
        newton.append({"nlev": nlev, "sha256": h(on)})
    out["apply_newton"] = {"nx": 9, "r_seed": 31, "scale": hx(1.01), "levels": newton}

    # ---- PCG solves (pcg.cpp:10-117) -----------------------------------------------------
    solves = []

    def rec_solve(tag, kind, nx, m, scale, csr=None, tol=1e-8, maxit=20000, bounds=None):
        a, b = bounds if bounds else R.analytic_extremes(3, nx)
        x, bvec, rep = R.pcg_solve(kind, a, b, m, scale, nx=nx, csr=csr, seed=SEED, tol=tol, maxit=maxit)
        xt = R.random_uniform(len(x), SEED)
        err = float(np.linalg.norm(x - xt) / np.linalg.norm(xt))
        solves.append({"tag": tag, "kind": kind, "nx": nx, "m": m, "scale": hx(scale), "tol": tol,
                       "maxit": maxit, "alpha": hx(a), "beta": hx(b),
                       "report": {k: (hx(v) if isinstance(v, float) else v) for k, v in rep.items()
                                  if k != "wall_time"},
                       "x_sha256": h(x), "b_sha256": h(bvec), "err": hx(err),
                       "x_norm": hx(float(np.linalg.norm(x)))})
        print(tag, rep["iters"], rep["ddot"], rep["matvec"], rep["rel_res"], err, file=sys.stderr)

    rec_solve("cfg1", "lap3d_assembled", 100, 20, 1.001)
    rec_solve("cfg1_s1", "lap3d_assembled", 100, 20, 1.0)
    rec_solve("cfg1_k0", "lap3d", 100, 0, 1.001)
    for m in (0, 1, 5, 10, 20, 40):
        rec_solve(f"lap24_m{m}", "lap3d", 24, m, 1.001)
    rec_solve("lap24_cg", "lap3d", 24, -1, 1.0)
    rec_solve("lap24_maxit", "lap3d", 24, 5, 1.001, maxit=3)
    rec_solve("lap32_m80", "lap3d", 32, 80, 1.001)
    rec_solve("csr300_m7", "csr", 0, 7, 1.01, csr=(rp, ci, va), bounds=(0.05, 1.9))
    out["pcg_solve"] = solves

    # ---- pcg_solve with NewtonPreconditioner (pcg.hpp:27-40) ---------------------------------
    nsolves = []
    for tag, kind, nx, nlev, scale, csr, bounds in [
            ("lap24_n3", "lap3d", 24, 3, 1.001, None, None),
            ("lap24_n5", "lap3d", 24, 5, 1.001, None, None),
            ("lap24_n0", "lap3d", 24, 0, 1.0, None, None),
            ("csr300_n3", "csr", 0, 3, 1.01, (rp, ci, va), (0.05, 1.9))]:
        a, b = bounds if bounds else R.analytic_extremes(3, nx)
        x, bvec, rep = R.pcg_solve_newton(kind, a, b, nlev, scale, nx=nx, csr=csr, seed=SEED)
        nsolves.append({"tag": tag, "kind": kind, "nx": nx, "nlev": nlev, "scale": hx(scale),
                        "alpha": hx(a), "beta": hx(b),
                        "report": {k: (hx(v) if isinstance(v, float) else v) for k, v in rep.items()
                                   if k != "wall_time"},
                        "x_sha256": h(x), "b_sha256": h(bvec)})
        print(tag, rep["iters"], rep["ddot"], rep["matvec"], rep["rel_res"], file=sys.stderr)
    out["pcg_solve_newton"] = nsolves

    # ---- Table 1 (spectrum.cpp:59-88) ------------------------------------
    t1 = {}
    for sol in ("ones", "random"):
        for s in (1.0, 1.01):
            rows = R.spectrum_table(78, [0, 1, 3, 7, 15, 31], s, sol)
            t1[f"{sol}:{s}"] = [[int(r[0]), int(r[1]), hx(r[2]), hx(r[3]), int(r[4]), hx(r[5])] for r in rows]
    out["table1"] = t1

    # ---- bound estimators (eigenest.cpp:48-167) ----------------------------------------
    eig = []
    for tag, kind, nx, csr, ptol, pmax, dtol, dmax in [
            ("lap10_default", "lap3d", 10, None, 1e-4, 200, 1e-2, 5000),
            ("lap24_tight", "lap3d", 24, None, 1e-8, 2000, 1e-4, 5000),
            ("csr300_default", "csr", 0, (rp, ci, va), 1e-4, 200, 1e-2, 5000)]:
        pm = R.power_method(kind, tol=ptol, maxit=pmax, nx=nx, csr=csr)
        dg = R.dacg_smallest(kind, tol=dtol, maxit=dmax, nx=nx, csr=csr)
        eig.append({"tag": tag, "kind": kind, "nx": nx, "power": {"tol": ptol, "maxit": pmax,
                    "value": hx(pm["value"]), "iters": pm["iters"], "matvecs": pm["matvecs"],
                    "converged": pm["converged"]},
                    "dacg": {"tol": dtol, "maxit": dmax, "value": hx(dg["value"]), "iters": dg["iters"],
                             "matvecs": dg["matvecs"], "converged": dg["converged"]}})
    out["eigen_estimators"] = eig

    # ---- load_matrix_market / save_matrix_market (matrix_market.cpp:55-199) ------------------
    from tests.golden.mm_cases import cases as mm_cases  # noqa: E402
    mm = {}
    for name, text in mm_cases().items():
        try:
            n, rp, ci, va = R.mm_load(text, "<" + name + ">")
        except OracleError as e:
            mm[name] = {"error": str(e)}
            continue
        saved = R.mm_save(n, rp, ci, va)
        mm[name] = {"n": int(n), "nnz": int(len(va)), "row_ptr": hashlib.sha256(rp.astype("<i8").tobytes()).hexdigest(),
                    "col_idx": hashlib.sha256(ci.astype("<i8").tobytes()).hexdigest(), "values": h(va),
                    "save_sha256": hashlib.sha256(saved.encode()).hexdigest()}
    out["matrix_market"] = mm

    with open(os.path.join(HERE, "reference_golden.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", os.path.join(HERE, "reference_golden.json"))


if __name__ == "__main__":
    main()
