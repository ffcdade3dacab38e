# SPDX-License-Identifier: Apache-2.0
"""TEST INFRASTRUCTURE ONLY — ctypes wrappers for the parity checkers.

* ``Oracle``  : oracle/_ref/liboracle.so, our plain-C restatement of the
  reference hot path (oracle/polycg_oracle.c).
* ``RefLib``  : oracle/_ref/libpolycg_ref.so, the reference library itself
  (/root/reference/proj/src compiled by oracle/Makefile) behind the flat C API
  of oracle/ref_driver.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module, and only as the checker or the CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_ref")

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)


def build(quiet: bool = True) -> None:
    """Compile the oracle (and the reference, when /root/reference exists)."""
    subprocess.run(["make", "-C", HERE, "-j8"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _ptr(a, t=_dp):
    return None if a is None else a.ctypes.data_as(t)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class InvalidArgument(OracleError):
    pass


class NumericalError(OracleError):
    pass


class ParseError(OracleError):
    pass


def _raise(code, msg):
    if code == 7:
        raise ParseError(code, msg)
    if code == 1:
        raise InvalidArgument(code, msg)
    if code == 2:
        raise NumericalError(code, msg)
    raise OracleError(code, msg)


class _OrOp(C.Structure):
    _fields_ = [("kind", C.c_int), ("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64),
                ("n", C.c_int64), ("row_ptr", _i64p), ("col_idx", _i64p), ("values", _dp),
                ("d", _dp)]


class Report(C.Structure):
    _fields_ = [("iters", C.c_int64), ("ddot", C.c_int64), ("matvec", C.c_int64),
                ("prec_applies", C.c_int64), ("rel_res", C.c_double),
                ("true_rel_res", C.c_double), ("wall_time", C.c_double),
                ("converged", C.c_int64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class OracleOp:
    """Operator description for the C oracle. kind: 'lap3d' | 'lap2d' | 'csr'.

    CSR arrays are int64 (the reference's Index); d = inv_sqrt_diag.
    """

    def __init__(self, kind, nx=0, ny=0, nz=0, row_ptr=None, col_idx=None, values=None, d=None):
        self.kind = kind
        self.keep = []
        k = {"lap3d": 0, "lap2d": 1, "csr": 2}[kind]
        s = _OrOp()
        s.kind = k
        s.nx, s.ny, s.nz = nx, (ny or nx), (nz or nx)
        if kind == "lap2d":
            s.nz = 1
        if kind == "csr":
            row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
            col_idx = np.ascontiguousarray(col_idx, dtype=np.int64)
            values = np.ascontiguousarray(values, dtype=np.float64)
            s.n = len(row_ptr) - 1
            s.row_ptr, s.col_idx, s.values = _ptr(row_ptr, _i64p), _ptr(col_idx, _i64p), _ptr(values)
            self.keep += [row_ptr, col_idx, values]
            if d is None:
                diag = csr_diagonal(row_ptr, col_idx, values)
                d = 1.0 / np.sqrt(diag)
        else:
            s.n = s.nx * s.ny * s.nz
        if d is not None:
            d = np.ascontiguousarray(d, dtype=np.float64)
            s.d = _ptr(d)
            self.keep.append(d)
        self.s = s
        self.n = s.n


def csr_diagonal(row_ptr, col_idx, values):
    """CsrMatrix::diagonal (proj/src/linop.cpp:189-197)."""
    n = len(row_ptr) - 1
    rows = np.repeat(np.arange(n), np.diff(row_ptr))
    d = np.zeros(n)
    m = col_idx == rows
    d[rows[m]] = values[m]
    return d


class Oracle:
    def __init__(self, path=None):
        path = path or os.path.join(OUT, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        self.L = L
        L.or_last_error.restype = C.c_char_p
        L.or_eval_poly.restype = C.c_double
        L.or_eval_poly.argtypes = [_dp, _dp, C.c_int, C.c_double]
        L.or_cheb_params.argtypes = [C.c_double, C.c_double, C.c_int, C.c_double, _dp, _dp]
        L.or_newton_params.argtypes = [C.c_double, C.c_double, C.c_int, C.c_double, _dp]
        L.or_analytic_extremes.argtypes = [C.c_int, C.c_int64, C.c_int, _dp, _dp]
        L.or_analytic_extremes_box.argtypes = [C.c_int64, C.c_int64, C.c_int64, _dp, _dp]
        L.or_random_uniform.argtypes = [C.c_int64, C.c_uint64, C.c_uint64, _dp]
        L.or_apply.argtypes = [C.POINTER(_OrOp), _dp, _dp]
        L.or_apply_inner.argtypes = [C.POINTER(_OrOp), _dp, _dp]
        L.or_apply_chebyshev.argtypes = [C.POINTER(_OrOp), _dp, _dp, C.c_int, _dp, _dp]
        L.or_apply_newton.argtypes = [C.POINTER(_OrOp), _dp, C.c_int, _dp, _dp]
        L.or_pcg_solve.argtypes = [C.POINTER(_OrOp), _dp, _dp, C.c_int, _dp, _dp, C.c_double,
                                   C.c_int, _dp, C.POINTER(Report)]
        L.or_pcg_solve_newton.argtypes = [C.POINTER(_OrOp), _dp, C.c_int, _dp, _dp, C.c_double,
                                          C.c_int, _dp, C.POINTER(Report)]
        L.or_lanczos.argtypes = [C.POINTER(_OrOp), C.c_int, C.c_uint64, _dp, _dp, _dp, _dp]
        L.or_tridiag_extremes.argtypes = [C.c_int, _dp, _dp, _dp, _dp]
        L.or_power_method.argtypes = [C.POINTER(_OrOp), C.c_double, C.c_int, C.c_uint64, _dp]
        L.or_dacg_smallest.argtypes = [C.POINTER(_OrOp), C.c_double, C.c_int, C.c_uint64, _dp]

    def _chk(self, code):
        if code:
            _raise(code, self.L.or_last_error().decode())

    def cheb_params(self, alpha, beta, m, scale=1.0):
        tds = np.zeros(3)
        rho = np.zeros(max(m, 0) + 1)
        self._chk(self.L.or_cheb_params(alpha, beta, m, scale, _ptr(tds), _ptr(rho)))
        return {"theta": tds[0], "delta": tds[1], "sigma": tds[2], "rho": rho, "m": m,
                "tds": tds}

    def eval_poly(self, params, lam):
        return self.L.or_eval_poly(_ptr(params["tds"]), _ptr(params["rho"]), params["m"], lam)

    def newton_params(self, alpha, beta, nlev, scale=1.0):
        z = np.zeros(nlev + 1)
        self._chk(self.L.or_newton_params(alpha, beta, nlev, scale, _ptr(z)))
        return z

    def analytic_extremes(self, dim, nx, scaled=True):
        lo, hi = C.c_double(), C.c_double()
        self.L.or_analytic_extremes(dim, nx, int(scaled), C.byref(lo), C.byref(hi))
        return lo.value, hi.value

    def analytic_extremes_box(self, nx, ny, nz):
        lo, hi = C.c_double(), C.c_double()
        self.L.or_analytic_extremes_box(nx, ny, nz, C.byref(lo), C.byref(hi))
        return lo.value, hi.value

    def random_uniform(self, n, seed, offset=0):
        out = np.empty(n)
        self.L.or_random_uniform(n, seed, offset, _ptr(out))
        return out

    def apply(self, op: OracleOp, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(op.n)
        self._chk(self.L.or_apply(C.byref(op.s), _ptr(x), _ptr(y)))
        return y

    def apply_inner(self, op: OracleOp, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(op.n)
        self._chk(self.L.or_apply_inner(C.byref(op.s), _ptr(x), _ptr(y)))
        return y

    def apply_chebyshev(self, op: OracleOp, params, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        out = np.empty(op.n)
        self._chk(self.L.or_apply_chebyshev(C.byref(op.s), _ptr(params["tds"]),
                                            _ptr(params["rho"]), params["m"], _ptr(r), _ptr(out)))
        return out

    def apply_newton(self, op: OracleOp, zeta, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        out = np.empty(op.n)
        self._chk(self.L.or_apply_newton(C.byref(op.s), _ptr(zeta), len(zeta) - 1, _ptr(r),
                                         _ptr(out)))
        return out

    def pcg_solve(self, op: OracleOp, params, b, tol=1e-8, maxit=20000, x0=None):
        """params None -> plain CG (prec == nullptr)."""
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty(op.n)
        rep = Report()
        if params is None:
            tds = np.zeros(3)
            rho = np.zeros(1)
            m = -1
        else:
            tds, rho, m = params["tds"], params["rho"], params["m"]
        x0p = None if x0 is None else np.ascontiguousarray(x0, dtype=np.float64)
        self._chk(self.L.or_pcg_solve(C.byref(op.s), _ptr(tds), _ptr(rho), m, _ptr(b),
                                      _ptr(x0p), tol, maxit, _ptr(x), C.byref(rep)))
        return x, rep.as_dict()

    def pcg_solve_newton(self, op: OracleOp, zeta, b, tol=1e-8, maxit=20000, x0=None):
        """pcg_solve with a NewtonPreconditioner (pcg.hpp:27-40)."""
        b = np.ascontiguousarray(b, dtype=np.float64)
        zeta = np.ascontiguousarray(zeta, dtype=np.float64)
        x = np.empty(op.n)
        rep = Report()
        x0p = None if x0 is None else np.ascontiguousarray(x0, dtype=np.float64)
        self._chk(self.L.or_pcg_solve_newton(C.byref(op.s), _ptr(zeta), len(zeta) - 1, _ptr(b),
                                             _ptr(x0p), tol, maxit, _ptr(x), C.byref(rep)))
        return x, rep.as_dict()

    def lanczos(self, op: OracleOp, steps, seed):
        a = np.zeros(steps)
        b = np.zeros(steps)
        lo, hi = C.c_double(), C.c_double()
        self._chk(self.L.or_lanczos(C.byref(op.s), steps, seed, C.byref(lo), C.byref(hi),
                                    _ptr(a), _ptr(b)))
        return lo.value, hi.value, a, b

    def _eig(self, fn, op, tol, maxit, seed):
        out = np.zeros(4)
        self._chk(getattr(self.L, fn)(C.byref(op.s), tol, maxit, seed, _ptr(out)))
        return {"value": out[0], "iters": int(out[1]), "matvecs": int(out[2]),
                "converged": bool(out[3])}

    def power_method(self, op, tol=1e-4, maxit=200, seed=20240801):
        return self._eig("or_power_method", op, tol, maxit, seed)

    def dacg_smallest(self, op, tol=1e-2, maxit=5000, seed=20240801):
        return self._eig("or_dacg_smallest", op, tol, maxit, seed)

    def tridiag_extremes(self, a, b):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        lo, hi = C.c_double(), C.c_double()
        self.L.or_tridiag_extremes(len(a), _ptr(a), _ptr(b), C.byref(lo), C.byref(hi))
        return lo.value, hi.value


# --------------------------------------------------------------------------- reference

REF_KIND = {"lap3d": 0, "lap2d": 1, "lap3d_assembled": 2, "csr": 3, "lap2d_assembled": 4}


class RefLib:
    """The reference library itself (oracle/_ref/libpolycg_ref.so)."""

    def __init__(self, path=None):
        path = path or os.path.join(OUT, "libpolycg_ref.so")
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        self.L = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_cheb_params.argtypes = [C.c_double, C.c_double, C.c_int, C.c_double, _dp, _dp]
        L.ref_eval_poly.argtypes = [C.c_double, C.c_double, C.c_int, C.c_double, _dp, C.c_int, _dp]
        L.ref_newton_params.argtypes = [C.c_double, C.c_double, C.c_int, C.c_double, _dp]
        L.ref_analytic_extremes.argtypes = [C.c_int, C.c_int64, C.c_int, _dp, _dp]
        L.ref_random_uniform.argtypes = [C.c_int64, C.c_uint64, _dp]
        L.ref_apply.argtypes = [C.c_int, C.c_int64, C.c_int64, _i64p, _i64p, _dp, _dp, _dp, C.c_int]
        L.ref_apply_chebyshev.argtypes = [C.c_int, C.c_int64, C.c_int64, _i64p, _i64p, _dp,
                                          C.c_double, C.c_double, C.c_int, C.c_double, _dp, _dp,
                                          C.POINTER(C.c_uint64)]
        L.ref_apply_newton.argtypes = [C.c_int, C.c_int64, C.c_int64, _i64p, _i64p, _dp,
                                       C.c_double, C.c_double, C.c_int, C.c_double, _dp, _dp]
        L.ref_pcg_solve.argtypes = [C.c_int, C.c_int64, C.c_int64, _i64p, _i64p, _dp, C.c_double,
                                    C.c_double, C.c_int, C.c_double, _dp, C.c_uint64, C.c_double,
                                    C.c_int, _dp, _dp, C.POINTER(Report)]
        L.ref_pcg_solve_newton.argtypes = L.ref_pcg_solve.argtypes
        L.ref_mm_load_text.argtypes = [C.c_char_p, C.c_int64, C.c_char_p, _i64p, _i64p]
        L.ref_mm_load_file.argtypes = [C.c_char_p, _i64p, _i64p]
        L.ref_mm_fetch.argtypes = [_i64p, _i64p, _dp]
        L.ref_mm_fetch.restype = None
        L.ref_mm_save_text.argtypes = [C.c_int64, _i64p, _i64p, _dp, C.POINTER(C.c_char_p),
                                       _i64p]
        L.ref_spectrum_table.argtypes = [C.c_int64, C.POINTER(C.c_int), C.c_int, C.c_double,
                                         C.c_int, C.c_uint64, _dp]
        L.ref_set_threads.argtypes = [C.c_int]
        for fn in ("ref_power_method", "ref_dacg_smallest"):
            getattr(L, fn).argtypes = [C.c_int, C.c_int64, C.c_int64, _i64p, _i64p, _dp, C.c_double,
                                       C.c_int, C.c_uint64, _dp]

    def _chk(self, code):
        if code:
            _raise(code, self.L.ref_last_error().decode())

    def set_threads(self, t):
        self.L.ref_set_threads(int(t))

    def cheb_params(self, alpha, beta, m, scale=1.0):
        tds = np.zeros(3)
        rho = np.zeros(max(m, 0) + 1)
        self._chk(self.L.ref_cheb_params(alpha, beta, m, scale, _ptr(tds), _ptr(rho)))
        return {"theta": tds[0], "delta": tds[1], "sigma": tds[2], "rho": rho, "m": m, "tds": tds}

    def eval_poly(self, alpha, beta, m, scale, lams):
        lams = np.ascontiguousarray(lams, dtype=np.float64)
        out = np.empty(len(lams))
        self._chk(self.L.ref_eval_poly(alpha, beta, m, scale, _ptr(lams), len(lams), _ptr(out)))
        return out

    def newton_params(self, alpha, beta, nlev, scale=1.0):
        z = np.zeros(nlev + 1)
        self._chk(self.L.ref_newton_params(alpha, beta, nlev, scale, _ptr(z)))
        return z

    def analytic_extremes(self, dim, nx, scaled=True):
        lo, hi = C.c_double(), C.c_double()
        self._chk(self.L.ref_analytic_extremes(0 if dim == 3 else 1, nx, int(scaled),
                                               C.byref(lo), C.byref(hi)))
        return lo.value, hi.value

    def random_uniform(self, n, seed):
        out = np.empty(n)
        self._chk(self.L.ref_random_uniform(n, seed, _ptr(out)))
        return out

    @staticmethod
    def _csr(csr):
        if csr is None:
            return 0, None, None, None, []
        rp = np.ascontiguousarray(csr[0], dtype=np.int64)
        ci = np.ascontiguousarray(csr[1], dtype=np.int64)
        va = np.ascontiguousarray(csr[2], dtype=np.float64)
        return len(rp) - 1, _ptr(rp, _i64p), _ptr(ci, _i64p), _ptr(va), [rp, ci, va]

    def _n(self, kind, nx, csr):
        if kind in ("lap3d", "lap3d_assembled"):
            return nx ** 3
        if kind in ("lap2d", "lap2d_assembled"):
            return nx ** 2
        return len(csr[0]) - 1

    def apply(self, kind, x, nx=0, csr=None, reps=1):
        n, rp, ci, va, keep = self._csr(csr)
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(self._n(kind, nx, csr))
        self._chk(self.L.ref_apply(REF_KIND[kind], nx, n, rp, ci, va, _ptr(x), _ptr(y), reps))
        return y

    def apply_chebyshev(self, kind, alpha, beta, m, scale, r, nx=0, csr=None):
        n, rp, ci, va, keep = self._csr(csr)
        r = np.ascontiguousarray(r, dtype=np.float64)
        out = np.empty(self._n(kind, nx, csr))
        mv = C.c_uint64()
        self._chk(self.L.ref_apply_chebyshev(REF_KIND[kind], nx, n, rp, ci, va, alpha, beta, m,
                                             scale, _ptr(r), _ptr(out), C.byref(mv)))
        return out, mv.value

    def apply_newton(self, kind, alpha, beta, nlev, scale, r, nx=0, csr=None):
        n, rp, ci, va, keep = self._csr(csr)
        r = np.ascontiguousarray(r, dtype=np.float64)
        out = np.empty(self._n(kind, nx, csr))
        self._chk(self.L.ref_apply_newton(REF_KIND[kind], nx, n, rp, ci, va, alpha, beta, nlev,
                                          scale, _ptr(r), _ptr(out)))
        return out

    def pcg_solve(self, kind, alpha, beta, m, scale, nx=0, csr=None, b=None, seed=20240801,
                  tol=1e-8, maxit=20000, want_x=True):
        """m < 0: plain CG. b None: b = A x_true, x_true = random_uniform_vector(n, seed)."""
        n, rp, ci, va, keep = self._csr(csr)
        N = self._n(kind, nx, csr)
        x = np.empty(N) if want_x else None
        b_out = np.empty(N) if (b is None and want_x) else None
        bp = None if b is None else np.ascontiguousarray(b, dtype=np.float64)
        rep = Report()
        self._chk(self.L.ref_pcg_solve(REF_KIND[kind], nx, n, rp, ci, va, alpha, beta, m, scale,
                                       _ptr(bp), seed, tol, maxit, _ptr(x), _ptr(b_out),
                                       C.byref(rep)))
        return x, (b_out if b is None else bp), rep.as_dict()

    def pcg_solve_newton(self, kind, alpha, beta, nlev, scale, nx=0, csr=None, b=None,
                         seed=20240801, tol=1e-8, maxit=20000):
        """pcg_solve with NewtonPreconditioner(newton_params(alpha, beta, nlev, scale))."""
        n, rp, ci, va, keep = self._csr(csr)
        N = self._n(kind, nx, csr)
        x = np.empty(N)
        b_out = np.empty(N) if b is None else None
        bp = None if b is None else np.ascontiguousarray(b, dtype=np.float64)
        rep = Report()
        self._chk(self.L.ref_pcg_solve_newton(REF_KIND[kind], nx, n, rp, ci, va, alpha, beta,
                                              nlev, scale, _ptr(bp), seed, tol, maxit, _ptr(x),
                                              _ptr(b_out), C.byref(rep)))
        return x, (b_out if b is None else bp), rep.as_dict()

    def mm_load(self, source, name=None):
        """load_matrix_market: text (with name) or a path -> (n, row_ptr, col_idx, values)."""
        n, nnz = C.c_int64(), C.c_int64()
        if name is not None:
            data = source.encode() if isinstance(source, str) else source
            self._chk(self.L.ref_mm_load_text(data, len(data), name.encode(), C.byref(n),
                                              C.byref(nnz)))
        else:
            self._chk(self.L.ref_mm_load_file(os.fsencode(source), C.byref(n), C.byref(nnz)))
        rp = np.empty(n.value + 1, dtype=np.int64)
        ci = np.empty(nnz.value, dtype=np.int64)
        va = np.empty(nnz.value)
        self.L.ref_mm_fetch(rp.ctypes.data_as(_i64p), ci.ctypes.data_as(_i64p), _ptr(va))
        return n.value, rp, ci, va

    def mm_save(self, n, rp, ci, va):
        """save_matrix_market(CsrMatrix(n, rp, ci, va), ostream) -> text."""
        rp = np.ascontiguousarray(rp, dtype=np.int64)
        ci = np.ascontiguousarray(ci, dtype=np.int64)
        va = np.ascontiguousarray(va, dtype=np.float64)
        t, ln = C.c_char_p(), C.c_int64()
        self._chk(self.L.ref_mm_save_text(n, rp.ctypes.data_as(_i64p), ci.ctypes.data_as(_i64p),
                                          _ptr(va), C.byref(t), C.byref(ln)))
        return C.string_at(t, ln.value).decode()

    def _eig(self, fn, kind, tol, maxit, seed, nx=0, csr=None):
        n, rp, ci, va, keep = self._csr(csr)
        out = np.zeros(4)
        self._chk(getattr(self.L, fn)(REF_KIND[kind], nx, n, rp, ci, va, tol, maxit, seed, _ptr(out)))
        return {"value": out[0], "iters": int(out[1]), "matvecs": int(out[2]),
                "converged": bool(out[3])}

    def power_method(self, kind, tol=1e-4, maxit=200, seed=20240801, nx=0, csr=None):
        return self._eig("ref_power_method", kind, tol, maxit, seed, nx, csr)

    def dacg_smallest(self, kind, tol=1e-2, maxit=5000, seed=20240801, nx=0, csr=None):
        return self._eig("ref_dacg_smallest", kind, tol, maxit, seed, nx, csr)

    def spectrum_table(self, nx, degrees, scale, solution="ones", seed=20240801):
        deg = (C.c_int * len(degrees))(*degrees)
        rows = np.zeros(6 * len(degrees))
        sol = {"ones": 0, "flat": 1, "random": 2}[solution]
        self._chk(self.L.ref_spectrum_table(nx, deg, len(degrees), scale, sol, seed, _ptr(rows)))
        return rows.reshape(-1, 6)
