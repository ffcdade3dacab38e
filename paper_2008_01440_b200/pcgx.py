# SPDX-License-Identifier: Apache-2.0
"""Python host binding of the B200 Chebyshev-PCG library (ctypes over include/pcgx.h).

This mirrors the reference's public C++ API (/root/reference/proj/include/polycg)
name for name so that parity tests read like the reference's own tests:

================================  =============================================
reference (polycg)                here
================================  =============================================
StencilOperator(lap3d, nx)        ``StencilOperator(nx, ny=None, nz=None)``
CsrMatrix(n, rp, ci, va)          ``CsrMatrix(n, row_ptr, col_idx, values)``
jacobi_scale(op)                  ``jacobi_scale(op, ctx) -> (ScaledOperator, d)``
LinearOperator::apply             ``ScaledOperator.apply(x)``
cheb_params / eval_poly           ``cheb_params`` / ``eval_poly``
apply_chebyshev                   ``apply_chebyshev(params, op, r)``
ChebyshevPreconditioner           ``ChebyshevPreconditioner(params)``
newton_params / chi_sequence      ``newton_params`` / ``chi_sequence``
apply_newton                      ``apply_newton(params, op, r)``
NewtonPreconditioner              ``NewtonPreconditioner(params)``
SolveOptions / SolveReport        ``SolveOptions`` / ``SolveReport``
pcg_solve(op, b, opts, prec)      ``pcg_solve(op, b, opts, prec)``
random_uniform_vector(n, seed)    ``random_uniform_vector(n, seed)``
analytic_extremes(kind, nx, s)    ``analytic_extremes(dim, nx, scaled)``
load/save_matrix_market           ``load_matrix_market`` / ``save_matrix_market``
std::invalid_argument             ``InvalidArgument`` (a ``ValueError``)
polycg::NumericalError            ``NumericalError``
polycg::ParseError                ``ParseError``
================================  =============================================

Every compute call runs the sm_100a kernels in ``libpcgx.so``; there is no CPU
fallback. Importing works without a GPU (host-only helpers such as
``cheb_params`` and the generators are usable); creating a ``Context`` on a
machine without a CUDA device raises ``CudaError``.
"""
from __future__ import annotations

import ctypes as C
import os
import weakref
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PCGX_LIB") or os.path.join(_HERE, "libpcgx.so")

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_vp = C.c_void_p


class PcgxError(RuntimeError):
    status = -1


class InvalidArgument(PcgxError, ValueError):
    status = 1


class NumericalError(PcgxError):
    status = 2


class CudaError(PcgxError):
    status = 3


class NcclError(PcgxError):
    status = 4


class OverflowError_(PcgxError):
    status = 5


class Unsupported(PcgxError):
    status = 6


class ParseError(PcgxError):
    """polycg::ParseError (types.hpp:16-21): unparsable input, message has file:line."""
    status = 7


class CallbackStop(PcgxError):
    """SolveOptions.on_iterate stopped the solve (its exception is chained)."""
    status = 8


_ERRS = {1: InvalidArgument, 2: NumericalError, 3: CudaError, 4: NcclError, 5: OverflowError_,
         6: Unsupported, 7: ParseError, 8: CallbackStop}


class _CsrHost(C.Structure):
    _fields_ = [("n", C.c_int64), ("nnz", C.c_int64), ("row_ptr", C.POINTER(C.c_int64)),
                ("col_idx", C.POINTER(C.c_int64)), ("values", C.POINTER(C.c_double))]


class _Cheb(C.Structure):
    _fields_ = [("m", C.c_int), ("theta", C.c_double), ("delta", C.c_double),
                ("sigma", C.c_double), ("rho", _dp)]


class _Newton(C.Structure):
    _fields_ = [("nlev", C.c_int), ("zeta", _dp)]


_ITERATE_FN = C.CFUNCTYPE(C.c_int, C.c_int64, _dp, C.c_int64, C.c_void_p)


class _Opts(C.Structure):
    _fields_ = [("tol", C.c_double), ("maxit", C.c_int), ("x0", _vp), ("flags", C.c_uint32),
                ("on_iterate", _ITERATE_FN), ("on_iterate_user", C.c_void_p)]


class _Report(C.Structure):
    _fields_ = [("iters", C.c_int64), ("ddot", C.c_int64), ("matvec", C.c_int64),
                ("prec_applies", C.c_int64), ("rel_res", C.c_double),
                ("true_rel_res", C.c_double), ("wall_time", C.c_double),
                ("converged", C.c_int64), ("kernel_launches", C.c_int64),
                ("wasted_matvec", C.c_int64), ("allreduces", C.c_int64),
                ("halo_bytes", C.c_int64), ("alg_bytes", C.c_double),
                ("spmv_equiv_bytes", C.c_double), ("step_ms", C.c_double),
                ("step_launches", C.c_int64), ("step_bytes", C.c_double),
                ("step_steps", C.c_int64)]


FLAG_TIME_KERNELS = 1
FLAG_NO_GRAPH = 2

# Exported symbols of include/pcgx.h (tests check the .so exports all of them).
SYMBOLS = [
    "pcgx_abi_version", "pcgx_last_error", "pcgx_context_create", "pcgx_nccl_unique_id",
    "pcgx_context_create_dist", "pcgx_local_group_create", "pcgx_context_create_host",
    "pcgx_context_create_ipc",
    "pcgx_context_destroy", "pcgx_context_rank",
    "pcgx_context_nranks", "pcgx_synchronize", "pcgx_kernel_launches", "pcgx_device_alloc",
    "pcgx_context_create_loopback",
    "pcgx_device_free", "pcgx_memcpy_h2d", "pcgx_memcpy_d2h", "pcgx_memcpy_d2d",
    "pcgx_host_alloc", "pcgx_host_free", "pcgx_timer_start", "pcgx_timer_stop",
    "pcgx_flush_l2", "pcgx_stencil7_create", "pcgx_slab_partition", "pcgx_chunk_plan", "pcgx_csr_create",
    "pcgx_csr_create_i32",
    "pcgx_csr_create_local",
    "pcgx_operator_destroy", "pcgx_operator_size", "pcgx_operator_local_size",
    "pcgx_operator_z0", "pcgx_operator_row0", "pcgx_operator_nnz", "pcgx_operator_storage", "pcgx_operator_matvec_count",
    "pcgx_operator_apply", "pcgx_operator_apply_device", "pcgx_cheb_params", "pcgx_cheb_eval",
    "pcgx_cheb_apply", "pcgx_cheb_apply_device", "pcgx_solve_opts_default", "pcgx_pcg_solve",
    "pcgx_pcg_solve_device", "pcgx_random_uniform_device", "pcgx_random_uniform",
    "pcgx_analytic_extremes", "pcgx_analytic_extremes_box", "pcgx_lanczos_bounds",
    "pcgx_power_method", "pcgx_dacg_smallest",
    "pcgx_gen_fe27_size", "pcgx_gen_fe27_fill", "pcgx_gen_elast27_size",
    "pcgx_gen_elast27_fill", "pcgx_newton_params", "pcgx_newton_eval", "pcgx_chi_sequence",
    "pcgx_newton_apply", "pcgx_newton_apply_device", "pcgx_pcg_solve_newton",
    "pcgx_pcg_solve_newton_device", "pcgx_mm_load", "pcgx_mm_load_text", "pcgx_csr_host_free",
    "pcgx_mm_save", "pcgx_mm_save_text", "pcgx_free_text", "pcgx_cheb_apply_steps",
]

_lib = None


def lib():
    """Load libpcgx.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2008_01440_b200.build` "
                          "(there is no CPU fallback)")
    if not os.environ.get("PCGX_NCCL_LIB"):
        # prefer the NCCL torch ships (same process may import torch later)
        import importlib.util
        spec = importlib.util.find_spec("nvidia")
        for base in (spec.submodule_search_locations or []) if spec else []:
            cand = os.path.join(base, "nccl", "lib", "libnccl.so.2")
            if os.path.exists(cand):
                os.environ["PCGX_NCCL_LIB"] = cand
                break
    L = C.CDLL(LIB_PATH)
    ctx = C.c_void_p
    op = C.c_void_p
    sig = {
        "pcgx_abi_version": (C.c_int, []),
        "pcgx_last_error": (C.c_char_p, [ctx]),
        "pcgx_context_create": (C.c_int, [C.c_int, C.POINTER(ctx)]),
        "pcgx_nccl_unique_id": (C.c_int, [C.c_void_p]),
        "pcgx_context_create_dist": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_void_p,
                                               C.POINTER(ctx)]),
        "pcgx_local_group_create": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(ctx)]),
        "pcgx_context_create_host": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_size_t,
                                               C.POINTER(ctx)]),
        "pcgx_context_create_loopback": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(ctx)]),
        "pcgx_context_create_ipc": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_size_t,
                                              C.POINTER(ctx)]),
        "pcgx_context_destroy": (None, [ctx]),
        "pcgx_context_rank": (C.c_int, [ctx]),
        "pcgx_context_nranks": (C.c_int, [ctx]),
        "pcgx_synchronize": (C.c_int, [ctx]),
        "pcgx_kernel_launches": (C.c_int64, [ctx]),
        "pcgx_device_alloc": (C.c_int, [ctx, C.c_size_t, C.POINTER(C.c_void_p)]),
        "pcgx_device_free": (C.c_int, [ctx, C.c_void_p]),
        "pcgx_memcpy_h2d": (C.c_int, [ctx, C.c_void_p, C.c_void_p, C.c_size_t]),
        "pcgx_memcpy_d2h": (C.c_int, [ctx, C.c_void_p, C.c_void_p, C.c_size_t]),
        "pcgx_memcpy_d2d": (C.c_int, [ctx, C.c_void_p, C.c_void_p, C.c_size_t]),
        "pcgx_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(C.c_void_p)]),
        "pcgx_host_free": (C.c_int, [C.c_void_p]),
        "pcgx_timer_start": (C.c_int, [ctx]),
        "pcgx_timer_stop": (C.c_int, [ctx, _dp]),
        "pcgx_flush_l2": (C.c_int, [ctx, C.c_size_t]),
        "pcgx_stencil7_create": (C.c_int, [ctx, C.c_int64, C.c_int64, C.c_int64, C.c_double,
                                           C.POINTER(op)]),
        "pcgx_csr_create": (C.c_int, [ctx, C.c_int64, _i64p, _i64p, _dp, _dp, C.POINTER(op)]),
        "pcgx_csr_create_i32": (C.c_int, [ctx, C.c_int64, _i32p, _i32p, _dp, _dp,
                                          C.POINTER(op)]),
        "pcgx_csr_create_local": (C.c_int, [ctx, C.c_int64, C.c_int64, C.c_int64, _i64p, _i64p, _dp, _dp,
                                            C.POINTER(op)]),
        "pcgx_slab_partition": (None, [C.c_int64, C.c_int, C.c_int, _i64p, _i64p]),
        "pcgx_chunk_plan": (C.c_int, [C.c_int, C.c_int64, C.c_int64, C.c_int, C.POINTER(C.c_int)]),
        "pcgx_operator_destroy": (None, [op]),
        "pcgx_operator_size": (C.c_int64, [op]),
        "pcgx_operator_local_size": (C.c_int64, [op]),
        "pcgx_operator_z0": (C.c_int64, [op]),
        "pcgx_operator_row0": (C.c_int64, [op]),
        "pcgx_operator_nnz": (C.c_int64, [op]),
        "pcgx_operator_storage": (C.c_int, [op]),
        "pcgx_operator_matvec_count": (C.c_uint64, [op]),
        "pcgx_operator_apply": (C.c_int, [ctx, op, _dp, _dp]),
        "pcgx_operator_apply_device": (C.c_int, [ctx, op, C.c_void_p, C.c_void_p]),
        "pcgx_cheb_params": (C.c_int, [C.c_double, C.c_double, C.c_int, C.c_double, _dp, _dp]),
        "pcgx_cheb_eval": (C.c_double, [C.POINTER(_Cheb), C.c_double]),
        "pcgx_cheb_apply": (C.c_int, [ctx, op, C.POINTER(_Cheb), _dp, _dp]),
        "pcgx_cheb_apply_device": (C.c_int, [ctx, op, C.POINTER(_Cheb), C.c_void_p, C.c_void_p]),
        "pcgx_cheb_apply_steps": (C.c_int, [ctx, op, C.POINTER(_Cheb), _dp, _dp]),
        "pcgx_newton_params": (C.c_int, [C.c_double, C.c_double, C.c_int, C.c_double, _dp]),
        "pcgx_newton_eval": (C.c_double, [C.POINTER(_Newton), C.c_double]),
        "pcgx_chi_sequence": (C.c_int, [C.c_double, C.c_double, C.c_int, _dp]),
        "pcgx_newton_apply": (C.c_int, [ctx, op, C.POINTER(_Newton), _dp, _dp]),
        "pcgx_newton_apply_device": (C.c_int, [ctx, op, C.POINTER(_Newton), C.c_void_p,
                                               C.c_void_p]),
        "pcgx_pcg_solve_newton": (C.c_int, [ctx, op, C.POINTER(_Newton), _dp, _dp,
                                            C.POINTER(_Opts), C.POINTER(_Report)]),
        "pcgx_pcg_solve_newton_device": (C.c_int, [ctx, op, C.POINTER(_Newton), C.c_void_p,
                                                   C.c_void_p, C.POINTER(_Opts),
                                                   C.POINTER(_Report)]),
        "pcgx_mm_load": (C.c_int, [C.c_char_p, C.POINTER(_CsrHost)]),
        "pcgx_mm_load_text": (C.c_int, [C.c_char_p, C.c_size_t, C.c_char_p, C.POINTER(_CsrHost)]),
        "pcgx_csr_host_free": (None, [C.POINTER(_CsrHost)]),
        "pcgx_mm_save": (C.c_int, [C.c_char_p, C.c_int64, _i64p, _i64p, _dp]),
        "pcgx_mm_save_text": (C.c_int, [C.c_int64, _i64p, _i64p, _dp, C.POINTER(C.c_void_p),
                                        C.POINTER(C.c_size_t)]),
        "pcgx_free_text": (None, [C.c_void_p]),
        "pcgx_solve_opts_default": (None, [C.POINTER(_Opts)]),
        "pcgx_pcg_solve": (C.c_int, [ctx, op, C.POINTER(_Cheb), _dp, _dp, C.POINTER(_Opts),
                                     C.POINTER(_Report)]),
        "pcgx_pcg_solve_device": (C.c_int, [ctx, op, C.POINTER(_Cheb), C.c_void_p, C.c_void_p,
                                            C.POINTER(_Opts), C.POINTER(_Report)]),
        "pcgx_random_uniform_device": (C.c_int, [ctx, C.c_int64, C.c_uint64, C.c_uint64,
                                                 C.c_void_p]),
        "pcgx_random_uniform": (None, [C.c_int64, C.c_uint64, C.c_uint64, _dp]),
        "pcgx_analytic_extremes": (None, [C.c_int, C.c_int64, C.c_int, _dp, _dp]),
        "pcgx_analytic_extremes_box": (None, [C.c_int64, C.c_int64, C.c_int64, _dp, _dp]),
        "pcgx_lanczos_bounds": (C.c_int, [ctx, op, C.c_int, C.c_int, C.c_uint64, _dp, _dp]),
        "pcgx_power_method": (C.c_int, [ctx, op, C.c_double, C.c_int, C.c_uint64, _dp]),
        "pcgx_dacg_smallest": (C.c_int, [ctx, op, C.c_double, C.c_int, C.c_uint64, _dp]),
        "pcgx_gen_fe27_size": (C.c_int, [C.c_int64, _i64p, _i64p]),
        "pcgx_gen_fe27_fill": (C.c_int, [C.c_int64, C.c_double, C.c_uint64, _i32p, _i32p, _dp]),
        "pcgx_gen_elast27_size": (C.c_int, [C.c_int64, _i64p, _i64p]),
        "pcgx_gen_elast27_fill": (C.c_int, [C.c_int64, C.c_double, C.c_double, C.c_double,
                                            C.c_uint64, _i32p, _i32p, _dp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    if L.pcgx_abi_version() != 1:
        raise ImportError("libpcgx ABI mismatch")
    _lib = L
    return L


def _ptr(a, t=_dp):
    return a.ctypes.data_as(t)


def _check(status, ctx_handle=None):
    if status == 0:
        return
    msg = lib().pcgx_last_error(ctx_handle).decode(errors="replace")
    raise _ERRS.get(status, PcgxError)(msg)


# ============================================================================ context

class Context:
    """One GPU (optionally one rank of a z-slab NCCL job). Mirrors the
    one-Preconditioner-per-solve ownership rule (pcg.hpp:16-19): a context runs
    one call at a time."""

    def __init__(self, device: int = 0, *, nranks: int = 1, rank: int = 0, nccl_id=None,
                 dist: bool = False, host_comm: str | None = None, ipc_comm: str | None = None,
                 mailbox_bytes: int = 0, loopback: bool = False,
                 _handle=None):
        L = lib()
        h = C.c_void_p()
        if _handle is not None:
            h = _handle
        elif loopback:
            # measurement only: a rank of a z-slab job whose neighbours are itself
            _check(L.pcgx_context_create_loopback(device, nranks, rank, C.byref(h)))
        elif host_comm is not None:
            # one rank of a multi-process job on one host, exchanging through the
            # shared-memory segment `host_comm` (pcgx_context_create_host)
            _check(L.pcgx_context_create_host(device, nranks, rank, host_comm.encode(), mailbox_bytes,
                                              C.byref(h)))
        elif ipc_comm is not None:
            # one rank of a multi-process job on one node exchanging through CUDA-IPC
            # device mailboxes, handshake segment `ipc_comm` (pcgx_context_create_ipc)
            _check(L.pcgx_context_create_ipc(device, nranks, rank, ipc_comm.encode(), mailbox_bytes,
                                             C.byref(h)))
        elif nranks == 1 and not dist:
            _check(L.pcgx_context_create(device, C.byref(h)))
        else:
            buf = C.create_string_buffer(bytes(nccl_id), 128)
            _check(L.pcgx_context_create_dist(device, nranks, rank, buf, C.byref(h)))
        self.h = h
        self.device = device
        self._children = weakref.WeakSet()  # operators / vectors to release before the context

    @classmethod
    def local_group(cls, nranks: int, devices=None):
        """P z-slab ranks in this process (drive each from its own thread)."""
        hs = (C.c_void_p * nranks)()
        devs = None if devices is None else (C.c_int * nranks)(*devices)
        _check(lib().pcgx_local_group_create(nranks, devs, hs))
        return [cls(devices[r] if devices else 0, _handle=C.c_void_p(hs[r])) for r in range(nranks)]

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(lib().pcgx_nccl_unique_id(buf))
        return buf.raw

    @property
    def rank(self):
        return lib().pcgx_context_rank(self.h)

    @property
    def nranks(self):
        return lib().pcgx_context_nranks(self.h)

    @property
    def kernel_launches(self) -> int:
        return lib().pcgx_kernel_launches(self.h)

    def synchronize(self):
        _check(lib().pcgx_synchronize(self.h), self.h)

    def timer_start(self):
        _check(lib().pcgx_timer_start(self.h), self.h)

    def timer_stop(self) -> float:
        ms = C.c_double()
        _check(lib().pcgx_timer_stop(self.h, C.byref(ms)), self.h)
        return ms.value

    def flush_l2(self, nbytes=256 << 20):
        _check(lib().pcgx_flush_l2(self.h, nbytes), self.h)

    def close(self):
        if self.h:
            for ch in list(self._children):
                ch.close()
            lib().pcgx_context_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class DeviceVector:
    """fp64 vector in HBM owned by a context."""

    def __init__(self, ctx: Context, n: int):
        self.ctx, self.n = ctx, int(n)
        p = C.c_void_p()
        _check(lib().pcgx_device_alloc(ctx.h, 8 * max(self.n, 1), C.byref(p)), ctx.h)
        self.ptr = p.value
        ctx._children.add(self)

    @classmethod
    def from_numpy(cls, ctx, a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        v = cls(ctx, a.size)
        _check(lib().pcgx_memcpy_h2d(ctx.h, v.ptr, a.ctypes.data, 8 * a.size), ctx.h)
        return v

    def numpy(self):
        out = np.empty(self.n)
        _check(lib().pcgx_memcpy_d2h(self.ctx.h, out.ctypes.data, self.ptr, 8 * self.n), self.ctx.h)
        return out

    def copy_from(self, other: "DeviceVector"):
        _check(lib().pcgx_memcpy_d2d(self.ctx.h, self.ptr, other.ptr, 8 * self.n), self.ctx.h)

    def free(self):
        if self.ptr and self.ctx.h:
            lib().pcgx_device_free(self.ctx.h, self.ptr)
        self.ptr = None

    close = free

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class PinnedBuffer:
    """Page-locked host fp64 buffer (numpy view) for the end-to-end path."""

    def __init__(self, n):
        p = C.c_void_p()
        _check(lib().pcgx_host_alloc(8 * max(int(n), 1), C.byref(p)))
        self.ptr = p.value
        self.array = np.ctypeslib.as_array(C.cast(p, _dp), shape=(int(n),))

    def free(self):
        if self.ptr:
            lib().pcgx_host_free(self.ptr)
            self.ptr = None


# ============================================================================ operators

@dataclass
class StencilOperator:
    """StencilOperator(lap3d, nx) (proj/include/polycg/linop.hpp:94-108); ny, nz
    default to nx (the builder allows boxes for config 5 weak scaling)."""
    nx: int
    ny: int | None = None
    nz: int | None = None

    def dims(self):
        return self.nx, self.ny or self.nx, self.nz or self.nx

    def size(self):
        a, b, c = self.dims()
        return a * b * c

    def diagonal(self):
        return np.full(self.size(), 6.0)


@dataclass
class CsrMatrix:
    """CsrMatrix(n, row_ptr, col_idx, values) (linop.hpp:60-85), host arrays."""
    n: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    def size(self):
        return self.n

    def nnz(self):
        return int(self.row_ptr[-1])

    def diagonal(self):
        rows = np.repeat(np.arange(self.n), np.diff(self.row_ptr))
        d = np.zeros(self.n)
        m = self.col_idx == rows
        d[rows[m]] = self.values[m]
        return d


def _csr_from_host(h: _CsrHost) -> CsrMatrix:
    n, nnz = int(h.n), int(h.nnz)
    rp = np.ctypeslib.as_array(h.row_ptr, shape=(n + 1,)).copy()
    ci = np.ctypeslib.as_array(h.col_idx, shape=(max(nnz, 1),))[:nnz].copy()
    va = np.ctypeslib.as_array(h.values, shape=(max(nnz, 1),))[:nnz].copy()
    return CsrMatrix(n, rp, ci, va)


def load_matrix_market(source, name: str | None = None) -> CsrMatrix:
    """load_matrix_market (matrix_market.cpp:55-166): a path, or (bytes/str) text with
    ``name`` used in messages like the reference's istream overload. Raises ParseError."""
    L = lib()
    h = _CsrHost()
    if isinstance(source, (bytes, str)) and name is not None:
        data = source.encode() if isinstance(source, str) else source
        st = L.pcgx_mm_load_text(data, len(data), name.encode(), C.byref(h))
    else:
        st = L.pcgx_mm_load(os.fsencode(source), C.byref(h))
    try:
        _check(st, None)
        return _csr_from_host(h)
    finally:
        L.pcgx_csr_host_free(C.byref(h))


def _csr_arrays(m: CsrMatrix):
    rp = np.ascontiguousarray(m.row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(m.col_idx, dtype=np.int64)
    va = np.ascontiguousarray(m.values, dtype=np.float64)
    return rp, ci, va


def save_matrix_market(m: CsrMatrix, path=None):
    """save_matrix_market (matrix_market.cpp:172-199). path None: return the text."""
    L = lib()
    rp, ci, va = _csr_arrays(m)
    args = (int(m.n), rp.ctypes.data_as(_i64p), ci.ctypes.data_as(_i64p), _ptr(va))
    if path is not None:
        _check(L.pcgx_mm_save(os.fsencode(path), *args), None)
        return None
    buf, ln = C.c_void_p(), C.c_size_t()
    _check(L.pcgx_mm_save_text(*args, C.byref(buf), C.byref(ln)), None)
    try:
        return C.string_at(buf, ln.value).decode()
    finally:
        L.pcgx_free_text(buf)


class ScaledOperator:
    """Device-resident D^{-1/2} A D^{-1/2} (ScaledOperator, linop.hpp:112-126)."""

    def __init__(self, ctx: Context, handle, inner):
        self.ctx, self.h, self.inner = ctx, handle, inner
        ctx._children.add(self)

    def size(self):
        return lib().pcgx_operator_size(self.h)

    def local_size(self):
        return lib().pcgx_operator_local_size(self.h)

    def z0(self):
        return lib().pcgx_operator_z0(self.h)

    def row0(self):
        """First global row owned by this rank (slab / block rows)."""
        return lib().pcgx_operator_row0(self.h)

    STORAGE = {0: "stencil", 1: "sell32", 2: "bsr3", 3: "csr_tiles", 4: "csr_chunked", 5: "dia", 6: "dia_grid", 7: "bsr3_grid"}

    def storage(self) -> str:
        """Device storage of the operator (pcgx_operator_storage)."""
        return self.STORAGE[lib().pcgx_operator_storage(self.h)]

    def nnz(self):
        return lib().pcgx_operator_nnz(self.h)

    def matvec_count(self):
        return lib().pcgx_operator_matvec_count(self.h)

    def apply(self, x):
        """y = A x. numpy in/out (host) or DeviceVector in/out (device)."""
        if isinstance(x, DeviceVector):
            y = DeviceVector(self.ctx, self.local_size())
            _check(lib().pcgx_operator_apply_device(self.ctx.h, self.h, x.ptr, y.ptr), self.ctx.h)
            return y
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.size != self.local_size():
            raise InvalidArgument(f"apply: vector length {x.size} does not match operator "
                                  f"dimension {self.local_size()}")
        y = np.empty(self.local_size())
        _check(lib().pcgx_operator_apply(self.ctx.h, self.h, _ptr(x), _ptr(y)), self.ctx.h)
        return y

    def close(self):
        if self.h and self.ctx.h:
            lib().pcgx_operator_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def jacobi_scale(op, ctx: Context):
    """jacobi_scale (proj/src/linop.cpp:340-351): returns (ScaledOperator, inv_sqrt_diag)."""
    L = lib()
    h = C.c_void_p()
    if isinstance(op, StencilOperator):
        nx, ny, nz = op.dims()
        _check(L.pcgx_stencil7_create(ctx.h, nx, ny, nz, 0.0, C.byref(h)), ctx.h)
        return ScaledOperator(ctx, h, op), None
    if isinstance(op, CsrMatrix):
        rp, ci = np.asarray(op.row_ptr), np.asarray(op.col_idx)
        va = np.ascontiguousarray(op.values, dtype=np.float64)
        if rp.dtype == np.int32 and ci.dtype == np.int32:
            _check(L.pcgx_csr_create_i32(ctx.h, op.n, _ptr(np.ascontiguousarray(rp), _i32p),
                                         _ptr(np.ascontiguousarray(ci), _i32p), _ptr(va), None,
                                         C.byref(h)), ctx.h)
        else:
            rp = np.ascontiguousarray(rp, dtype=np.int64)
            ci = np.ascontiguousarray(ci, dtype=np.int64)
            _check(L.pcgx_csr_create(ctx.h, op.n, _ptr(rp, _i64p), _ptr(ci, _i64p), _ptr(va),
                                     None, C.byref(h)), ctx.h)
        return ScaledOperator(ctx, h, op), None
    raise InvalidArgument("jacobi_scale: unsupported operator type")


def csr_block_rows(ctx: Context, n, row_ptr, col_idx, values, row0=None):
    """Jacobi-scaled block-row CsrMatrix from this rank's rows only
    (pcgx_csr_create_local): row_ptr (n_local + 1, any base) / col_idx (global) /
    values of rows [row0, row0 + n_local): the pcgx_slab_partition block of the rows
    (row0 None), or on every rank whole 3 x 3 block rows / whole node planes of a
    cubic grid (the partitions that keep BSR-3 / the offset storage)."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int64)
    va = np.ascontiguousarray(values, dtype=np.float64)
    nl = len(rp) - 1
    if row0 is None:
        row0, _ = slab_partition(n, ctx.nranks, ctx.rank)
    h = C.c_void_p()
    _check(lib().pcgx_csr_create_local(ctx.h, n, row0, nl, _ptr(rp, _i64p), _ptr(ci, _i64p), _ptr(va), None,
                                       C.byref(h)), ctx.h)
    return ScaledOperator(ctx, h, None)


# ============================================================================ polynomial

@dataclass
class ChebyshevParams:
    """ChebyshevParams (polyprec.hpp:36-45)."""
    m: int
    alpha: float
    beta: float
    scale: float
    theta: float
    delta: float
    sigma: float
    rho: np.ndarray = field(repr=False)

    def _c(self):
        s = _Cheb()
        s.m, s.theta, s.delta, s.sigma = self.m, self.theta, self.delta, self.sigma
        self._rho_keep = np.ascontiguousarray(self.rho, dtype=np.float64)
        s.rho = _ptr(self._rho_keep)
        return s


def cheb_params(alpha, beta, m, scale=1.0) -> ChebyshevParams:
    """cheb_params (polyprec.cpp:56-79), bit-exact, with the positivity check."""
    tds = np.zeros(3)
    rho = np.zeros(max(int(m), 0) + 1)
    st = lib().pcgx_cheb_params(alpha, beta, int(m), scale, _ptr(tds), _ptr(rho))
    _check(st, None)
    return ChebyshevParams(int(m), alpha, beta, scale, tds[0], tds[1], tds[2], rho)


def eval_poly(params, lam: float) -> float:
    """eval_poly (polyprec.cpp:81-100), Chebyshev or Newton form."""
    if isinstance(params, NewtonParams):
        return lib().pcgx_newton_eval(C.byref(params._c()), lam)
    return lib().pcgx_cheb_eval(C.byref(params._c()), lam)


@dataclass
class NewtonParams:
    """NewtonParams (polyprec.hpp:22-31)."""
    nlev: int
    alpha0: float
    beta0: float
    scale: float
    zeta: np.ndarray = field(repr=False)

    def degree(self):
        return (1 << self.nlev) - 1

    def _c(self):
        s = _Newton()
        s.nlev = self.nlev
        self._zeta_keep = np.ascontiguousarray(self.zeta, dtype=np.float64)
        s.zeta = _ptr(self._zeta_keep)
        return s


def newton_params(alpha0, beta0, nlev, scale=1.0) -> NewtonParams:
    """newton_params (polyprec.cpp:27-54), bit-exact, with the positivity check."""
    zeta = np.zeros(max(int(nlev), 0) + 1)
    _check(lib().pcgx_newton_params(alpha0, beta0, int(nlev), scale, _ptr(zeta)), None)
    return NewtonParams(int(nlev), alpha0, beta0, scale, zeta)


def chi_sequence(alpha, beta, nlev) -> np.ndarray:
    """chi_sequence (polyprec.cpp:102-123)."""
    chi = np.zeros(max(int(nlev), 0))
    _check(lib().pcgx_chi_sequence(alpha, beta, int(nlev), _ptr(chi)), None)
    return chi


class ChebyshevPreconditioner:
    """ChebyshevPreconditioner (pcg.hpp:42-55)."""

    def __init__(self, params: ChebyshevParams):
        self._params = params

    def params(self):
        return self._params

    def degree(self):
        return self._params.m

    def apply(self, op: ScaledOperator, r):
        return apply_chebyshev(self._params, op, r)


def apply_chebyshev(params: ChebyshevParams, op: ScaledOperator, r):
    """out = p_m(A) r (polyprec.cpp:169-198) on the device."""
    cp = params._c()
    if isinstance(r, DeviceVector):
        out = DeviceVector(op.ctx, op.local_size())
        _check(lib().pcgx_cheb_apply_device(op.ctx.h, op.h, C.byref(cp), r.ptr, out.ptr), op.ctx.h)
        return out
    r = np.ascontiguousarray(r, dtype=np.float64)
    if r.size != op.local_size():
        raise InvalidArgument("apply_chebyshev: vector length mismatch")
    out = np.empty(op.local_size())
    _check(lib().pcgx_cheb_apply(op.ctx.h, op.h, C.byref(cp), _ptr(r), _ptr(out)), op.ctx.h)
    return out


class NewtonPreconditioner:
    """NewtonPreconditioner (pcg.hpp:27-40)."""

    def __init__(self, params: NewtonParams):
        self._params = params

    def params(self):
        return self._params

    def degree(self):
        return self._params.degree()

    def apply(self, op: ScaledOperator, r):
        return apply_newton(self._params, op, r)


def apply_newton(params: NewtonParams, op: ScaledOperator, r):
    """out = P_nlev(A) r (polyprec.cpp:135-160) on the device: 2^nlev - 1 matvecs."""
    cp = params._c()
    if isinstance(r, DeviceVector):
        out = DeviceVector(op.ctx, op.local_size())
        _check(lib().pcgx_newton_apply_device(op.ctx.h, op.h, C.byref(cp), r.ptr, out.ptr),
               op.ctx.h)
        return out
    r = np.ascontiguousarray(r, dtype=np.float64)
    if r.size != op.local_size():
        raise InvalidArgument("apply_newton: vector length mismatch")
    out = np.empty(op.local_size())
    _check(lib().pcgx_newton_apply(op.ctx.h, op.h, C.byref(cp), _ptr(r), _ptr(out)), op.ctx.h)
    return out


def apply_chebyshev_steps(params: ChebyshevParams, op: ScaledOperator, r) -> np.ndarray:
    """Every degree step x_1..x_m of apply_chebyshev (the parity entry): shape (m, n)."""
    r = np.ascontiguousarray(r, dtype=np.float64)
    if r.size != op.local_size():
        raise InvalidArgument("apply_chebyshev: vector length mismatch")
    out = np.empty((max(params.m, 0), op.local_size()))
    cp = params._c()
    _check(lib().pcgx_cheb_apply_steps(op.ctx.h, op.h, C.byref(cp), _ptr(r), _ptr(out)), op.ctx.h)
    return out


# ============================================================================ solver

@dataclass
class SolveOptions:
    """SolveOptions (pcg.hpp:57-64). on_iterate(it, x) is called after every
    iteration (pcg.cpp:88) with a host numpy copy of the current x (the rank's part
    on a multi-rank context); an exception it raises stops the solve and propagates."""
    tol: float = 1e-8
    maxit: int = 20000
    x0: object = None
    flags: int = 0
    on_iterate: object = None


@dataclass
class SolveReport:
    """SolveReport (pcg.hpp:73-82) + device extensions."""
    iters: int = 0
    ddot: int = 0
    matvec: int = 0
    prec_applies: int = 0
    rel_res: float = 0.0
    true_rel_res: float = 0.0
    wall_time: float = 0.0
    converged: bool = False
    kernel_launches: int = 0
    wasted_matvec: int = 0
    allreduces: int = 0
    halo_bytes: int = 0
    alg_bytes: float = 0.0
    spmv_equiv_bytes: float = 0.0
    step_ms: float = 0.0
    step_launches: int = 0
    step_bytes: float = 0.0
    step_steps: int = 0

    @classmethod
    def _from(cls, r: _Report):
        d = {f: getattr(r, f) for f, _ in _Report._fields_}
        d["converged"] = bool(d["converged"])
        return cls(**d)


def pcg_solve(op: ScaledOperator, b, opts: SolveOptions | None = None,
              prec: ChebyshevPreconditioner | NewtonPreconditioner | None = None, x_out=None):
    """pcg_solve (pcg.cpp:10-117) on the GPU.

    b numpy -> host entry (b copied in, x copied out inside the call; returns
    numpy x). b DeviceVector -> device entry (returns a DeviceVector x, or
    writes into x_out).
    """
    opts = opts or SolveOptions()
    L = lib()
    o = _Opts()
    L.pcgx_solve_opts_default(C.byref(o))
    o.tol, o.maxit, o.flags = opts.tol, opts.maxit, opts.flags
    caught = []
    if opts.on_iterate is not None:
        def _tramp(it, xp, n, _user):
            try:
                opts.on_iterate(int(it), np.ctypeslib.as_array(xp, shape=(n,)).copy())
                return 0
            except BaseException as e:  # noqa: BLE001 - rethrown after the C call
                caught.append(e)
                return 1
        o.on_iterate = _ITERATE_FN(_tramp)
    rep = _Report()
    newton = isinstance(prec, NewtonPreconditioner)
    cp = C.byref(prec.params()._c()) if prec is not None else None
    f_dev = L.pcgx_pcg_solve_newton_device if newton else L.pcgx_pcg_solve_device
    f_host = L.pcgx_pcg_solve_newton if newton else L.pcgx_pcg_solve
    if isinstance(b, DeviceVector):
        if x_out is not None and (not isinstance(x_out, DeviceVector) or x_out.n != op.local_size()):
            raise InvalidArgument("pcg_solve: x_out must be a DeviceVector of "
                                  f"{op.local_size()} elements for a device rhs")
        x = x_out or DeviceVector(op.ctx, op.local_size())
        if opts.x0 is not None:
            o.x0 = opts.x0.ptr
        st = f_dev(op.ctx.h, op.h, cp, b.ptr, x.ptr, C.byref(o), C.byref(rep))
        if caught:
            raise caught[0]
        _check(st, op.ctx.h)
        return x, SolveReport._from(rep)
    b = np.ascontiguousarray(b, dtype=np.float64)
    if b.size != op.local_size():
        raise InvalidArgument("pcg_solve: rhs length mismatch")
    if x_out is None:
        x = np.empty(op.local_size())
    else:
        x = x_out
        if (not isinstance(x, np.ndarray) or x.dtype != np.float64 or not x.flags.c_contiguous
                or not x.flags.writeable or x.size != op.local_size()):
            raise InvalidArgument("pcg_solve: x_out must be a writeable C-contiguous float64 array of "
                                  f"{op.local_size()} elements")
    x0 = None
    if opts.x0 is not None:
        x0 = np.ascontiguousarray(opts.x0, dtype=np.float64)
        if x0.size != b.size:
            raise InvalidArgument("pcg_solve: x0 length mismatch")
        o.x0 = x0.ctypes.data
    st = f_host(op.ctx.h, op.h, cp, _ptr(b), x.ctypes.data_as(_dp), C.byref(o), C.byref(rep))
    if caught:
        raise caught[0]
    _check(st, op.ctx.h)
    return x, SolveReport._from(rep)


def lanczos_bounds(op: ScaledOperator, steps_hi=20, steps=30, seed=20240801):
    lo, hi = C.c_double(), C.c_double()
    _check(lib().pcgx_lanczos_bounds(op.ctx.h, op.h, steps_hi, steps, seed, C.byref(lo),
                                     C.byref(hi)), op.ctx.h)
    return lo.value, hi.value


@dataclass
class EigResult:
    """EigResult (eigenest.hpp:21-30; the per-iteration trace is not kept)."""
    value: float
    iters: int
    matvecs: int
    converged: bool


@dataclass
class EigOptions:
    """EigOptions (eigenest.hpp:15-19)."""
    tol: float = 1e-4
    maxit: int = 200
    seed: int = 20240801


def _eig(fn, op, opts):
    out = np.zeros(4)
    _check(getattr(lib(), fn)(op.ctx.h, op.h, opts.tol, opts.maxit, opts.seed, _ptr(out)), op.ctx.h)
    return EigResult(float(out[0]), int(out[1]), int(out[2]), bool(out[3]))


def power_method(op: ScaledOperator, opts: EigOptions | None = None) -> EigResult:
    """power_method (eigenest.cpp:48-79) on the device."""
    return _eig("pcgx_power_method", op, opts or EigOptions())


def dacg_smallest(op: ScaledOperator, opts: EigOptions | None = None) -> EigResult:
    """dacg_smallest (eigenest.cpp:81-167) on the device."""
    return _eig("pcgx_dacg_smallest", op, opts or EigOptions(tol=1e-2, maxit=5000))


def estimate_bounds(op: ScaledOperator, power_opts: EigOptions | None = None,
                    dacg_opts: EigOptions | None = None):
    """estimate_bounds (eigenest.cpp:169-185): (alpha0, beta0, power result, dacg result)."""
    hi = power_method(op, power_opts)
    lo = dacg_smallest(op, dacg_opts)
    if not (lo.value > 0.0) or lo.value > hi.value:
        raise NumericalError("estimate_bounds: estimates violate 0 < alpha0 <= beta0")
    return lo.value, hi.value, hi, lo


# ============================================================================ inputs

def random_uniform_vector(n, seed, offset=0, ctx: Context | None = None):
    """random_uniform_vector (eigenest.cpp:22-30). Host numpy, or a DeviceVector
    generated on the GPU when ctx is given (bit-identical)."""
    if ctx is None:
        out = np.empty(int(n))
        lib().pcgx_random_uniform(int(n), seed, offset, _ptr(out))
        return out
    v = DeviceVector(ctx, n)
    _check(lib().pcgx_random_uniform_device(ctx.h, int(n), seed, offset, v.ptr), ctx.h)
    return v


def slab_partition(nz, nranks, rank):
    """(z0, nz_local) of rank's z-slab (the partition every pcgx rank uses)."""
    z0, nl = C.c_int64(), C.c_int64()
    lib().pcgx_slab_partition(nz, nranks, rank, C.byref(z0), C.byref(nl))
    return z0.value, nl.value


def chunk_plan(span, tiles, slots=148, long_chunks=True):
    """Chunk heights of a temporally blocked pass over `span` planes (pcgx_chunk_plan)."""
    h = (C.c_int * 48)()
    n = lib().pcgx_chunk_plan(span, tiles, slots, 1 if long_chunks else 0, h)
    return [h[i] for i in range(n)]


def analytic_extremes(dim, nx, scaled=True):
    lo, hi = C.c_double(), C.c_double()
    lib().pcgx_analytic_extremes(dim, nx, int(scaled), C.byref(lo), C.byref(hi))
    return lo.value, hi.value


def analytic_extremes_box(nx, ny, nz):
    lo, hi = C.c_double(), C.c_double()
    lib().pcgx_analytic_extremes_box(nx, ny, nz, C.byref(lo), C.byref(hi))
    return lo.value, hi.value


def gen_fe27(nx, sigma=1.0, seed=20240801) -> CsrMatrix:
    """Config 3 matrix (int32 CSR): Q1 heterogeneous diffusion, lognormal cells."""
    n, nnz = C.c_int64(), C.c_int64()
    _check(lib().pcgx_gen_fe27_size(nx, C.byref(n), C.byref(nnz)))
    rp = np.empty(n.value + 1, dtype=np.int32)
    ci = np.empty(nnz.value, dtype=np.int32)
    va = np.empty(nnz.value)
    _check(lib().pcgx_gen_fe27_fill(nx, sigma, seed, _ptr(rp, _i32p), _ptr(ci, _i32p), _ptr(va)))
    return CsrMatrix(n.value, rp, ci, va)


def gen_elast27(nx, lam=1.0, mu=0.5, eps=0.1, seed=20240801) -> CsrMatrix:
    """Config 4 matrix (int32 CSR): 3-dof Q1 elasticity, 3x3 blocks, per-cell scaling."""
    n, nnz = C.c_int64(), C.c_int64()
    _check(lib().pcgx_gen_elast27_size(nx, C.byref(n), C.byref(nnz)))
    rp = np.empty(n.value + 1, dtype=np.int32)
    ci = np.empty(nnz.value, dtype=np.int32)
    va = np.empty(nnz.value)
    _check(lib().pcgx_gen_elast27_fill(nx, lam, mu, eps, seed, _ptr(rp, _i32p), _ptr(ci, _i32p),
                                       _ptr(va)))
    return CsrMatrix(n.value, rp, ci, va)
