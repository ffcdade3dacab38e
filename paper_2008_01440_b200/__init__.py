# SPDX-License-Identifier: Apache-2.0
"""B200-native Chebyshev-polynomial-preconditioned CG (arxiv 2008.01440 hot path).

The product is the native library ``libpcgx.so`` (sm_100a kernels + C++ host
orchestration behind the C ABI in include/pcgx.h). This package holds its
sources (csrc/), its build recipe (build.py) and the Python host binding
(pcgx.py) that mirrors the reference's polycg API.
"""
from .pcgx import (  # noqa: F401
    ChebyshevParams, ChebyshevPreconditioner, Context, CsrMatrix, CudaError, DeviceVector,
    InvalidArgument, NumericalError, PcgxError, PinnedBuffer, ScaledOperator, SolveOptions,
    SolveReport, StencilOperator, analytic_extremes, analytic_extremes_box, apply_chebyshev,
    FLAG_NO_GRAPH, FLAG_TIME_KERNELS, cheb_params, eval_poly, gen_elast27, gen_fe27, jacobi_scale, lanczos_bounds, lib,
    pcg_solve, random_uniform_vector, slab_partition, EigOptions, EigResult, power_method,
    dacg_smallest, estimate_bounds, NewtonParams, NewtonPreconditioner, apply_newton,
    newton_params, chi_sequence, ParseError, load_matrix_market, save_matrix_market,
    apply_chebyshev_steps,
)
