/* SPDX-License-Identifier: Apache-2.0
 *
 * TEST INFRASTRUCTURE ONLY. A plain-C, single-threaded restatement of the
 * reference's Chebyshev-PCG hot path (/root/reference/proj), used by tests/ as
 * the parity checker and by bench.py's cpu_baseline leg. Nothing in the
 * product (paper_2008_01440_b200/) links, loads or calls it.
 *
 * Pinned against the reference itself (oracle/_ref/libpolycg_ref.so built from
 * the reference sources) through tests/golden/ fixtures; see tests/test_oracle.py.
 */
#ifndef POLYCG_ORACLE_H
#define POLYCG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes mirror the reference's exception classes:
 * 0 ok, 1 std::invalid_argument, 2 polycg::NumericalError. */
enum { OR_OK = 0, OR_INVALID = 1, OR_NUMERICAL = 2 };

const char* or_last_error(void);

/* Operator = D^{-1/2} A D^{-1/2} (ScaledOperator over the inner operator).
 *  kind 0: 3D 7-point FD Laplacian on nx*ny*nz (diag 6, off -1, Dirichlet),
 *          i fastest, then j, then k (proj/src/linop.cpp:236-258);
 *  kind 1: 2D 5-point on nx*ny (proj/src/linop.cpp:218-235);
 *  kind 2: CSR, int64 row_ptr/col_idx, fp64 values (proj/src/linop.cpp:171-187).
 * d = inv_sqrt_diag (n entries). For kinds 0/1 d may be NULL: every entry is
 * then 1/sqrt(6) resp. 1/sqrt(4), exactly what jacobi_scale computes from the
 * constant StencilOperator::diagonal (linop.cpp:209-211, 340-351). */
typedef struct {
  int kind;
  int64_t nx, ny, nz;
  int64_t n;
  const int64_t* row_ptr;
  const int64_t* col_idx;
  const double* values;
  const double* d;
} or_op;

typedef struct {
  int64_t iters, ddot, matvec, prec_applies;
  double rel_res, true_rel_res, wall_time;
  int64_t converged;
} or_report;

/* cheb_params (proj/src/polyprec.cpp:56-79). tds = {theta, delta, sigma}, rho[m+1]. */
int or_cheb_params(double alpha, double beta, int m, double scale, double* tds, double* rho);
/* eval_poly, Chebyshev form (polyprec.cpp:89-100). */
double or_eval_poly(const double* tds, const double* rho, int m, double lambda);
/* newton_params (polyprec.cpp:27-54): zeta[nlev+1]. */
int or_newton_params(double alpha0, double beta0, int nlev, double scale, double* zeta);

/* analytic_extremes (linop.cpp:382-390), dim 2 or 3, cubic grid. */
void or_analytic_extremes(int dim, int64_t nx, int scaled, double* lo, double* hi);
/* Builder generalisation to a 3D box nx*ny*nz (scaled): the extremes of
 * (1/3) * sum_d 2*(2 sin^2(pi k_d h_d / 2)). Equals or_analytic_extremes at
 * nx = ny = nz up to rounding (not bitwise; the cubic form is used there). */
void or_analytic_extremes_box(int64_t nx, int64_t ny, int64_t nz, double* lo, double* hi);

/* random_uniform_vector (eigenest.cpp:13-30) elements [offset, offset+n). */
void or_random_uniform(int64_t n, uint64_t seed, uint64_t offset, double* out);

/* y = (D^{-1/2} A D^{-1/2}) x  (ScaledOperator::apply_impl, linop.cpp:271-275). */
int or_apply(const or_op* op, const double* x, double* y);
/* y = A x, unscaled inner operator. */
int or_apply_inner(const or_op* op, const double* x, double* y);

/* out = p_m(A) r (apply_chebyshev, polyprec.cpp:169-198). */
int or_apply_chebyshev(const or_op* op, const double* tds, const double* rho, int m,
                       const double* r, double* out);
/* apply_newton (polyprec.cpp:135-167). */
int or_apply_newton(const or_op* op, const double* zeta, int nlev, const double* r, double* out);

/* pcg_solve (pcg.cpp:10-117). m < 0: no preconditioner. x0 may be NULL. */
int or_pcg_solve(const or_op* op, const double* tds, const double* rho, int m, const double* b,
                 const double* x0, double tol, int maxit, double* x, or_report* rep);

/* pcg_solve with a NewtonPreconditioner (pcg.hpp:27-40): zeta[nlev+1]. */
int or_pcg_solve_newton(const or_op* op, const double* zeta, int nlev, const double* b,
                        const double* x0, double tol, int maxit, double* x, or_report* rep);

/* power_method / dacg_smallest (eigenest.cpp:48-167): out = {value, iters,
 * matvecs, converged}. */
int or_power_method(const or_op* op, double tol, int maxit, uint64_t seed, double* out);
int or_dacg_smallest(const or_op* op, double tol, int maxit, uint64_t seed, double* out);

/* Lanczos extremal Ritz values (builder-defined bound estimator, not in the
 * reference; the product's pcgx_lanczos_bounds follows the same algorithm).
 * start = seeded random_uniform_vector(n, seed) normalised; `steps` steps of the
 * three-term recurrence WITHOUT reorthogonalisation; Ritz values of the steps x
 * steps tridiagonal by Sturm bisection. lo/hi = smallest/largest Ritz value. */
int or_lanczos(const or_op* op, int steps, uint64_t seed, double* lo, double* hi,
               double* alphas, double* betas);
/* Extremal eigenvalues of a symmetric tridiagonal (diag a[k], offdiag b[k], k<k-1)
 * by Sturm bisection to full precision. */
void or_tridiag_extremes(int k, const double* a, const double* b, double* lo, double* hi);

#ifdef __cplusplus
}
#endif
#endif
