/* SPDX-License-Identifier: Apache-2.0
 *
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference hot path, used
 * as the parity checker (tests/) and the cpu_baseline leg (bench.py). Never
 * linked into the product. Every function cites the reference lines it follows.
 *
 * Arithmetic discipline: one IEEE binary64 op per reference operator, in the
 * reference's evaluation order, built with -ffp-contract=off (no FMA), exactly
 * as the reference's Release build on baseline x86-64 (proj/CMakeLists.txt:6-8).
 * Reductions (dot, norm) are sequential left-to-right: Eigen's own packet order
 * is not reproducible without Eigen (absent from the image); this is the same
 * order oracle/eigen_shim gives the compiled reference, so the two agree
 * bitwise (tests/test_oracle.py pins that).
 */
#include "polycg_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static char g_err[512];
const char* or_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

/* ---------------------------------------------------------------- params */

/* polyprec.cpp:89-100 */
double or_eval_poly(const double* tds, const double* rho, int m, double lambda) {
  const double theta = tds[0], delta = tds[1], sigma = tds[2];
  double p_prev = 0.0;
  double p = 1.0 / theta;
  for (int k = 1; k <= m; ++k) {
    /* rho[k] * (2.0*sigma*(1.0 - lambda/theta)*p - rho[k-1]*p_prev + 2.0/delta) */
    const double t1 = ((2.0 * sigma) * (1.0 - lambda / theta)) * p;
    const double t2 = rho[k - 1] * p_prev;
    const double p_new = rho[k] * ((t1 - t2) + 2.0 / delta);
    p_prev = p;
    p = p_new;
  }
  return p;
}

/* polyprec.cpp:56-79, positivity check :13-23 */
int or_cheb_params(double alpha, double beta, int m, double scale, double* tds, double* rho) {
  if (!(alpha > 0.0)) return fail(OR_INVALID, "cheb_params: alpha must be positive");
  if (!(beta > alpha))
    return fail(OR_INVALID, "cheb_params: need alpha < beta (delta = 0 divides by zero)");
  if (m < 0) return fail(OR_INVALID, "cheb_params: m must be >= 0");
  if (!(scale >= 1.0)) return fail(OR_INVALID, "cheb_params: scale must be >= 1");
  const double theta = (scale * 0.5) * (alpha + beta); /* :69, left-assoc */
  const double delta = 0.5 * (beta - alpha);           /* :70 */
  const double sigma = theta / delta;                  /* :71 */
  tds[0] = theta;
  tds[1] = delta;
  tds[2] = sigma;
  rho[0] = 1.0 / sigma;
  for (int k = 1; k <= m; ++k) rho[k] = 1.0 / (2.0 * sigma - rho[k - 1]);
  for (int g = 0; g < 1000; ++g) {
    const double lam = alpha + (beta - alpha) * (double)g / (1000 - 1);
    if (!(or_eval_poly(tds, rho, m, lam) > 0.0)) {
      snprintf(g_err, sizeof g_err, "polynomial preconditioner not positive at lambda = %f", lam);
      return OR_NUMERICAL;
    }
  }
  return OR_OK;
}

static double newton_eval(const double* zeta, int nlev, double lambda) { /* polyprec.cpp:81-87 */
  double r = zeta[0];
  for (int j = 1; j <= nlev; ++j) r = zeta[j] * (2.0 * r - (lambda * r) * r);
  return r;
}

/* polyprec.cpp:27-54 */
int or_newton_params(double alpha0, double beta0, int nlev, double scale, double* zeta) {
  if (!(alpha0 > 0.0) || !(beta0 >= alpha0))
    return fail(OR_INVALID, "newton_params: need 0 < alpha0 <= beta0");
  if (nlev < 0) return fail(OR_INVALID, "newton_params: nlev must be >= 0");
  if (!(scale >= 1.0)) return fail(OR_INVALID, "newton_params: scale must be >= 1");
  const double theta = 0.5 * (alpha0 + beta0);
  const double delta = 0.5 * (beta0 - alpha0);
  zeta[0] = 1.0 / (scale * theta);
  if (nlev >= 1) {
    const double t = (scale * theta - delta) * zeta[0];
    zeta[1] = 2.0 / ((1.0 + 2.0 * t) - t * t);
    for (int j = 2; j <= nlev; ++j) {
      const double z = zeta[j - 1];
      zeta[j] = 2.0 / ((1.0 + 2.0 * z) - z * z);
    }
  }
  for (int g = 0; g < 1000; ++g) {
    const double lam = alpha0 + (beta0 - alpha0) * (double)g / (1000 - 1);
    if (!(newton_eval(zeta, nlev, lam) > 0.0)) {
      snprintf(g_err, sizeof g_err, "polynomial preconditioner not positive at lambda = %f", lam);
      return OR_NUMERICAL;
    }
  }
  return OR_OK;
}

/* linop.cpp:382-390 */
void or_analytic_extremes(int dim, int64_t nx, int scaled, double* lo, double* hi) {
  const double pi = 3.14159265358979323846;
  const double h = 1.0 / (double)(nx + 1);
  const double s = sin(pi * h / 2.0);
  const double c = cos(pi * h / 2.0);
  const double factor = ((scaled ? 2.0 / (double)(2 * dim) : 2.0) * 2.0) * (double)dim;
  *lo = (factor * s) * s;
  *hi = (factor * c) * c;
}

void or_analytic_extremes_box(int64_t nx, int64_t ny, int64_t nz, double* lo, double* hi) {
  const double pi = 3.14159265358979323846;
  const int64_t dims[3] = {nx, ny, nz};
  double smin = 0.0, smax = 0.0;
  for (int d = 0; d < 3; ++d) {
    const double h = 1.0 / (double)(dims[d] + 1);
    const double s = sin(pi * h / 2.0);
    const double c = cos(pi * h / 2.0);
    smin += s * s;
    smax += c * c;
  }
  /* scaled eigenvalue (1/6) sum_d 4 sin^2(pi k_d h_d / 2) = (2/3) sum_d sin^2 */
  *lo = (2.0 / 3.0) * smin;
  *hi = (2.0 / 3.0) * smax;
}

/* eigenest.cpp:13-30: v_i = 2u-1, u = (splitmix64 >> 11) * 2^-53, state += gamma per draw */
void or_random_uniform(int64_t n, uint64_t seed, uint64_t offset, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    uint64_t z = seed + ((uint64_t)(offset + (uint64_t)i) + 1u) * 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    z = z ^ (z >> 31);
    const double u = (double)(z >> 11) * 0x1.0p-53;
    out[i] = 2.0 * u - 1.0;
  }
}

/* ---------------------------------------------------------------- operators */

static int64_t op_n(const or_op* op) {
  if (op->kind == 0) return op->nx * op->ny * op->nz;
  if (op->kind == 1) return op->nx * op->ny;
  return op->n;
}

/* linop.cpp:236-258 (3D) and :218-235 (2D): terms skipped at the boundary,
 * ascending column order k-1, j-1, i-1, centre, i+1, j+1, k+1. */
static void inner_apply(const or_op* op, const double* t, double* y) {
  if (op->kind == 0) {
    const int64_t nx = op->nx, ny = op->ny, nz = op->nz, nxy = nx * ny;
    for (int64_t k = 0; k < nz; ++k)
      for (int64_t j = 0; j < ny; ++j)
        for (int64_t i = 0; i < nx; ++i) {
          const int64_t r = k * nxy + j * nx + i;
          double sum = 0.0;
          if (k > 0) sum += -t[r - nxy];
          if (j > 0) sum += -t[r - nx];
          if (i > 0) sum += -t[r - 1];
          sum += 6.0 * t[r];
          if (i < nx - 1) sum += -t[r + 1];
          if (j < ny - 1) sum += -t[r + nx];
          if (k < nz - 1) sum += -t[r + nxy];
          y[r] = sum;
        }
  } else if (op->kind == 1) {
    const int64_t nx = op->nx, ny = op->ny;
    for (int64_t j = 0; j < ny; ++j)
      for (int64_t i = 0; i < nx; ++i) {
        const int64_t r = j * nx + i;
        double sum = 0.0;
        if (j > 0) sum += -t[r - nx];
        if (i > 0) sum += -t[r - 1];
        sum += 4.0 * t[r];
        if (i < nx - 1) sum += -t[r + 1];
        if (j < ny - 1) sum += -t[r + nx];
        y[r] = sum;
      }
  } else { /* linop.cpp:171-187 */
    const int64_t n = op->n;
    for (int64_t i = 0; i < n; ++i) {
      double sum = 0.0;
      for (int64_t k = op->row_ptr[i]; k < op->row_ptr[i + 1]; ++k)
        sum += op->values[k] * t[op->col_idx[k]];
      y[i] = sum;
    }
  }
}

static double op_d(const or_op* op, int64_t i) {
  if (op->d) return op->d[i];
  return 1.0 / sqrt(op->kind == 0 ? 6.0 : 4.0); /* jacobi_scale, linop.cpp:348 */
}

int or_apply_inner(const or_op* op, const double* x, double* y) {
  inner_apply(op, x, y);
  return OR_OK;
}

/* ScaledOperator::apply_impl, linop.cpp:271-275: t = d.*x; y = A t; y .*= d */
int or_apply(const or_op* op, const double* x, double* y) {
  const int64_t n = op_n(op);
  if (op->kind == 2 && !op->d) return fail(OR_INVALID, "or_apply: CSR needs d");
  double* t = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
  for (int64_t i = 0; i < n; ++i) t[i] = op_d(op, i) * x[i];
  inner_apply(op, t, y);
  for (int64_t i = 0; i < n; ++i) y[i] = y[i] * op_d(op, i);
  free(t);
  return OR_OK;
}

static double dot(int64_t n, const double* a, const double* b) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

/* ---------------------------------------------------------------- polynomial */

/* apply_chebyshev, polyprec.cpp:169-198 */
int or_apply_chebyshev(const or_op* op, const double* tds, const double* rho, int m,
                       const double* r, double* out) {
  const int64_t n = op_n(op);
  const double theta = tds[0], delta = tds[1], sigma = tds[2];
  if (m == 0) {
    for (int64_t i = 0; i < n; ++i) out[i] = r[i] / theta;
    return OR_OK;
  }
  double* x_old = (double*)malloc(sizeof(double) * (size_t)n);
  double* x = (double*)malloc(sizeof(double) * (size_t)n);
  double* z = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) x_old[i] = r[i] / theta;
  or_apply(op, r, z);
  const double c1 = 2.0 * rho[1] / delta;
  for (int64_t i = 0; i < n; ++i) x[i] = c1 * (2.0 * r[i] - z[i] / theta);
  const double c2 = 2.0 / delta, c3 = 2.0 * sigma;
  for (int k = 2; k <= m; ++k) {
    or_apply(op, x, z);
    for (int64_t i = 0; i < n; ++i) z[i] = c2 * (r[i] - z[i]);
    for (int64_t i = 0; i < n; ++i) x_old[i] = rho[k] * ((c3 * x[i] - rho[k - 1] * x_old[i]) + z[i]);
    double* tmp = x_old;
    x_old = x;
    x = tmp;
  }
  memcpy(out, x, sizeof(double) * (size_t)n);
  free(x_old);
  free(x);
  free(z);
  return OR_OK;
}

/* newton_rec / apply_newton, polyprec.cpp:135-167 */
static void newton_rec(const or_op* op, const double* zeta, int j, const double* r_in,
                       double* out, double** level, int64_t n) {
  if (j == 0) {
    for (int64_t i = 0; i < n; ++i) out[i] = zeta[0] * r_in[i];
    return;
  }
  double* u = level[j - 1];
  newton_rec(op, zeta, j - 1, r_in, u, level, n);
  or_apply(op, u, out);
  newton_rec(op, zeta, j - 1, out, out, level, n);
  for (int64_t i = 0; i < n; ++i) out[i] = zeta[j] * (2.0 * u[i] - out[i]);
}

int or_apply_newton(const or_op* op, const double* zeta, int nlev, const double* r, double* out) {
  const int64_t n = op_n(op);
  double** level = (double**)calloc((size_t)(nlev + 1), sizeof(double*));
  for (int j = 0; j < nlev; ++j) level[j] = (double*)malloc(sizeof(double) * (size_t)n);
  newton_rec(op, zeta, nlev, r, out, level, n);
  for (int j = 0; j < nlev; ++j) free(level[j]);
  free(level);
  return OR_OK;
}

/* ---------------------------------------------------------------- solver */

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* The preconditioner of a solve: Chebyshev (pcg.hpp:42-55) or Newton form
 * (pcg.hpp:27-40); m < 0 = none. */
typedef struct {
  int newton;
  const double* tds;
  const double* rho;
  const double* zeta;
  int m;  /* Chebyshev degree, or Newton nlev */
} prec_t;

static void prec_apply(const or_op* op, const prec_t* P, const double* r, double* z) {
  if (P->newton) or_apply_newton(op, P->zeta, P->m, r, z);
  else or_apply_chebyshev(op, P->tds, P->rho, P->m, r, z);
}

static int pcg_solve_impl(const or_op* op, const prec_t* P, const double* b, const double* x0,
                          double tol, int maxit, double* x, or_report* rep);

/* pcg_solve, pcg.cpp:10-117 (counters at :33,41,44,58-59,65,73,75,84,96-97,102,113,115) */
int or_pcg_solve(const or_op* op, const double* tds, const double* rho_c, int m, const double* b,
                 const double* x0, double tol, int maxit, double* x, or_report* rep) {
  const prec_t P = {0, tds, rho_c, NULL, m};
  return pcg_solve_impl(op, &P, b, x0, tol, maxit, x, rep);
}

/* pcg_solve with a NewtonPreconditioner (degree 2^nlev - 1). */
int or_pcg_solve_newton(const or_op* op, const double* zeta, int nlev, const double* b,
                        const double* x0, double tol, int maxit, double* x, or_report* rep) {
  if (nlev < 0) return fail(OR_INVALID, "apply_newton: nlev must be >= 0");
  const prec_t P = {1, NULL, NULL, zeta, nlev};
  return pcg_solve_impl(op, &P, b, x0, tol, maxit, x, rep);
}

static int pcg_solve_impl(const or_op* op, const prec_t* P, const double* b, const double* x0,
                          double tol, int maxit, double* x, or_report* rep) {
  const int m = P->m;
  const int64_t n = op_n(op);
  if (!(tol > 0.0)) return fail(OR_INVALID, "pcg_solve: tol must be positive");
  if (maxit < 1) return fail(OR_INVALID, "pcg_solve: maxit must be >= 1");
  const int mdeg = m < 0 ? 0 : (P->newton ? (1 << m) - 1 : m);
  const double t0 = now_s();
  memset(rep, 0, sizeof *rep);
  double* r = (double*)malloc(sizeof(double) * (size_t)n);
  double* z = (double*)malloc(sizeof(double) * (size_t)n);
  double* p = (double*)malloc(sizeof(double) * (size_t)n);
  double* q = (double*)malloc(sizeof(double) * (size_t)n);
  int status = OR_OK;
  if (x0) memcpy(x, x0, sizeof(double) * (size_t)n);
  else memset(x, 0, sizeof(double) * (size_t)n);

  const double bnorm = sqrt(dot(n, b, b));
  rep->ddot++;
  if (bnorm == 0.0) {
    rep->converged = 1;
    memset(x, 0, sizeof(double) * (size_t)n);
    goto done;
  }
  if (x0) {
    or_apply(op, x, r);
    rep->matvec++;
    for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
    const double rnorm = sqrt(dot(n, r, r));
    rep->ddot++;
    rep->rel_res = rnorm / bnorm;
    if (rep->rel_res <= tol) {
      rep->converged = 1;
      rep->true_rel_res = rep->rel_res;
      goto done;
    }
  } else {
    memcpy(r, b, sizeof(double) * (size_t)n);
    rep->rel_res = 1.0;
  }
  if (m >= 0) {
    prec_apply(op, P, r, z);
    rep->prec_applies++;
    rep->matvec += mdeg;
  } else {
    memcpy(z, r, sizeof(double) * (size_t)n);
  }
  memcpy(p, z, sizeof(double) * (size_t)n);
  double rho = dot(n, r, z);
  rep->ddot++;
  if (!isfinite(rho) || rho <= 0.0) {
    snprintf(g_err, sizeof g_err, "pcg_solve: r'z = %f at setup (preconditioner not SPD?)", rho);
    status = OR_NUMERICAL;
    goto done;
  }
  for (int it = 1; it <= maxit; ++it) {
    or_apply(op, p, q);
    rep->matvec++;
    const double pq = dot(n, p, q);
    rep->ddot++;
    if (!isfinite(pq) || pq <= 0.0) {
      snprintf(g_err, sizeof g_err, "pcg_solve: p'Ap = %f (operator not SPD?)", pq);
      status = OR_NUMERICAL;
      goto done;
    }
    const double alpha = rho / pq;
    for (int64_t i = 0; i < n; ++i) x[i] = x[i] + alpha * p[i];
    for (int64_t i = 0; i < n; ++i) r[i] = r[i] - alpha * q[i];
    const double rnorm = sqrt(dot(n, r, r));
    rep->ddot++;
    if (!isfinite(rnorm)) {
      status = fail(OR_NUMERICAL, "pcg_solve: residual norm is not finite");
      goto done;
    }
    rep->iters = it;
    rep->rel_res = rnorm / bnorm;
    if (rep->rel_res <= tol) {
      rep->converged = 1;
      break;
    }
    if (it == maxit) break;
    if (m >= 0) {
      prec_apply(op, P, r, z);
      rep->prec_applies++;
      rep->matvec += mdeg;
    } else {
      memcpy(z, r, sizeof(double) * (size_t)n);
    }
    const double rho_new = dot(n, r, z);
    rep->ddot++;
    if (!isfinite(rho_new) || rho_new <= 0.0) {
      snprintf(g_err, sizeof g_err, "pcg_solve: r'z = %f (preconditioner not SPD?)", rho_new);
      status = OR_NUMERICAL;
      goto done;
    }
    const double beta = rho_new / rho;
    for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    rho = rho_new;
  }
  or_apply(op, x, q);
  rep->matvec++;
  for (int64_t i = 0; i < n; ++i) q[i] = b[i] - q[i];
  rep->true_rel_res = sqrt(dot(n, q, q)) / bnorm;
  rep->ddot++;
done:
  rep->wall_time = now_s() - t0;
  free(r);
  free(z);
  free(p);
  free(q);
  return status;
}

/* ---------------------------------------------------------------- Lanczos */

/* Number of eigenvalues of T strictly below x (Sturm count, LDL^T pivots). */
static int sturm_count(int k, const double* a, const double* b, double x) {
  int cnt = 0;
  double d = 1.0;
  for (int i = 0; i < k; ++i) {
    const double bb = i > 0 ? b[i - 1] * b[i - 1] : 0.0;
    d = (a[i] - x) - (i > 0 ? bb / d : 0.0);
    if (d == 0.0) d = -1e-300;
    if (d < 0.0) ++cnt;
  }
  return cnt;
}

void or_tridiag_extremes(int k, const double* a, const double* b, double* lo, double* hi) {
  double gl = a[0], gu = a[0];
  for (int i = 0; i < k; ++i) {
    const double r = (i > 0 ? fabs(b[i - 1]) : 0.0) + (i < k - 1 ? fabs(b[i]) : 0.0);
    if (a[i] - r < gl) gl = a[i] - r;
    if (a[i] + r > gu) gu = a[i] + r;
  }
  for (int which = 0; which < 2; ++which) {
    double l = gl, u = gu;
    const int target = which == 0 ? 1 : k; /* count(<x) >= target */
    for (int it = 0; it < 200; ++it) {
      const double mid = 0.5 * (l + u);
      if (mid <= l || mid >= u) break;
      if (sturm_count(k, a, b, mid) >= target) u = mid;
      else l = mid;
    }
    if (which == 0) *lo = 0.5 * (l + u);
    else *hi = 0.5 * (l + u);
  }
}

int or_lanczos(const or_op* op, int steps, uint64_t seed, double* lo, double* hi,
               double* alphas, double* betas) {
  const int64_t n = op_n(op);
  if (steps < 1) return fail(OR_INVALID, "lanczos: steps must be >= 1");
  double* v = (double*)malloc(sizeof(double) * (size_t)n);
  double* v_prev = (double*)calloc((size_t)n, sizeof(double));
  double* w = (double*)malloc(sizeof(double) * (size_t)n);
  or_random_uniform(n, seed, 0, v);
  const double nv = sqrt(dot(n, v, v));
  for (int64_t i = 0; i < n; ++i) v[i] = v[i] / nv;
  double beta_prev = 0.0;
  int k = 0;
  for (int j = 0; j < steps; ++j) {
    or_apply(op, v, w);
    const double a = dot(n, w, v);
    for (int64_t i = 0; i < n; ++i) w[i] = (w[i] - a * v[i]) - beta_prev * v_prev[i];
    const double bnext = sqrt(dot(n, w, w));
    alphas[j] = a;
    betas[j] = bnext;
    k = j + 1;
    if (bnext == 0.0) break;
    for (int64_t i = 0; i < n; ++i) {
      v_prev[i] = v[i];
      v[i] = w[i] / bnext;
    }
    beta_prev = bnext;
  }
  or_tridiag_extremes(k, alphas, betas, lo, hi);
  free(v);
  free(v_prev);
  free(w);
  return OR_OK;
}

/* ---------------------------------------------------------------- power / DACG */

/* start_vector (eigenest.cpp:35-46): seeded uniform, normalised; seed+1 once if zero */
static int start_vector(const or_op* op, uint64_t seed, const char* who, double* v) {
  const int64_t n = op_n(op);
  or_random_uniform(n, seed, 0, v);
  double nrm = sqrt(dot(n, v, v));
  if (nrm == 0.0) {
    or_random_uniform(n, seed + 1, 0, v);
    nrm = sqrt(dot(n, v, v));
    if (nrm == 0.0) {
      snprintf(g_err, sizeof g_err, "%s: zero starting vector", who);
      return OR_NUMERICAL;
    }
  }
  for (int64_t i = 0; i < n; ++i) v[i] = v[i] / nrm;
  return OR_OK;
}

/* power_method, eigenest.cpp:48-79 */
int or_power_method(const or_op* op, double tol, int maxit, uint64_t seed, double* out) {
  const int64_t n = op_n(op);
  if (!(tol > 0.0)) return fail(OR_INVALID, "power_method: tol must be positive");
  double* v = (double*)malloc(sizeof(double) * (size_t)n);
  double* w = (double*)malloc(sizeof(double) * (size_t)n);
  double value = 0.0, matvecs = 0.0;
  int iters = 0, conv = 0, st = start_vector(op, seed, "power_method", v);
  double beta_old = 0.0;
  for (int it = 1; st == OR_OK && it <= maxit; ++it) {
    or_apply(op, v, w);
    matvecs += 1.0;
    const double beta = dot(n, v, w);
    value = beta;
    iters = it;
    if (it > 1 && fabs(beta - beta_old) <= tol * fabs(beta)) {
      conv = 1;
      break;
    }
    beta_old = beta;
    const double wnorm = sqrt(dot(n, w, w));
    if (wnorm == 0.0) {
      st = start_vector(op, seed + 1, "power_method", v);
      if (st) break;
      or_apply(op, v, w);
      matvecs += 1.0;
      if (sqrt(dot(n, w, w)) == 0.0) {
        st = fail(OR_NUMERICAL, "power_method: operator annihilates the start vector");
        break;
      }
    }
    const double wn = sqrt(dot(n, w, w));
    for (int64_t i = 0; i < n; ++i) v[i] = w[i] / wn;
  }
  out[0] = value;
  out[1] = iters;
  out[2] = matvecs;
  out[3] = conv;
  free(v);
  free(w);
  return st;
}

/* dacg_smallest, eigenest.cpp:81-167 */
int or_dacg_smallest(const or_op* op, double tol, int maxit, uint64_t seed, double* out) {
  const int64_t n = op_n(op);
  if (!(tol > 0.0)) return fail(OR_INVALID, "dacg_smallest: tol must be positive");
  double* x = (double*)malloc(sizeof(double) * (size_t)n);
  double* ax = (double*)malloc(sizeof(double) * (size_t)n);
  double* p = (double*)calloc((size_t)n, sizeof(double));
  double* ap = (double*)malloc(sizeof(double) * (size_t)n);
  double* g = (double*)malloc(sizeof(double) * (size_t)n);
  double* e = (double*)malloc(sizeof(double) * (size_t)n);
  double value = 0.0, matvecs = 0.0;
  int iters = 0, conv = 0;
  int st = start_vector(op, seed, "dacg_smallest", x);
  if (st) goto done;
  or_apply(op, x, ax);
  matvecs += 1.0;
  double q = dot(n, x, ax);
  if (!(q > 0.0)) {
    st = fail(OR_NUMERICAL, "dacg_smallest: x'Ax <= 0, operator not positive definite");
    goto done;
  }
  double g_old_sq = 0.0;
  int have_p = 0;
  for (int it = 0; it <= maxit; ++it) {
    value = q;
    iters = it;
    for (int64_t i = 0; i < n; ++i) {
      e[i] = ax[i] - q * x[i];
      g[i] = 2.0 * e[i];
    }
    const double resid = sqrt(dot(n, e, e)) / q;
    if (resid <= tol) {
      conv = 1;
      break;
    }
    if (it == maxit) break;
    const double gsq = dot(n, g, g);
    if (!have_p || it % 50 == 0) {
      for (int64_t i = 0; i < n; ++i) p[i] = -g[i];
    } else {
      const double c = gsq / g_old_sq;
      for (int64_t i = 0; i < n; ++i) p[i] = -g[i] + c * p[i];
    }
    have_p = 1;
    g_old_sq = gsq;
    or_apply(op, p, ap);
    matvecs += 1.0;
    const double hxx = q, hxp = dot(n, x, ap), hpp = dot(n, p, ap);
    const double mxx = 1.0, mxp = dot(n, x, p), mpp = dot(n, p, p);
    if (!(hpp > 0.0)) {
      st = fail(OR_NUMERICAL, "dacg_smallest: p'Ap <= 0, operator not positive definite");
      goto done;
    }
    const double a2 = mxx * mpp - mxp * mxp;
    const double a1 = -((hxx * mpp + hpp * mxx) - 2.0 * hxp * mxp);
    const double a0 = hxx * hpp - hxp * hxp;
    const double disc = sqrt(fmax(0.0, a1 * a1 - 4.0 * a2 * a0));
    const double lambda = (-a1 - disc) / (2.0 * a2);
    const double r11 = hxx - lambda * mxx, r12 = hxp - lambda * mxp;
    const double r22 = hpp - lambda * mpp;
    double cx, cp;
    if (fabs(r12) + fabs(r22) > fabs(r11) + fabs(r12)) {
      cx = -r22;
      cp = r12;
    } else {
      cx = -r12;
      cp = r11;
    }
    if (cx == 0.0 && cp == 0.0) {
      cx = 1.0;
      cp = 0.0;
    }
    for (int64_t i = 0; i < n; ++i) {
      x[i] = cx * x[i] + cp * p[i];
      ax[i] = cx * ax[i] + cp * ap[i];
    }
    const double xnorm = sqrt(dot(n, x, x));
    if (xnorm == 0.0) {
      st = fail(OR_NUMERICAL, "dacg_smallest: line search collapsed");
      goto done;
    }
    for (int64_t i = 0; i < n; ++i) {
      x[i] = x[i] / xnorm;
      ax[i] = ax[i] / xnorm;
    }
    const double q_prev = q;
    q = dot(n, x, ax);
    if (!(q > 0.0)) {
      st = fail(OR_NUMERICAL, "dacg_smallest: x'Ax <= 0, operator not positive definite");
      goto done;
    }
    if (q > q_prev * (1.0 + 1e-12)) {
      st = fail(OR_NUMERICAL, "dacg_smallest: Rayleigh quotient increased");
      goto done;
    }
  }
done:
  out[0] = value;
  out[1] = iters;
  out[2] = matvecs;
  out[3] = conv;
  free(x);
  free(ax);
  free(p);
  free(ap);
  free(g);
  free(e);
  return st;
}
