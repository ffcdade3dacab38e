// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE ONLY — the checker and the CPU-baseline arm, never the
// product. Built by oracle/Makefile into oracle/_ref/libpolycg_ref.so.
//
// A flat C API over the UNMODIFIED reference library `polycg` (compiled from
// /root/reference/proj/src where the sources lie, against oracle/eigen_shim and
// a build-time copy of linop.hpp with one added copy constructor; see the
// Makefile). Every entry point constructs reference objects and calls the
// reference's own functions, so results ARE the reference's results:
//
//   ref_cheb_params       -> polycg::cheb_params          (proj/src/polyprec.cpp:56-79)
//   ref_eval_poly         -> polycg::eval_poly            (proj/src/polyprec.cpp:89-100)
//   ref_analytic_extremes -> polycg::analytic_extremes    (proj/src/linop.cpp:382-390)
//   ref_random_uniform    -> polycg::random_uniform_vector(proj/src/eigenest.cpp:22-30)
//   ref_apply             -> ScaledOperator::apply        (proj/src/linop.cpp:271-275)
//   ref_apply_chebyshev   -> polycg::apply_chebyshev      (proj/src/polyprec.cpp:169-198)
//   ref_apply_newton      -> polycg::apply_newton         (proj/src/polyprec.cpp:148-160)
//   ref_pcg_solve         -> polycg::pcg_solve            (proj/src/pcg.cpp:10-117)
//   ref_pcg_solve_newton  -> polycg::pcg_solve with NewtonPreconditioner (pcg.hpp:27-40)
//   ref_spectrum_table    -> polycg::spectrum_table       (proj/src/spectrum.cpp:59-88)
//
// Operators: kind 0 = StencilOperator(lap3d, nx), kind 1 = StencilOperator(lap2d, nx),
// kind 2 = assembled CsrMatrix (assemble_laplacian lap3d), kind 3 = user CSR (int64
// arrays). All are Jacobi-scaled with jacobi_scale (proj/src/linop.cpp:340-351),
// exactly as the reference CLI's build_problem does (tools/polycg.cpp:192-204).

#include "polycg/eigenest.hpp"
#include "polycg/linop.hpp"
#include "polycg/matrix_market.hpp"
#include "polycg/pcg.hpp"
#include "polycg/polyprec.hpp"
#include "polycg/spectrum.hpp"

#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

using namespace polycg;

namespace {

thread_local std::string g_err;

// 0 ok, 1 invalid_argument, 2 NumericalError, 3 other.
template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const NumericalError& e) {
    g_err = e.what();
    return 2;
  } catch (const ParseError& e) {
    g_err = e.what();
    return 7;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

struct RefProblem {
  std::unique_ptr<LinearOperator> inner;
  std::unique_ptr<ScaledOperator> scaled;
};

RefProblem make_problem(int kind, std::int64_t nx, std::int64_t n, const std::int64_t* rp,
                        const std::int64_t* ci, const double* va) {
  RefProblem p;
  if (kind == 0) {
    p.inner = fd_laplacian(StencilKind::lap3d, nx, OperatorForm::stencil);
  } else if (kind == 1) {
    p.inner = fd_laplacian(StencilKind::lap2d, nx, OperatorForm::stencil);
  } else if (kind == 2) {
    p.inner = fd_laplacian(StencilKind::lap3d, nx, OperatorForm::assembled);
  } else if (kind == 4) {
    p.inner = fd_laplacian(StencilKind::lap2d, nx, OperatorForm::assembled);
  } else if (kind == 3) {
    const std::int64_t nnz = rp[n];
    p.inner = std::make_unique<CsrMatrix>(
        n, std::vector<Index>(rp, rp + n + 1), std::vector<Index>(ci, ci + nnz),
        std::vector<double>(va, va + nnz), 0.0);
  } else {
    throw std::invalid_argument("ref: unknown operator kind");
  }
  auto [scaled, inv_sqrt] = jacobi_scale(*p.inner);
  p.scaled = std::make_unique<ScaledOperator>(std::move(scaled));
  return p;
}

Vector to_vec(const double* p, std::int64_t n) {
  Vector v(n);
  std::memcpy(v.data(), p, sizeof(double) * static_cast<std::size_t>(n));
  return v;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// load_matrix_market(istream, name) (matrix_market.cpp:61-166) / (path) (:55-59):
// sizes now, arrays by ref_mm_fetch (the matrix is kept per thread in between).
thread_local std::unique_ptr<CsrMatrix> g_mm;
int ref_mm_load_text(const char* text, std::int64_t len, const char* name, std::int64_t* n,
                     std::int64_t* nnz) {
  return guarded([&] {
    std::istringstream in(std::string(text, static_cast<std::size_t>(len)));
    g_mm = std::make_unique<CsrMatrix>(load_matrix_market(in, name));
    *n = g_mm->size();
    *nnz = g_mm->nnz();
  });
}
int ref_mm_load_file(const char* path, std::int64_t* n, std::int64_t* nnz) {
  return guarded([&] {
    g_mm = std::make_unique<CsrMatrix>(load_matrix_market(std::string(path)));
    *n = g_mm->size();
    *nnz = g_mm->nnz();
  });
}
void ref_mm_fetch(std::int64_t* rp, std::int64_t* ci, double* va) {
  std::memcpy(rp, g_mm->row_ptr().data(), sizeof(std::int64_t) * g_mm->row_ptr().size());
  std::memcpy(ci, g_mm->col_idx().data(), sizeof(std::int64_t) * g_mm->col_idx().size());
  std::memcpy(va, g_mm->values().data(), sizeof(double) * g_mm->values().size());
  g_mm.reset();
}
// save_matrix_market(m, ostream) (matrix_market.cpp:178-199); the text stays valid
// until the next call on this thread.
thread_local std::string g_mm_text;
int ref_mm_save_text(std::int64_t n, const std::int64_t* rp, const std::int64_t* ci,
                     const double* va, const char** text, std::int64_t* len) {
  return guarded([&] {
    const std::int64_t nnz = rp[n];
    CsrMatrix m(n, std::vector<Index>(rp, rp + n + 1), std::vector<Index>(ci, ci + nnz),
                std::vector<double>(va, va + nnz));
    std::ostringstream out;
    save_matrix_market(m, out);
    g_mm_text = out.str();
    *text = g_mm_text.c_str();
    *len = static_cast<std::int64_t>(g_mm_text.size());
  });
}

void ref_set_threads(int t) { set_apply_threads(t); }
int ref_get_threads() { return apply_threads(); }

// out_tds = {theta, delta, sigma}; rho has m+1 slots.
int ref_cheb_params(double alpha, double beta, int m, double scale, double* out_tds, double* rho) {
  return guarded([&] {
    const ChebyshevParams p = cheb_params(alpha, beta, m, scale);
    out_tds[0] = p.theta;
    out_tds[1] = p.delta;
    out_tds[2] = p.sigma;
    for (int k = 0; k <= m; ++k) rho[k] = p.rho[static_cast<std::size_t>(k)];
  });
}

int ref_eval_poly(double alpha, double beta, int m, double scale, const double* lam, int nl,
                  double* out) {
  return guarded([&] {
    const ChebyshevParams p = cheb_params(alpha, beta, m, scale);
    for (int i = 0; i < nl; ++i) out[i] = eval_poly(p, lam[i]);
  });
}

int ref_newton_params(double alpha, double beta, int nlev, double scale, double* zeta) {
  return guarded([&] {
    const NewtonParams p = newton_params(alpha, beta, nlev, scale);
    for (int j = 0; j <= nlev; ++j) zeta[j] = p.zeta[static_cast<std::size_t>(j)];
  });
}

// kind: 0 lap3d, 1 lap2d
int ref_analytic_extremes(int kind, std::int64_t nx, int scaled, double* lo, double* hi) {
  return guarded([&] {
    const auto [a, b] =
        analytic_extremes(kind == 0 ? StencilKind::lap3d : StencilKind::lap2d, nx, scaled != 0);
    *lo = a;
    *hi = b;
  });
}

int ref_random_uniform(std::int64_t n, std::uint64_t seed, double* out) {
  return guarded([&] {
    const Vector v = random_uniform_vector(n, seed);
    std::memcpy(out, v.data(), sizeof(double) * static_cast<std::size_t>(n));
  });
}

// y = (D^{-1/2} A D^{-1/2}) x; reps applications back to back (timing use).
int ref_apply(int kind, std::int64_t nx, std::int64_t n, const std::int64_t* rp,
              const std::int64_t* ci, const double* va, const double* x, double* y, int reps) {
  return guarded([&] {
    RefProblem p = make_problem(kind, nx, n, rp, ci, va);
    const Vector xv = to_vec(x, p.scaled->size());
    Vector yv(p.scaled->size());
    for (int r = 0; r < (reps < 1 ? 1 : reps); ++r) p.scaled->apply(xv, yv);
    std::memcpy(y, yv.data(), sizeof(double) * static_cast<std::size_t>(yv.size()));
  });
}

// out = p_m(A) r on the scaled operator; matvecs receives the operator's counter.
int ref_apply_chebyshev(int kind, std::int64_t nx, std::int64_t n, const std::int64_t* rp,
                        const std::int64_t* ci, const double* va, double alpha, double beta,
                        int m, double scale, const double* r, double* out,
                        std::uint64_t* matvecs) {
  return guarded([&] {
    RefProblem p = make_problem(kind, nx, n, rp, ci, va);
    const ChebyshevParams prm = cheb_params(alpha, beta, m, scale);
    const Vector rv = to_vec(r, p.scaled->size());
    p.scaled->reset_matvec_count();
    const Vector o = apply_chebyshev(prm, *p.scaled, rv);
    if (matvecs) *matvecs = p.scaled->matvec_count();
    std::memcpy(out, o.data(), sizeof(double) * static_cast<std::size_t>(o.size()));
  });
}

int ref_apply_newton(int kind, std::int64_t nx, std::int64_t n, const std::int64_t* rp,
                     const std::int64_t* ci, const double* va, double alpha, double beta,
                     int nlev, double scale, const double* r, double* out) {
  return guarded([&] {
    RefProblem p = make_problem(kind, nx, n, rp, ci, va);
    const NewtonParams prm = newton_params(alpha, beta, nlev, scale);
    const Vector rv = to_vec(r, p.scaled->size());
    const Vector o = apply_newton(prm, *p.scaled, rv);
    std::memcpy(out, o.data(), sizeof(double) * static_cast<std::size_t>(o.size()));
  });
}

// report: iters, ddot, matvec, prec_applies, rel_res, true_rel_res, wall_time, converged
struct RefReport {
  std::int64_t iters, ddot, matvec, prec_applies;
  double rel_res, true_rel_res, wall_time;
  std::int64_t converged;
};

// m < 0 -> no preconditioner (plain CG). b may be NULL -> b = A x_true with
// x_true = random_uniform_vector(n, seed) (tools/polycg.cpp:266-278,375-376).
// newton = 0: ChebyshevPreconditioner(cheb_params(alpha, beta, m, scale)), m < 0 none;
// newton = 1: NewtonPreconditioner(newton_params(alpha, beta, m = nlev, scale)).
int ref_pcg_solve_prec(int kind, std::int64_t nx, std::int64_t n, const std::int64_t* rp,
                       const std::int64_t* ci, const double* va, double alpha, double beta, int m,
                       double scale, int newton, const double* b, std::uint64_t seed, double tol,
                       int maxit, double* x_out, double* b_out, RefReport* rep);

int ref_pcg_solve(int kind, std::int64_t nx, std::int64_t n, const std::int64_t* rp,
                  const std::int64_t* ci, const double* va, double alpha, double beta, int m,
                  double scale, const double* b, std::uint64_t seed, double tol, int maxit,
                  double* x_out, double* b_out, RefReport* rep) {
  return ref_pcg_solve_prec(kind, nx, n, rp, ci, va, alpha, beta, m, scale, 0, b, seed, tol, maxit,
                            x_out, b_out, rep);
}

int ref_pcg_solve_newton(int kind, std::int64_t nx, std::int64_t n, const std::int64_t* rp,
                         const std::int64_t* ci, const double* va, double alpha, double beta,
                         int nlev, double scale, const double* b, std::uint64_t seed, double tol,
                         int maxit, double* x_out, double* b_out, RefReport* rep) {
  return ref_pcg_solve_prec(kind, nx, n, rp, ci, va, alpha, beta, nlev, scale, 1, b, seed, tol,
                            maxit, x_out, b_out, rep);
}

int ref_pcg_solve_prec(int kind, std::int64_t nx, std::int64_t n, const std::int64_t* rp,
                       const std::int64_t* ci, const double* va, double alpha, double beta, int m,
                       double scale, int newton, const double* b, std::uint64_t seed, double tol,
                       int maxit, double* x_out, double* b_out, RefReport* rep) {
  return guarded([&] {
    RefProblem p = make_problem(kind, nx, n, rp, ci, va);
    const Index N = p.scaled->size();
    Vector bv;
    if (b) {
      bv = to_vec(b, N);
    } else {
      const Vector exact = random_uniform_vector(N, seed);
      bv = p.scaled->apply(exact);
    }
    if (b_out) std::memcpy(b_out, bv.data(), sizeof(double) * static_cast<std::size_t>(N));
    SolveOptions opts;
    opts.tol = tol;
    opts.maxit = maxit;
    std::unique_ptr<Preconditioner> prec;
    if (newton) prec = std::make_unique<NewtonPreconditioner>(newton_params(alpha, beta, m, scale));
    else if (m >= 0) prec = std::make_unique<ChebyshevPreconditioner>(cheb_params(alpha, beta, m, scale));
    auto [x, report] = pcg_solve(*p.scaled, bv, opts, prec.get());
    if (x_out) std::memcpy(x_out, x.data(), sizeof(double) * static_cast<std::size_t>(N));
    rep->iters = report.iters;
    rep->ddot = static_cast<std::int64_t>(report.ddot);
    rep->matvec = static_cast<std::int64_t>(report.matvec);
    rep->prec_applies = static_cast<std::int64_t>(report.prec_applies);
    rep->rel_res = report.rel_res;
    rep->true_rel_res = report.true_rel_res;
    rep->wall_time = report.wall_time;
    rep->converged = report.converged ? 1 : 0;
  });
}

// power_method / dacg_smallest (eigenest.cpp:48-167) on the scaled operator.
// out: {value, iters, matvecs, converged}
int ref_power_method(int kind, std::int64_t nx, std::int64_t n, const std::int64_t* rp,
                     const std::int64_t* ci, const double* va, double tol, int maxit,
                     std::uint64_t seed, double* out) {
  return guarded([&] {
    RefProblem p = make_problem(kind, nx, n, rp, ci, va);
    const EigResult r = power_method(*p.scaled, EigOptions{tol, maxit, seed});
    out[0] = r.value;
    out[1] = r.iters;
    out[2] = static_cast<double>(r.matvecs);
    out[3] = r.converged ? 1.0 : 0.0;
  });
}

int ref_dacg_smallest(int kind, std::int64_t nx, std::int64_t n, const std::int64_t* rp,
                      const std::int64_t* ci, const double* va, double tol, int maxit,
                      std::uint64_t seed, double* out) {
  return guarded([&] {
    RefProblem p = make_problem(kind, nx, n, rp, ci, va);
    const EigResult r = dacg_smallest(*p.scaled, EigOptions{tol, maxit, seed});
    out[0] = r.value;
    out[1] = r.iters;
    out[2] = static_cast<double>(r.matvecs);
    out[3] = r.converged ? 1.0 : 0.0;
  });
}

// rows: 6 doubles each {m, iters, mu_max, mu_min, l, kappa}; solution 0 ones, 1 flat, 2 random
int ref_spectrum_table(std::int64_t nx, const int* degrees, int nd, double scale, int solution,
                       std::uint64_t seed, double* rows) {
  return guarded([&] {
    TableOptions opts;
    opts.solution = solution == 0 ? SolutionKind::ones
                                  : (solution == 1 ? SolutionKind::flat : SolutionKind::random);
    opts.seed = seed;
    const auto out = spectrum_table(nx, std::vector<int>(degrees, degrees + nd), scale, opts);
    for (std::size_t i = 0; i < out.size(); ++i) {
      rows[6 * i + 0] = out[i].m;
      rows[6 * i + 1] = out[i].iters;
      rows[6 * i + 2] = out[i].mu_max;
      rows[6 * i + 3] = out[i].mu_min;
      rows[6 * i + 4] = static_cast<double>(out[i].l);
      rows[6 * i + 5] = out[i].kappa;
    }
  });
}

}  // extern "C"
