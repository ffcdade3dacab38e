// SPDX-License-Identifier: Apache-2.0
//
// Host-side scalar math of the hot path. Compiled with -ffp-contract=off and no
// -march so every expression rounds exactly as the reference's Release build
// (proj/CMakeLists.txt:6-8): the coefficients are bit-exact by construction.
#include <cmath>
#include <cstdio>
#include <string>

#include "pcgx.h"
#include "host_math.hpp"

namespace pcgx {

// polyprec.cpp:89-100 (Chebyshev-form scalar mirror of the vector recursion)
double cheb_eval(double theta, double delta, double sigma, const double* rho, int m,
                 double lambda) {
  double p_prev = 0.0;
  double p = 1.0 / theta;
  for (int k = 1; k <= m; ++k) {
    const double p_new =
        rho[k] * (2.0 * sigma * (1.0 - lambda / theta) * p - rho[k - 1] * p_prev + 2.0 / delta);
    p_prev = p;
    p = p_new;
  }
  return p;
}

// polyprec.cpp:56-79 with check_positivity :13-23. Returns 0, or the status
// with `msg` set to the reference's exception text.
int cheb_params(double alpha, double beta, int m, double scale, double* tds, double* rho,
                std::string* msg) {
  if (!(alpha > 0.0)) {
    *msg = "cheb_params: alpha must be positive";
    return PCGX_ERR_INVALID;
  }
  if (!(beta > alpha)) {
    *msg = "cheb_params: need alpha < beta (delta = 0 divides by zero)";
    return PCGX_ERR_INVALID;
  }
  if (m < 0) {
    *msg = "cheb_params: m must be >= 0";
    return PCGX_ERR_INVALID;
  }
  if (!(scale >= 1.0)) {
    *msg = "cheb_params: scale must be >= 1";
    return PCGX_ERR_INVALID;
  }
  const double theta = scale * 0.5 * (alpha + beta);
  const double delta = 0.5 * (beta - alpha);
  const double sigma = theta / delta;
  tds[0] = theta;
  tds[1] = delta;
  tds[2] = sigma;
  rho[0] = 1.0 / sigma;
  for (int k = 1; k <= m; ++k) rho[k] = 1.0 / (2.0 * sigma - rho[k - 1]);
  constexpr int kGrid = 1000;
  for (int g = 0; g < kGrid; ++g) {
    const double lam = alpha + (beta - alpha) * static_cast<double>(g) / (kGrid - 1);
    if (!(cheb_eval(theta, delta, sigma, rho, m, lam) > 0.0)) {
      *msg = "polynomial preconditioner not positive at lambda = " + std::to_string(lam);
      return PCGX_ERR_NUMERICAL;
    }
  }
  return 0;
}

// eval_poly, Newton form (polyprec.cpp:81-87): the scalar mirror of the recursion.
double newton_eval(const double* zeta, int nlev, double lambda) {
  double r = zeta[0];
  for (int j = 1; j <= nlev; ++j) r = zeta[j] * (2.0 * r - lambda * r * r);
  return r;
}

// newton_params (polyprec.cpp:27-54): zeta[0..nlev]; same validation and
// positivity check (1000-point grid on [alpha0, beta0]) as the reference.
int newton_params(double alpha0, double beta0, int nlev, double scale, double* zeta,
                  std::string* msg) {
  if (!(alpha0 > 0.0) || !(beta0 >= alpha0)) {
    *msg = "newton_params: need 0 < alpha0 <= beta0";
    return PCGX_ERR_INVALID;
  }
  if (nlev < 0) {
    *msg = "newton_params: nlev must be >= 0";
    return PCGX_ERR_INVALID;
  }
  if (!(scale >= 1.0)) {
    *msg = "newton_params: scale must be >= 1";
    return PCGX_ERR_INVALID;
  }
  const double theta = 0.5 * (alpha0 + beta0);
  const double delta = 0.5 * (beta0 - alpha0);
  zeta[0] = 1.0 / (scale * theta);
  if (nlev >= 1) {
    const double t = (scale * theta - delta) * zeta[0];
    zeta[1] = 2.0 / (1.0 + 2.0 * t - t * t);
    for (int j = 2; j <= nlev; ++j) {
      const double z = zeta[j - 1];
      zeta[j] = 2.0 / (1.0 + 2.0 * z - z * z);
    }
  }
  constexpr int kGrid = 1000;
  for (int g = 0; g < kGrid; ++g) {
    const double lam = alpha0 + (beta0 - alpha0) * static_cast<double>(g) / (kGrid - 1);
    if (!(newton_eval(zeta, nlev, lam) > 0.0)) {
      *msg = "polynomial preconditioner not positive at lambda = " + std::to_string(lam);
      return PCGX_ERR_NUMERICAL;
    }
  }
  return 0;
}

// chi_sequence (polyprec.cpp:102-123): chi_j = 2 sigma_k^2 / sigma_{2k}.
int chi_sequence(double alpha, double beta, int nlev, double* chi, std::string* msg) {
  if (!(alpha > 0.0) || !(beta > alpha)) {
    *msg = "chi_sequence: need 0 < alpha < beta";
    return PCGX_ERR_INVALID;
  }
  if (nlev < 0 || nlev > 30) {
    *msg = "chi_sequence: nlev must be in [0, 30]";
    return PCGX_ERR_INVALID;
  }
  double sigma_k = (alpha + beta) / (beta - alpha);
  bool huge = false;
  for (int j = 0; j < nlev; ++j) {
    if (huge || sigma_k > 1e150) {  // 2 sigma_k^2 would overflow; chi is 1 from here on
      huge = true;
      chi[j] = 1.0;
      continue;
    }
    const double sigma_2k = 2.0 * sigma_k * sigma_k - 1.0;
    chi[j] = 2.0 * sigma_k * sigma_k / sigma_2k;
    sigma_k = sigma_2k;
  }
  return 0;
}

// linop.cpp:382-390
void analytic_extremes(int dim, long long nx, int scaled, double* lo, double* hi) {
  const double pi = 3.141592653589793238462643383279502884;
  const double h = 1.0 / static_cast<double>(nx + 1);
  const double s = std::sin(pi * h / 2.0);
  const double c = std::cos(pi * h / 2.0);
  const double factor =
      (scaled ? 2.0 / static_cast<double>(2 * dim) : 2.0) * 2.0 * static_cast<double>(dim);
  *lo = factor * s * s;
  *hi = factor * c * c;
}

void analytic_extremes_box(long long nx, long long ny, long long nz, double* lo, double* hi) {
  const double pi = 3.141592653589793238462643383279502884;
  const long long dims[3] = {nx, ny, nz};
  double smin = 0.0, smax = 0.0;
  for (int d = 0; d < 3; ++d) {
    const double h = 1.0 / static_cast<double>(dims[d] + 1);
    const double s = std::sin(pi * h / 2.0);
    const double c = std::cos(pi * h / 2.0);
    smin += s * s;
    smax += c * c;
  }
  *lo = (2.0 / 3.0) * smin;
  *hi = (2.0 / 3.0) * smax;
}

// eigenest.cpp:13-30
void random_uniform_host(long long n, unsigned long long seed, unsigned long long offset,
                         double* out) {
  for (long long i = 0; i < n; ++i) {
    unsigned long long z = seed + (offset + static_cast<unsigned long long>(i) + 1ull) *
                                      0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z = z ^ (z >> 31);
    const double u = static_cast<double>(z >> 11) * 0x1.0p-53;
    out[i] = 2.0 * u - 1.0;
  }
}

// Sturm count of eigenvalues of the symmetric tridiagonal (a, b) below x.
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

void tridiag_extremes(int k, const double* a, const double* b, double* lo, double* hi) {
  double gl = a[0], gu = a[0];
  for (int i = 0; i < k; ++i) {
    const double r = (i > 0 ? std::fabs(b[i - 1]) : 0.0) + (i < k - 1 ? std::fabs(b[i]) : 0.0);
    if (a[i] - r < gl) gl = a[i] - r;
    if (a[i] + r > gu) gu = a[i] + r;
  }
  for (int which = 0; which < 2; ++which) {
    double l = gl, u = gu;
    const int target = which == 0 ? 1 : k;
    for (int it = 0; it < 200; ++it) {
      const double mid = 0.5 * (l + u);
      if (mid <= l || mid >= u) break;
      if (sturm_count(k, a, b, mid) >= target) u = mid;
      else l = mid;
    }
    (which == 0 ? *lo : *hi) = 0.5 * (l + u);
  }
}

}  // namespace pcgx
