// SPDX-License-Identifier: Apache-2.0
#pragma once
#include <cstddef>
#include <string>

#include "pcgx.h"

namespace pcgx {
double cheb_eval(double theta, double delta, double sigma, const double* rho, int m, double lambda);
int cheb_params(double alpha, double beta, int m, double scale, double* tds, double* rho,
                std::string* msg);
double newton_eval(const double* zeta, int nlev, double lambda);
int newton_params(double alpha0, double beta0, int nlev, double scale, double* zeta,
                  std::string* msg);
int chi_sequence(double alpha, double beta, int nlev, double* chi, std::string* msg);
void analytic_extremes(int dim, long long nx, int scaled, double* lo, double* hi);
void analytic_extremes_box(long long nx, long long ny, long long nz, double* lo, double* hi);
void random_uniform_host(long long n, unsigned long long seed, unsigned long long offset,
                         double* out);
int mm_load(const char* path, pcgx_csr_host* out, std::string* msg);
int mm_load_text(const char* text, size_t len, const char* name, pcgx_csr_host* out,
                 std::string* msg);
int mm_save_text(int64_t n, const int64_t* rp, const int64_t* ci, const double* va,
                 std::string* text);
void tridiag_extremes(int k, const double* a, const double* b, double* lo, double* hi);
}  // namespace pcgx
