// SPDX-License-Identifier: Apache-2.0
//
// TEST: the reference-side C++ binding (include/polycg_gpu/adapter.hpp) used
// exactly as a maintainer would, against the reference library itself
// (oracle/_ref objects, built from /root/reference/proj/src). Built by
// `make -C oracle adapter_test`; run by tests/test_adapter.py on a GPU box.
//
// For each case the SAME ScaledOperator, rhs and ChebyshevPreconditioner go to
// polycg::pcg_solve (CPU reference) and polycg::gpu::pcg_solve (B200), and the
// program prints one JSON line per case with both reports and the solution
// difference; exit code 0 iff every case meets the parity bar.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "polycg/eigenest.hpp"
#include "polycg/linop.hpp"
#include "polycg/pcg.hpp"
#include "polycg/polyprec.hpp"
#include "polycg_gpu/adapter.hpp"

using namespace polycg;

static int run_case(const char* tag, const LinearOperator& inner, Index nx, int m, double s,
                    polycg::gpu::Session& sess) {
  auto [scaled, inv_sqrt] = jacobi_scale(inner);
  const auto [a0, b0] = analytic_extremes(StencilKind::lap3d, nx, true);
  const Vector exact = random_uniform_vector(scaled.size(), 20240801);
  const Vector b = scaled.apply(exact);
  SolveOptions opts;
  ChebyshevPreconditioner p_cpu(cheb_params(a0, b0, m, s));
  ChebyshevPreconditioner p_gpu(cheb_params(a0, b0, m, s));
  auto [x_ref, r_ref] = pcg_solve(scaled, b, opts, &p_cpu);
  polycg::gpu::DeviceOperator dop(sess, scaled);
  auto [x_gpu, r_gpu] = polycg::gpu::pcg_solve(sess, dop, scaled, b, opts, &p_gpu);
  double dn = 0.0, xn = 0.0;
  for (Index i = 0; i < x_ref.size(); ++i) {
    dn += (x_gpu[i] - x_ref[i]) * (x_gpu[i] - x_ref[i]);
    xn += x_ref[i] * x_ref[i];
  }
  const double rel = std::sqrt(dn / xn);
  // per-step Chebyshev parity through the adapter (bitwise expected)
  Vector r0 = random_uniform_vector(scaled.size(), 4242), o_cpu, o_gpu;
  o_cpu = apply_chebyshev(cheb_params(a0, b0, 7, s), scaled, r0);
  polycg::gpu::apply_chebyshev(sess, dop, cheb_params(a0, b0, 7, s), r0, o_gpu);
  bool bitwise = true;
  for (Index i = 0; i < r0.size(); ++i) bitwise = bitwise && (o_cpu[i] == o_gpu[i]);
  const bool ok = std::abs(r_gpu.iters - r_ref.iters) <= 1 && rel <= 1e-10 && bitwise &&
                  r_gpu.ddot == r_ref.ddot && r_gpu.matvec == r_ref.matvec &&
                  r_gpu.converged == r_ref.converged;
  std::printf(
      "{\"case\": \"%s\", \"ok\": %s, \"iters\": [%d, %d], \"ddot\": [%llu, %llu], "
      "\"matvec\": [%llu, %llu], \"rel_res\": [%.17g, %.17g], \"x_rel_diff\": %.3e, "
      "\"cheb7_bitwise\": %s, \"wall_time\": [%.6f, %.6f]}\n",
      tag, ok ? "true" : "false", r_ref.iters, r_gpu.iters, (unsigned long long)r_ref.ddot,
      (unsigned long long)r_gpu.ddot, (unsigned long long)r_ref.matvec,
      (unsigned long long)r_gpu.matvec, r_ref.rel_res, r_gpu.rel_res, rel,
      bitwise ? "true" : "false", r_ref.wall_time, r_gpu.wall_time);
  return ok ? 0 : 1;
}

static bool same_bits(const Vector& a, const Vector& b) {
  if (a.size() != b.size()) return false;
  for (Index i = 0; i < a.size(); ++i)
    if (std::memcmp(a.data() + i, b.data() + i, sizeof(double)) != 0) return false;
  return true;
}

static bool same_report(const SolveReport& a, const SolveReport& b) {
  return a.iters == b.iters && a.ddot == b.ddot && a.matvec == b.matvec &&
         a.prec_applies == b.prec_applies && a.rel_res == b.rel_res &&
         a.true_rel_res == b.true_rel_res && a.converged == b.converged;
}

// The reference's own extension points (linop.hpp:21-47, pcg.hpp:20-25): the
// reference's pcg_solve / power_method / dacg_smallest run unchanged with the
// device operator and the device preconditioners plugged in. The device SpMV and
// Chebyshev / Newton applies are bitwise the reference's and the reductions are
// the reference's own (host), so x, every counter and every residual must be
// bit-identical to the all-CPU run.
static int plugin_cases(polycg::gpu::Session& sess) {
  int bad = 0;
  auto run = [&](const char* tag, const LinearOperator& inner, Index nx, int m, bool newton) {
    auto [scaled, d] = jacobi_scale(inner);
    const auto [a0, b0] = analytic_extremes(StencilKind::lap3d, nx, true);
    const Vector b = scaled.apply(random_uniform_vector(scaled.size(), 20240801));
    std::unique_ptr<Preconditioner> p_cpu, p_gpu, p_gpu2;
    if (newton) {
      p_cpu = std::make_unique<NewtonPreconditioner>(newton_params(a0, b0, m, 1.001));
      p_gpu = std::make_unique<polycg::gpu::NewtonPreconditioner>(sess, newton_params(a0, b0, m, 1.001));
      p_gpu2 = std::make_unique<polycg::gpu::NewtonPreconditioner>(sess, newton_params(a0, b0, m, 1.001));
    } else {
      p_cpu = std::make_unique<ChebyshevPreconditioner>(cheb_params(a0, b0, m, 1.001));
      p_gpu = std::make_unique<polycg::gpu::ChebyshevPreconditioner>(sess, cheb_params(a0, b0, m, 1.001));
      p_gpu2 = std::make_unique<polycg::gpu::ChebyshevPreconditioner>(sess, cheb_params(a0, b0, m, 1.001));
    }
    auto [x_ref, r_ref] = polycg::pcg_solve(scaled, b, {}, p_cpu.get());
    // (1) device operator + device preconditioner under the reference's pcg_solve
    polycg::gpu::DeviceLinearOperator dlo(sess, scaled);
    auto [x_dev, r_dev] = polycg::pcg_solve(dlo, b, {}, p_gpu.get());
    // (2) the device preconditioner with the host operator (cached upload)
    const int up0 = sess.uploads();
    auto [x_mix, r_mix] = polycg::pcg_solve(scaled, b, {}, p_gpu2.get());
    auto [x_mix2, r_mix2] = polycg::pcg_solve(scaled, b, {}, p_gpu2.get());
    const int reup = sess.uploads() - up0;
    const bool ok = same_bits(x_ref, x_dev) && same_report(r_ref, r_dev) && same_bits(x_ref, x_mix) &&
                    same_report(r_ref, r_mix) && same_bits(x_ref, x_mix2) && reup == 0 &&
                    dlo.matvec_count() == static_cast<std::uint64_t>(r_ref.iters + 1);
    std::printf("{\"case\": \"%s\", \"ok\": %s, \"iters\": [%d, %d], \"matvec\": [%llu, %llu], "
                "\"x_bitwise\": [%s, %s], \"report_equal\": [%s, %s], \"reuploads\": %d, "
                "\"dlo_matvec_count\": %llu}\n",
                tag, ok ? "true" : "false", r_ref.iters, r_dev.iters, (unsigned long long)r_ref.matvec,
                (unsigned long long)r_dev.matvec, same_bits(x_ref, x_dev) ? "true" : "false",
                same_bits(x_ref, x_mix) ? "true" : "false", same_report(r_ref, r_dev) ? "true" : "false",
                same_report(r_ref, r_mix) ? "true" : "false", reup,
                (unsigned long long)dlo.matvec_count());
    return ok ? 0 : 1;
  };
  const StencilOperator st32(StencilKind::lap3d, 32);
  bad += run("plugin_ref_pcg_stencil32_cheb10", st32, 32, 10, false);
  const CsrMatrix cs24 = assemble_laplacian(StencilKind::lap3d, 24);
  bad += run("plugin_ref_pcg_csr24_cheb7", cs24, 24, 7, false);
  bad += run("plugin_ref_pcg_stencil32_newton3", st32, 32, 3, true);
  // power_method / dacg_smallest (eigenest.cpp:48-167) on the device operator
  {
    auto [scaled, d] = jacobi_scale(st32);
    polycg::gpu::DeviceLinearOperator dlo(sess, scaled);
    const EigResult pc = polycg::power_method(scaled), pg = polycg::power_method(dlo);
    EigOptions dopt;
    dopt.tol = 1e-2;
    dopt.maxit = 5000;
    const EigResult dc = polycg::dacg_smallest(scaled, dopt), dg = polycg::dacg_smallest(dlo, dopt);
    const bool ok = pc.value == pg.value && pc.iters == pg.iters && pc.matvecs == pg.matvecs &&
                    dc.value == dg.value && dc.iters == dg.iters && dc.matvecs == dg.matvecs &&
                    pc.trace == pg.trace && dc.trace == dg.trace;
    std::printf("{\"case\": \"plugin_ref_power_dacg_stencil32\", \"ok\": %s, \"power\": [%.17g, %.17g], "
                "\"dacg\": [%.17g, %.17g], \"iters\": [%d, %d, %d, %d]}\n",
                ok ? "true" : "false", pc.value, pg.value, dc.value, dg.value, pc.iters, pg.iters, dc.iters,
                dg.iters);
    bad += ok ? 0 : 1;
  }
  // the one-shot drop-in pcg_solve caches its session and operator upload
  {
    auto [scaled, d] = jacobi_scale(st32);
    const auto [a0, b0] = analytic_extremes(StencilKind::lap3d, 32, true);
    const Vector b = scaled.apply(random_uniform_vector(scaled.size(), 20240801));
    ChebyshevPreconditioner p(cheb_params(a0, b0, 10, 1.001));
    auto& ds = polycg::gpu::default_session(0);
    const int u0 = ds.uploads();
    auto [x1, r1] = polycg::gpu::pcg_solve(scaled, b, {}, &p);
    auto [x2, r2] = polycg::gpu::pcg_solve(scaled, b, {}, &p);
    const int ups = ds.uploads() - u0;
    const bool ok = ups == 1 && same_bits(x1, x2) && r1.iters == r2.iters;
    std::printf("{\"case\": \"oneshot_upload_cached\", \"ok\": %s, \"uploads\": %d}\n",
                ok ? "true" : "false", ups);
    bad += ok ? 0 : 1;
  }
  return bad;
}

int main() {
  set_apply_threads(8);
  polycg::gpu::Session sess(0);
  int bad = 0;
  const StencilOperator st40(StencilKind::lap3d, 40);
  bad += run_case("stencil40_m10", st40, 40, 10, 1.001, sess);
  const CsrMatrix cs30 = assemble_laplacian(StencilKind::lap3d, 30);
  bad += run_case("csr30_m20", cs30, 30, 20, 1.001, sess);
  // NewtonPreconditioner (pcg.hpp:27-40): same call, same answer
  {
    auto [scaled, d] = jacobi_scale(st40);
    const auto [a0, b0] = analytic_extremes(StencilKind::lap3d, 40, true);
    const Vector b = scaled.apply(random_uniform_vector(scaled.size(), 20240801));
    NewtonPreconditioner p_cpu(newton_params(a0, b0, 3, 1.001));
    NewtonPreconditioner p_gpu(newton_params(a0, b0, 3, 1.001));
    auto [x_ref, r_ref] = pcg_solve(scaled, b, {}, &p_cpu);
    polycg::gpu::DeviceOperator dop(sess, scaled);
    auto [x_gpu, r_gpu] = polycg::gpu::pcg_solve(sess, dop, scaled, b, {}, &p_gpu);
    double dn = 0.0, xn = 0.0;
    for (Index i = 0; i < x_ref.size(); ++i) {
      dn += (x_gpu[i] - x_ref[i]) * (x_gpu[i] - x_ref[i]);
      xn += x_ref[i] * x_ref[i];
    }
    const double rel = std::sqrt(dn / xn);
    Vector r0 = random_uniform_vector(scaled.size(), 4242), o_gpu;
    const Vector o_cpu = apply_newton(newton_params(a0, b0, 4, 1.001), scaled, r0);
    polycg::gpu::apply_newton(sess, dop, newton_params(a0, b0, 4, 1.001), r0, o_gpu);
    bool bitwise = true;
    for (Index i = 0; i < r0.size(); ++i) bitwise = bitwise && (o_cpu[i] == o_gpu[i]);
    const bool ok = std::abs(r_gpu.iters - r_ref.iters) <= 1 && rel <= 1e-10 && bitwise &&
                    r_gpu.ddot == r_ref.ddot && r_gpu.matvec == r_ref.matvec;
    std::printf("{\"case\": \"stencil40_newton3\", \"ok\": %s, \"iters\": [%d, %d], "
                "\"x_rel_diff\": %.3e, \"newton4_bitwise\": %s}\n",
                ok ? "true" : "false", r_ref.iters, r_gpu.iters, rel, bitwise ? "true" : "false");
    bad += ok ? 0 : 1;
  }
  // SolveOptions::on_iterate (pcg.hpp:62-63, pcg.cpp:88): the same (iteration, x)
  // sequence as the reference; an exception thrown by the callback propagates
  {
    const StencilOperator st24(StencilKind::lap3d, 24);
    auto [scaled, d] = jacobi_scale(st24);
    const auto [a0, b0] = analytic_extremes(StencilKind::lap3d, 24, true);
    const Vector b = scaled.apply(random_uniform_vector(scaled.size(), 20240801));
    ChebyshevPreconditioner p_cpu(cheb_params(a0, b0, 6, 1.001));
    ChebyshevPreconditioner p_gpu(cheb_params(a0, b0, 6, 1.001));
    std::vector<std::pair<int, Vector>> seq_cpu, seq_gpu;
    SolveOptions o_cpu, o_gpu;
    o_cpu.on_iterate = [&](int it, const Vector& x) { seq_cpu.emplace_back(it, x); };
    o_gpu.on_iterate = [&](int it, const Vector& x) { seq_gpu.emplace_back(it, x); };
    auto [x_ref, r_ref] = pcg_solve(scaled, b, o_cpu, &p_cpu);
    polycg::gpu::DeviceOperator dop(sess, scaled);
    auto [x_gpu, r_gpu] = polycg::gpu::pcg_solve(sess, dop, scaled, b, o_gpu, &p_gpu);
    bool ok = seq_cpu.size() == seq_gpu.size() && (int)seq_gpu.size() == r_gpu.iters;
    double worst = 0.0;
    for (size_t k = 0; ok && k < seq_cpu.size(); ++k) {
      ok = seq_cpu[k].first == seq_gpu[k].first;
      double dn = 0.0, xn = 0.0;
      for (Index i = 0; i < seq_cpu[k].second.size(); ++i) {
        const double e = seq_gpu[k].second[i] - seq_cpu[k].second[i];
        dn += e * e;
        xn += seq_cpu[k].second[i] * seq_cpu[k].second[i];
      }
      worst = std::max(worst, std::sqrt(dn / xn));
    }
    bool last_is_x = !seq_gpu.empty();
    for (Index i = 0; last_is_x && i < x_gpu.size(); ++i) last_is_x = seq_gpu.back().second[i] == x_gpu[i];
    ok = ok && worst <= 1e-10 && last_is_x;
    bool thrown = false;
    SolveOptions o_stop;
    o_stop.on_iterate = [](int it, const Vector&) {
      if (it == 3) throw std::runtime_error("stop at 3");
    };
    try {
      polycg::gpu::pcg_solve(sess, dop, scaled, b, o_stop, &p_gpu);
    } catch (const std::runtime_error& e) {
      thrown = std::string(e.what()) == "stop at 3";
    }
    auto [x_again, r_again] = polycg::gpu::pcg_solve(sess, dop, scaled, b, {}, &p_gpu);
    ok = ok && thrown && r_again.converged && r_again.iters == r_gpu.iters;
    std::printf("{\"case\": \"on_iterate_stencil24_m6\", \"ok\": %s, \"calls\": [%zu, %zu], "
                "\"worst_x_rel_diff\": %.3e, \"exception_propagated\": %s}\n",
                ok ? "true" : "false", seq_cpu.size(), seq_gpu.size(), worst, thrown ? "true" : "false");
    bad += ok ? 0 : 1;
  }
  // error path: an unknown preconditioner type is rejected like a bad argument
  struct Half : Preconditioner {
    void apply(const LinearOperator&, const Vector& r, Vector& z) override { z = 0.5 * r; }
    int degree() const override { return 0; }
  } half;
  try {
    auto [scaled, d] = jacobi_scale(st40);
    polycg::gpu::pcg_solve(scaled, Vector::Ones(scaled.size()), {}, &half);
    bad += 1;
  } catch (const std::invalid_argument&) {
    std::printf("{\"case\": \"reject_custom_prec\", \"ok\": true}\n");
  }
  bad += plugin_cases(sess);
  return bad == 0 ? 0 : 1;
}
