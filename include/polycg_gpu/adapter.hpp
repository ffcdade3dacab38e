// SPDX-License-Identifier: Apache-2.0
//
// polycg::gpu — the reference-side binding of the B200 library (header-only).
//
// A maintainer of the reference (`polycg`, /root/reference/proj) adds this header
// and links libpcgx.so; call sites then switch from
//     polycg::pcg_solve(op, b, opts, &prec)              (include/polycg/pcg.hpp:89-91)
// to
//     polycg::gpu::pcg_solve(op, b, opts, &prec)
// with the same arguments, the same return type and the same exceptions.
//
// Supported inputs — exactly what the hot path covers:
//   op   : ScaledOperator over StencilOperator(lap3d, nx) or CsrMatrix
//          (what jacobi_scale returns, src/linop.cpp:340-351)
//   prec : ChebyshevPreconditioner (pcg.hpp:42-55), NewtonPreconditioner
//          (pcg.hpp:27-40) or nullptr (plain CG)
// Anything else throws std::invalid_argument (there is no silent CPU fallback).
//
// Depends on the reference's headers (polycg/linop.hpp, polycg/pcg.hpp) and on
// include/pcgx.h. One Session owns a device context; like the reference's
// Preconditioner, use one per concurrent solve (pcg.hpp:16-19).
#ifndef POLYCG_GPU_ADAPTER_HPP
#define POLYCG_GPU_ADAPTER_HPP

#include <algorithm>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>

#include "pcgx.h"
#include "polycg/linop.hpp"
#include "polycg/pcg.hpp"
#include "polycg/polyprec.hpp"

namespace polycg::gpu {

[[noreturn]] inline void rethrow(pcgx_status st, const char* msg) {
  if (st == PCGX_ERR_NUMERICAL) throw NumericalError(msg);
  if (st == PCGX_ERR_INVALID || st == PCGX_ERR_UNSUPPORTED || st == PCGX_ERR_OVERFLOW)
    throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

inline void check(pcgx_status st, pcgx_context ctx) {
  if (st != PCGX_OK) rethrow(st, pcgx_last_error(ctx));
}

class Session {
 public:
  explicit Session(int device = 0) { check(pcgx_context_create(device, &ctx_), nullptr); }
  ~Session() { pcgx_context_destroy(ctx_); }
  Session(const Session&) = delete;
  Session& operator=(const Session&) = delete;
  pcgx_context get() const { return ctx_; }

 private:
  pcgx_context ctx_ = nullptr;
};

// Uploads a reference operator (ScaledOperator over a 3D stencil or a CSR).
class DeviceOperator {
 public:
  DeviceOperator(const Session& s, const LinearOperator& op) : ctx_(s.get()) {
    const auto* scaled = dynamic_cast<const ScaledOperator*>(&op);
    if (!scaled)
      throw std::invalid_argument("gpu::pcg_solve: operator must be a ScaledOperator (jacobi_scale)");
    const Vector& d = scaled->inv_sqrt_diag();
    if (const auto* st = dynamic_cast<const StencilOperator*>(&scaled->inner())) {
      if (st->kind() != StencilKind::lap3d)
        throw std::invalid_argument("gpu::pcg_solve: only the 3D 7-point stencil is accelerated");
      for (Index i = 1; i < d.size(); ++i)
        if (!(d[i] == d[0]))
          throw std::invalid_argument("gpu::pcg_solve: stencil scaling must be constant");
      check(pcgx_stencil7_create(ctx_, st->nx(), st->nx(), st->nx(), d.size() ? d[0] : 0.0, &h_),
            ctx_);
    } else if (const auto* csr = dynamic_cast<const CsrMatrix*>(&scaled->inner())) {
      static_assert(sizeof(Index) == sizeof(int64_t), "polycg::Index is int64");
      check(pcgx_csr_create(ctx_, csr->size(),
                            reinterpret_cast<const int64_t*>(csr->row_ptr().data()),
                            reinterpret_cast<const int64_t*>(csr->col_idx().data()),
                            csr->values().data(), d.data(), &h_),
            ctx_);
    } else {
      throw std::invalid_argument("gpu::pcg_solve: inner operator must be StencilOperator or CsrMatrix");
    }
  }
  ~DeviceOperator() { pcgx_operator_destroy(h_); }
  DeviceOperator(const DeviceOperator&) = delete;
  DeviceOperator& operator=(const DeviceOperator&) = delete;
  pcgx_operator get() const { return h_; }

 private:
  pcgx_context ctx_;
  pcgx_operator h_ = nullptr;
};

// Same contract as polycg::pcg_solve (src/pcg.cpp:10-117).
inline std::pair<Vector, SolveReport> pcg_solve(const Session& s, const DeviceOperator& dop,
                                                const LinearOperator& op, const Vector& b,
                                                const SolveOptions& opts = {},
                                                Preconditioner* prec = nullptr) {
  const Index n = op.size();
  if (b.size() != n) throw std::invalid_argument("pcg_solve: rhs length mismatch");
  if (opts.x0 && opts.x0->size() != n) throw std::invalid_argument("pcg_solve: x0 length mismatch");
  pcgx_cheb cheb{};
  const pcgx_cheb* cp = nullptr;
  pcgx_newton newton{};
  const pcgx_newton* np = nullptr;
  if (prec) {
    if (auto* c = dynamic_cast<ChebyshevPreconditioner*>(prec)) {
      const ChebyshevParams& p = c->params();
      cheb.m = p.m;
      cheb.theta = p.theta;
      cheb.delta = p.delta;
      cheb.sigma = p.sigma;
      cheb.rho = p.rho.data();
      cp = &cheb;
    } else if (auto* nw = dynamic_cast<NewtonPreconditioner*>(prec)) {
      newton.nlev = nw->params().nlev;
      newton.zeta = nw->params().zeta.data();
      np = &newton;
    } else {
      throw std::invalid_argument(
          "gpu::pcg_solve: only ChebyshevPreconditioner and NewtonPreconditioner are accelerated");
    }
  }
  pcgx_solve_opts o;
  pcgx_solve_opts_default(&o);
  o.tol = opts.tol;
  o.maxit = opts.maxit;
  o.x0 = opts.x0 ? opts.x0->data() : nullptr;
  // on_iterate(it, x) (pcg.cpp:88): the library hands a host copy of x; an
  // exception the callback throws is held here and rethrown after the C call
  struct Iterate {
    const SolveOptions* opts;
    Vector xv;
    std::exception_ptr err;
  } it_state{&opts, Vector(), nullptr};
  if (opts.on_iterate) {
    o.on_iterate = [](int64_t it, const double* xh, int64_t nx, void* user) -> int {
      auto* st = static_cast<Iterate*>(user);
      try {
        st->xv.resize(static_cast<Index>(nx));
        std::copy(xh, xh + nx, st->xv.data());
        st->opts->on_iterate(static_cast<int>(it), st->xv);
        return 0;
      } catch (...) {
        st->err = std::current_exception();
        return 1;
      }
    };
    o.on_iterate_user = &it_state;
  }
  pcgx_report r{};
  Vector x(n);
  const pcgx_status st = np ? pcgx_pcg_solve_newton(s.get(), dop.get(), np, b.data(), x.data(), &o, &r)
                            : pcgx_pcg_solve(s.get(), dop.get(), cp, b.data(), x.data(), &o, &r);
  if (it_state.err) std::rethrow_exception(it_state.err);
  check(st, s.get());
  SolveReport rep;
  rep.iters = static_cast<int>(r.iters);
  rep.ddot = static_cast<std::uint64_t>(r.ddot);
  rep.matvec = static_cast<std::uint64_t>(r.matvec);
  rep.prec_applies = static_cast<std::uint64_t>(r.prec_applies);
  rep.rel_res = r.rel_res;
  rep.true_rel_res = r.true_rel_res;
  rep.wall_time = r.wall_time;
  rep.converged = r.converged != 0;
  return {std::move(x), rep};
}

// Drop-in overload: uploads the operator for this one call.
inline std::pair<Vector, SolveReport> pcg_solve(const LinearOperator& op, const Vector& b,
                                                const SolveOptions& opts = {},
                                                Preconditioner* prec = nullptr, int device = 0) {
  Session s(device);
  DeviceOperator dop(s, op);
  return pcg_solve(s, dop, op, b, opts, prec);
}

// out = p_m(A) r on the device (apply_chebyshev, src/polyprec.cpp:169-198).
inline void apply_chebyshev(const Session& s, const DeviceOperator& dop,
                            const ChebyshevParams& p, const Vector& r, Vector& out) {
  const pcgx_cheb cheb{p.m, p.theta, p.delta, p.sigma, p.rho.data()};
  out.resize(r.size());
  check(pcgx_cheb_apply(s.get(), dop.get(), &cheb, r.data(), out.data()), s.get());
}

// out = P_nlev(A) r on the device (apply_newton, src/polyprec.cpp:148-160).
inline void apply_newton(const Session& s, const DeviceOperator& dop, const NewtonParams& p,
                         const Vector& r, Vector& out) {
  const pcgx_newton nw{p.nlev, p.zeta.data()};
  out.resize(r.size());
  check(pcgx_newton_apply(s.get(), dop.get(), &nw, r.data(), out.data()), s.get());
}

}  // namespace polycg::gpu

#endif  // POLYCG_GPU_ADAPTER_HPP
