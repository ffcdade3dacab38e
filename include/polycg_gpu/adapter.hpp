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
//
// The reference's own extension points are served as well, so callers that keep
// polycg::pcg_solve / power_method / dacg_smallest run their operator and
// preconditioner work on the GPU:
//   DeviceLinearOperator : LinearOperator   (include/polycg/linop.hpp:21-47)
//       apply_impl = one device SpMV (host vectors in and out per call)
//   ChebyshevPreconditioner / NewtonPreconditioner : Preconditioner
//       (include/polycg/pcg.hpp:20-55) apply = p_m(A) r on the device
// Both are bitwise the reference's operator / apply_chebyshev / apply_newton, so
// polycg::pcg_solve(DeviceLinearOperator, b, opts, &gpu::ChebyshevPreconditioner)
// returns the reference's x bit for bit (its reductions still run on the host).
// Sessions upload each operator once (cache keyed by the operator's identity and
// a fingerprint of its data; operators are immutable, linop.hpp:17-20).
#ifndef POLYCG_GPU_ADAPTER_HPP
#define POLYCG_GPU_ADAPTER_HPP

#include <algorithm>
#include <cstdint>
#include <exception>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>
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

class DeviceOperator;

class Session {
 public:
  explicit Session(int device = 0) { check(pcgx_context_create(device, &ctx_), nullptr); }
  ~Session();
  Session(const Session&) = delete;
  Session& operator=(const Session&) = delete;
  pcgx_context get() const { return ctx_; }
  // The device copy of a reference operator, uploaded on first use and kept for
  // the session's lifetime (operators are immutable after construction).
  const DeviceOperator& upload(const LinearOperator& op);
  // Number of operator uploads this session performed (cache misses).
  int uploads() const { return uploads_; }
  // Serialises calls on the context (a context runs one call at a time).
  std::mutex& mutex() { return mu_; }

 private:
  pcgx_context ctx_ = nullptr;
  std::mutex mu_;
  int uploads_ = 0;
  using Key = std::tuple<const void*, const void*, const void*, Index, std::uint64_t>;
  std::map<Key, std::unique_ptr<DeviceOperator>> cache_;
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

inline Session::~Session() {
  cache_.clear();  // operators before their context
  pcgx_context_destroy(ctx_);
}

// Identity + fingerprint of a reference operator: the addresses of the operator,
// its inner operator and its data, the size, and a hash of the scaling and of 64
// sampled CSR entries (a freed-and-reallocated operator at the same address with
// other data misses the cache).
inline const DeviceOperator& Session::upload(const LinearOperator& op) {
  const auto* scaled = dynamic_cast<const ScaledOperator*>(&op);
  const void* inner = scaled ? static_cast<const void*>(&scaled->inner()) : nullptr;
  const void* data = nullptr;
  std::uint64_t h = 1469598103934665603ull;
  auto mix = [&h](const void* p, std::size_t nb) {
    const auto* c = static_cast<const unsigned char*>(p);
    for (std::size_t i = 0; i < nb; ++i) h = (h ^ c[i]) * 1099511628211ull;
  };
  if (scaled) {
    const Vector& d = scaled->inv_sqrt_diag();
    if (d.size()) {
      mix(d.data(), sizeof(double));
      mix(d.data() + (d.size() - 1), sizeof(double));
    }
    if (const auto* csr = dynamic_cast<const CsrMatrix*>(&scaled->inner())) {
      data = csr->values().data();
      const Index nnz = csr->nnz();
      for (int k = 0; k < 64 && nnz > 0; ++k) {
        const Index e = static_cast<Index>((static_cast<std::uint64_t>(k) * 2654435761u) % nnz);
        mix(&csr->values()[e], sizeof(double));
        mix(&csr->col_idx()[e], sizeof(Index));
      }
    } else if (const auto* st = dynamic_cast<const StencilOperator*>(&scaled->inner())) {
      const Index nx = st->nx();
      mix(&nx, sizeof nx);
    }
  }
  const Key key{static_cast<const void*>(&op), inner, data, op.size(), h};
  std::lock_guard<std::mutex> lk(mu_);
  auto it = cache_.find(key);
  if (it == cache_.end()) {
    it = cache_.emplace(key, std::make_unique<DeviceOperator>(*this, op)).first;
    ++uploads_;
  }
  return *it->second;
}

// The process-wide session of a device, created on first use and kept until exit
// (never destroyed: CUDA may already be torn down when static destructors run).
inline Session& default_session(int device = 0) {
  static std::mutex mu;
  static std::map<int, Session*> sessions;
  std::lock_guard<std::mutex> lk(mu);
  Session*& s = sessions[device];
  if (!s) s = new Session(device);
  return *s;
}

// LinearOperator (linop.hpp:21-47) whose apply is one device SpMV of the wrapped
// reference operator (ScaledOperator over StencilOperator(lap3d) or CsrMatrix):
// bitwise ScaledOperator::apply (linop.cpp:271-275). Host vectors cross per call,
// so the reference's own algorithms (pcg_solve, power_method, dacg_smallest)
// run unchanged on top of it. diagonal() is the wrapped operator's. The wrapped
// operator must outlive this one (like ScaledOperator's inner, linop.hpp:110-111).
// Note: LinearOperator::matvec_count of THIS object counts its applies; the
// device SpMVs of a gpu::ChebyshevPreconditioner are counted by the device
// operator (pcgx_operator_matvec_count) and by pcg_solve's SolveReport.
class DeviceLinearOperator : public LinearOperator {
 public:
  DeviceLinearOperator(Session& s, const LinearOperator& op)
      : LinearOperator(op.size()), s_(&s), ref_(&op), dop_(&s.upload(op)) {}
  explicit DeviceLinearOperator(const LinearOperator& op, int device = 0)
      : DeviceLinearOperator(default_session(device), op) {}

  Vector diagonal() const override { return ref_->diagonal(); }
  Session& session() const { return *s_; }
  const DeviceOperator& device() const { return *dop_; }

 private:
  void apply_impl(const Vector& x, Vector& y) const override {
    std::lock_guard<std::mutex> lk(s_->mutex());
    check(pcgx_operator_apply(s_->get(), dop_->get(), x.data(), y.data()), s_->get());
  }

  Session* s_;
  const LinearOperator* ref_;
  const DeviceOperator* dop_;
};

namespace detail {
// The device copy of the operator a preconditioner is applied with: a
// DeviceLinearOperator's own, else the session's cached upload.
inline const DeviceOperator& device_of(Session& s, const LinearOperator& op) {
  if (const auto* d = dynamic_cast<const DeviceLinearOperator*>(&op))
    if (&d->session() == &s) return d->device();
  return s.upload(op);
}
}  // namespace detail

// Preconditioner (pcg.hpp:20-25) applying p_m(A) r on the device: bitwise
// apply_chebyshev (polyprec.cpp:169-198) for the operator pcg_solve passes in.
class ChebyshevPreconditioner : public Preconditioner {
 public:
  ChebyshevPreconditioner(Session& s, ChebyshevParams params) : s_(&s), params_(std::move(params)) {}
  explicit ChebyshevPreconditioner(ChebyshevParams params, int device = 0)
      : ChebyshevPreconditioner(default_session(device), std::move(params)) {}

  void apply(const LinearOperator& op, const Vector& r, Vector& z) override {
    if (r.size() != op.size()) throw std::invalid_argument("apply_chebyshev: size mismatch");
    const DeviceOperator& dop = detail::device_of(*s_, op);
    const pcgx_cheb c{params_.m, params_.theta, params_.delta, params_.sigma, params_.rho.data()};
    z.resize(r.size());
    std::lock_guard<std::mutex> lk(s_->mutex());
    check(pcgx_cheb_apply(s_->get(), dop.get(), &c, r.data(), z.data()), s_->get());
  }
  int degree() const override { return params_.m; }
  const ChebyshevParams& params() const { return params_; }

 private:
  Session* s_;
  ChebyshevParams params_;
};
using GpuChebyshevPreconditioner = ChebyshevPreconditioner;

// Preconditioner applying the Newton form P_nlev(A) r on the device: bitwise
// apply_newton (polyprec.cpp:135-160).
class NewtonPreconditioner : public Preconditioner {
 public:
  NewtonPreconditioner(Session& s, NewtonParams params) : s_(&s), params_(std::move(params)) {}
  explicit NewtonPreconditioner(NewtonParams params, int device = 0)
      : NewtonPreconditioner(default_session(device), std::move(params)) {}

  void apply(const LinearOperator& op, const Vector& r, Vector& z) override {
    if (r.size() != op.size()) throw std::invalid_argument("apply_newton: size mismatch");
    const DeviceOperator& dop = detail::device_of(*s_, op);
    const pcgx_newton nw{params_.nlev, params_.zeta.data()};
    z.resize(r.size());
    std::lock_guard<std::mutex> lk(s_->mutex());
    check(pcgx_newton_apply(s_->get(), dop.get(), &nw, r.data(), z.data()), s_->get());
  }
  int degree() const override { return params_.degree(); }
  const NewtonParams& params() const { return params_; }

 private:
  Session* s_;
  NewtonParams params_;
};
using GpuNewtonPreconditioner = NewtonPreconditioner;

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
    const ChebyshevParams* cpar = nullptr;
    const NewtonParams* npar = nullptr;
    if (auto* c = dynamic_cast<polycg::ChebyshevPreconditioner*>(prec)) cpar = &c->params();
    else if (auto* g = dynamic_cast<ChebyshevPreconditioner*>(prec)) cpar = &g->params();
    else if (auto* nw = dynamic_cast<polycg::NewtonPreconditioner*>(prec)) npar = &nw->params();
    else if (auto* gn = dynamic_cast<NewtonPreconditioner*>(prec)) npar = &gn->params();
    if (cpar) {
      const ChebyshevParams& p = *cpar;
      cheb.m = p.m;
      cheb.theta = p.theta;
      cheb.delta = p.delta;
      cheb.sigma = p.sigma;
      cheb.rho = p.rho.data();
      cp = &cheb;
    } else if (npar) {
      newton.nlev = npar->nlev;
      newton.zeta = npar->zeta.data();
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

// Drop-in overload: the device's default session, the operator uploaded once per
// session (cached), so repeated solves on one operator pay no re-upload.
inline std::pair<Vector, SolveReport> pcg_solve(const LinearOperator& op, const Vector& b,
                                                const SolveOptions& opts = {},
                                                Preconditioner* prec = nullptr, int device = 0) {
  Session& s = default_session(device);
  const DeviceOperator& dop = detail::device_of(s, op);
  std::lock_guard<std::mutex> lk(s.mutex());
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
