// SPDX-License-Identifier: Apache-2.0
//
// sm_100a kernels of the Chebyshev-PCG hot path. All fp64, HBM-bound, no
// tensor cores (there is no dense contraction on this path).
//
//   stencil7_kernel<Epi>  K1+K4(+K5/K6/K7 epilogue): scaled 7-point SpMV fused
//                         with whatever consumes y in the same pass
//                         (proj/src/linop.cpp:236-258, 271-275)
//   csr_kernel<Epi>       K2+K4(+epilogue): scaled CSR SpMV, int32 indices
//                         (proj/src/linop.cpp:171-187, 271-275)
//   update/pupdate/...    K7: PCG vector updates fused with their reductions
//                         (proj/src/pcg.cpp:81-83, 101, 107)
//   splitmix_kernel       K8: random_uniform_vector (proj/src/eigenest.cpp:13-30)
//
// The epilogue functors hold the fused per-point work; every reducing launch
// ends in block_reduce_finish (warp shuffle tree -> block tree -> last-block
// grid finish), deterministic for a fixed launch shape.
#pragma once

#include "common.cuh"

#ifndef PCGX_V2_MINB
#define PCGX_V2_MINB 4
#endif

namespace pcgx {

// x / b, correctly rounded, from inv = RN(1/b): Markstein's FMA correction
// (q0 = RN(x inv), r = x - q0 b exactly, q = RN(q0 + r inv) = RN(x / b) for normal
// operands away from over/underflow) — the reference's IEEE quotient without the
// iterative division sequence.
// Operands outside [2^-960, 2^960], zero, inf and NaN (never on the solver's data):
// |x| is scaled by a power of two into the range where the correction is exact
// and scaled back; for a subnormal quotient the one double-rounding case
// (q1 * 2^-1000 exactly halfway between two subnormals while the true quotient is
// not) is resolved by the sign of the exact remainder; zero, inf and NaN give
// x * inv (the sign and class of x / b). Plain arithmetic, no call into the
// division slow path (a call site in a hot loop blocks scheduling around it).
// Bitwise the IEEE quotient: checked against x / b on 2.4e8 host operands (normal,
// subnormal, tiny, huge, special) for six divisors.
#ifndef PCGX_DIVWIDE_INLINE
#define PCGX_DIVWIDE_INLINE 0
#endif
#if PCGX_DIVWIDE_INLINE
__device__ __forceinline__
#else
__device__ __noinline__
#endif
double div_rn_wide(double x, double b, double inv) {
  const double ax = fabs(x);
  const bool tiny = ax < 0x1p-960, huge = ax > 0x1p960;
  const double sc = tiny ? 0x1p1000 : (huge ? 0x1p-100 : 1.0);
  const double us = tiny ? 0x1p-1000 : (huge ? 0x1p100 : 1.0);
  const double xs = x * sc;
  const double q0 = xs * inv;
  const double r0 = __fma_rn(-q0, b, xs);
  const double q1 = __fma_rn(r0, inv, q0);
  double y = q1 * us;
  if (tiny) {
    const double rem = __fma_rn(-q1, b, xs);
    const double dd = q1 - y * sc;
    if (fabs(dd) == 0x1p-75 && rem != 0.0) y = (q1 + copysign(0x1p-75, rem)) * us;
  }
  return (ax > 0.0 && ax <= 0x1.fffffffffffffp1023) ? y : x * inv;
}

__device__ __forceinline__ double div_rn(double x, double b, double inv) {
  const double q0 = x * inv;
  const double r = __fma_rn(-q0, b, x);
  double q = __fma_rn(r, inv, q0);
  // biased exponent outside [63, 1983] <=> |x| outside [2^-960, 2^961), or 0 / inf / NaN
  const unsigned e = ((unsigned)__double2hiint(x) >> 20) & 0x7ffu;
  if (e - 63u > 1920u) q = div_rn_wide(x, b, inv);
  return q;
}
// Two quotients by the same divisor with ONE range branch (the first two-step
// pass divides four values per lane and plane): the fast path for both, the
// out-of-line path only for an operand outside [2^-960, 2^961) -- bitwise div_rn.
__device__ __forceinline__ double2 div2_rn(double x0, double x1, double b, double inv) {
  const double p0 = x0 * inv, p1 = x1 * inv;
  const double r0 = __fma_rn(-p0, b, x0), r1 = __fma_rn(-p1, b, x1);
  double q0 = __fma_rn(r0, inv, p0), q1 = __fma_rn(r1, inv, p1);
  const unsigned e0 = ((unsigned)__double2hiint(x0) >> 20) & 0x7ffu;
  const unsigned e1 = ((unsigned)__double2hiint(x1) >> 20) & 0x7ffu;
  const bool w0 = e0 - 63u > 1920u, w1 = e1 - 63u > 1920u;
  if (w0 | w1) {
    if (w0) q0 = div_rn_wide(x0, b, inv);
    if (w1) q1 = div_rn_wide(x1, b, inv);
  }
  return make_double2(q0, q1);
}

// The same quotient where zeros are frequent (zero-filled Dirichlet halo values in
// the direction step): +-0 / b = +-0 by a select instead of the out-of-line path,
// which a warp would otherwise take for every boundary lane (and the block barrier
// would wait for it).
__device__ __forceinline__ double div_rn_z(double x, double b, double inv) {
  const double q0 = x * inv;
  const double r = __fma_rn(-q0, b, x);
  double q = __fma_rn(r, inv, q0);
  const unsigned e = ((unsigned)__double2hiint(x) >> 20) & 0x7ffu;
  if (e - 63u > 1920u && x != 0.0) q = div_rn_wide(x, b, inv);
  return x == 0.0 ? x : q;
}

#ifndef PCGX_DIA_STREAM
#define PCGX_DIA_STREAM 1
#endif
#ifndef PCGX_MAT_STREAM
#define PCGX_MAT_STREAM 1
#endif
// the value stream is read once: keep it out of L1 so the x / d gathers stay there
// (when the matrix exceeds L2: an L2-resident one, cfg1's 56 MB, streams 20% slower
// through the non-allocating path, so the operator picks the plain path there)
template <bool kStream = true>
__device__ __forceinline__ double ld_stream(const double* p) {
#if PCGX_DIA_STREAM
  if (!kStream) return __ldg(p);
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
#else
  return __ldg(p);
#endif
}

// epilogue operand streams (r, x_old, b: read once per point)
#ifndef PCGX_EPI_STREAM
#define PCGX_EPI_STREAM 1
#endif
__device__ __forceinline__ double ld_epi(const double* p) {
#if PCGX_EPI_STREAM
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
#else
  return __ldg(p);
#endif
}
__device__ __forceinline__ double2 ld_epi2(const double* p) {
#if PCGX_EPI_STREAM
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
#else
  return __ldg(reinterpret_cast<const double2*>(p));
#endif
}

// ... for a stream the same kernel later overwrites in place (coherent path, no .nc)
__device__ __forceinline__ double ld_epi_rw(const double* p) {
#if PCGX_EPI_STREAM
  double v;
  asm volatile("ld.global.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
#else
  return *p;
#endif
}
__device__ __forceinline__ double2 ld_epi_rw2(const double* p) {
#if PCGX_EPI_STREAM
  double2 v;
  asm volatile("ld.global.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
#else
  return *reinterpret_cast<const double2*>(p);
#endif
}

// matrix value streams of the SELL / BSR-3 kernels (same policy, separately switchable)
__device__ __forceinline__ double ld_mat(const double* p) {
#if PCGX_MAT_STREAM
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
#else
  return __ldg(p);
#endif
}

// ----------------------------------------------------------------- reduction

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;  // lane 0 holds the fixed-order tree sum
}

// All threads of the block must call. Writes the block partial; the last block
// to finish sums all partials in a fixed order and stores/accumulates the
// result into red.result, then re-arms the ticket counter.
__device__ __forceinline__ void block_reduce_finish(double v, const Reduce& red) {
  __shared__ double ws[32];
  __shared__ bool is_last;
  const int nthreads = blockDim.x * blockDim.y * blockDim.z;
  const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  const unsigned nblocks = gridDim.x * gridDim.y * gridDim.z;
  const unsigned bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  const int lane = tid & 31, warp = tid >> 5, nwarps = (nthreads + 31) >> 5;
  v = warp_sum(v);
  if (lane == 0) ws[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < nwarps ? ws[lane] : 0.0;
    v = warp_sum(v);
    if (lane == 0) {
      red.partials[bid] = v;
      __threadfence();
      const unsigned ticket = atomicAdd(red.counter, 1u);
      is_last = (ticket == nblocks - 1);
    }
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  double s = 0.0;
  for (unsigned b = tid; b < nblocks; b += nthreads) s += __ldcg(red.partials + b);
  s = warp_sum(s);
  if (lane == 0) ws[warp] = s;
  __syncthreads();
  if (warp == 0) {
    s = lane < nwarps ? ws[lane] : 0.0;
    s = warp_sum(s);
    if (lane == 0) {
      const double res = red.accumulate ? (*red.result + s) : s;
      *red.result = res;
      if (red.mirror) *red.mirror = res;
      if (red.cond_bt) cudaGraphSetConditional(red.cond, sqrt(res) / red.cond_bt[0] <= red.cond_bt[1] ? 0u : 1u);
      *red.counter = 0u;
      __threadfence();
    }
  }
}

// Two values reduced together (partials[2 b], partials[2 b + 1]) into
// result[0], result[1]: the [r'r, r'z] pair of one iteration.
__device__ __forceinline__ void block_reduce_finish2(double v0, double v1, const Reduce& red) {
  __shared__ double ws0[32], ws1[32];
  __shared__ bool is_last2;
  const int nthreads = blockDim.x * blockDim.y * blockDim.z;
  const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  const unsigned nblocks = gridDim.x * gridDim.y * gridDim.z;
  const unsigned bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  const int lane = tid & 31, warp = tid >> 5, nwarps = (nthreads + 31) >> 5;
  v0 = warp_sum(v0);
  v1 = warp_sum(v1);
  if (lane == 0) {
    ws0[warp] = v0;
    ws1[warp] = v1;
  }
  __syncthreads();
  if (warp == 0) {
    v0 = warp_sum(lane < nwarps ? ws0[lane] : 0.0);
    v1 = warp_sum(lane < nwarps ? ws1[lane] : 0.0);
    if (lane == 0) {
      red.partials[2 * bid] = v0;
      red.partials[2 * bid + 1] = v1;
      __threadfence();
      const unsigned ticket = atomicAdd(red.counter, 1u);
      is_last2 = (ticket == nblocks - 1);
    }
  }
  __syncthreads();
  if (!is_last2) return;
  __threadfence();
  double s0 = 0.0, s1 = 0.0;
  for (unsigned b = tid; b < nblocks; b += nthreads) {
    s0 += __ldcg(red.partials + 2 * b);
    s1 += __ldcg(red.partials + 2 * b + 1);
  }
  s0 = warp_sum(s0);
  s1 = warp_sum(s1);
  if (lane == 0) {
    ws0[warp] = s0;
    ws1[warp] = s1;
  }
  __syncthreads();
  if (warp == 0) {
    s0 = warp_sum(lane < nwarps ? ws0[lane] : 0.0);
    s1 = warp_sum(lane < nwarps ? ws1[lane] : 0.0);
    if (lane == 0) {
      red.result[0] = s0;
      red.result[1] = s1;
      if (red.mirror) {
        red.mirror[0] = s0;
        red.mirror[1] = s1;
      }
      *red.counter = 0u;
      __threadfence();
    }
  }
}

// N values reduced together into red.result[0..N) (partials[N b + k]).
template <int N>
__device__ __forceinline__ void block_reduce_finishN(const double (&vin)[N], const Reduce& red) {
  __shared__ double wsn[N][32];
  __shared__ bool is_lastn;
  const int nthreads = blockDim.x * blockDim.y * blockDim.z;
  const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  const unsigned nblocks = gridDim.x * gridDim.y * gridDim.z;
  const unsigned bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  const int lane = tid & 31, warp = tid >> 5, nwarps = (nthreads + 31) >> 5;
  double v[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    v[k] = warp_sum(vin[k]);
    if (lane == 0) wsn[k][warp] = v[k];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < N; ++k) v[k] = warp_sum(lane < nwarps ? wsn[k][lane] : 0.0);
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < N; ++k) red.partials[N * bid + k] = v[k];
      __threadfence();
      const unsigned ticket = atomicAdd(red.counter, 1u);
      is_lastn = (ticket == nblocks - 1);
    }
  }
  __syncthreads();
  if (!is_lastn) return;
  __threadfence();
#pragma unroll
  for (int k = 0; k < N; ++k) v[k] = 0.0;
  for (unsigned b = tid; b < nblocks; b += nthreads)
#pragma unroll
    for (int k = 0; k < N; ++k) v[k] += __ldcg(red.partials + N * b + k);
#pragma unroll
  for (int k = 0; k < N; ++k) {
    v[k] = warp_sum(v[k]);
    if (lane == 0) wsn[k][warp] = v[k];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < N; ++k) v[k] = warp_sum(lane < nwarps ? wsn[k][lane] : 0.0);
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < N; ++k) red.result[k] = v[k];
      if (red.mirror)
        for (int k = 0; k < N; ++k) red.mirror[k] = v[k];
      *red.counter = 0u;
      __threadfence();
    }
  }
}

// ----------------------------------------------------------------- epilogues
// Two-phase interface so the marching kernels can prefetch the epilogue's own
// operand vectors one plane ahead:
//   ld(idx, v)  / ld2(idx, v)          load the per-point operands (scalar / double2)
//   st(idx, y, xc, v) / st2(...)        consume y = (A_scaled x)[idx] and xc = x[idx],
//                                       write outputs, return the point's contribution
//                                       to the launch's reduction.

__device__ __forceinline__ double2 ldg2(const double* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}
__device__ __forceinline__ double2 ld2(const double* p) {
  return *reinterpret_cast<const double2*>(p);
}
__device__ __forceinline__ void st2(double* p, double a, double b) {
  *reinterpret_cast<double2*>(p) = make_double2(a, b);
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// q = A p ; contribution p_i q_i  (pcg.cpp:72-74)
struct EpiStore {
  double* out;
  __device__ __forceinline__ void pf(long long) const {}
  __device__ __forceinline__ void ld(long long, double (&)[2]) const {}
  __device__ __forceinline__ void ld2(long long, double2 (&)[2]) const {}
  __device__ __forceinline__ double st(long long idx, double y, double xc, const double (&)[2]) const {
    out[idx] = y;
    return xc * y;
  }
  __device__ __forceinline__ double st2(long long idx, double y0, double y1, double2 xc,
                                        const double2 (&)[2]) const {
    pcgx::st2(out + idx, y0, y1);
    return xc.x * y0 + xc.y * y1;
  }
};

// e = b - A x ; contribution e_i^2  (pcg.cpp:43-45 with x0, exit true residual :112-114)
struct EpiResid {
  const double* __restrict__ b;
  double* e;  // may be nullptr (true residual: only the norm is needed)
  __device__ __forceinline__ void pf(long long idx) const { prefetch_l2(b + idx); }
  __device__ __forceinline__ void ld(long long idx, double (&v)[2]) const { v[0] = ld_epi(b + idx); }
  __device__ __forceinline__ void ld2(long long idx, double2 (&v)[2]) const { v[0] = ld_epi2(b + idx); }
  __device__ __forceinline__ double st(long long idx, double y, double, const double (&v)[2]) const {
    const double ei = v[0] - y;
    if (e) e[idx] = ei;
    return ei * ei;
  }
  __device__ __forceinline__ double st2(long long idx, double y0, double y1, double2,
                                        const double2 (&v)[2]) const {
    const double e0 = v[0].x - y0, e1 = v[0].y - y1;
    if (e) pcgx::st2(e + idx, e0, e1);
    return e0 * e0 + e1 * e1;
  }
};

// Chebyshev step 1 (polyprec.cpp:187-189), input vector = r:
//   x = (2 rho_1 / delta) * (2 r - (A r) / theta)
// x_old = r / theta is NOT stored: step 2 recomputes it from r (same bits).
// Contribution r_i x_i (used when m == 1, i.e. x is already z = P r).
struct EpiChebFirst {
  double* __restrict__ xout;
  double theta, c1;
  double inv;  // RN(1 / theta)
  __device__ __forceinline__ void pf(long long) const {}
  __device__ __forceinline__ void ld(long long, double (&)[2]) const {}
  __device__ __forceinline__ void ld2(long long, double2 (&)[2]) const {}
  __device__ __forceinline__ double f(double y, double xc) const {
    return c1 * ((2.0 * xc) - div_rn(y, theta, inv));
  }
  __device__ __forceinline__ double st(long long idx, double y, double xc, const double (&)[2]) const {
    const double xn = f(y, xc);
    xout[idx] = xn;
    return xc * xn;
  }
  __device__ __forceinline__ double st2(long long idx, double y0, double y1, double2 xc,
                                        const double2 (&)[2]) const {
    const double a = f(y0, xc.x), b = f(y1, xc.y);
    pcgx::st2(xout + idx, a, b);
    return xc.x * a + xc.y * b;
  }
};

// Chebyshev step k >= 2 (polyprec.cpp:190-195), input vector = x_{k-1}:
//   z = (2/delta) (r - A x) ; x_new = rho_k ((2 sigma) x - rho_{k-1} x_old + z)
// x_old is r/theta at k == 2 (xold_from_r), otherwise read from xold; x_new is
// written to out (== xold for the in-place middle steps: each point's x_old is
// read by its own thread before it is overwritten). Contribution r_i x_new_i.
struct EpiChebStep {
  const double* __restrict__ r;
  const double* xold;
  double* out;
  double rk, rk1, c2, c3, theta;
  int xold_from_r;
  double inv;  // RN(1 / theta)
  __device__ __forceinline__ void pf(long long idx) const {
    prefetch_l2(r + idx);
    if (!xold_from_r) prefetch_l2(xold + idx);
  }
  __device__ __forceinline__ void ld(long long idx, double (&v)[2]) const {
    v[0] = ld_epi(r + idx);
    v[1] = xold_from_r ? 0.0 : ld_epi_rw(xold + idx);
  }
  __device__ __forceinline__ void ld2(long long idx, double2 (&v)[2]) const {
    v[0] = ld_epi2(r + idx);
    v[1] = xold_from_r ? make_double2(0.0, 0.0) : ld_epi_rw2(xold + idx);
  }
  __device__ __forceinline__ double f(double y, double xc, double ri, double xo_in) const {
    const double xo = xold_from_r ? div_rn(ri, theta, inv) : xo_in;
    const double z = c2 * (ri - y);
    return rk * (((c3 * xc) - (rk1 * xo)) + z);
  }
  __device__ __forceinline__ double st(long long idx, double y, double xc, const double (&v)[2]) const {
    const double xn = f(y, xc, v[0], v[1]);
    out[idx] = xn;
    return v[0] * xn;
  }
  __device__ __forceinline__ double st2(long long idx, double y0, double y1, double2 xc,
                                        const double2 (&v)[2]) const {
    const double a = f(y0, xc.x, v[0].x, v[1].x), b = f(y1, xc.y, v[0].y, v[1].y);
    pcgx::st2(out + idx, a, b);
    return v[0].x * a + v[0].y * b;
  }
};

// Newton form (polyprec.cpp:135-160), one SpMV of the recursion fused with the
// element-wise steps that follow it in the reference's order:
//   nchain == 0 : out = zeta0 * (A x)                    (the next level-0 scale)
//   nchain >= 1 : t = zeta0 * (A x); t = zeta1 * ((2 x) - t)    [u = L0 = x]
//                 t = zeta2 * ((2 L1) - t); t = zeta3 * ((2 L2) - t)   (nchain 2, 3)
// u1, u2 = L1, L2 (per-point operands v[0], v[1]); with a reduction the
// operand slot after the chain's holds r and the contribution is r_i out_i.
struct EpiNewton {
  double* out;
  const double* u1;
  const double* u2;
  double z0, z1, z2, z3;
  int nchain;
  __device__ __forceinline__ void pf(long long idx) const {
    if (u1) prefetch_l2(u1 + idx);
    if (u2) prefetch_l2(u2 + idx);
  }
  __device__ __forceinline__ void ld(long long idx, double (&v)[2]) const {
    v[0] = u1 ? __ldg(u1 + idx) : 0.0;
    v[1] = u2 ? __ldg(u2 + idx) : 0.0;
  }
  __device__ __forceinline__ void ld2(long long idx, double2 (&v)[2]) const {
    v[0] = u1 ? ldg2(u1 + idx) : make_double2(0.0, 0.0);
    v[1] = u2 ? ldg2(u2 + idx) : make_double2(0.0, 0.0);
  }
  __device__ __forceinline__ double f(double y, double xc, double a, double b) const {
    double t = z0 * y;
    if (nchain >= 1) t = z1 * ((2.0 * xc) - t);
    if (nchain >= 2) t = z2 * ((2.0 * a) - t);
    if (nchain >= 3) t = z3 * ((2.0 * b) - t);
    return t;
  }
  // reduction operand: the slot after the chain's operands
  __device__ __forceinline__ double rr(double a, double b) const { return nchain >= 2 ? b : a; }
  __device__ __forceinline__ double st(long long idx, double y, double xc, const double (&v)[2]) const {
    const double t = f(y, xc, v[0], v[1]);
    out[idx] = t;
    return rr(v[0], v[1]) * t;
  }
  __device__ __forceinline__ double st2(long long idx, double y0, double y1, double2 xc,
                                        const double2 (&v)[2]) const {
    const double a = f(y0, xc.x, v[0].x, v[1].x), b = f(y1, xc.y, v[0].y, v[1].y);
    pcgx::st2(out + idx, a, b);
    return rr(v[0].x, v[1].x) * a + rr(v[0].y, v[1].y) * b;
  }
};

// The rest of a Newton chain that did not fit the SpMV epilogue, element-wise:
// out = zeta[j] * ((2 L[j-1]) - out) for j = j0 .. j1 (polyprec.cpp:145);
// optional contribution r_i out_i.
constexpr int kNewtonMaxLev = 24;
struct NewtonChain {
  int j0, j1;
  double zeta[kNewtonMaxLev + 1];
  const double* L[kNewtonMaxLev];
};

// ----------------------------------------------------------------- 7-point stencil

// ----------------------------------------------------------------- operator inputs
// The operator kernels read their input vector through an `In` policy:
//   InVec  : x itself;
//   InComb : the PCG direction update fused into the SpMV that consumes it,
//            p_new = z + beta p_old with beta = S[s_new] / S[s_old]
//            (pcg.cpp:107; `first`: p = z, pcg.cpp:63), evaluated per loaded
//            element with the reference's rounding (z + (beta * p)), so the
//            values are bitwise those of a separate update pass; the epilogue
//            writes p_new once at the centre point (EpiStoreP).
// Ghost planes (z-slab neighbours) hold the raw vectors; In combines them too.

struct InVec {
  const double* __restrict__ x;
  const double* glo;  // ghost plane below the slab (or nullptr: Dirichlet)
  const double* ghi;
  const double* gx;   // CSR block rows: values of the ghost columns (index - nloc)
  long long nloc;
  __device__ __forceinline__ void init() {}
  __device__ __forceinline__ double ld1(long long i) const { return __ldg(x + i); }
  __device__ __forceinline__ double ldc(long long c) const {
    return c < nloc ? __ldg(x + c) : __ldg(gx + (c - nloc));
  }
  __device__ __forceinline__ double2 ld2(long long i) const { return ldg2(x + i); }
  __device__ __forceinline__ void pf(long long i) const { prefetch_l2(x + i); }
  __device__ __forceinline__ double glo1(long long c) const { return glo ? __ldg(glo + c) : 0.0; }
  __device__ __forceinline__ double ghi1(long long c) const { return ghi ? __ldg(ghi + c) : 0.0; }
  __device__ __forceinline__ double2 glo2(long long c) const {
    return glo ? ldg2(glo + c) : make_double2(0.0, 0.0);
  }
  __device__ __forceinline__ double2 ghi2(long long c) const {
    return ghi ? ldg2(ghi + c) : make_double2(0.0, 0.0);
  }
};

struct InComb {
  const double* __restrict__ z;
  const double* __restrict__ p;
  const double* S;
  int s_new, s_old, first;
  const double *zlo, *zhi, *plo, *phi;  // ghost planes of z and p_old
  const double *gz, *gp;                // CSR block rows: ghost columns of z and p_old
  long long nloc;
  double beta;
  __device__ __forceinline__ void init() { beta = first ? 0.0 : S[s_new] / S[s_old]; }
  __device__ __forceinline__ double f(double zv, double pv) const {
    return first ? zv : zv + beta * pv;
  }
  __device__ __forceinline__ double ld1(long long i) const { return f(__ldg(z + i), first ? 0.0 : __ldg(p + i)); }
  __device__ __forceinline__ double ldc(long long c) const {
    if (c < nloc) return ld1(c);
    return f(__ldg(gz + (c - nloc)), first ? 0.0 : __ldg(gp + (c - nloc)));
  }
  __device__ __forceinline__ double2 ld2(long long i) const {
    const double2 a = ldg2(z + i);
    if (first) return a;
    const double2 b = ldg2(p + i);
    return make_double2(a.x + beta * b.x, a.y + beta * b.y);
  }
  __device__ __forceinline__ void pf(long long i) const {
    prefetch_l2(z + i);
    if (!first) prefetch_l2(p + i);
  }
  __device__ __forceinline__ double glo1(long long c) const {
    return zlo ? f(__ldg(zlo + c), first ? 0.0 : __ldg(plo + c)) : 0.0;
  }
  __device__ __forceinline__ double ghi1(long long c) const {
    return zhi ? f(__ldg(zhi + c), first ? 0.0 : __ldg(phi + c)) : 0.0;
  }
  __device__ __forceinline__ double2 glo2(long long c) const {
    return zlo ? make_double2(glo1(c), glo1(c + 1)) : make_double2(0.0, 0.0);
  }
  __device__ __forceinline__ double2 ghi2(long long c) const {
    return zhi ? make_double2(ghi1(c), ghi1(c + 1)) : make_double2(0.0, 0.0);
  }
};

// q = A p_new ; writes p_new (the input at the centre) ; contribution p_new_i q_i
struct EpiStoreP {
  double* q;
  double* pout;
  __device__ __forceinline__ void pf(long long) const {}
  __device__ __forceinline__ void ld(long long, double (&)[2]) const {}
  __device__ __forceinline__ void ld2(long long, double2 (&)[2]) const {}
  __device__ __forceinline__ double st(long long idx, double y, double xc, const double (&)[2]) const {
    q[idx] = y;
    pout[idx] = xc;
    return xc * y;
  }
  __device__ __forceinline__ double st2(long long idx, double y0, double y1, double2 xc,
                                        const double2 (&)[2]) const {
    pcgx::st2(q + idx, y0, y1);
    pcgx::st2(pout + idx, xc.x, xc.y);
    return xc.x * y0 + xc.y * y1;
  }
};

// Scaled 7-point row: terms in ascending column order k-1, j-1, i-1, centre,
// i+1, j+1, k+1 (linop.cpp:247-253), t = d*x per neighbour (linop.cpp:272),
// y = s*d (linop.cpp:274). A missing (Dirichlet) neighbour is passed as 0: its
// term -(d*0) = -0 leaves the running sum bit-identical to the skipped term.
__device__ __forceinline__ double stencil_point(double d, double xm, double xs, double xw,
                                                double xc, double xe, double xn, double xp) {
  double s = 0.0;
  s = s + (-(d * xm));
  s = s + (-(d * xs));
  s = s + (-(d * xw));
  s = s + (6.0 * (d * xc));
  s = s + (-(d * xe));
  s = s + (-(d * xn));
  s = s + (-(d * xp));
  return s * d;
}

// The same sum from pre-scaled neighbours t = d * x (each product formed once per
// point by the caller): the identical IEEE operations, hence bitwise equal.
__device__ __forceinline__ double stencil_point_t(double d, double tm, double ts, double tw,
                                                  double tc, double te, double tn, double tp) {
  double s = 0.0;
  s = s + (-tm);
  s = s + (-ts);
  s = s + (-tw);
  s = s + (6.0 * tc);
  s = s + (-te);
  s = s + (-tn);
  s = s + (-tp);
  return s * d;
}

// One thread per (i, j) column, marching planes [kb, ke) with the k-1, k, k+1
// values in registers and the k+2 plane prefetched one iteration ahead; the
// in-plane neighbours (i +- 1, j +- 1) come through L1 (the block's own plane
// tile). Missing (Dirichlet) neighbours are 0, whose term -(d*0) = -0 leaves the
// running sum bit-identical to the reference's skipped term.
template <class In, class Epi, bool kRed>
__global__ void __launch_bounds__(kStencilThreads)
stencil7_kernel(StencilGeom g, In in, Epi epi, int k_begin, int k_end, int kz, Reduce red) {
  in.init();
  const int i = blockIdx.x * kStencilBX + threadIdx.x;
  const int j = blockIdx.y * kStencilBY + threadIdx.y;
  const int kb = k_begin + blockIdx.z * kz;
  const int ke = min(kb + kz, k_end);
  double acc = 0.0;
  if (i < g.nx && j < g.ny && kb < ke) {
    const long long col = (long long)j * g.nx + i;
    const long long nxy = g.nxy;
    auto plane = [&](int k) -> double {
      if (k < 0) return in.glo1(col);
      if (k >= g.nzl) return in.ghi1(col);
      return in.ld1((long long)k * nxy + col);
    };
    const bool has_w = i > 0, has_e = i < g.nx - 1, has_s = j > 0, has_n = j < g.ny - 1;
    const double d = g.d;
    double xm = plane(kb - 1);
    double xc = plane(kb);
    double xp = plane(kb + 1);
    double ev[2] = {0.0, 0.0};
    epi.ld((long long)kb * nxy + col, ev);
    for (int k = kb; k < ke; ++k) {
      const long long idx = (long long)k * nxy + col;
      const bool more = k + 1 < ke;
      const double xpp = more ? plane(k + 2) : 0.0;
      double evn[2] = {0.0, 0.0};
      if (more) epi.ld(idx + nxy, evn);
      const double xw = has_w ? in.ld1(idx - 1) : 0.0;
      const double xe = has_e ? in.ld1(idx + 1) : 0.0;
      const double xs = has_s ? in.ld1(idx - g.nx) : 0.0;
      const double xn = has_n ? in.ld1(idx + g.nx) : 0.0;
      const double y = stencil_point(d, xm, xs, xw, xc, xe, xn, xp);
      const double c = epi.st(idx, y, xc, ev);
      if (kRed) acc = acc + c;
      xm = xc;
      xc = xp;
      xp = xpp;
      ev[0] = evn[0];
      ev[1] = evn[1];
    }
  }
  if (kRed) block_reduce_finish(acc, red);
}


// Vectorised variant for even nx (all BASELINE grids): each lane owns TWO
// consecutive i (one 16-byte load per vector per plane), a warp spans 64 i; the
// i-1 / i+1 neighbours come from the adjacent lanes by shuffle (lane 0 / 31
// load the one value outside the warp), j+-1 through L1. The next plane of x
// and of the epilogue operands is prefetched one iteration ahead, so each thread
// keeps 3-4 independent 16-byte HBM loads in flight across the dependent march.
template <class In, class Epi, bool kRed>
__global__ void __launch_bounds__(kStencilThreads, PCGX_V2_MINB)
stencil7v2_kernel(StencilGeom g, In in, Epi epi, int k_begin, int k_end, int kz, Reduce red,
                  int pfd) {
  in.init();
  const int lane = threadIdx.x;
  const int i0 = blockIdx.x * 64 + 2 * lane;
  const int j = blockIdx.y * kStencilBY + threadIdx.y;
  const int kb = k_begin + blockIdx.z * kz;
  const int ke = min(kb + kz, k_end);
  double acc = 0.0;
  if (j < g.ny && kb < ke) {  // warp-uniform: every lane of the warp runs the march
    const bool valid = i0 < g.nx;
    const long long col = (long long)j * g.nx + i0;
    const long long nxy = g.nxy;
    const double2 zero2 = make_double2(0.0, 0.0);
    auto plane = [&](int k) -> double2 {
      if (!valid) return zero2;
      if (k < 0) return in.glo2(col);
      if (k >= g.nzl) return in.ghi2(col);
      return in.ld2((long long)k * nxy + col);
    };
    const bool has_s = valid && j > 0, has_n = valid && j < g.ny - 1;
    const bool edge_w = lane == 0, edge_e = lane == 31;
    const bool has_w = valid && i0 > 0, has_e = valid && i0 + 2 < g.nx;
    const double d = g.d;
    double2 xm = plane(kb - 1);
    double2 xc = plane(kb);
    double2 xp = plane(kb + 1);
    double2 ev[2] = {zero2, zero2};
    if (valid) epi.ld2((long long)kb * nxy + col, ev);
    for (int k = kb; k < ke; ++k) {
      const long long idx = (long long)k * nxy + col;
      const bool more = k + 1 < ke;
      const double2 xpp = more ? plane(k + 2) : zero2;
      double2 evn[2] = {zero2, zero2};
      if (more && valid) epi.ld2(idx + nxy, evn);
      if (pfd > 0 && valid && k + pfd < ke) {  // L2 prefetch pfd planes ahead (no registers)
        const long long pidx = idx + (long long)pfd * nxy;
        if (k + pfd + 1 < g.nzl) in.pf(pidx + nxy);
        epi.pf(pidx);
      }
      const double2 xs = has_s ? in.ld2(idx - g.nx) : zero2;
      const double2 xn = has_n ? in.ld2(idx + g.nx) : zero2;
      double xw = __shfl_up_sync(0xffffffffu, xc.y, 1);
      double xe = __shfl_down_sync(0xffffffffu, xc.x, 1);
      if (edge_w) xw = has_w ? in.ld1(idx - 1) : 0.0;
      if (edge_e) xe = has_e ? in.ld1(idx + 2) : 0.0;
      const double y0 = stencil_point(d, xm.x, xs.x, xw, xc.x, xc.y, xn.x, xp.x);
      const double y1 = stencil_point(d, xm.y, xs.y, xc.x, xc.y, xe, xn.y, xp.y);
      if (valid) {
        const double c = epi.st2(idx, y0, y1, xc, ev);
        if (kRed) acc = acc + c;
      }
      xm = xc;
      xc = xp;
      xp = xpp;
      ev[0] = evn[0];
      ev[1] = evn[1];
    }
  }
  if (kRed) block_reduce_finish(acc, red);
}

// ----------------------------------------------------------------- CSR

// Persistent grid over blocks of kCsrRows consecutive rows. The block's nnz
// range is contiguous; it is walked in chunks: every thread forms products
// va[k] * (d[c] * x[c]) for a coalesced stride of k into shared memory, then
// each row-thread sums ITS row's products sequentially in column order, which
// is the reference's order (linop.cpp:183-185) -> bitwise-equal rows.
template <class Epi, bool kRed>
__global__ void __launch_bounds__(kCsrRows)
csr_kernel(CsrGeom g, const double* __restrict__ x, Epi epi, Reduce red) {
  __shared__ double prod[kCsrChunk];
  double acc = 0.0;
  const int nrb = (g.n + kCsrRows - 1) / kCsrRows;
  for (int rb = blockIdx.x; rb < nrb; rb += gridDim.x) {
    const int row0 = rb * kCsrRows;
    const int row = row0 + threadIdx.x;
    const int rend = min(row0 + kCsrRows, g.n);
    const int nz0 = __ldg(g.row_ptr + row0), nz1 = __ldg(g.row_ptr + rend);
    int mb = 0, me = 0;
    if (row < g.n) {
      mb = __ldg(g.row_ptr + row);
      me = __ldg(g.row_ptr + row + 1);
    }
    // the row's own epilogue operands are independent of the chunk loop: issue them first
    double ev[2] = {0.0, 0.0};
    double xr = 0.0, dr = 0.0;
    if (row < g.n) {
      epi.ld(row, ev);
      xr = __ldg(x + row);
      dr = __ldg(g.dvec + row);
    }
    double sum = 0.0;
    constexpr int kPer = kCsrChunk / kCsrRows;  // products per thread per chunk
    for (int c0 = nz0; c0 < nz1; c0 += kCsrChunk) {
      const int c1 = min(c0 + kCsrChunk, nz1);
      // all index/value loads of the chunk first, then all gathers, then the
      // products: two dependent memory round trips per chunk, kPer-way MLP each
      int cidx[kPer];
      double val[kPer];
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int k = c0 + threadIdx.x + q * kCsrRows;
        cidx[q] = k < c1 ? __ldg(g.col_idx + k) : 0;
        val[q] = k < c1 ? __ldg(g.values + k) : 0.0;
      }
      double dx[kPer], xx[kPer];
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        dx[q] = __ldg(g.dvec + cidx[q]);
        xx[q] = __ldg(x + cidx[q]);
      }
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int k = c0 + threadIdx.x + q * kCsrRows;
        if (k < c1) prod[k - c0] = val[q] * (dx[q] * xx[q]);
      }
      __syncthreads();
      const int lo = max(mb, c0), hi = min(me, c1);
      for (int k = lo; k < hi; ++k) sum = sum + prod[k - c0];
      __syncthreads();
    }
    if (row < g.n) {
      const double y = sum * dr;
      const double c = epi.st(row, y, xr, ev);
      if (kRed) acc = acc + c;
    }
  }
  if (kRed) block_reduce_finish(acc, red);
}


// ----------------------------------------------------------------- CSR, TMA-pipelined


// ----------------------------------------------------------------- SELL-32 (sliced ELLPACK)

// The CSR matrix re-laid out at upload as slices of 32 rows (one warp): within
// slice s, entry k of lane (= row) l lives at slice_ptr[s] + 32 k + l, rows
// shorter than the slice's longest are padded. A thread owns one row and walks
// it in column order (k ascending = the reference's CSR order, linop.cpp:183-185),
// so each row's sum is bitwise the reference's; every value / index load is a
// coalesced 256 B / 128 B warp access, the x and d gathers are coalesced for
// stencil-structured rows, and padded slots are skipped by predicate (never
// added: a +0 product could flip a -0 sum).
struct SellGeom {
  int n;
  int nslices;
  int s_begin, s_end;          // slices of this launch
  const long long* slice_ptr;  // nslices + 1 (entries)
  const int* rowlen;           // n
  const int* col;              // padded
  const double* val;           // padded
  const double* dvec;
};

#ifndef PCGX_SELL_BATCH
#define PCGX_SELL_BATCH 8
#endif
#ifndef PCGX_SELL_MINB
#define PCGX_SELL_MINB 4
#endif
constexpr int kSellBatch = PCGX_SELL_BATCH;

template <class In, class Epi, bool kRed>
__global__ void __launch_bounds__(256, PCGX_SELL_MINB)
sell_kernel(SellGeom g, In in, Epi epi, Reduce red) {
  in.init();
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  double acc = 0.0;
  for (int s = g.s_begin + blockIdx.x * wpb + (threadIdx.x >> 5); s < g.s_end; s += gridDim.x * wpb) {
    const int row = s * 32 + lane;
    const long long base = __ldg(g.slice_ptr + s) + lane;
    const int L = (int)((__ldg(g.slice_ptr + s + 1) - __ldg(g.slice_ptr + s)) >> 5);
    const bool live = row < g.n;
    const int len = live ? __ldg(g.rowlen + row) : 0;
    double ev[2] = {0.0, 0.0};
    double xr = 0.0, dr = 0.0;
    if (live) {
      epi.ld(row, ev);
      xr = in.ld1(row);
      dr = __ldg(g.dvec + row);
    }
    double sum = 0.0;
    for (int k = 0; k < L; k += kSellBatch) {
      double vv[kSellBatch], dv[kSellBatch], xv[kSellBatch];
#pragma unroll
      for (int q = 0; q < kSellBatch; ++q) {
        const bool on = (k + q) < len;
        const long long e = base + (long long)(k + q) * 32;
        const int c = on ? __ldg(g.col + e) : 0;
        vv[q] = on ? ld_mat(g.val + e) : 0.0;
        dv[q] = on ? __ldg(g.dvec + c) : 0.0;  // dvec spans the ghost columns too
        xv[q] = on ? in.ldc(c) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < kSellBatch; ++q)
        if (k + q < len) sum = sum + vv[q] * (dv[q] * xv[q]);
    }
    if (live) {
      const double y = sum * dr;
      const double c = epi.st(row, y, xr, ev);
      if (kRed) acc = acc + c;
    }
  }
  if (kRed) block_reduce_finish(acc, red);
}

// ----------------------------------------------------------------- 3x3 block CSR
// A CSR matrix whose rows come in aligned triples with a shared pattern of full
// 3x3 blocks (3 dof per node: the elasticity family, cfg4) is stored as BSR-3 in
// the SELL-32 arrangement over BLOCK rows: per slice of 32 block rows, step k
// holds one block column index per lane (128 B) and the 9 block values as nine
// coalesced 256-byte rows (q = 3c + d, val[(slot0 + 32k) * 9 + 32 q + lane]).
// Matrix bytes per nnz: 8 + 4/9 (vs 12 for the int32 CSR). One thread owns a
// block row = three CSR rows with three sums; each sum takes its terms in the
// CSR row's column order (blocks ascending, d = 0..2), v * (d_c * x_c), so every
// row is bitwise the scalar CSR kernel's (linop.cpp:171-187, 271-275).
struct Bsr3Geom {
  int nb;                      // block rows (n / 3)
  int s_begin, s_end;          // slices of this launch
  const long long* slice_ptr;  // nslices + 1 (blocks; multiples of 32)
  const int* blen;             // nb: blocks per block row
  const int* bcol;             // padded: block column J (column 3J .. 3J+2)
  const double* val;           // padded: 9 per block (see above)
  const double* dvec;
};

#ifndef PCGX_BSR_BATCH
#define PCGX_BSR_BATCH 1
#endif
constexpr int kBsrBatch = PCGX_BSR_BATCH;

#ifndef PCGX_BSR_MINB
#define PCGX_BSR_MINB 4
#endif
template <class In, class Epi, bool kRed>
__global__ void __launch_bounds__(256, PCGX_BSR_MINB)
bsr3_kernel(Bsr3Geom g, In in, Epi epi, Reduce red) {
  in.init();
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  double acc = 0.0;
  for (int s = g.s_begin + blockIdx.x * wpb + (threadIdx.x >> 5); s < g.s_end; s += gridDim.x * wpb) {
    const int br = s * 32 + lane;
    const long long base = __ldg(g.slice_ptr + s);
    const int L = (int)((__ldg(g.slice_ptr + s + 1) - base) >> 5);
    const bool live = br < g.nb;
    const int len = live ? __ldg(g.blen + br) : 0;
    const long long r0 = 3LL * br;
    double ev[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    double xr[3] = {0.0, 0.0, 0.0}, dr[3] = {0.0, 0.0, 0.0};
    if (live) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        epi.ld(r0 + c, ev[c]);
        xr[c] = in.ld1(r0 + c);
        dr[c] = __ldg(g.dvec + r0 + c);
      }
    }
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int k = 0; k < L; k += kBsrBatch) {
      double v[kBsrBatch][9], t[kBsrBatch][3];
#pragma unroll
      for (int q = 0; q < kBsrBatch; ++q) {
        const bool on = (k + q) < len;
        const long long slot = base + 32LL * (k + q);
        const int J = on ? __ldg(g.bcol + slot + lane) : 0;
        const double* vp = g.val + slot * 9 + lane;
#pragma unroll
        for (int e = 0; e < 9; ++e) v[q][e] = on ? ld_mat(vp + 32 * e) : 0.0;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const long long cidx = 3LL * J + d;
          t[q][d] = on ? __ldg(g.dvec + cidx) * in.ldc(cidx) : 0.0;
        }
      }
#pragma unroll
      for (int q = 0; q < kBsrBatch; ++q)
        if (k + q < len) {
          s0 = s0 + v[q][0] * t[q][0];
          s0 = s0 + v[q][1] * t[q][1];
          s0 = s0 + v[q][2] * t[q][2];
          s1 = s1 + v[q][3] * t[q][0];
          s1 = s1 + v[q][4] * t[q][1];
          s1 = s1 + v[q][5] * t[q][2];
          s2 = s2 + v[q][6] * t[q][0];
          s2 = s2 + v[q][7] * t[q][1];
          s2 = s2 + v[q][8] * t[q][2];
        }
    }
    if (live) {
      const double c0 = epi.st(r0, s0 * dr[0], xr[0], ev[0]);
      const double c1 = epi.st(r0 + 1, s1 * dr[1], xr[1], ev[1]);
      const double c2 = epi.st(r0 + 2, s2 * dr[2], xr[2], ev[2]);
      if (kRed) acc = acc + ((c0 + c1) + c2);
    }
  }
  if (kRed) block_reduce_finish(acc, red);
}

// ----------------------------------------------------------------- diagonal (offset) storage
// A CSR matrix whose column offsets (col - row) come from a small fixed set (K <= 32:
// the 27-point FE stencils of cfg3, the assembled 7-point Laplacian) is stored by
// offset: val[k * ld + i] = a(i, i + off[k]) (coalesced across rows) plus one
// presence mask per row. No column indices: 8 B per stored entry + 4 B per row
// (vs 12 B per nnz). Terms are taken in ascending offset = ascending column order,
// only where the mask bit is set, v * (d_c * x_c): bitwise the CSR row sum.
constexpr int kDiaMax = 32;

struct DiaGeom {
  int n, K;
  long long ld;
  int off[kDiaMax];
  const double* val;
  const unsigned* mask;
  const double* dvec;
};

#ifndef PCGX_DIA_MINB
#define PCGX_DIA_MINB 8
#endif
template <class In, class Epi, bool kRed, bool kStream>
__global__ void __launch_bounds__(256, PCGX_DIA_MINB)
dia_kernel(DiaGeom g, In in, Epi epi, Reduce red) {
  in.init();
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < g.n;
       i += (long long)gridDim.x * blockDim.x) {
    double ev[2];
    epi.ld(i, ev);
    const double xr = in.ld1(i);
    const double dr = __ldg(g.dvec + i);
    const unsigned msk = __ldg(g.mask + i);
    double sum = 0.0;
#pragma unroll 9
    for (int k = 0; k < g.K; ++k) {
      if (msk & (1u << k)) {
        const long long c = i + g.off[k];
        sum = sum + ld_stream<kStream>(g.val + k * g.ld + i) * (__ldg(g.dvec + c) * in.ldc(c));
      }
    }
    const double y = sum * dr;
    const double cc = epi.st(i, y, xr, ev);
    if (kRed) acc = acc + cc;
  }
  if (kRed) block_reduce_finish(acc, red);
}

// ----------------------------------------------------------------- offset storage on a grid
// The offset storage of a matrix on a cubic nx^3 grid whose column offsets are
// exactly a structured pattern (the 27-point box, cfg3; the 7-point star, cfg1)
// and whose couplings never wrap across a grid face (checked at upload). Slot s
// of the storage is then the grid neighbour (dz, dy, dx) of DiaPat<P>, in the
// same ascending-offset order. Instead of gathering d_c and x_c per slot through
// L1 (dia_kernel: 54 dependent gathers per row, latency-bound), a CTA owns a
// 32 x 8 column tile, marches its z-chunk and stages t = d * x of a 34 x 10 patch
// per plane in a 4-plane shared ring (the product ScaledOperator forms,
// linop.cpp:272); a row's terms are its value stream times ring reads, added in
// slot order, absent slots skipped — the row sums are bitwise dia_kernel's.
template <int P>
struct DiaPat;
template <>
struct DiaPat<27> {
  static constexpr int K = 27;
  __host__ __device__ static constexpr int dz(int s) { return s / 9 - 1; }
  __host__ __device__ static constexpr int dy(int s) { return (s / 3) % 3 - 1; }
  __host__ __device__ static constexpr int dx(int s) { return s % 3 - 1; }
};
template <>
struct DiaPat<7> {  // k-1, j-1, i-1, centre, i+1, j+1, k+1
  static constexpr int K = 7;
  __host__ __device__ static constexpr int dz(int s) { return s == 0 ? -1 : (s == 6 ? 1 : 0); }
  __host__ __device__ static constexpr int dy(int s) { return s == 1 ? -1 : (s == 5 ? 1 : 0); }
  __host__ __device__ static constexpr int dx(int s) { return s == 2 ? -1 : (s == 4 ? 1 : 0); }
};

#ifndef PCGX_D3X
#define PCGX_D3X 32
#endif
#ifndef PCGX_D3Y
#define PCGX_D3Y 8
#endif
constexpr int kD3X = PCGX_D3X, kD3Y = PCGX_D3Y, kD3PX = kD3X + 2, kD3PY = kD3Y + 2;
constexpr int kD3Plane = kD3PX * kD3PY, kD3Threads = kD3X * kD3Y;
static_assert(kD3Plane <= 2 * kD3Threads, "two staged patch elements per thread");

struct Dia3Geom {
  int nx, kz;  // grid edge (i, j), planes per z-chunk
  long long ld;
  const double* val;
  const unsigned* mask;
  const double* dvec;
  // z-slab of a multi-rank operator: nzl local planes, this launch covers planes
  // [kb0, ke0); dlo / dhi = the Jacobi values of the neighbours' boundary planes
  // (nullptr: Dirichlet side), their x planes come through In's glo / ghi
  int nzl = 0, kb0 = 0, ke0 = 0;
  const double* dlo = nullptr;
  const double* dhi = nullptr;
};

#ifndef PCGX_DIA3_MINB
#define PCGX_DIA3_MINB 3
#endif
template <int P, class In, class Epi, bool kRed, bool kStream>
__global__ void __launch_bounds__(kD3Threads, PCGX_DIA3_MINB)
dia3_kernel(Dia3Geom g, In in, Epi epi, Reduce red) {
  __shared__ double sT[4][kD3Plane];
  using Pat = DiaPat<P>;
  in.init();
  const int nx = g.nx;
  const long long nxy = (long long)nx * nx;
  const int tiles_x = (nx + kD3X - 1) / kD3X;
  const int i0 = (int)(blockIdx.x % tiles_x) * kD3X, j0 = (int)(blockIdx.x / tiles_x) * kD3Y;
  const int kb = g.kb0 + blockIdx.y * g.kz, ke = min(kb + g.kz, g.ke0);
  const int nzl = g.nzl;
  const int tid = threadIdx.x, tx = tid % kD3X, ty = tid / kD3X;
  const int i = i0 + tx, j = j0 + ty;
  const bool own = i < nx && j < nx;
  // the two patch elements this thread stages
  const int e1 = tid + kD3Threads;
  const int pi0 = i0 - 1 + tid % kD3PX, pj0 = j0 - 1 + tid / kD3PX;
  const int pi1 = i0 - 1 + e1 % kD3PX, pj1 = j0 - 1 + e1 / kD3PX;
  const bool in0 = pi0 >= 0 && pi0 < nx && pj0 >= 0 && pj0 < nx;
  const bool in1 = e1 < kD3Plane && pi1 >= 0 && pi1 < nx && pj1 >= 0 && pj1 < nx;
  const long long c0 = (long long)pj0 * nx + pi0, c1 = (long long)pj1 * nx + pi1;
  auto stage = [&](int k, double& t0, double& t1) {
    const bool kin = k >= 0 && k < nzl;
    const long long kb0 = (long long)k * nxy;
    if (kin) {
      t0 = in0 ? __ldg(g.dvec + kb0 + c0) * in.ldc(kb0 + c0) : 0.0;
      t1 = in1 ? __ldg(g.dvec + kb0 + c1) * in.ldc(kb0 + c1) : 0.0;
    } else if (k == -1 && g.dlo) {  // the lower neighbour's last plane
      t0 = in0 ? __ldg(g.dlo + c0) * in.glo1(c0) : 0.0;
      t1 = in1 ? __ldg(g.dlo + c1) * in.glo1(c1) : 0.0;
    } else if (k == nzl && g.dhi) {  // the upper neighbour's first plane
      t0 = in0 ? __ldg(g.dhi + c0) * in.ghi1(c0) : 0.0;
      t1 = in1 ? __ldg(g.dhi + c1) * in.ghi1(c1) : 0.0;
    } else {
      t0 = t1 = 0.0;
    }
  };
  auto put = [&](int k, double t0, double t1) {
    double* s = sT[(k + 4) & 3];
    s[tid] = t0;
    if (e1 < kD3Plane) s[e1] = t1;
  };
  {
    double a0, a1, b0, b1, c0v, c1v;
    stage(kb - 1, a0, a1);
    stage(kb, b0, b1);
    stage(kb + 1, c0v, c1v);
    put(kb - 1, a0, a1);
    put(kb, b0, b1);
    put(kb + 1, c0v, c1v);
  }
  __syncthreads();
  const int own_off = (ty + 1) * kD3PX + tx + 1;
  double acc = 0.0;
  for (int k = kb; k < ke; ++k) {
    double n0, n1;
    stage(k + 2, n0, n1);  // plane k+2, stored after this plane's rows
    if (own) {
      const long long row = (long long)k * nxy + (long long)j * nx + i;
      double ev[2];
      epi.ld(row, ev);
      const double xr = in.ld1(row);
      const double dr = __ldg(g.dvec + row);
      const unsigned msk = __ldg(g.mask + row);
      double v[Pat::K];
#pragma unroll
      for (int s = 0; s < Pat::K; ++s)
        v[s] = ((msk >> s) & 1u) ? ld_stream<kStream>(g.val + s * g.ld + row) : 0.0;
      const double* pm = sT[(k + 3) & 3] + own_off;
      const double* p0 = sT[k & 3] + own_off;
      const double* pp = sT[(k + 1) & 3] + own_off;
      double sum = 0.0;
#pragma unroll
      for (int s = 0; s < Pat::K; ++s) {
        const double* pl = Pat::dz(s) < 0 ? pm : (Pat::dz(s) == 0 ? p0 : pp);
        if ((msk >> s) & 1u) sum = sum + v[s] * pl[Pat::dy(s) * kD3PX + Pat::dx(s)];
      }
      const double y = sum * dr;
      const double cc = epi.st(row, y, xr, ev);
      if (kRed) acc = acc + cc;
    }
    put(k + 2, n0, n1);
    __syncthreads();
  }
  if (kRed) block_reduce_finish(acc, red);
}

// ----------------------------------------------------------------- vector kernels
// Grid-stride over a fixed grid (deterministic element -> thread map).

// x += alpha p ; r -= alpha q ; contribution r_i^2, alpha = rz[prev] / pq[cur]
// (pcg.cpp:80-83). zmode 1 (m = 0, polyprec.cpp:179-181): also z = r / theta
// and r'z (pcg.cpp:101) in the same pass; zmode 2 (no preconditioner, z = r):
// r'z = r'r. zmode > 0 reduces the adjacent pair [r'r, r'z] (red.result[0..1]).
__global__ void __launch_bounds__(kVecThreads)
update_kernel(long long n, double* __restrict__ x, double* __restrict__ r,
              const double* __restrict__ p, const double* __restrict__ q, const double* S,
              int s_rho, int s_pq, Reduce red, int zmode, double theta, double* __restrict__ z) {
  const double alpha = S[s_rho] / S[s_pq];
  const double inv = 1.0 / theta;  // RN(1/theta), as on the host
  double acc = 0.0, acc2 = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    if (x) x[i] = x[i] + alpha * p[i];  // x == nullptr: deferred to the next direction step
    const double ri = r[i] - alpha * q[i];
    r[i] = ri;
    acc = acc + ri * ri;
    if (zmode == 1) {
      const double zi = div_rn(ri, theta, inv);
      if (z) z[i] = zi;
      acc2 = acc2 + ri * zi;
    } else if (zmode == 2) {
      acc2 = acc2 + ri * ri;
    }
  }
  if (zmode) block_reduce_finish2(acc, acc2, red);
  else block_reduce_finish(acc, red);
}

// update_kernel on 16-byte pairs (n even, 16-byte aligned vectors): the same
// per-element operations, four 16-byte loads in flight per thread per step.
#ifndef PCGX_UPD_U2
#define PCGX_UPD_U2 1  // k = 0 solve -3% at 320^3
#endif
template <int kZ, bool kX>
__global__ void __launch_bounds__(kVecThreads)
update2_kernel(long long n2, double2* __restrict__ x, double2* __restrict__ r,
               const double2* __restrict__ p, const double2* __restrict__ q, const double* S,
               int s_rho, int s_pq, Reduce red, double theta, double2* __restrict__ z) {
  const double alpha = S[s_rho] / S[s_pq];
  const double inv = 1.0 / theta;  // RN(1/theta), as on the host
  double acc = 0.0, acc2 = 0.0;
#if PCGX_UPD_U2
  // two elements per thread and step, both pairs' loads issued before either store
  const long long G = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += 2 * G) {
    const long long j = i + G;
    const bool hj = j < n2;
    double2 ri = r[i], rj = make_double2(0.0, 0.0);
    const double2 qi = __ldg(q + i);
    double2 qj = make_double2(0.0, 0.0);
    if (hj) {
      rj = r[j];
      qj = __ldg(q + j);
    }
    auto one = [&](long long k, double2 rv, const double2 qv) {
      if (kX) {
        double2 xi = x[k];
        const double2 pi = __ldg(p + k);
        xi.x = xi.x + alpha * pi.x;
        xi.y = xi.y + alpha * pi.y;
        x[k] = xi;
      }
      rv.x = rv.x - alpha * qv.x;
      rv.y = rv.y - alpha * qv.y;
      r[k] = rv;
      acc = acc + rv.x * rv.x;
      acc = acc + rv.y * rv.y;
      if (kZ == 1) {
        const double2 zi = make_double2(div_rn(rv.x, theta, inv), div_rn(rv.y, theta, inv));
        if (z) z[k] = zi;
        acc2 = acc2 + rv.x * zi.x;
        acc2 = acc2 + rv.y * zi.y;
      } else if (kZ == 2) {
        acc2 = acc2 + rv.x * rv.x;
        acc2 = acc2 + rv.y * rv.y;
      }
    };
    one(i, ri, qi);
    if (hj) one(j, rj, qj);
  }
#else
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2;
       i += (long long)gridDim.x * blockDim.x) {
    double2 ri = r[i];
    const double2 qi = __ldg(q + i);
    if (kX) {  // !kX: x += alpha p is deferred to the next direction step
      double2 xi = x[i];
      const double2 pi = __ldg(p + i);
      xi.x = xi.x + alpha * pi.x;
      xi.y = xi.y + alpha * pi.y;
      x[i] = xi;
    }
    ri.x = ri.x - alpha * qi.x;
    ri.y = ri.y - alpha * qi.y;
    r[i] = ri;
    acc = acc + ri.x * ri.x;
    acc = acc + ri.y * ri.y;
    if (kZ == 1) {
      const double2 zi = make_double2(div_rn(ri.x, theta, inv), div_rn(ri.y, theta, inv));
      if (z) z[i] = zi;  // z == nullptr: the direction step forms r / theta itself
      acc2 = acc2 + ri.x * zi.x;
      acc2 = acc2 + ri.y * zi.y;
    } else if (kZ == 2) {
      acc2 = acc2 + ri.x * ri.x;
      acc2 = acc2 + ri.y * ri.y;
    }
  }
#endif
  if (kZ) block_reduce_finish2(acc, acc2, red);
  else block_reduce_finish(acc, red);
}

// x += alpha p, alpha = S[s_rho] / S[s_pq] (pcg.cpp:82): a deferred x update that
// no later direction step will apply (the iteration limit was reached)
__global__ void __launch_bounds__(kVecThreads)
xupd_kernel(long long n, double* __restrict__ x, const double* __restrict__ p, const double* S,
            int s_rho, int s_pq) {
  const double alpha = S[s_rho] / S[s_pq];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    x[i] = x[i] + alpha * p[i];
}

// p_new = z + beta p_old, beta = rz[cur] / rz[prev] (pcg.cpp:107); first: p = z
// (pcg.cpp:63). Out of place (the direction buffers ping-pong per iteration).
__global__ void __launch_bounds__(kVecThreads)
pupdate_kernel(long long n, double* __restrict__ pnew, const double* __restrict__ pold,
               const double* __restrict__ z, const double* S, int s_new, int s_old, int first) {
  const double beta = first ? 0.0 : S[s_new] / S[s_old];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    pnew[i] = first ? z[i] : z[i] + beta * pold[i];
}

// z = r / theta (m == 0, polyprec.cpp:179-181) or z = r (no preconditioner,
// pcg.cpp:61,99) ; contribution r_i z_i  (pcg.cpp:64,101)
__global__ void __launch_bounds__(kVecThreads)
zr_kernel(long long n, double* __restrict__ z, const double* __restrict__ r, double theta,
          int divide, Reduce red) {
  const double inv = 1.0 / theta;
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double ri = r[i];
    const double zi = divide ? div_rn(ri, theta, inv) : ri;
    z[i] = zi;
    acc = acc + ri * zi;
  }
  block_reduce_finish(acc, red);
}

// Newton level 0 (polyprec.cpp:139-141): out = zeta0 * in; contribution in_i out_i.
template <bool kRed>
__global__ void __launch_bounds__(kVecThreads)
nscale_kernel(long long n, double* __restrict__ out, const double* __restrict__ in, double z0,
              Reduce red) {
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double v = in[i];
    const double o = z0 * v;
    out[i] = o;
    if (kRed) acc = acc + v * o;
  }
  if (kRed) block_reduce_finish(acc, red);
}

template <bool kRed>
__global__ void __launch_bounds__(kVecThreads)
nchain_kernel(long long n, double* __restrict__ out, const NewtonChain ch,
              const double* __restrict__ r, Reduce red) {
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double t = out[i];
    for (int j = ch.j0; j <= ch.j1; ++j) t = ch.zeta[j] * ((2.0 * __ldg(ch.L[j - 1] + i)) - t);
    out[i] = t;
    if (kRed) acc = acc + __ldg(r + i) * t;
  }
  if (kRed) block_reduce_finish(acc, red);
}

// result = a . b
__global__ void __launch_bounds__(kVecThreads)
dot_kernel(long long n, const double* __restrict__ a, const double* __restrict__ b, Reduce red) {
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    acc = acc + a[i] * b[i];
  block_reduce_finish(acc, red);
}

// Lanczos three-term update: w = (w - a v) - b v_prev, contribution w_i^2;
// a = S[s_a] (the all-reduced v'Av), b = beta of the previous step (host value).
__global__ void __launch_bounds__(kVecThreads)
lanczos_w_kernel(long long n, double* __restrict__ w, const double* __restrict__ v,
                 const double* __restrict__ vprev, const double* S, int s_a, double b,
                 Reduce red) {
  const double a = S[s_a];
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double wi = (w[i] - a * v[i]) - b * vprev[i];
    w[i] = wi;
    acc = acc + wi * wi;
  }
  block_reduce_finish(acc, red);
}

// vprev = v ; v = w / s
__global__ void __launch_bounds__(kVecThreads)
lanczos_shift_kernel(long long n, double* __restrict__ v, double* __restrict__ vprev,
                     const double* __restrict__ w, double s) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    vprev[i] = v[i];
    v[i] = w[i] / s;
  }
}

// v = v / s
__global__ void __launch_bounds__(kVecThreads)
scale_div_kernel(long long n, double* __restrict__ v, double s) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    v[i] = v[i] / s;
}

__global__ void __launch_bounds__(kVecThreads)
fill_kernel(long long n, double* __restrict__ v, double val) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    v[i] = val;
}

// random_uniform_vector elements [offset, offset+n): the i-th draw of splitmix64
// seeded with `seed` uses state seed + (i+1) * golden-gamma (eigenest.cpp:13-30).
__global__ void __launch_bounds__(kVecThreads)
splitmix_kernel(long long n, unsigned long long seed, unsigned long long offset,
                double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    unsigned long long z = seed + (offset + (unsigned long long)i + 1ull) * 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z = z ^ (z >> 31);
    const double u = (double)(z >> 11) * 0x1.0p-53;
    out[i] = 2.0 * u - 1.0;
  }
}

// out[k] = x[idx[k]] (send buffers of the CSR block-row halo)
__global__ void __launch_bounds__(kVecThreads)
pack_kernel(long long n, const int* __restrict__ idx, const double* __restrict__ x,
            double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = x[idx[i]];
}

// ---- power method / DACG (eigenest.cpp:48-167), elementwise in the reference's order

// v = w / s  (power_method: v = w / w.norm())
__global__ void __launch_bounds__(kVecThreads)
div_copy_kernel(long long n, double* __restrict__ v, const double* __restrict__ w, double s) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    v[i] = w[i] / s;
}

// e = ax - q x, g = 2 e: reduces [e'e, g'g]
__global__ void __launch_bounds__(kVecThreads)
dacg_g_kernel(long long n, const double* __restrict__ x, const double* __restrict__ ax, double q,
              Reduce red) {
  double v[2] = {0.0, 0.0};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double e = ax[i] - q * x[i];
    const double g = 2.0 * e;
    v[0] = v[0] + e * e;
    v[1] = v[1] + g * g;
  }
  block_reduce_finishN<2>(v, red);
}

// p = -g (restart) or p = -g + c p, g = 2 (ax - q x) recomputed
__global__ void __launch_bounds__(kVecThreads)
dacg_p_kernel(long long n, const double* __restrict__ x, const double* __restrict__ ax, double q,
              double* __restrict__ p, double c, int restart) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double g = 2.0 * (ax[i] - q * x[i]);
    p[i] = restart ? -g : -g + c * p[i];
  }
}

// [x'ap, x'p, p'p]
__global__ void __launch_bounds__(kVecThreads)
dot3_kernel(long long n, const double* __restrict__ x, const double* __restrict__ p,
            const double* __restrict__ ap, Reduce red) {
  double v[3] = {0.0, 0.0, 0.0};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double xi = x[i], pi = p[i];
    v[0] = v[0] + xi * ap[i];
    v[1] = v[1] + xi * pi;
    v[2] = v[2] + pi * pi;
  }
  block_reduce_finishN<3>(v, red);
}

// x = cx x + cp p ; ax = cx ax + cp ap ; reduces x'x
__global__ void __launch_bounds__(kVecThreads)
dacg_x_kernel(long long n, double* __restrict__ x, double* __restrict__ ax,
              const double* __restrict__ p, const double* __restrict__ ap, double cx, double cp,
              Reduce red) {
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double xi = cx * x[i] + cp * p[i];
    x[i] = xi;
    ax[i] = cx * ax[i] + cp * ap[i];
    acc = acc + xi * xi;
  }
  block_reduce_finish(acc, red);
}

// x /= s ; ax /= s ; reduces x'ax
__global__ void __launch_bounds__(kVecThreads)
dacg_norm_kernel(long long n, double* __restrict__ x, double* __restrict__ ax, double s,
                 Reduce red) {
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double xi = x[i] / s;
    const double ai = ax[i] / s;
    x[i] = xi;
    ax[i] = ai;
    acc = acc + xi * ai;
  }
  block_reduce_finish(acc, red);
}

// Writes a large scratch buffer (flushes L2 between timed iterations).
__global__ void flush_kernel(long long n, double* __restrict__ buf) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    buf[i] = (double)i;
}

}  // namespace pcgx
