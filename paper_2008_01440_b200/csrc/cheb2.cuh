// SPDX-License-Identifier: Apache-2.0
//
// Shared definitions of the temporally blocked Chebyshev passes:
// the pass parameters and the mbarrier / TMA primitives the two-step
// (cheb2f.cuh), three-step (cheb3.cuh) and direction-step (dir_tma.cuh) kernels
// use. Two steps per pass:
//
//   stage 1: C = x_k     = rho_k     ((2s) A - rho_{k-1} B + (2/d)(R - S A))
//   stage 2: E = x_{k+1} = rho_{k+1} ((2s) C - rho_k     A + (2/d)(R - S C))
// with A = x_{k-1}, B = x_{k-2}, R = r, S the scaled 7-point operator
// (polyprec.cpp:190-195). kFirst: the pass is steps (1, 2): stage 1 is
// x_1 = c1 (2 r - (S r)/theta) with A = R = r (polyprec.cpp:187-189) and stage 2
// uses x_old = x_0 = r/theta. HBM traffic per point per TWO steps: read A, B, R +
// write C, E = 40 B (vs 64 B for two single-step passes).
#pragma once

#include <cuda.h>

#include "kernels.cuh"

namespace pcgx {

constexpr int kC2TX = 64;          // output tile width (i); one warp = 32 lanes x 2 points
constexpr int kC2W = kC2TX + 4;    // row width of the 1-halo planes: tile-i t <-> column t+2
#ifndef PCGX_C2UNROLL
#define PCGX_C2UNROLL 4
#endif
constexpr int kC2Unroll = PCGX_C2UNROLL;  // plane-loop unroll

struct Cheb2Params {
  int nx, ny, nzl;          // local grid
  // z-slabs: loaded planes must lie in [a_lo, a_hi) (A, B, R; the slab plus the
  // neighbours' planes exchanged into the vectors' padding), C is computed on
  // [c_lo, c_hi) and is 0 (Dirichlet) elsewhere; tensor z = plane + zoff.
  int a_lo, a_hi, c_lo, c_hi, zoff;
  long long nxy;
  double d;                 // inv sqrt diag
  double theta;
  // stage 1 (step k) and stage 2 (step k+1) coefficients
  double rk1, rk1m1;        // rho_k, rho_{k-1}      (stage 1, STEP)
  double c1;                // 2 rho_1 / delta       (stage 1, FIRST)
  double rk2, rk2m1;        // rho_{k+1}, rho_k      (stage 2)
  double c2, c3;            // 2/delta, 2 sigma
  double* outC;             // x_k   (interior tile points)
  double* outE;             // x_{k+1}
  // fused PCG update (pipelined kernel, kFirst): A = r_old and the Q map hold
  // r(it-1) and q(it); r = r_old - alpha q (pcg.cpp:83), alpha = S[s_rho] / S[s_pq],
  // is formed in shared memory, written to rout and reduced as r'r
  const double* S;
  int s_rho, s_pq;
  double* rout;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

}  // namespace pcgx
