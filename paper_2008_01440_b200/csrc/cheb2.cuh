// SPDX-License-Identifier: Apache-2.0
//
// Temporal blocking of the Chebyshev recurrence: TWO degree steps per pass over
// HBM, TMA-staged.
//
//   stage 1: C = x_k     = rho_k     ((2s) A - rho_{k-1} B + (2/d)(R - S A))
//   stage 2: E = x_{k+1} = rho_{k+1} ((2s) C - rho_k     A + (2/d)(R - S C))
// with A = x_{k-1}, B = x_{k-2}, R = r, S the scaled 7-point operator
// (polyprec.cpp:190-195). kFirst: the pass is steps (1, 2): stage 1 is
// x_1 = c1 (2 r - (S r)/theta) with A = R = r (polyprec.cpp:187-189) and stage 2
// uses x_old = x_0 = r/theta.
//
// One CTA owns a 64 x 8 (i x j) output tile and marches a z-chunk. Per plane it
// TMA-loads A with a 2-deep halo (68 x 12 box), B and R with a 1-deep halo
// (66 x 10); out-of-domain box elements arrive zero-filled, which is exactly the
// homogeneous Dirichlet boundary. (B and R use 68 x 10 boxes from i0-2.) Stage 1 computes C on the 66 x 10 extended
// tile (the halo redundantly) into a 3-plane shared ring; stage 2 reads C from
// there. HBM traffic per point per TWO steps: read A, B, R + write C, E = 40 B
// (vs 64 B for two single-step passes); halo re-reads are served by L2.
// Loads run D = 3 planes ahead through a ring of mbarriers; one elected thread
// issues them. Per-point arithmetic is the single-step kernel's (bitwise parity).
#pragma once

#include <cuda.h>

#include "kernels.cuh"

namespace pcgx {

constexpr int kC2TX = 64, kC2TY = 8;                 // output tile
constexpr int kC2AX = kC2TX + 4, kC2AY = kC2TY + 4;  // A box (2-halo)
constexpr int kC2EX = kC2TX + 2, kC2EY = kC2TY + 2;  // extended tile (1-halo)
// B and R boxes start at i0-2 (not i0-1): the innermost TMA box coordinate must
// be 16-byte aligned, i.e. even for fp64 (tools/tma_probe: odd -> illegal instruction).
constexpr int kC2BX = kC2TX + 4, kC2BY = kC2TY + 2;
constexpr int kC2D = 3;                              // prefetch distance (planes)
constexpr int kC2NA = kC2D + 2, kC2NB = kC2D, kC2NR = kC2D + 1, kC2NC = 3;
constexpr int kC2APlane = kC2AX * kC2AY;             // doubles (6528 B = 51 x 128 B)
constexpr int kC2EPlane = kC2EX * kC2EY;             // doubles used per extended plane
constexpr int kC2EStride = 688;                      // slot stride: 5504 B = 43 x 128 B (TMA dst alignment)
constexpr int kC2BPlane = kC2BX * kC2BY;             // doubles loaded per B / R plane (5440 B)
constexpr int kC2Threads = 256;
constexpr size_t kC2Smem =
    sizeof(double) * (size_t)(kC2NA * kC2APlane + (kC2NB + kC2NR + kC2NC) * kC2EStride) +
    16 * (kC2D + 1) + 128;

struct Cheb2Params {
  int nx, ny, nzl;          // local grid
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

// grid: (ceil(nx/64), ceil(ny/8), ceil(nzl/kz)); block: 256 threads; dynamic smem kC2Smem.
template <bool kFirst, bool kRed>
__global__ void __launch_bounds__(kC2Threads, 2)
stencil7_cheb2_kernel(const __grid_constant__ CUtensorMap mapA,  // A (68 x 12 box)
                      const __grid_constant__ CUtensorMap mapB,  // B (68 x 10 box)
                      const __grid_constant__ CUtensorMap mapR,  // R (68 x 10 box)
                      Cheb2Params p, int kz, Reduce red) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sA = reinterpret_cast<double*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  double* sB = sA + kC2NA * kC2APlane;
  double* sR = sB + kC2NB * kC2EStride;
  double* sC = sR + kC2NR * kC2EStride;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sC + kC2NC * kC2EStride);  // kC2D unit bars + 1 prologue

  const int tid = threadIdx.x;
  const int i0 = blockIdx.x * kC2TX, j0 = blockIdx.y * kC2TY;
  const int kb = blockIdx.z * kz;
  const int ke = min(kb + kz, p.nzl);
  const unsigned bytesA = kC2APlane * 8, bytesE = kC2BPlane * 8;
  const unsigned unit_bytes = kFirst ? bytesA : bytesA + 2 * bytesE;

  if (tid == 0) {
    for (int q = 0; q <= kC2D; ++q) mbar_init(&bars[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // load unit u (stage-1 plane u): A[u+1], B[u], R[u]. Planes outside [0, nzl)
  // are never loaded (a box lying wholly outside the tensor faults on sm_100a
  // instead of zero-filling); their few readers substitute 0 = Dirichlet.
  auto in_z = [&](int z) { return z >= 0 && z < p.nzl; };
  auto issue_unit = [&](int u) {
    uint64_t* bar = &bars[(u - (kb - 1)) % kC2D];
    const bool la = in_z(u + 1), lbr = !kFirst && in_z(u);
    mbar_expect_tx(bar, (la ? bytesA : 0u) + (lbr ? 2 * bytesE : 0u));
    if (la)
      tma_load_3d(sA + ((u + 1 - (kb - 2)) % kC2NA) * kC2APlane, &mapA, i0 - 2, j0 - 2, u + 1, bar);
    if (lbr) {
      tma_load_3d(sB + ((u - (kb - 1)) % kC2NB) * kC2EStride, &mapB, i0 - 2, j0 - 1, u, bar);
      tma_load_3d(sR + ((u - (kb - 1)) % kC2NR) * kC2EStride, &mapR, i0 - 2, j0 - 1, u, bar);
    }
  };
  const int u_last = ke;  // stage 1 runs u = kb-1 .. ke
  if (tid == 0) {
    uint64_t* pb = &bars[kC2D];
    mbar_expect_tx(pb, (in_z(kb - 2) ? bytesA : 0u) + (in_z(kb - 1) ? bytesA : 0u));
    if (in_z(kb - 2)) tma_load_3d(sA + 0 * kC2APlane, &mapA, i0 - 2, j0 - 2, kb - 2, pb);
    if (in_z(kb - 1)) tma_load_3d(sA + 1 * kC2APlane, &mapA, i0 - 2, j0 - 2, kb - 1, pb);
    for (int u = kb - 1; u < kb - 1 + kC2D && u <= u_last; ++u) issue_unit(u);
  }
  mbar_wait(&bars[kC2D], 0);

  const double d = p.d;
  double acc = 0.0;
  for (int u = kb - 1; u <= u_last; ++u) {
    const int ui = u - (kb - 1);
    mbar_wait(&bars[ui % kC2D], (ui / kC2D) & 1);
    // ---------------- stage 1: C[u] on the 66 x 10 extended tile
    const double* Am = sA + ((u - 1 - (kb - 2)) % kC2NA) * kC2APlane;
    const double* Ac = sA + ((u - (kb - 2)) % kC2NA) * kC2APlane;
    const double* Ap = sA + ((u + 1 - (kb - 2)) % kC2NA) * kC2APlane;
    const double* Bs = sB + (ui % kC2NB) * kC2EStride;
    const double* Rs = sR + (ui % kC2NR) * kC2EStride;
    double* Cs = sC + (((u % kC2NC) + kC2NC) % kC2NC) * kC2EStride;
    const bool write_c = (u >= kb) && (u < ke);  // halo planes belong to the neighbouring chunks
    const bool plane_in = (u >= 0) && (u < p.nzl);
    const bool has_m = u - 1 >= 0, has_p = u + 1 < p.nzl;
    for (int e = tid; e < kC2EPlane; e += kC2Threads) {
      const int ii = e % kC2EX, jj = e / kC2EX;
      const int gi = i0 - 1 + ii, gj = j0 - 1 + jj;
      double cval = 0.0;
      if (plane_in && gi >= 0 && gi < p.nx && gj >= 0 && gj < p.ny) {
        const int a = (jj + 1) * kC2AX + (ii + 1);  // centre in A-box coordinates
        const double xc = Ac[a];
        const double y = stencil_point(d, has_m ? Am[a] : 0.0, Ac[a - kC2AX], Ac[a - 1], xc,
                                       Ac[a + 1], Ac[a + kC2AX], has_p ? Ap[a] : 0.0);
        if (kFirst) {
          cval = p.c1 * ((2.0 * xc) - (y / p.theta));
        } else {
          const int be = jj * kC2BX + ii + 1;  // B/R box coordinates
          const double ri = Rs[be];
          const double z = p.c2 * (ri - y);
          cval = p.rk1 * (((p.c3 * xc) - (p.rk1m1 * Bs[be])) + z);
        }
        if (write_c && ii >= 1 && ii <= kC2TX && jj >= 1 && jj <= kC2TY)
          p.outC[(long long)u * p.nxy + (long long)gj * p.nx + gi] = cval;
      }
      Cs[e] = cval;
    }
    __syncthreads();
    // ---------------- stage 2: E[u-1] on the 64 x 8 tile
    const int v = u - 1;
    if (v >= kb) {
      const double* Cm = sC + ((((v - 1) % kC2NC) + kC2NC) % kC2NC) * kC2EStride;
      const double* Cc = sC + (((v % kC2NC) + kC2NC) % kC2NC) * kC2EStride;
      const double* Cp = Cs;
      const double* Aold = sA + ((v - (kb - 2)) % kC2NA) * kC2APlane;    // A[v]
      const double* Rv = sR + ((v - (kb - 1)) % kC2NR) * kC2EStride;     // R[v]
      for (int e = tid; e < kC2TX * kC2TY; e += kC2Threads) {
        const int ii = e % kC2TX, jj = e / kC2TX;
        const int gi = i0 + ii, gj = j0 + jj;
        if (gi < p.nx && gj < p.ny) {
          const int c = (jj + 1) * kC2EX + (ii + 1);  // centre in extended-tile coordinates
          const double xc = Cc[c];
          const double y = stencil_point(d, Cm[c], Cc[c - kC2EX], Cc[c - 1], xc, Cc[c + 1],
                                         Cc[c + kC2EX], Cp[c]);
          const int a = (jj + 2) * kC2AX + (ii + 2);
          double ri, xo;
          if (kFirst) {
            ri = Aold[a];            // A == R == r
            xo = ri / p.theta;       // x_0 = r / theta
          } else {
            ri = Rv[(jj + 1) * kC2BX + ii + 2];
            xo = Aold[a];            // x_{k-1}
          }
          const double z = p.c2 * (ri - y);
          const double xn = p.rk2 * (((p.c3 * xc) - (p.rk2m1 * xo)) + z);
          p.outE[(long long)v * p.nxy + (long long)gj * p.nx + gi] = xn;
          if (kRed) acc = acc + ri * xn;
        }
      }
    }
    __syncthreads();
    if (tid == 0 && u + kC2D <= u_last) issue_unit(u + kC2D);
  }
  if (kRed) block_reduce_finish(acc, red);
}

}  // namespace pcgx
