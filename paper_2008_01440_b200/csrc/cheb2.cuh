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
// TMA-loads A with a 2-deep j halo (68 x 12 box), B and R with a 1-deep one
// (68 x 10); out-of-domain box elements arrive zero-filled (the homogeneous
// Dirichlet boundary). Stage 1 computes C on the 66 x 10 extended tile (the halo
// redundantly) into a 3-plane shared ring; stage 2 reads C from there. HBM traffic per point per TWO steps: read A, B, R + write C, E = 40 B
// (vs 64 B for two single-step passes); halo re-reads are served by L2.
// Loads run D = 4 planes ahead through a ring of mbarriers; one elected thread
// issues them. One block barrier per plane (the ring refill rides on it). Per-point arithmetic is the single-step kernel's (bitwise parity).
#pragma once

#include <cuda.h>

#include "kernels.cuh"

namespace pcgx {

#ifndef PCGX_C2TY
#define PCGX_C2TY 8
#endif
constexpr int kC2TX = 64, kC2TY = PCGX_C2TY;         // output tile (i x j)
constexpr int kC2W = kC2TX + 4;                      // row width of every smem plane (tile-i t <-> col t+2)
constexpr int kC2AY = kC2TY + 4;                     // A box rows (2-halo in j)
constexpr int kC2BY = kC2TY + 2;                     // B, R boxes and the C ring: 1-halo rows
// Every TMA box starts at i0-2: the innermost box coordinate must be 16-byte
// aligned, i.e. even for fp64 (tools/tma_probe: an odd origin is an illegal
// instruction on sm_100a). A box 68 x 12 (6528 B), B/R boxes 68 x 10 (5440 B).
constexpr int kC2AX = kC2W, kC2BX = kC2W;
#ifndef PCGX_C2D
#define PCGX_C2D 4
#endif
#ifndef PCGX_C2MINB
#define PCGX_C2MINB 2
#endif
#ifndef PCGX_C2UNROLL
#define PCGX_C2UNROLL 4
#endif
constexpr int kC2Unroll = PCGX_C2UNROLL;             // plane-loop unroll
constexpr int kC2D = PCGX_C2D;                       // prefetch distance (planes)
constexpr int kC2NA = kC2D + 2, kC2NB = kC2D, kC2NR = kC2D + 1, kC2NC = 3;
constexpr int kC2APlane = kC2W * kC2AY;              // 816 doubles = 51 x 128 B
constexpr int kC2BPlane = kC2W * kC2BY;              // 680 doubles
constexpr int kC2EStride = (kC2W * kC2BY + 15) / 16 * 16;  // B/R slot stride, 128-byte multiple (TMA dst)
constexpr int kC2CStride = kC2BPlane;                // C ring slot (plain shared stores)
constexpr int kC2Warps = kC2TY + 2;                  // one warp per extended row in stage 1
constexpr int kC2Threads = 32 * kC2Warps;            // 320 at the default 64 x 8 tile
constexpr size_t kC2Smem = sizeof(double) * (size_t)(kC2NA * kC2APlane + (kC2NB + kC2NR) * kC2EStride +
                                                     kC2NC * kC2CStride) +
                           16 * (kC2D + 1) + 128;

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

// grid: (ceil(nx/64), ceil(ny/8), ceil(nzl/kz)); block: 320 threads; dynamic smem kC2Smem.
//
// Stage 1: warp w owns extended row w (tile row w-1); lane l owns the point
// pair tile-i (2l, 2l+1). The k-1 / k+1 neighbours of the pairs live in per-lane
// register queues, i-1 / i+1 come by shuffle, only j-1 / j+1 and the operands
// are read from shared memory (16-byte LDS). Ring slots rotate by one per plane
// and are tracked with incremented indices (no modulo).
//
// Stage 2 (kV = 0): warp w < 8 owns tile row w, reading its C centre, the A and
// R operands from shared memory; warps 8 and 9 compute the two halo columns
// (tile-i -1 and 64) of C for the plane stage 1 just produced (first read by
// stage 2 one iteration later).
// Stage 2 (kV >= 1, "own row"): warp w in 1..8 computes E for the row it produced
// in stage 1, so the C centre queue (k-1, k, k+1), x_{k-1} and the i-neighbours
// are its own registers; only C's j +- 1 rows come from shared memory. Warps 0
// and 9 (the j-halo rows) compute the halo columns.
// kV = 2 additionally keeps t = d * x instead of x in the stencil queues and in
// the C ring: each product d * x is formed once per point instead of once per
// use (7x), so a stencil costs 1-3 DMUL + 7 DADD instead of 9 DMUL + 7 DADD; the
// IEEE products are the same, hence bitwise the same sums.
template <bool kFirst, bool kRed, int kV>
__global__ void __launch_bounds__(kC2Threads, PCGX_C2MINB)
stencil7_cheb2_kernel(const __grid_constant__ CUtensorMap mapA,  // A (68 x 12 box)
                      const __grid_constant__ CUtensorMap mapB,  // B (68 x 10 box)
                      const __grid_constant__ CUtensorMap mapR,  // R (68 x 10 box)
                      Cheb2Params p, int k_begin, int k_end, int kz, Reduce red) {
  constexpr bool kOwn = kV >= 1, kT = kV >= 2;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // 128-byte aligned base, kept as a shared-space pointer (LDS, not generic LD)
  double* sA = reinterpret_cast<double*>(smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u));
  double* sB = sA + kC2NA * kC2APlane;
  double* sR = sB + kC2NB * kC2EStride;
  double* sC = sR + kC2NR * kC2EStride;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sC + kC2NC * kC2CStride);  // kC2D unit bars + 1 prologue

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int i0 = blockIdx.x * kC2TX, j0 = blockIdx.y * kC2TY;
  const int kb = k_begin + blockIdx.z * kz;
  const int ke = min(kb + kz, k_end);
  const unsigned bytesA = kC2APlane * 8, bytesB = kC2BPlane * 8;

  if (tid == 0) {
    for (int q = 0; q <= kC2D; ++q) mbar_init(&bars[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // Load unit u (stage-1 plane u): A[u+1], B[u], R[u]. Planes outside [0, nzl)
  // are never loaded (their readers substitute 0 = Dirichlet).
  auto in_z = [&](int z) { return z >= p.a_lo && z < p.a_hi; };
  const int zo = p.zoff;
  auto issue_unit = [&](int u) {
    uint64_t* bar = &bars[(u - (kb - 1)) % kC2D];
    const bool la = in_z(u + 1), lbr = !kFirst && in_z(u);
    mbar_expect_tx(bar, (la ? bytesA : 0u) + (lbr ? 2 * bytesB : 0u));
    if (la) tma_load_3d(sA + ((u + 1 - (kb - 2)) % kC2NA) * kC2APlane, &mapA, i0 - 2, j0 - 2, u + 1 + zo, bar);
    if (lbr) {
      tma_load_3d(sB + ((u - (kb - 1)) % kC2NB) * kC2EStride, &mapB, i0 - 2, j0 - 1, u + zo, bar);
      tma_load_3d(sR + ((u - (kb - 1)) % kC2NR) * kC2EStride, &mapR, i0 - 2, j0 - 1, u + zo, bar);
    }
  };
  const int u_last = ke;  // stage 1 runs u = kb-1 .. ke
  if (tid == 0) {
    uint64_t* pb = &bars[kC2D];
    mbar_expect_tx(pb, (in_z(kb - 2) ? bytesA : 0u) + (in_z(kb - 1) ? bytesA : 0u));
    if (in_z(kb - 2)) tma_load_3d(sA, &mapA, i0 - 2, j0 - 2, kb - 2 + zo, pb);
    if (in_z(kb - 1)) tma_load_3d(sA + kC2APlane, &mapA, i0 - 2, j0 - 2, kb - 1 + zo, pb);
    for (int u = kb - 1; u < kb - 1 + kC2D && u <= u_last; ++u) issue_unit(u);
  }
  mbar_wait(&bars[kC2D], 0);

  const double d = p.d;
  const double inv_t = 1.0 / p.theta;  // RN(1/theta): quotients by theta via div_rn
  const double2 zero2 = make_double2(0.0, 0.0);
  const int col = 2 * lane + 2;                    // smem column of the lane's pair
  const int gi = i0 + 2 * lane;                    // global i of the pair's first point
  const bool pair_in = gi < p.nx;                  // nx even: both points or none
  // stage 1 (extended row `warp`)
  const int gj1 = j0 - 1 + warp;
  const bool row1_in = gj1 >= 0 && gj1 < p.ny;
  const bool do1 = row1_in && pair_in;
  const int offA1 = (warp + 1) * kC2W + col;       // A-box offset of the pair
  const int offB1 = warp * kC2W + col;             // B/R/C offset of the pair
  const bool c_interior = warp >= 1 && warp <= kC2TY;
  double* gC = p.outC + (long long)gj1 * p.nx + gi;  // + u * nxy
  // stage 2: tile row `warp` for warps 0..7 (kV = 0) or own row for warps 1..8
  const bool stage2 = kOwn ? c_interior : warp < kC2TY;
  const int gj2 = kOwn ? gj1 : j0 + warp;
  const bool do2 = stage2 && gj2 < p.ny && pair_in;
  const int offC2 = kOwn ? offB1 : (warp + 1) * kC2W + col;
  const int offA2 = kOwn ? offA1 : (warp + 2) * kC2W + col;
  double* gE = p.outE + (long long)gj2 * p.nx + gi;  // + v * nxy
  // halo columns (lanes 0..9 of two warps): column tile-i -1 or 64
  const int hw0 = kOwn ? 0 : kC2TY, hw1 = kOwn ? kC2TY + 1 : kC2TY + 1;
  const bool do_h = (warp == hw0 || warp == hw1) && lane < kC2BY;
  const int hcol = warp == hw0 ? 1 : kC2TX + 2;
  const int hgi = warp == hw0 ? i0 - 1 : i0 + kC2TX;
  const int hgj = j0 - 1 + lane;
  const bool h_in = do_h && hgi >= 0 && hgi < p.nx && hgj >= 0 && hgj < p.ny;
  const int offAh = (lane + 1) * kC2W + hcol, offBh = lane * kC2W + hcol;

  // Ring slots of plane u, as rotating shared pointers (one add + select per ring
  // per plane): A[u-1], A[u], A[u+1]; B[u]; R[u-1], R[u]; C[u-1], C[u].
  const double* const sAend = sA + kC2NA * kC2APlane;
  const double* const sBend = sB + kC2NB * kC2EStride;
  const double* const sRend = sR + kC2NR * kC2EStride;
  double* const sCend = sC + kC2NC * kC2CStride;
  const double* pAm = sA;                      // A[kb-2]
  const double* pAu = sA + kC2APlane;          // A[kb-1]
  const double* pAp = sA + 2 * kC2APlane;      // A[kb]
  const double* pBu = sB;                      // B[kb-1]
  const double* pRu = sR;                      // R[kb-1]
  const double* pRm = sR + (kC2NR - 1) * kC2EStride;  // R[kb-2] (never read)
  const int sc0 = (((kb - 1) % kC2NC) + kC2NC) % kC2NC;
  double* pCu = sC + sc0 * kC2CStride;         // C[kb-1]
  double* pCm = sC + ((sc0 + kC2NC - 1) % kC2NC) * kC2CStride;
  int bslot = 0;                               // unit barrier of plane u
  unsigned bphase = 0;
  double* gCu = gC + (long long)(kb - 1) * p.nxy;  // this lane's C pair at plane u
  double* gEv = gE + (long long)(kb - 2) * p.nxy;  // this lane's E pair at plane u-1

  auto mul2 = [&](double2 v) { return make_double2(d * v.x, d * v.y); };
  // stage-1 queue: A (x, or t = d x when kT) of planes u-1, u
  double2 am = in_z(kb - 2) ? *reinterpret_cast<const double2*>(sA + offA1) : zero2;
  double2 ac = in_z(kb - 1) ? *reinterpret_cast<const double2*>(sA + kC2APlane + offA1) : zero2;
  if (kT) {
    am = mul2(am);
    ac = mul2(ac);
  }
  double2 cm = zero2, cc = zero2;     // stage-2 C (x, or t when kT) of planes v-1, v
  double2 cx = zero2;                 // kT: C x of plane v (own row)
  double acc = 0.0;

#pragma unroll kC2Unroll
  for (int u = kb - 1; u <= u_last; ++u) {
    mbar_wait(&bars[bslot], bphase);
    const double* Au = pAu;
    const double* Ap = pAp;
    const double* Bu = pBu;
    const double* Ru = pRu;
    double* Cu = pCu;
    const bool plane_in = u >= p.c_lo && u < p.c_hi, has_p = in_z(u + 1);
    // ---------------- stage 1: C[u] pairs of the extended tile
    double2 ap, cv = zero2;
    {
      ap = has_p ? *reinterpret_cast<const double2*>(Ap + offA1) : zero2;
      if (kT) ap = mul2(ap);
      double aw = __shfl_up_sync(0xffffffffu, ac.y, 1);
      double ae = __shfl_down_sync(0xffffffffu, ac.x, 1);
      if (lane == 0) aw = kT ? d * Au[offA1 - 1] : Au[offA1 - 1];
      if (lane == 31) ae = kT ? d * Au[offA1 + 2] : Au[offA1 + 2];
      if (plane_in && do1) {
        const double2 as = *reinterpret_cast<const double2*>(Au + offA1 - kC2W);
        const double2 an = *reinterpret_cast<const double2*>(Au + offA1 + kC2W);
        double y0, y1;
        double2 xc;
        if (kT) {
          xc = *reinterpret_cast<const double2*>(Au + offA1);
          y0 = stencil_point_t(d, am.x, d * as.x, aw, ac.x, ac.y, d * an.x, ap.x);
          y1 = stencil_point_t(d, am.y, d * as.y, ac.x, ac.y, ae, d * an.y, ap.y);
        } else {
          xc = ac;
          y0 = stencil_point(d, am.x, as.x, aw, ac.x, ac.y, an.x, ap.x);
          y1 = stencil_point(d, am.y, as.y, ac.x, ac.y, ae, an.y, ap.y);
        }
        if (kFirst) {
          cv.x = p.c1 * ((2.0 * xc.x) - div_rn(y0, p.theta, inv_t));
          cv.y = p.c1 * ((2.0 * xc.y) - div_rn(y1, p.theta, inv_t));
        } else {
          const double2 bb = *reinterpret_cast<const double2*>(Bu + offB1);
          const double2 rr = *reinterpret_cast<const double2*>(Ru + offB1);
          cv.x = p.rk1 * (((p.c3 * xc.x) - (p.rk1m1 * bb.x)) + p.c2 * (rr.x - y0));
          cv.y = p.rk1 * (((p.c3 * xc.y) - (p.rk1m1 * bb.y)) + p.c2 * (rr.y - y1));
        }
        if (c_interior && u >= kb && u < ke) st2(gCu, cv.x, cv.y);
      }
      *reinterpret_cast<double2*>(Cu + offB1) = kT ? mul2(cv) : cv;
      if (!kOwn) {
        am = ac;
        ac = ap;
      }
    }
    __syncthreads();
    // Refill the ring slots of unit u-1 with unit u-1+D: every warp is past
    // stage 2 / the halo of iteration u-1, the last readers of A[u-2], B[u-1],
    // R[u-2]. This is the only block barrier of the iteration: a warp runs on
    // from its stage 2 of u into stage 1 of u+1 without waiting for the others.
    if (tid == 0 && u >= kb && u - 1 + kC2D <= u_last) issue_unit(u - 1 + kC2D);
    // ---------------- stage 2: E[u-1] on the tile | halo columns of C[u]
    if (stage2) {
      const int v = u - 1;
      const double* Cv = pCm;
      double2 cp;  // C (x or t) of plane v+1 = u
      if (kOwn) cp = kT ? mul2(cv) : cv;
      else cp = *reinterpret_cast<const double2*>(Cu + offC2);
      double cw = __shfl_up_sync(0xffffffffu, cc.y, 1);
      double ce = __shfl_down_sync(0xffffffffu, cc.x, 1);
      if (lane == 0) cw = Cv[offC2 - 1];
      if (lane == 31) ce = Cv[offC2 + 2];
      if (v >= kb && do2) {
        const double2 cs = *reinterpret_cast<const double2*>(Cv + offC2 - kC2W);
        const double2 cn = *reinterpret_cast<const double2*>(Cv + offC2 + kC2W);
        double y0, y1;
        double2 ccx;
        if (kT) {
          y0 = stencil_point_t(d, cm.x, cs.x, cw, cc.x, cc.y, cn.x, cp.x);
          y1 = stencil_point_t(d, cm.y, cs.y, cc.x, cc.y, ce, cn.y, cp.y);
          ccx = cx;
        } else {
          y0 = stencil_point(d, cm.x, cs.x, cw, cc.x, cc.y, cn.x, cp.x);
          y1 = stencil_point(d, cm.y, cs.y, cc.x, cc.y, ce, cn.y, cp.y);
          ccx = cc;
        }
        // A[v] = A[u-1]: the stage-1 queue's previous centre (own row, x only)
        const double2 av = (kOwn && !kT) ? am : *reinterpret_cast<const double2*>(pAm + offA2);
        double2 rv, xo;
        if (kFirst) {
          rv = av;  // A == R == r
          xo = make_double2(div_rn(av.x, p.theta, inv_t), div_rn(av.y, p.theta, inv_t));  // x_0 = r / theta
        } else {
          rv = *reinterpret_cast<const double2*>(pRm + offC2);  // R[v]
          xo = av;  // x_{k-1}
        }
        const double e0 = p.rk2 * (((p.c3 * ccx.x) - (p.rk2m1 * xo.x)) + p.c2 * (rv.x - y0));
        const double e1 = p.rk2 * (((p.c3 * ccx.y) - (p.rk2m1 * xo.y)) + p.c2 * (rv.y - y1));
        st2(gEv, e0, e1);
        if (kRed) acc = acc + (rv.x * e0 + rv.y * e1);
      }
      cm = cc;
      cc = cp;
      if (kT) cx = cv;
    } else if (do_h) {
      double hx = 0.0;
      if (plane_in && h_in) {
        const double xc = Au[offAh];
        const double y = stencil_point(d, in_z(u - 1) ? pAm[offAh] : 0.0, Au[offAh - kC2W],
                                       Au[offAh - 1], xc, Au[offAh + 1], Au[offAh + kC2W],
                                       has_p ? Ap[offAh] : 0.0);
        if (kFirst) hx = p.c1 * ((2.0 * xc) - div_rn(y, p.theta, inv_t));
        else hx = p.rk1 * (((p.c3 * xc) - (p.rk1m1 * Bu[offBh])) + p.c2 * (Ru[offBh] - y));
      }
      Cu[offBh] = kT ? d * hx : hx;
    }
    if (kOwn) {
      am = ac;
      ac = ap;
    }
    // rotate the rings and global pointers by one plane
    pAm = pAu;
    pAu = pAp;
    pAp = (pAp + kC2APlane == sAend) ? sA : pAp + kC2APlane;
    pBu = (pBu + kC2EStride == sBend) ? sB : pBu + kC2EStride;
    pRm = pRu;
    pRu = (pRu + kC2EStride == sRend) ? sR : pRu + kC2EStride;
    pCm = pCu;
    pCu = (pCu + kC2CStride == sCend) ? sC : pCu + kC2CStride;
    if (++bslot == kC2D) {
      bslot = 0;
      bphase ^= 1u;
    }
    gCu += p.nxy;
    gEv += p.nxy;
  }
  if (kRed) block_reduce_finish(acc, red);
}

}  // namespace pcgx
