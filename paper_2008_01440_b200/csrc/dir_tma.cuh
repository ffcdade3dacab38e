// SPDX-License-Identifier: Apache-2.0
//
// The PCG direction step on the 7-point stencil, TMA-staged:
//   p_new = z + beta p_old   (pcg.cpp:107; first iteration p = z, pcg.cpp:63)
//   q     = A_scaled p_new   (pcg.cpp:72, linop.cpp:236-258, 271-275)
//   p_new . q                (pcg.cpp:74, the first reduction point)
// The register-queue kernel (stencil7v2 with InComb) re-forms z + beta p for every
// neighbour it loads (three combines and six loads per point); here each plane of
// z and p_old arrives once as a 68 x 10 TMA box, every element is combined ONCE
// into a shared p_new plane, and the stencil reads its j-neighbours from there
// (k-neighbours from a per-lane register queue, i-neighbours by shuffle). Same
// per-element operations in the same order as the other paths, so p_new and q are
// bitwise theirs. HBM: read z, p_old; write p_new, q = 32 B per point.
#pragma once

#include "cheb2f.cuh"

namespace pcgx {

// Tile 64 x kDTY (default: the pipelined two-step kernel's 64 x 20, one CTA of
// 22 warps per SM, so both share the 68 x 22 tensor maps): fewer redundant halo
// rows than 64 x 8 (22 box rows per 20 output rows instead of 10 per 8).
#ifndef PCGX_DIRTY
#define PCGX_DIRTY PCGX_C2FTY
#endif
#ifndef PCGX_DIRMINB
#define PCGX_DIRMINB 1
#endif
// (the x tiles of the deferred x += alpha p_old arrive by TMA in the z / p_old units;
// a register load one plane ahead left warps waiting at the plane barrier: removed)
#ifndef PCGX_DIRNS
#define PCGX_DIRNS 5
#endif
constexpr int kDTY = PCGX_DIRTY;
constexpr int kDBY = kDTY + 2;                          // box rows (1-halo)
constexpr int kDBPlane = kC2W * kDBY;
constexpr int kDEStride = (kDBPlane + 15) / 16 * 16;    // TMA destinations: 128-byte multiples
constexpr int kDirNS = PCGX_DIRNS;        // z / p_old ring slots (NS - 2 planes ahead)
constexpr int kDirNC = 3;                 // p_new planes
#ifndef PCGX_DIRUNROLL
#define PCGX_DIRUNROLL 2
#endif
constexpr int kDirUnroll = PCGX_DIRUNROLL; // plane-loop unroll
constexpr int kDirThreads = 32 * (kDTY + 2);  // one warp per extended row (tile rows + 2 halo rows)
constexpr bool kDirXTma = true;
constexpr int kDXStride = kC2TX * kDTY;  // x tile (64 x kDTY), a 128-byte multiple
constexpr size_t kDirSmem =
    sizeof(double) * (size_t)(2 * kDirNS * kDEStride + kDirNC * kDBPlane + (kDirXTma ? kDirNS * kDXStride : 0)) +
    8 * kDirNS + 128;

struct DirParams {
  int nx, ny, nzl;
  // z-slab ranks: z / p_old planes exist on [a_lo, a_hi) (the slab plus the
  // neighbours' boundary planes exchanged into the vectors' padding); tensor z of
  // plane u is u + zoff
  int a_lo, a_hi, zoff;
  long long nxy;
  double d;
  const double* S;
  int s_new, s_old, first;
  double* x;     // != nullptr: also the previous iteration's x += alpha p_old (pcg.cpp:82),
  int s_pq;      //   alpha = S[s_old] / S[s_pq] (deferred from the update kernel)
  double* q;     // A p_new
  double* pout;  // p_new
  double ztheta; // > 0: the z input is r and z = r / ztheta is formed here (m = 0, pcg.cpp:64)
};

// grid: (tiles, plan.n); block kDirThreads; dynamic smem kDirSmem.
__global__ void __launch_bounds__(kDirThreads, PCGX_DIRMINB)
stencil7_dir_kernel(const __grid_constant__ CUtensorMap mapZ, const __grid_constant__ CUtensorMap mapP,
                    const __grid_constant__ CUtensorMap mapX, DirParams p, int k_begin, int k_end,
                    const __grid_constant__ ChunkPlan plan, Reduce red) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sZ = reinterpret_cast<double*>(smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u));
  double* sP = sZ + kDirNS * kDEStride;
  double* sX = sP + kDirNS * kDEStride;  // kDirXTma: x tiles, one per unit (128-byte aligned)
  double* sN = sX + (kDirXTma ? kDirNS * kDXStride : 0);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sN + kDirNC * kDBPlane);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tiles_x = (p.nx + kC2TX - 1) / kC2TX;
  const int i0 = (int)(blockIdx.x % tiles_x) * kC2TX, j0 = (int)(blockIdx.x / tiles_x) * kDTY;
  const int kb = k_begin + plan.start[blockIdx.y];
  const int ke = min(k_begin + plan.start[blockIdx.y + 1], k_end);
  if ((plan.skip >> blockIdx.y) & 1ull) {  // a masked chunk (ChunkPlan::skip) only joins the reduction
    block_reduce_finish(0.0, red);
    return;
  }
  const bool first = p.first != 0;
  const double beta = first ? 0.0 : p.S[p.s_new] / p.S[p.s_old];
  const unsigned bytes = kDBPlane * 8;  // box bytes
  auto in_z = [&](int z) { return z >= p.a_lo && z < p.a_hi; };
  const bool xupd = p.x != nullptr && !first;
  // unit u: the z (and p_old) boxes of plane u, slot / barrier (u - (kb-1)) % NS
  auto issue = [&](int u) {
    const int q = (u - (kb - 1)) % kDirNS;
    const bool ld = in_z(u);
    const bool lx = kDirXTma && xupd && u >= kb && u < ke;
    mbar_expect_tx(&bars[q], (ld ? (first ? bytes : 2 * bytes) : 0u) + (lx ? kDXStride * 8u : 0u));
    if (ld) {
      tma_load_3d(sZ + q * kDEStride, &mapZ, i0 - 2, j0 - 1, u + p.zoff, &bars[q]);
      if (!first) tma_load_3d(sP + q * kDEStride, &mapP, i0 - 2, j0 - 1, u + p.zoff, &bars[q]);
    }
    if (lx) tma_load_3d(sX + q * kDXStride, &mapX, i0, j0, u, &bars[q]);
  };
  if (tid == 0) {
    for (int q = 0; q < kDirNS; ++q) mbar_init(&bars[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int u = kb - 1; u < kb - 1 + kDirNS && u <= ke; ++u) issue(u);
  }
  __syncthreads();

  const double d = p.d;
  const double2 zero2 = make_double2(0.0, 0.0);
  const int col = 2 * lane + 2;
  const int gi = i0 + 2 * lane;
  const bool pair_in = gi < p.nx;
  const int gj = j0 - 1 + warp;
  const bool do1 = gj >= 0 && gj < p.ny && pair_in;
  const bool tile_row = warp >= 1 && warp <= kDTY;
  const int off = warp * kC2W + col;
  const int eoff = lane == 0 ? -1 : 64 - 2 * lane;  // lane 0: west of its pair; else lane 31's east
  const long long goff = (long long)gj * p.nx + gi;
  const bool zdiv = p.ztheta > 0.0;
  const double zinv = zdiv ? 1.0 / p.ztheta : 0.0;  // RN(1/theta), as on the host
  auto zval = [&](double v) { return zdiv ? div_rn_z(v, p.ztheta, zinv) : v; };
  auto comb = [&](double zv, double pv) {
    zv = zval(zv);
    return first ? zv : zv + beta * pv;
  };
  const double alpha = xupd ? p.S[p.s_old] / p.S[p.s_pq] : 0.0;

  double2 pm = zero2, pc = zero2;  // p_new of the warp's row at planes u-2, u-1
  double acc = 0.0;
  int slot = 0;
  unsigned phase = 0;
  int sc = 0;  // p_new ring slot of plane u
#pragma unroll kDirUnroll
  for (int u = kb - 1; u <= ke; ++u) {
    // the x pair of plane u-1 (deferred update below): issued before the waits of
    // this iteration so its latency hides behind them
    double2 xv = zero2;
    const bool xdo = xupd && tile_row && do1 && u - 1 >= kb;
    mbar_wait(&bars[slot], phase);
    const double* Zu = sZ + slot * kDEStride;
    const double* Pu = sP + slot * kDEStride;
    double2 pn = zero2;
    if (in_z(u) && do1) {
      const double2 zv = *reinterpret_cast<const double2*>(Zu + off);
      if (first) {
        pn = make_double2(zval(zv.x), zval(zv.y));
      } else {
        const double2 pv = *reinterpret_cast<const double2*>(Pu + off);
        pn = make_double2(comb(zv.x, pv.x), comb(zv.y, pv.y));
      }
    }
    double* Nu = sN + sc * kDBPlane;
    *reinterpret_cast<double2*>(Nu + off) = pn;
    __syncthreads();
    // the slot of plane u-2 is free (its last readers are behind this barrier)
    if (tid == 0 && u >= kb + 1 && u - 2 + kDirNS <= ke) issue(u - 2 + kDirNS);
    const int v = u - 1;
    if (tile_row && v >= kb) {
      // p_new of plane v: the warp's own pair (pc), i-neighbours by shuffle, the
      // lane-0 / lane-31 outer neighbours combined from plane v's boxes (zero-filled
      // outside the domain), j-neighbours from the shared plane
      const int sv = slot == 0 ? kDirNS - 1 : slot - 1;
      const double* Zv = sZ + sv * kDEStride;
      const double* Pv = sP + sv * kDEStride;
      const double* Nv = sN + (sc == 0 ? kDirNC - 1 : sc - 1) * kDBPlane;
      double pw = __shfl_up_sync(0xffffffffu, pc.y, 1);
      double pe = __shfl_down_sync(0xffffffffu, pc.x, 1);
      {
        // one combine for the warp (lane 0: its west, the others: broadcast of lane
        // 31's east) instead of two divergent ones
        const double e = comb(Zv[off + eoff], first ? 0.0 : Pv[off + eoff]);
        pw = lane == 0 ? e : pw;
        pe = lane == 31 ? e : pe;
      }
      if (do1) {
        const double2 ps = *reinterpret_cast<const double2*>(Nv + off - kC2W);
        const double2 pnn = *reinterpret_cast<const double2*>(Nv + off + kC2W);
        const double y0 = stencil_point(d, pm.x, ps.x, pw, pc.x, pc.y, pnn.x, pn.x);
        const double y1 = stencil_point(d, pm.y, ps.y, pc.x, pc.y, pe, pnn.y, pn.y);
        const long long idx = (long long)v * p.nxy + goff;
        PCGX_DCHECK(idx >= -(long long)p.zoff * p.nxy && idx + 2 <= (long long)(p.nzl + p.zoff) * p.nxy);
        st2(p.q + idx, y0, y1);
        st2(p.pout + idx, pc.x, pc.y);
        acc = acc + (pc.x * y0 + pc.y * y1);
        if (xdo) {
          xv = *reinterpret_cast<const double2*>(sX + sv * kDXStride + (warp - 1) * kC2TX + 2 * lane);
          const double2 po = *reinterpret_cast<const double2*>(Pv + off);
          xv.x = xv.x + alpha * po.x;
          xv.y = xv.y + alpha * po.y;
          st2(p.x + idx, xv.x, xv.y);
        }
      }
    }
    pm = pc;
    pc = pn;
    if (++slot == kDirNS) {
      slot = 0;
      phase ^= 1u;
    }
    sc = (sc + 1 == kDirNC) ? 0 : sc + 1;
  }
  block_reduce_finish(acc, red);
}

}  // namespace pcgx
