// SPDX-License-Identifier: Apache-2.0
//
// The regular Chebyshev degree step (polyprec.cpp:190-195) on 3x3-block matrices
// whose nodes sit on a cubic nx^3 grid with the 27-point block box (config 4:
// 3-dof Q1 elasticity): the dia3t design for blocks. Next to the BSR-3 arrays
// (SELL-32 over block rows) the upload keeps a grid copy of the values,
// gval[(s * 9 + e) * ldn + node] (slot s = grid neighbour (dz, dy, dx) in
// ascending-offset order, e = 3c + d the block entry), and a 27-bit presence mask
// per node. A CTA owns a 32 x 4 node tile and marches its z-chunk; per plane it
// takes nine 4D value boxes (32 x 4 x 1 x 27: one (dz, dy) row of three slots)
// through a 4-stage ring and one auxiliary unit (masks, r, x_old of the plane,
// the 36 x 6 node patches of x and d of the next plane, dofs interleaved) through
// a 2-stage ring. t = d * x of the patches goes to a 4-plane shared ring; each
// thread sums its node's three rows over the present slots, block columns in
// ascending order, d = 0..2 within a block: the bsr3_kernel's (and the CSR's)
// sequence of roundings, then the recurrence and the in-place store.
#pragma once

#include "dia3t.cuh"

namespace pcgx {

constexpr int kB3X = 32, kB3Y = 4;                  // node tile
constexpr int kB3Threads = kB3X * kB3Y;             // one node (three rows) per thread
constexpr int kB3PX = 3 * (kB3X + 4), kB3PY = kB3Y + 2;  // patch: 36 nodes x 3 dofs, 6 rows
constexpr int kB3Patch = kB3PX * kB3PY;             // 648 doubles
constexpr int kB3Tile = kB3X * kB3Y;                // 128 nodes
constexpr int kB3VBox = 27 * kB3Tile;               // one value unit: 3 slots x 9 entries
constexpr int kB3NV = 4, kB3NA = 2, kB3TR = 4;
// aux stage layout (doubles, TMA destinations 128-byte aligned)
constexpr int kB3OffM = 0;                           // 128 u32 masks = 64 doubles
constexpr int kB3OffR = 64;
constexpr int kB3OffO = kB3OffR + 3 * kB3Tile;
constexpr int kB3OffX = kB3OffO + 3 * kB3Tile;
constexpr int kB3PatchS = (kB3Patch + 15) / 16 * 16;
constexpr int kB3OffD = kB3OffX + kB3PatchS;
constexpr int kB3OffP = kB3OffD + kB3PatchS;  // direction step: p_old patch
constexpr int kB3Aux = kB3OffP + kB3PatchS;
static_assert(kB3OffX % 16 == 0 && kB3OffD % 16 == 0 && kB3OffP % 16 == 0 && kB3Aux % 16 == 0,
              "128-byte TMA destinations");
constexpr size_t kBsr3tSmem =
    sizeof(double) * ((size_t)kB3NV * kB3VBox + (size_t)kB3NA * kB3Aux + (size_t)kB3TR * kB3Patch) +
    8 * (kB3NV + kB3NA) + 128;

struct Bsr3tMaps {
  CUtensorMap val;   // 4D (nx, nx, nx, 243) fp64, box (32, 4, 1, 27)
  CUtensorMap mask;  // 3D (nx, nx, nx) u32, box (32, 4, 1)
  CUtensorMap r, xo; // 3D (3 nx, nx, nx) fp64, box (96, 4, 1)
  CUtensorMap x, d;  // 3D (3 nx, nx, nx) fp64, box (108, 6, 1)
  CUtensorMap p;     // direction step: p_old patches
};

// Epi as in dia3t_kernel: EpiChebStep, EpiChebFirst, or EpiStoreP with In = InComb.
template <bool kRed, class Epi, class In = InVec>
__global__ void __launch_bounds__(kB3Threads, 1)
bsr3t_kernel(const __grid_constant__ Bsr3tMaps maps, int nx, int kz, Epi epi, Reduce red, In in) {
  constexpr bool kFirst = std::is_same<Epi, EpiChebFirst>::value;
  constexpr bool kDir = std::is_same<Epi, EpiStoreP>::value;
  in.init();
  bool first_dir = false;
  if constexpr (kDir) first_dir = in.first != 0;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sV = reinterpret_cast<double*>(smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u));
  double* sA = sV + kB3NV * kB3VBox;
  double* tr = sA + kB3NA * kB3Aux;
  uint64_t* barV = reinterpret_cast<uint64_t*>(tr + kB3TR * kB3Patch);
  uint64_t* barA = barV + kB3NV;
  const int tid = threadIdx.x, tx = tid % kB3X, ty = tid / kB3X;
  const int tiles_x = (nx + kB3X - 1) / kB3X;
  const int i0 = (int)(blockIdx.x % tiles_x) * kB3X, j0 = (int)(blockIdx.x / tiles_x) * kB3Y;
  const int kb = blockIdx.y * kz, ke = min(kb + kz, nx);
  const int i = i0 + tx, j = j0 + ty;
  const bool own = i < nx && j < nx;
  const long long nxy = (long long)nx * nx;
  bool need_xo = false;
  if constexpr (!kFirst && !kDir) need_xo = !epi.xold_from_r;
  const unsigned bytes_patch = kB3Patch * 8;
  const unsigned bytes_aux = kB3Tile * 4 + (kFirst || kDir ? 0u : 3 * kB3Tile * 8 * (need_xo ? 2 : 1));
  const unsigned npatch = (kDir && !first_dir) ? 3u : 2u;
  const int u0 = kb - 2;  // first aux unit: patch of plane kb-1
  const int nvu = (ke - kb) * 9;

  // aux unit u: masks, r, x_old of plane u (kb <= u < ke), x / d patches of plane u+1
  auto issue_aux = [&](int u) {
    const int q = (u - u0) % kB3NA;
    double* s = sA + q * kB3Aux;
    const bool vals = u >= kb && u < ke, pat = u + 1 >= 0 && u + 1 < nx;
    mbar_expect_tx(&barA[q], (vals ? bytes_aux : 0u) + (pat ? npatch * bytes_patch : 0u));
    if (vals) {
      tma_load_3d(s + kB3OffM, &maps.mask, i0, j0, u, &barA[q]);
      if (!kFirst && !kDir) tma_load_3d(s + kB3OffR, &maps.r, 3 * i0, j0, u, &barA[q]);
      if (need_xo) tma_load_3d(s + kB3OffO, &maps.xo, 3 * i0, j0, u, &barA[q]);
    }
    if (pat) {
      tma_load_3d(s + kB3OffX, &maps.x, 3 * (i0 - 2), j0 - 1, u + 1, &barA[q]);
      tma_load_3d(s + kB3OffD, &maps.d, 3 * (i0 - 2), j0 - 1, u + 1, &barA[q]);
      if (kDir && !first_dir) tma_load_3d(s + kB3OffP, &maps.p, 3 * (i0 - 2), j0 - 1, u + 1, &barA[q]);
    }
  };
  // value unit v: plane kb + v / 9, slot group g = v % 9 (slots 3g .. 3g+2)
  auto issue_val = [&](int v) {
    const int q = v % kB3NV;
    mbar_expect_tx(&barV[q], (unsigned)(kB3VBox * 8));
    tma_load_4d(sV + q * kB3VBox, &maps.val, i0, j0, kb + v / 9, 27 * (v % 9), &barV[q]);
  };
  auto wait_aux = [&](int u) {
    const int q = u - u0;
    mbar_wait(&barA[q % kB3NA], (unsigned)(q / kB3NA) & 1u);
  };
  auto wait_val = [&](int v) { mbar_wait(&barV[v % kB3NV], (unsigned)(v / kB3NV) & 1u); };
  // t = d * x of plane u+1 into the t ring (zeros outside the grid); the own node's
  // x and d of that plane
  const int own_p = (ty + 1) * kB3PX + 3 * (tx + 2);
  auto put_t = [&](int u, double (&xo_)[3], double (&do_)[3]) {
    const double* s = sA + ((u - u0) % kB3NA) * kB3Aux;
    double* tp = tr + ((u + 1 + kB3TR) & 3) * kB3Patch;
    const bool pat = u + 1 >= 0 && u + 1 < nx;
    if constexpr (kDir) {  // p = z + beta p_old, combined once per element (InComb::f)
      for (int e = tid; e < kB3Patch; e += kB3Threads)
        tp[e] = pat ? s[kB3OffD + e] * in.f(s[kB3OffX + e], first_dir ? 0.0 : s[kB3OffP + e]) : 0.0;
    } else {
      for (int e = tid; e < kB3Patch; e += kB3Threads) tp[e] = pat ? s[kB3OffD + e] * s[kB3OffX + e] : 0.0;
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double xv = pat ? s[kB3OffX + own_p + c] : 0.0;
      if constexpr (kDir) xv = pat ? in.f(xv, first_dir ? 0.0 : s[kB3OffP + own_p + c]) : 0.0;
      xo_[c] = xv;
      do_[c] = pat ? s[kB3OffD + own_p + c] : 0.0;
    }
  };

  if (tid == 0) {
    for (int q = 0; q < kB3NV; ++q) mbar_init(&barV[q], 1);
    for (int q = 0; q < kB3NA; ++q) mbar_init(&barA[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    issue_aux(u0);
    issue_aux(u0 + 1);
    for (int v = 0; v < kB3NV && v < nvu; ++v) issue_val(v);
  }
  double xr[3], dr[3], xn_[3], dn_[3];
  wait_aux(u0);
  put_t(u0, xn_, dn_);  // t of plane kb-1
  wait_aux(u0 + 1);
  put_t(u0 + 1, xr, dr);  // t, x, d of plane kb
  __syncthreads();
  if (tid == 0) issue_aux(kb);  // into the stage of unit kb-2

  double acc = 0.0;
  int v = 0;  // value units consumed
  for (int k = kb; k < ke; ++k) {
    wait_aux(k);
    put_t(k, xn_, dn_);  // plane k+1
    __syncthreads();
    // the aux stage of unit k-1 was last read before this barrier
    if (tid == 0 && k + 1 <= ke - 1) issue_aux(k + 1);
    const double* sa = sA + ((k - u0) % kB3NA) * kB3Aux;
    const unsigned msk = reinterpret_cast<const unsigned*>(sa + kB3OffM)[tid];
    const double* tpl[3] = {tr + ((k + 3) & 3) * kB3Patch + own_p, tr + (k & 3) * kB3Patch + own_p,
                            tr + ((k + 1) & 3) * kB3Patch + own_p};
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int g = 0; g < 9; ++g, ++v) {
      wait_val(v);
      const double* sv = sV + (v % kB3NV) * kB3VBox + tid;
      const double* tp = tpl[g / 3] + (g % 3 - 1) * kB3PX;  // plane dz, row dy
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        if ((msk >> (3 * g + q)) & 1u) {
          const double* t = tp + 3 * (q - 1);  // column dx
          const double t0 = t[0], t1 = t[1], t2 = t[2];
          const double* w = sv + q * 9 * kB3Tile;
          s0 = s0 + w[0 * kB3Tile] * t0;
          s0 = s0 + w[1 * kB3Tile] * t1;
          s0 = s0 + w[2 * kB3Tile] * t2;
          s1 = s1 + w[3 * kB3Tile] * t0;
          s1 = s1 + w[4 * kB3Tile] * t1;
          s1 = s1 + w[5 * kB3Tile] * t2;
          s2 = s2 + w[6 * kB3Tile] * t0;
          s2 = s2 + w[7 * kB3Tile] * t1;
          s2 = s2 + w[8 * kB3Tile] * t2;
        }
      }
      __syncthreads();
      if (tid == 0 && v + kB3NV < nvu) issue_val(v + kB3NV);
    }
    if (own) {
      const double sum[3] = {s0, s1, s2};
      const long long row = 3 * ((long long)k * nxy + (long long)j * nx + i);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double y = sum[c] * dr[c];
        if constexpr (kDir) {
          epi.q[row + c] = y;
          epi.pout[row + c] = xr[c];
          if (kRed) acc = acc + xr[c] * y;
        } else if constexpr (kFirst) {
          const double xnew = epi.f(y, xr[c]);
          epi.xout[row + c] = xnew;
          if (kRed) acc = acc + xr[c] * xnew;
        } else {
          const double ri = sa[kB3OffR + 3 * tid + c];
          const double xo = need_xo ? sa[kB3OffO + 3 * tid + c] : 0.0;
          const double xnew = epi.f(y, xr[c], ri, xo);
          epi.out[row + c] = xnew;
          if (kRed) acc = acc + ri * xnew;
        }
      }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      xr[c] = xn_[c];
      dr[c] = dn_[c];
    }
  }
  if (kRed) block_reduce_finish(acc, red);
}

}  // namespace pcgx
