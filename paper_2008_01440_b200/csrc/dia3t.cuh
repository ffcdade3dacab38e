// SPDX-License-Identifier: Apache-2.0
//
// The regular Chebyshev degree step (polyprec.cpp:190-195) on offset storage
// over grid tiles with every operand streamed by TMA: dia3_kernel's tile and
// arithmetic (bitwise the same row sums and recurrence), but the 27 value slots
// of a plane arrive as ONE 4D box (32 i x 8 j x 1 k x 27 slots) instead of 27
// predicated loads per thread held in registers (80 registers, 24 warps per SM,
// a spill), together with the presence masks, r, x_old and the 36 x 10 patches of
// x and d of the next plane, through a 3-stage mbarrier ring. The warps only
// compute: t = d * x of plane k+1 into a 4-plane shared ring, then per point the
// present terms v * t in slot order, y = sum * d, the recurrence, the store of
// x_new (in place over x_old: each point's x_old arrived before its own store)
// and the r * x_new partial (last step).
//
// Box origins are even (an odd fp64 box origin is an illegal instruction on
// sm_100a) and planes outside the grid are never requested (a box wholly outside
// the tensor faults instead of zero-filling): their t plane is zeroed instead.
#pragma once

#include "cheb2.cuh"
#include "kernels.cuh"

namespace pcgx {

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

constexpr int kT3K = 27;                  // slots (the 27-point box)
constexpr int kT3PX = kD3X + 4;           // patch columns: tile-i t <-> column t + 2 (even box origin)
constexpr int kT3PY = kD3Y + 2;
constexpr int kT3Patch = kT3PX * kT3PY;   // 360
constexpr int kT3Tile = kD3X * kD3Y;      // 256
constexpr int kT3D = 3;                   // ring stages
// stage layout (doubles; every TMA destination 128-byte aligned)
constexpr int kT3OffV = 0;
constexpr int kT3OffM = kT3OffV + kT3K * kT3Tile;         // masks: 256 x u32 = 128 doubles
constexpr int kT3OffR = kT3OffM + kT3Tile / 2;
constexpr int kT3OffO = kT3OffR + kT3Tile;
constexpr int kT3OffX = kT3OffO + kT3Tile;
constexpr int kT3OffD = kT3OffX + (kT3Patch + 15) / 16 * 16;
constexpr int kT3OffP = kT3OffD + (kT3Patch + 15) / 16 * 16;  // direction step: p_old patch
constexpr int kT3Stage = kT3OffP + (kT3Patch + 15) / 16 * 16;
constexpr int kT3TRing = 4;
constexpr size_t kDia3tSmem =
    sizeof(double) * ((size_t)kT3D * kT3Stage + (size_t)kT3TRing * kT3Patch) + 16 * kT3D + 128;
static_assert(kT3Tile == kD3Threads, "one point per thread");
static_assert(kT3Patch <= 2 * kD3Threads, "two patch elements per thread");

struct Dia3tMaps {
  CUtensorMap val;   // 4D (nx, nx, nx, 27) fp64, box (32, 8, 1, 27)
  CUtensorMap mask;  // 3D (nx, nx, nx) u32, box (32, 8, 1)
  CUtensorMap r, xo; // 3D fp64, box (32, 8, 1)
  CUtensorMap x, d;  // 3D fp64, box (36, 10, 1)
  CUtensorMap p;     // direction step: p_old patches (36, 10, 1)
};

// Epi: EpiChebStep (regular step: r and x_old tiles by TMA), EpiChebFirst (step 1,
// polyprec.cpp:187-189: x_1 = c1 ((2 r) - (A r) / theta), the input IS r, no tiles)
// or EpiStoreP with In = InComb (the PCG direction step, pcg.cpp:63,72-74,107: the
// patches of z and p_old combine into p = z + beta p_old before t = d p; q = A p,
// p written at the own points, p . q reduced)
template <bool kRed, class Epi, class In = InVec>
__global__ void __launch_bounds__(kD3Threads, 1)
dia3t_kernel(const __grid_constant__ Dia3tMaps maps, int nx, int kz, Epi epi, Reduce red, In in) {
  constexpr bool kFirst = std::is_same<Epi, EpiChebFirst>::value;
  constexpr bool kDir = std::is_same<Epi, EpiStoreP>::value;
  in.init();
  bool first_dir = false;
  if constexpr (kDir) first_dir = in.first != 0;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* st0 = reinterpret_cast<double*>(smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u));
  double* tr = st0 + kT3D * kT3Stage;  // t ring, 4 planes
  uint64_t* bars = reinterpret_cast<uint64_t*>(tr + kT3TRing * kT3Patch);
  const int tid = threadIdx.x, tx = tid % kD3X, ty = tid / kD3X;
  const int tiles_x = (nx + kD3X - 1) / kD3X;
  const int i0 = (int)(blockIdx.x % tiles_x) * kD3X, j0 = (int)(blockIdx.x / tiles_x) * kD3Y;
  const int kb = blockIdx.y * kz, ke = min(kb + kz, nx);
  const int i = i0 + tx, j = j0 + ty;
  const bool own = i < nx && j < nx;
  const long long nxy = (long long)nx * nx;
  bool need_xo = false;
  if constexpr (!kFirst && !kDir) need_xo = !epi.xold_from_r;
  const unsigned bytes_tile = kT3Tile * 8, bytes_patch = kT3Patch * 8;
  const unsigned bytes_vals =
      (unsigned)(kT3K * kT3Tile * 8) + bytes_tile / 2 + (kFirst || kDir ? 0u : bytes_tile * (need_xo ? 2 : 1));
  const unsigned npatch = (kDir && !first_dir) ? 3u : 2u;
  const int u0 = kb - 2;  // first unit

  // unit u: values, masks, r, x_old of plane u (kb <= u < ke) and the x, d
  // patches of plane u + 1 (inside the grid); stage (u - u0) % kT3D
  auto issue = [&](int u) {
    const int sidx = (u - u0) % kT3D;
    double* s = st0 + sidx * kT3Stage;
    uint64_t* bar = &bars[sidx];
    const bool vals = u >= kb && u < ke, pat = u + 1 >= 0 && u + 1 < nx;
    mbar_expect_tx(bar, (vals ? bytes_vals : 0u) + (pat ? npatch * bytes_patch : 0u));
    if (vals) {
      tma_load_4d(s + kT3OffV, &maps.val, i0, j0, u, 0, bar);
      tma_load_3d(s + kT3OffM, &maps.mask, i0, j0, u, bar);
      if (!kFirst && !kDir) tma_load_3d(s + kT3OffR, &maps.r, i0, j0, u, bar);
      if (need_xo) tma_load_3d(s + kT3OffO, &maps.xo, i0, j0, u, bar);
    }
    if (pat) {
      tma_load_3d(s + kT3OffX, &maps.x, i0 - 2, j0 - 1, u + 1, bar);
      tma_load_3d(s + kT3OffD, &maps.d, i0 - 2, j0 - 1, u + 1, bar);
      if (kDir && !first_dir) tma_load_3d(s + kT3OffP, &maps.p, i0 - 2, j0 - 1, u + 1, bar);
    }
  };
  auto wait_unit = [&](int u) {
    const int q = u - u0;
    mbar_wait(&bars[q % kT3D], (unsigned)(q / kT3D) & 1u);
  };
  // t = d * x of plane u + 1 from unit u's patches into the t ring (zeros outside
  // the grid); returns the own point's x and d of that plane
  const int own_p = (ty + 1) * kT3PX + tx + 2;
  auto put_t = [&](int u, double& xo_, double& do_) {
    const double* s = st0 + ((u - u0) % kT3D) * kT3Stage;
    double* tp = tr + ((u + 1 + kT3TRing) & 3) * kT3Patch;
    const bool pat = u + 1 >= 0 && u + 1 < nx;
    if constexpr (kDir) {  // p = z + beta p_old, combined once per element (InComb::f)
      for (int e = tid; e < kT3Patch; e += kD3Threads)
        tp[e] = pat ? s[kT3OffD + e] * in.f(s[kT3OffX + e], first_dir ? 0.0 : s[kT3OffP + e]) : 0.0;
      xo_ = pat ? in.f(s[kT3OffX + own_p], first_dir ? 0.0 : s[kT3OffP + own_p]) : 0.0;
    } else {
      for (int e = tid; e < kT3Patch; e += kD3Threads) tp[e] = pat ? s[kT3OffD + e] * s[kT3OffX + e] : 0.0;
      xo_ = pat ? s[kT3OffX + own_p] : 0.0;
    }
    do_ = pat ? s[kT3OffD + own_p] : 0.0;
  };

  if (tid == 0) {
    for (int q = 0; q < kT3D; ++q) mbar_init(&bars[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int u = u0; u < u0 + kT3D && u <= ke - 1; ++u) issue(u);
  double xr, dr, xn_, dn_;
  wait_unit(u0);
  put_t(u0, xn_, dn_);  // t of plane kb - 1
  wait_unit(u0 + 1);
  put_t(u0 + 1, xr, dr);  // t, x, d of plane kb
  __syncthreads();
  if (tid == 0 && u0 + kT3D <= ke - 1) issue(u0 + kT3D);

  const double* const tbase = tr + own_p;
  double acc = 0.0;
  for (int k = kb; k < ke; ++k) {
    wait_unit(k);
    put_t(k, xn_, dn_);  // plane k + 1
    __syncthreads();
    // the stage of unit k-1 was last read before this barrier
    if (tid == 0 && k - 1 + kT3D <= ke - 1) issue(k - 1 + kT3D);
    if (own) {
      const double* s = st0 + ((k - u0) % kT3D) * kT3Stage;
      const unsigned msk = reinterpret_cast<const unsigned*>(s + kT3OffM)[tid];
      const double* pm = tbase + ((k + 3) & 3) * kT3Patch;  // planes k-1, k, k+1
      const double* p0 = tbase + (k & 3) * kT3Patch;
      const double* pp = tbase + ((k + 1) & 3) * kT3Patch;
      double sum = 0.0;
#pragma unroll
      for (int q = 0; q < kT3K; ++q) {
        using Pat = DiaPat<27>;
        const double* pl = Pat::dz(q) < 0 ? pm : (Pat::dz(q) == 0 ? p0 : pp);
        if ((msk >> q) & 1u) sum = sum + s[kT3OffV + q * kT3Tile + tid] * pl[Pat::dy(q) * kT3PX + Pat::dx(q)];
      }
      const double y = sum * dr;
      const long long row = (long long)k * nxy + (long long)j * nx + i;
      if constexpr (kDir) {
        PCGX_DCHECK(row >= 0);
        epi.q[row] = y;
        epi.pout[row] = xr;
        if (kRed) acc = acc + xr * y;  // EpiStoreP: p . q
      } else if constexpr (kFirst) {
        const double xnew = epi.f(y, xr);
        epi.xout[row] = xnew;
        if (kRed) acc = acc + xr * xnew;  // EpiChebFirst: r . x_1 (m == 1)
      } else {
        const double ri = s[kT3OffR + tid];
        const double xo = need_xo ? s[kT3OffO + tid] : 0.0;
        const double xnew = epi.f(y, xr, ri, xo);
        epi.out[row] = xnew;
        if (kRed) acc = acc + ri * xnew;
      }
    }
    xr = xn_;
    dr = dn_;
  }
  if (kRed) block_reduce_finish(acc, red);
}

}  // namespace pcgx
