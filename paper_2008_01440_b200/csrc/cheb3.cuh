// SPDX-License-Identifier: Apache-2.0
//
// THREE Chebyshev degree steps per HBM pass (temporal blocking):
//
//   stage 1: C = x_k     = rho_k     ((2s) A - rho_{k-1} B + (2/d)(R - S A))
//   stage 2: E = x_{k+1} = rho_{k+1} ((2s) C - rho_k     A + (2/d)(R - S C))
//   stage 3: F = x_{k+2} = rho_{k+2} ((2s) E - rho_{k+1} C + (2/d)(R - S E))
//
// with A = x_{k-1}, B = x_{k-2}, R = r and S the scaled 7-point operator
// (polyprec.cpp:190-195). The pass reads A, B, R and writes only the two iterates
// the next pass needs, E and F: 40 B per unknown per THREE steps (13.3 per step;
// the two-step pass of cheb2f.cuh moves 40 per two). C never leaves the SM. In a
// last pass (outE == nullptr) E is not written either: 32 B per unknown.
//
// Layout: one CTA owns a 64 x kTY (i x j) output tile and marches a z-chunk; kTY +
// 4 warps, warp w owns extended row j0 - 2 + w and lane l the point pair i0 + 2l,
// i0 + 2l + 1 of every stage on that row. Iteration t computes stage 1 of plane t
// on rows j0-2 .. j0+kTY+1, stage 2 of plane t-2 on rows j0-1 .. j0+kTY and stage
// 3 of plane t-4 on the tile rows; the three are independent inside an iteration
// (each reads only planes finished before the previous block barrier), so every
// lane carries up to six independent stencil + recurrence chains per barrier.
// The i-halo columns: stage 1 needs the pairs (i0-2, i0-1) and (i0+64, i0+65) on
// every extended row -- warps 0 and kTY+3 (stage 1 only) take them, one row per
// lane; stage 2 needs the points i0-1 and i0+64 -- warps 1 and kTY+2 (no stage 3)
// take them. Operands by TMA (zero-filled outside the domain: the Dirichlet
// boundary, whose -(d*0) terms leave every sum bit-identical): A as a 72 x (kTY+6)
// box (3-deep halo; origin i0-4, even as fp64 boxes must be), B and R as 68 x
// (kTY+4) boxes, D planes ahead through an mbarrier ring. Own-pair values travel
// in per-lane register queues along z (A: t+1..t-2, C: t..t-3, E: t-2..t-5);
// the in-plane neighbours, C[t-4], R and the halo positions are read from the
// shared rings. Per-point arithmetic is the single-step kernel's, in the
// reference's order: bitwise the reference's apply_chebyshev at every step.
#pragma once

#include <type_traits>

#include "cheb2f.cuh"

namespace pcgx {

// Default 64 x 12 tiles: 16 warps, so 128 registers per thread hold the six z
// queues without spills; rings three planes deep.
#ifndef PCGX_C3TY
#define PCGX_C3TY 12
#endif
#ifndef PCGX_C3D
#define PCGX_C3D 3
#endif
#ifndef PCGX_C3UNROLL
#define PCGX_C3UNROLL 4
#endif
#ifndef PCGX_C3MAXREG
#define PCGX_C3MAXREG 128
#endif
constexpr int k3TY = PCGX_C3TY;
constexpr int k3D = PCGX_C3D;
constexpr int k3Unroll = PCGX_C3UNROLL;
constexpr int k3W = kC2TX + 4;   // 68: B/R/C/E plane rows, tile-i t <-> column t + 2
constexpr int k3AW = kC2TX + 8;  // 72: A box rows, tile-i t <-> column t + 4
constexpr int k3R = k3TY + 4;    // B/R/C/E plane rows (tile-j t <-> row t + 2)
constexpr int k3AR = k3TY + 6;   // A box rows (tile-j t <-> row t + 3)
constexpr int k3APlane = (k3AW * k3AR + 15) / 16 * 16;  // 128-byte multiples (TMA destinations)
constexpr int k3Plane = (k3W * k3R + 15) / 16 * 16;
constexpr int k3Warps = k3TY + 4, k3Threads = 32 * k3Warps;
constexpr int k3NA = k3D + 3, k3NB = k3D, k3NR = k3D + 4, k3NC = 5, k3NE = 3;
// + a guard of 2 rows after the E ring: the stage-2/3 loads of the warps that do
// not need them (rows -1 and kTY+4 of a slot) must stay inside the allocation
constexpr int k3Guard = 2 * k3W;
constexpr size_t k3Smem =
    sizeof(double) * (size_t)(k3NA * k3APlane + (k3NB + k3NR + k3NC + k3NE) * k3Plane + k3Guard) +
    16 * (k3D + 1) + 128;
static_assert(k3Smem <= 232448, "three-step pass: shared memory over the sm_100a limit");
static_assert(k3TY + 4 <= 32, "halo lanes: one extended row per lane");

struct Cheb3Params {
  int nx, ny, nzl;
  int a_lo, a_hi, c_lo, c_hi, zoff;  // as Cheb2Params (single slab: 0, nzl, 0, nzl, 0)
  long long nxy;
  double d;
  double rk1, rk1m1, rk2, rk2m1, rk3, rk3m1;  // rho_k, rho_{k-1}, rho_{k+1}, rho_k, rho_{k+2}, rho_{k+1}
  double c2, c3;                              // 2/delta, 2 sigma
  double* outE;                               // x_{k+1} (nullptr: not needed, last pass)
  double* outF;                               // x_{k+2}
};

__device__ __forceinline__ double2 ld2s(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void st2s(double* p, double2 v) { *reinterpret_cast<double2*>(p) = v; }

// one recurrence step x_new = rk ((c3 x) - (rkm1 x_old) + c2 (r - y)) (polyprec.cpp:192-194)
__device__ __forceinline__ double cheb_rec(double rk, double rkm1, double c2, double c3, double x, double xo,
                                           double r, double y) {
  return rk * (((c3 * x) - (rkm1 * xo)) + c2 * (r - y));
}

template <bool kRed>
__global__ void __maxnreg__(PCGX_C3MAXREG)
stencil7_cheb3_kernel(const __grid_constant__ CUtensorMap mapA,  // A, box 72 x (kTY+6)
                      const __grid_constant__ CUtensorMap mapB,  // B, box 68 x (kTY+4)
                      const __grid_constant__ CUtensorMap mapR,  // R, box 68 x (kTY+4)
                      Cheb3Params p, int k_begin, int k_end, const __grid_constant__ ChunkPlan plan,
                      Reduce red) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sA = reinterpret_cast<double*>(smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u));
  double* sB = sA + k3NA * k3APlane;
  double* sR = sB + k3NB * k3Plane;
  double* sC = sR + k3NR * k3Plane;
  double* sE = sC + k3NC * k3Plane;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sE + k3NE * k3Plane + k3Guard);  // k3D unit bars + 1 prologue

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned bytesA = k3AW * k3AR * 8, bytesB = k3W * k3R * 8;
  const int tiles_x = (p.nx + kC2TX - 1) / kC2TX;
  const int i0 = (int)(blockIdx.x % tiles_x) * kC2TX, j0 = (int)(blockIdx.x / tiles_x) * k3TY;
  const int kb = k_begin + plan.start[blockIdx.y];
  const int ke = min(k_begin + plan.start[blockIdx.y + 1], k_end);
  if (tid == 0) {
    for (int q = 0; q <= k3D; ++q) mbar_init(&bars[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // plane slots: A (z - (kb-3)) % NA, B / R (z - (kb-2)) % N; unit u = {A[u+1], B[u], R[u]}
  auto in_z = [&](int z) { return z >= p.a_lo && z < p.a_hi; };
  const int zo = p.zoff;
  auto issue_unit = [&](int u) {
    uint64_t* bar = &bars[(u - (kb - 2)) % k3D];
    const bool la = in_z(u + 1), lbr = in_z(u);
    mbar_expect_tx(bar, (la ? bytesA : 0u) + (lbr ? 2 * bytesB : 0u));
    if (la) tma_load_3d(sA + ((u + 1 - (kb - 3)) % k3NA) * k3APlane, &mapA, i0 - 4, j0 - 3, u + 1 + zo, bar);
    if (lbr) {
      tma_load_3d(sB + ((u - (kb - 2)) % k3NB) * k3Plane, &mapB, i0 - 2, j0 - 2, u + zo, bar);
      tma_load_3d(sR + ((u - (kb - 2)) % k3NR) * k3Plane, &mapR, i0 - 2, j0 - 2, u + zo, bar);
    }
  };
  // stage 1 runs t = kb-2 .. ke+1, stage 2 (v = t-2) kb+1 .. ke+2, stage 3 (w = t-4) kb+4 .. ke+3
  const int u_last = ke + 1;
  if (tid == 0) {
    uint64_t* pb = &bars[k3D];
    mbar_expect_tx(pb, (in_z(kb - 3) ? bytesA : 0u) + (in_z(kb - 2) ? bytesA : 0u));
    if (in_z(kb - 3)) tma_load_3d(sA, &mapA, i0 - 4, j0 - 3, kb - 3 + zo, pb);
    if (in_z(kb - 2)) tma_load_3d(sA + k3APlane, &mapA, i0 - 4, j0 - 3, kb - 2 + zo, pb);
    for (int u = kb - 2; u < kb - 2 + k3D && u <= u_last; ++u) issue_unit(u);
  }
  mbar_wait(&bars[k3D], 0);

  const double d = p.d;
  const double2 zero2 = make_double2(0.0, 0.0);
  // own pair
  const int gi = i0 + 2 * lane;
  const bool pair_in = gi < p.nx;
  const int gj = j0 - 2 + warp;
  const bool own_in = pair_in && gj >= 0 && gj < p.ny;
  const int offA = (warp + 1) * k3AW + 2 * lane + 4;
  const int offB = warp * k3W + 2 * lane + 2;
  // stage-1 halo pairs: warp 0 the left (i0-2, i0-1), warp kTY+3 the right (i0+64, i0+65), row `lane`
  const int h1gi = warp == 0 ? i0 - 2 : i0 + kC2TX, h1gj = j0 - 2 + lane;
  const bool h1_in = h1gi >= 0 && h1gi < p.nx && h1gj >= 0 && h1gj < p.ny;
  // stage-2 halo points: warp 1 the left (i0-1), warp kTY+2 the right (i0+64), row `lane` + 1
  const int h2gi = warp == 1 ? i0 - 1 : i0 + kC2TX, h2gj = j0 - 1 + lane;
  const bool h2_in = h2gi >= 0 && h2gi < p.nx && h2gj >= 0 && h2gj < p.ny;

  PCGX_DCHECK(offA - k3AW - 1 >= 0 && offA + k3AW + 2 <= k3AW * k3AR);
  PCGX_DCHECK(offB - k3W - 1 >= -k3W && offB + k3W + 2 <= k3Plane + k3W);  // +-1 row: rings / guard
  [[maybe_unused]] const long long g_hi = (long long)p.nzl * p.nxy;  // PCGX_DCHECK bound
  const double* const sAend = sA + k3NA * k3APlane;
  const double* const sBend = sB + k3NB * k3Plane;
  const double* const sRend = sR + k3NR * k3Plane;
  auto nextA = [&](const double* q) { return q + k3APlane == sAend ? sA : q + k3APlane; };
  auto nextB = [&](const double* q) { return q + k3Plane == sBend ? sB : q + k3Plane; };
  auto nextR = [&](const double* q) { return q + k3Plane == sRend ? sR : q + k3Plane; };
  const long long gown = (long long)gj * p.nx + gi;
  double acc = 0.0;

  // The plane march, specialised per warp class (a warp-uniform dispatch below):
  //   kCls 3 (the tile rows): stages 1, 2, 3 of the own pair;
  //   kCls 2 (warps 1, kTY+2): stages 1, 2 + the stage-2 i-halo point of row `lane`;
  //   kCls 1 (warps 0, kTY+3): stage 1 + the stage-1 i-halo pair of row `lane`.
  // Every class's work is one basic block per plane: all operands are loaded from
  // valid ring slots first (a stale slot only feeds a result the selects discard),
  // then the independent stencil + recurrence chains, then the stores -- so the
  // compiler interleaves the chains -- and the classes carry similar work to the
  // one block barrier per plane.
  auto march = [&](auto cls) {
    constexpr int kCls = decltype(cls)::value;
    // ring slots of the planes iteration t touches (t = kb-2 here): A t-2 .. t+1
    // (slot of z: (z - (kb-3)) % NA), B t, R t, t-2, t-4 ((z - (kb-2)) % N), C t .. t-4,
    // E t-2 .. t-4 (both any consistent rotation)
    const double* pA2 = sA + (k3NA - 1) * k3APlane;
    const double* pAm = sA;
    const double* pAu = sA + k3APlane;
    const double* pAp = sA + 2 * k3APlane;
    const double* pBu = sB;
    const double* pRu = sR;
    const double* pR2 = sR + (k3NR - 2) * k3Plane;
    const double* pR4 = sR + (k3NR - 4) * k3Plane;
    double* pC0 = sC;
    double* pC1 = sC + 4 * k3Plane;
    double* pC2 = sC + 3 * k3Plane;
    double* pC3 = sC + 2 * k3Plane;
    double* pC4 = sC + 1 * k3Plane;
    double* pE0 = sE;
    double* pE1 = sE + 2 * k3Plane;
    double* pE2 = sE + k3Plane;
    int bslot = 0;
    unsigned bphase = 0;
    double* gE = p.outE ? p.outE + gown + (long long)(kb - 4) * p.nxy : nullptr;  // E pair at plane t-2
    double* gF = p.outF + gown + (long long)(kb - 6) * p.nxy;                    // F pair at plane t-4
    // Own-pair z queues, each a 4-register rotation (the loop is unrolled by 4, so
    // the rotations are renamings, not moves): A[t+1] .. A[t-2], C[t] .. C[t-3],
    // E[t-2] .. E[t-5]. C[t-4] and R come from their shared rings.
    double2 am = in_z(kb - 3) ? ld2s(sA + offA) : zero2;
    double2 ac = in_z(kb - 2) ? ld2s(sA + k3APlane + offA) : zero2;
    double2 a2 = zero2;
    double2 cm1 = zero2, cm2 = zero2, cm3 = zero2;  // C[t-1] .. C[t-3]
    double2 em3 = zero2, em4 = zero2, em5 = zero2;  // E[t-3] .. E[t-5]
    // halo positions (valid ring offsets for every lane; only the live ones are stored)
    const int hrow1 = lane < k3R ? lane : 0;
    const int offA_h = (hrow1 + 1) * k3AW + (warp == 0 ? 2 : kC2TX + 4);
    const int offB_h = hrow1 * k3W + (warp == 0 ? 0 : kC2TX + 2);
    const bool h_live1 = kCls == 1 && lane < k3R;
    const int hrow2 = lane < k3TY + 2 ? lane + 1 : 1;
    const int offB_p = hrow2 * k3W + (warp == 1 ? 1 : kC2TX + 2);
    const int offA_p = (hrow2 + 1) * k3AW + (warp == 1 ? 3 : kC2TX + 4);
    const bool h_live2 = kCls == 2 && lane < k3TY + 2;

#pragma unroll k3Unroll
    for (int t = kb - 2; t <= ke + 3; ++t) {
      if (tid == 0 && t >= kb - 1 && t - 1 + k3D <= u_last) issue_unit(t - 1 + k3D);
      const bool s1 = t <= ke + 1;
      const bool s2 = t >= kb + 1 && t <= ke + 2;
      const bool s3 = t >= kb + 4;
      if (s1) mbar_wait(&bars[bslot], bphase);
      const bool p1 = s1 && t >= p.c_lo && t < p.c_hi, has_p = in_z(t + 1);
      const bool p2 = s2 && t - 2 >= p.c_lo && t - 2 < p.c_hi;
      // ---- loads
      const double2 apl = ld2s(pAp + offA);
      const double2 ap = has_p ? apl : zero2;
      const double aw = pAu[offA - 1], ae = pAu[offA + 2];
      const double2 as = ld2s(pAu + offA - k3AW), an = ld2s(pAu + offA + k3AW);
      const double2 bb = ld2s(pBu + offB), rr = ld2s(pRu + offB);
      double cw = 0, ce = 0, ew = 0, ee = 0;
      double2 cs = zero2, cn = zero2, rv = zero2, es = zero2, en = zero2, r4 = zero2, c4 = zero2;
      if constexpr (kCls >= 2) {
        cw = pC2[offB - 1];
        ce = pC2[offB + 2];
        cs = ld2s(pC2 + offB - k3W);
        cn = ld2s(pC2 + offB + k3W);
        rv = ld2s(pR2 + offB);
      }
      if constexpr (kCls == 3) {
        ew = pE2[offB - 1];
        ee = pE2[offB + 2];
        es = ld2s(pE2 + offB - k3W);
        en = ld2s(pE2 + offB + k3W);
        r4 = ld2s(pR4 + offB);
        c4 = ld2s(pC4 + offB);
      }
      // stage-1 halo pair (kCls 1)
      double2 hm = zero2, hp = zero2, hc = zero2, hs = zero2, hn = zero2, hb = zero2, hr = zero2;
      double hw = 0, he = 0;
      if constexpr (kCls == 1) {
        const double2 hml = ld2s(pAm + offA_h), hpl = ld2s(pAp + offA_h);
        hm = in_z(t - 1) ? hml : zero2;
        hp = has_p ? hpl : zero2;
        hc = ld2s(pAu + offA_h);
        hs = ld2s(pAu + offA_h - k3AW);
        hn = ld2s(pAu + offA_h + k3AW);
        hw = pAu[offA_h - 1];
        he = pAu[offA_h + 2];
        hb = ld2s(pBu + offB_h);
        hr = ld2s(pRu + offB_h);
      }
      // stage-2 halo point (kCls 2)
      double qm = 0, qs = 0, qw = 0, qc = 0, qe = 0, qn = 0, qp = 0, qx = 0, qr = 0;
      if constexpr (kCls == 2) {
        qm = pC3[offB_p];
        qs = pC2[offB_p - k3W];
        qw = pC2[offB_p - 1];
        qc = pC2[offB_p];
        qe = pC2[offB_p + 1];
        qn = pC2[offB_p + k3W];
        qp = pC1[offB_p];
        qx = pA2[offA_p];
        qr = pR2[offB_p];
      }
      // ---- arithmetic: stage 1 on the extended rows
      const double y10 = stencil_point(d, am.x, as.x, aw, ac.x, ac.y, an.x, ap.x);
      const double y11 = stencil_point(d, am.y, as.y, ac.x, ac.y, ae, an.y, ap.y);
      const double c0 = cheb_rec(p.rk1, p.rk1m1, p.c2, p.c3, ac.x, bb.x, rr.x, y10);
      const double c1 = cheb_rec(p.rk1, p.rk1m1, p.c2, p.c3, ac.y, bb.y, rr.y, y11);
      const bool l1 = p1 && own_in;
      const double2 cv = make_double2(l1 ? c0 : 0.0, l1 ? c1 : 0.0);
      double2 ev = zero2, hv = zero2;
      double f0 = 0, f1 = 0, qv = 0;
      if constexpr (kCls >= 2) {  // stage 2 on rows j0-1 .. j0+kTY
        const double y20 = stencil_point(d, cm3.x, cs.x, cw, cm2.x, cm2.y, cn.x, cm1.x);
        const double y21 = stencil_point(d, cm3.y, cs.y, cm2.x, cm2.y, ce, cn.y, cm1.y);
        const double e0 = cheb_rec(p.rk2, p.rk2m1, p.c2, p.c3, cm2.x, a2.x, rv.x, y20);
        const double e1 = cheb_rec(p.rk2, p.rk2m1, p.c2, p.c3, cm2.y, a2.y, rv.y, y21);
        const bool l2 = p2 && own_in;
        ev = make_double2(l2 ? e0 : 0.0, l2 ? e1 : 0.0);
      }
      if constexpr (kCls == 3) {  // stage 3 on the tile rows
        const double y30 = stencil_point(d, em5.x, es.x, ew, em4.x, em4.y, en.x, em3.x);
        const double y31 = stencil_point(d, em5.y, es.y, em4.x, em4.y, ee, en.y, em3.y);
        f0 = cheb_rec(p.rk3, p.rk3m1, p.c2, p.c3, em4.x, c4.x, r4.x, y30);
        f1 = cheb_rec(p.rk3, p.rk3m1, p.c2, p.c3, em4.y, c4.y, r4.y, y31);
      }
      if constexpr (kCls == 1) {
        const double z0 = stencil_point(d, hm.x, hs.x, hw, hc.x, hc.y, hn.x, hp.x);
        const double z1 = stencil_point(d, hm.y, hs.y, hc.x, hc.y, he, hn.y, hp.y);
        const double v0 = cheb_rec(p.rk1, p.rk1m1, p.c2, p.c3, hc.x, hb.x, hr.x, z0);
        const double v1 = cheb_rec(p.rk1, p.rk1m1, p.c2, p.c3, hc.y, hb.y, hr.y, z1);
        const bool lh = p1 && h1_in;
        hv = make_double2(lh ? v0 : 0.0, lh ? v1 : 0.0);
      }
      if constexpr (kCls == 2) {
        const double y = stencil_point(d, qm, qs, qw, qc, qe, qn, qp);
        const double v = cheb_rec(p.rk2, p.rk2m1, p.c2, p.c3, qc, qx, qr, y);
        qv = (p2 && h2_in) ? v : 0.0;
      }
      // ---- stores
      if (s1) st2s(pC0 + offB, cv);
      if constexpr (kCls == 1) {
        if (s1 && h_live1) st2s(pC0 + offB_h, hv);
      }
      if constexpr (kCls >= 2) {
        if (s2) {
          st2s(pE0 + offB, ev);
          if (kCls == 3 && gE && own_in && t - 2 >= kb && t - 2 < ke) {
            PCGX_DCHECK(gE - p.outE >= 0 && gE - p.outE + 2 <= g_hi);
            st2(gE, ev.x, ev.y);
          }
        }
      }
      if constexpr (kCls == 2) {
        if (s2 && h_live2) pE0[offB_p] = qv;
      }
      if constexpr (kCls == 3) {
        if (s3 && own_in) {
          PCGX_DCHECK(gF - p.outF >= 0 && gF - p.outF + 2 <= g_hi);
          st2(gF, f0, f1);
          if (kRed) acc = acc + (r4.x * f0 + r4.y * f1);
        }
      }
      __syncthreads();
      // rotate the register queues, the rings and the global pointers by one plane
      a2 = am;
      am = ac;
      ac = ap;
      cm3 = cm2;
      cm2 = cm1;
      cm1 = cv;
      em5 = em4;
      em4 = em3;
      em3 = ev;
      pA2 = pAm;
      pAm = pAu;
      pAu = pAp;
      pAp = nextA(pAp);
      pBu = nextB(pBu);
      pRu = nextR(pRu);
      pR2 = nextR(pR2);
      pR4 = nextR(pR4);
      double* const c4s = pC4;
      pC4 = pC3;
      pC3 = pC2;
      pC2 = pC1;
      pC1 = pC0;
      pC0 = c4s;
      double* const e2s = pE2;
      pE2 = pE1;
      pE1 = pE0;
      pE0 = e2s;
      if (++bslot == k3D) {
        bslot = 0;
        bphase ^= 1u;
      }
      if (gE) gE += p.nxy;
      gF += p.nxy;
    }
  };
  if (warp >= 2 && warp <= k3TY + 1) march(std::integral_constant<int, 3>{});
  else if (warp == 1 || warp == k3TY + 2) march(std::integral_constant<int, 2>{});
  else march(std::integral_constant<int, 1>{});
  if (kRed) block_reduce_finish(acc, red);
}

}  // namespace pcgx
