// SPDX-License-Identifier: Apache-2.0
//
// Software-pipelined variant of the two-step Chebyshev pass (cheb2.cuh): the
// same two fused degree steps per HBM pass, the same tile, TMA boxes and
// per-point arithmetic (bitwise identical outputs), but iteration t of the plane
// loop computes stage 1 of plane t AND stage 2 of plane t-2 between the same pair
// of block barriers. The two stages are independent there (stage 2 of t-2 reads
// C[t-3..t-1], all complete at the previous barrier), so each lane carries four
// independent stencil + recurrence dependency chains instead of two: ncu showed
// the two-step kernel stalled mostly on fixed-latency fp64 dependencies ("wait")
// and barriers, not on HBM.
//
// Stage 2 is computed by the warp that produced the row in stage 1 ("own row":
// warps 1..8; warps 0 and 9 own the j-halo rows and compute the two i-halo
// columns of C), so the C centres of planes t-3, t-2, t-1 are registers; only
// C's j +- 1 rows and the lane-0/31 i-neighbours come from the C ring.
//
// Rings (D = prefetch distance in planes, load unit u = A[u+1], B[u], R[u]):
// A holds planes t-1 .. t+D (D+2 slots; A[t-2] of stage 2 is a register), B
// t .. t+D-1 (D), R t-2 .. t+D-1 (D+2), C t-2 .. t (3). The refill of unit
// t-1+D is issued at the top of iteration t: the slots it overwrites (A[t-2],
// B[t-1], R[t-3]) were last read in iteration t-1, before its closing barrier.
#pragma once

#include "cheb2.cuh"

namespace pcgx {

// Power / ceiling experiment only (tools/build_variant.py nomath -DPCGX_C2F_NOMATH=1;
// NOT bitwise, never the product): the stencil sums replaced by an integer XOR of
// the same seven operands, so the pass keeps every TMA box, shared load and store
// but drops ~15 of its ~22 fp64 operations per point-step.
#ifndef PCGX_C2F_NOMATH
#define PCGX_C2F_NOMATH 0
#endif
// Power-ceiling experiments (tools/build_variant.py, never the product, NOT bitwise):
// 1: no j-neighbour shared loads; 2: no i-neighbour loads either; 3: + no i-halo
// columns; 4: + no stencil arithmetic (the pass keeps its TMA boxes, one shared
// load per operand, the recurrence and the stores); 5: + the recurrence replaced by
// three additions; 6: + no C ring stores; 7: + no shared loads at all (TMA boxes in,
// constant stores out)
#ifndef PCGX_C2F_EXP
#define PCGX_C2F_EXP 0
#endif
__device__ __forceinline__ double c2f_stencil(double d, double a, double b, double c, double e, double f,
                                              double g, double h) {
#if PCGX_C2F_EXP >= 4
  return d * e + (a * 0.0 + b * 0.0 + c * 0.0 + f * 0.0 + g * 0.0 + h * 0.0) * 0.0 == 0.0 ? d * e : e;
#elif PCGX_C2F_NOMATH
  (void)d;
  const long long x = __double_as_longlong(a) ^ __double_as_longlong(b) ^ __double_as_longlong(c) ^
                      __double_as_longlong(e) ^ __double_as_longlong(f) ^ __double_as_longlong(g) ^
                      __double_as_longlong(h);
  return __longlong_as_double(x & 0x3fffffffffffffffll);
#else
  return stencil_point(d, a, b, c, e, f, g, h);
#endif
}

// Tile 64 x kFTY, kFTY + 2 warps. Default: 64 x 20 (22 warps, ONE CTA per SM,
// 80 registers), rings four planes deep (206 KB), R of stage 2 in registers.
// Measured at 320^3 against the alternatives (tools/kbench_cheb2.py, one box):
// 64 x 8 with 3 CTAs/SM and D = 2: +5%; 64 x 12, 2 CTAs/SM, D = 3: +1%;
// 64 x 20 with D = 3: +4%; 64 x 16, D = 5: +6%; 64 x 24, D = 3: +4%. Fewer
// redundant stage-1 rows (22 per 20 output rows) and a deep prefetch both pay.
#ifndef PCGX_C2FTY
#define PCGX_C2FTY 20
#endif
#ifndef PCGX_C2FD
#define PCGX_C2FD 4
#endif
#ifndef PCGX_C2FMINB
#define PCGX_C2FMINB 1
#endif
// register cap with one CTA per SM: 22 warps put 6 on one SM sub-partition (16K
// registers each), so 64 x 20 tiles allow 80
// kUpd: r(it) = r(it-1) - alpha q(it) formed ONCE per element, in place in the A
// slot, when the plane arrives (own pairs by their warps, the box's outer rows and
// columns by the two halo warps); every later read is a plain load
// (i-neighbours of every lane come straight from shared memory, two 8-byte LDS per
// stage; R of stage 2 travels in a register queue. The shuffle / edge-select and
// R-ring alternatives measured slower or equal in round 1 and were removed.)
#ifndef PCGX_C2FMAXREG
#define PCGX_C2FMAXREG 80
#endif
constexpr int kFTY = PCGX_C2FTY;
constexpr int kFW = kC2W;                            // 68: tile-i t <-> smem column t+2
constexpr int kFAY = kFTY + 4, kFBY = kFTY + 2;      // A box rows (2-halo), B/R/C rows (1-halo)
constexpr int kFAPlane = (kFW * kFAY + 15) / 16 * 16;  // A slot stride (128-byte TMA destinations)
constexpr int kFBPlane = kFW * kFBY;
constexpr int kFEStride = (kFBPlane + 15) / 16 * 16;  // TMA destinations: 128-byte multiples
constexpr int kFCStride = kFBPlane;
constexpr int kFWarps = kFTY + 2, kFThreads = 32 * kFWarps;
constexpr int kFD = PCGX_C2FD;
constexpr int kFNA = kFD + 2, kFNB = kFD, kFNR = kFD, kFNC = 3;
constexpr size_t kC2FSmem = sizeof(double) * (size_t)(kFNA * kFAPlane + (kFNB + kFNR) * kFEStride +
                                                      kFNC * kFCStride) +
                            16 * (kFD + 1) + 128;

// z-chunking of a launch: chunk c covers planes [k_begin + start[c], k_begin + start[c+1]).
// Chunks are dispatched chunk-major (all tiles of chunk 0 first), so the CTAs in
// flight are neighbouring tiles at similar z and their halo re-reads hit L2;
// the host shrinks the last chunks so the final wave ends evenly.
struct ChunkPlan {
  static constexpr int kMax = 48;
  int n;
  int start[kMax + 1];
  // chunks whose bit is set are not computed (their CTAs only join the reductions): a
  // slab rank's two boundary strips as ONE launch with the interior chunk masked
  unsigned long long skip;
};

template <bool kFirst, bool kRed, bool kUpd = false>
#if PCGX_C2FMINB == 1
__global__ void __maxnreg__(PCGX_C2FMAXREG)
#else
__global__ void __launch_bounds__(kFThreads, PCGX_C2FMINB)
#endif
stencil7_cheb2f_kernel(const __grid_constant__ CUtensorMap mapA,  // A (68 x (kFTY+4) box)
                       const __grid_constant__ CUtensorMap mapB,  // B (68 x (kFTY+2) box); kUpd: Q (A's box)
                       const __grid_constant__ CUtensorMap mapR,  // R (68 x (kFTY+2) box)
                       Cheb2Params p, int k_begin, int k_end, const __grid_constant__ ChunkPlan plan, Reduce red,
                       Reduce red_rr) {
  static_assert(!kUpd || (kFirst && !kRed), "the PCG update is fused into a non-reducing first pass only");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sA = reinterpret_cast<double*>(smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u));
  double* sB = sA + kFNA * kFAPlane;
  double* sR = sB + kFNB * kFEStride;
  double* sC = sR + kFNR * kFEStride;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sC + kFNC * kFCStride);  // kFD unit bars + 1 prologue
  // kUpd: the q ring (A's slots and box) lives where the first pass has no B / R
  static_assert(kFNA * kFAPlane <= (kFNB + kFNR) * kFEStride, "q ring does not fit the B / R rings");
  double* sQ = sB;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned bytesA = kFW * kFAY * 8, bytesB = kFBPlane * 8;  // box bytes (slots may be padded)
  const int tiles_x = (p.nx + kC2TX - 1) / kC2TX;
  const int i0 = (int)(blockIdx.x % tiles_x) * kC2TX, j0 = (int)(blockIdx.x / tiles_x) * kFTY;
  const int kb = k_begin + plan.start[blockIdx.y];
  const int ke = min(k_begin + plan.start[blockIdx.y + 1], k_end);
  if ((plan.skip >> blockIdx.y) & 1ull) {  // block-uniform; a masked chunk still joins the reductions
    if (kRed) block_reduce_finish(0.0, red);
    if (kUpd) block_reduce_finish(0.0, red_rr);
    return;
  }
  if (tid == 0) {
    for (int q = 0; q <= kFD; ++q) mbar_init(&bars[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // slot of plane z: A (z - (kb-2)) % NA, B and R (z - (kb-1)) % N, C (z - (kb-1)) % 3
  auto in_z = [&](int z) { return z >= p.a_lo && z < p.a_hi; };
  const int zo = p.zoff;
  auto issue_unit = [&](int u) {
    uint64_t* bar = &bars[(u - (kb - 1)) % kFD];
    const bool la = in_z(u + 1), lbr = !kFirst && in_z(u);
    mbar_expect_tx(bar, (la ? (kUpd ? 2 : 1) * bytesA : 0u) + (lbr ? 2 * bytesB : 0u));
    if (la) tma_load_3d(sA + ((u + 1 - (kb - 2)) % kFNA) * kFAPlane, &mapA, i0 - 2, j0 - 2, u + 1 + zo, bar);
    if (kUpd && la)
      tma_load_3d(sQ + ((u + 1 - (kb - 2)) % kFNA) * kFAPlane, &mapB, i0 - 2, j0 - 2, u + 1 + zo, bar);
    if (lbr) {
      tma_load_3d(sB + ((u - (kb - 1)) % kFNB) * kFEStride, &mapB, i0 - 2, j0 - 1, u + zo, bar);
      tma_load_3d(sR + ((u - (kb - 1)) % kFNR) * kFEStride, &mapR, i0 - 2, j0 - 1, u + zo, bar);
    }
  };
  const int u_last = ke;  // stage 1 runs t = kb-1 .. ke, stage 2 v = t-2 = kb .. ke-1
  if (tid == 0) {
    uint64_t* pb = &bars[kFD];
    const unsigned ba = (kUpd ? 2 : 1) * bytesA;
    mbar_expect_tx(pb, (in_z(kb - 2) ? ba : 0u) + (in_z(kb - 1) ? ba : 0u));
    if (in_z(kb - 2)) tma_load_3d(sA, &mapA, i0 - 2, j0 - 2, kb - 2 + zo, pb);
    if (in_z(kb - 1)) tma_load_3d(sA + kFAPlane, &mapA, i0 - 2, j0 - 2, kb - 1 + zo, pb);
    if (kUpd && in_z(kb - 2)) tma_load_3d(sQ, &mapB, i0 - 2, j0 - 2, kb - 2 + zo, pb);
    if (kUpd && in_z(kb - 1)) tma_load_3d(sQ + kFAPlane, &mapB, i0 - 2, j0 - 2, kb - 1 + zo, pb);
    for (int u = kb - 1; u < kb - 1 + kFD && u <= u_last; ++u) issue_unit(u);
  }
  mbar_wait(&bars[kFD], 0);

  // kUpd: every A value (r(it-1)) is read together with q(it) at the same offset of
  // the q ring and combined on the fly into r(it) = r(it-1) - alpha q(it), the update
  // kernel's element operation (pcg.cpp:83); the own row's new plane goes to rout
  // and into r'r (each interior point once, when its plane enters the queue).
  double acc_rr = 0.0;
  const double alpha = kUpd ? p.S[p.s_rho] / p.S[p.s_pq] : 0.0;
  const double* const sA0 = sA;
  auto rq2 = [&](const double* a, int off) {
    const double2 v = *reinterpret_cast<const double2*>(a + off);
    if (!kUpd) return v;
    const double2 w = *reinterpret_cast<const double2*>(sQ + (a - sA0) + off);
    return make_double2(v.x - alpha * w.x, v.y - alpha * w.y);
  };
  constexpr bool kIP = kUpd;
  // reads of planes already combined in place (kUpd) or plain (otherwise)
  auto rqx = [&](const double* a, int off) { return a[off]; };
  auto rqx2 = [&](const double* a, int off) { return *reinterpret_cast<const double2*>(a + off); };
  // kIP: element e of an A slot combined in place
  auto combine_slot = [&](double* a, int e) {
    a[e] = a[e] - alpha * sQ[(a - sA0) + e];
  };
  if (kIP) {  // the prologue planes kb-2, kb-1, whole boxes
    // (combining each plane's whole box one iteration ahead, by all threads
    // uniformly, instead of the own pairs + border split below: 291 -> 312 us)
    for (int e = tid; e < kFW * kFAY; e += kFThreads) {
      if (in_z(kb - 2)) combine_slot(sA, e);
      if (in_z(kb - 1)) combine_slot(sA + kFAPlane, e);
    }
    __syncthreads();
  }

  const double d = p.d;
  const double inv_t = 1.0 / p.theta;
  const double2 zero2 = make_double2(0.0, 0.0);
  const int col = 2 * lane + 2;
  const int gi = i0 + 2 * lane;
  const bool pair_in = gi < p.nx;
  const int gj = j0 - 1 + warp;                    // this warp's (extended) row
  const bool do1 = gj >= 0 && gj < p.ny && pair_in;
  const int offA = (warp + 1) * kFW + col;        // A-box offset of the pair
  const int offB = warp * kFW + col;              // B/R/C offset of the pair
  const bool interior = warp >= 1 && warp <= kFTY;  // a tile row: stage 2 here
  const bool do2 = interior && do1;
  double* gC = p.outC + (long long)gj * p.nx + gi;
  double* gE = p.outE + (long long)gj * p.nx + gi;
  // halo columns: warp 0 -> tile-i -1, warp 9 -> tile-i 64; lanes 0..9 = rows
  const bool do_h = (warp == 0 || warp == kFTY + 1) && lane < kFBY;
  const int hcol = warp == 0 ? 1 : kC2TX + 2;
  const int hgi = warp == 0 ? i0 - 1 : i0 + kC2TX;
  const int hgj = j0 - 1 + lane;
  const bool h_in = do_h && hgi >= 0 && hgi < p.nx && hgj >= 0 && hgj < p.ny;
  const int offAh = (lane + 1) * kFW + hcol, offBh = lane * kFW + hcol;
  // every shared offset this thread reads / writes lies inside its slot
  PCGX_DCHECK(offA - kFW - 1 >= 0 && offA + kFW + 2 < kFW * kFAY);
  PCGX_DCHECK(offB - kFW - 1 >= 0 || warp == 0);
  PCGX_DCHECK(offB + 2 <= kFBPlane && (warp == kFTY + 1 || offB + kFW + 2 <= kFBPlane));
  PCGX_DCHECK(!do_h || (offAh - kFW - 1 >= 0 && offAh + kFW + 1 < kFW * kFAY && offBh < kFBPlane));
  [[maybe_unused]] const long long g_lo = -(long long)p.zoff * p.nxy;  // PCGX_DCHECK bounds
  [[maybe_unused]] const long long g_hi = (long long)(p.nzl + p.zoff) * p.nxy;

  const double* const sAend = sA + kFNA * kFAPlane;
  const double* const sBend = sB + kFNB * kFEStride;
  const double* const sRend = sR + kFNR * kFEStride;
  const double* pAm = sA;                           // A[t-1]
  const double* pAu = sA + kFAPlane;               // A[t]
  const double* pAp = sA + 2 * kFAPlane;           // A[t+1]
  const double* pBu = sB;                           // B[t]
  const double* pRu = sR;                           // R[t]
  double2 r1 = zero2, r2 = zero2;                  // R[t-1], R[t-2] (own row)
  double* pCu = sC;                                 // C[t]
  double* pC1 = sC + 2 * kFCStride;                // C[t-1]
  double* pC2 = sC + kFCStride;                    // C[t-2]
  int bslot = 0;
  unsigned bphase = 0;
  double* gCt = gC + (long long)(kb - 1) * p.nxy;   // C pair at plane t
  double* gEv = gE + (long long)(kb - 3) * p.nxy;   // E pair at plane t-2

  double2 am = in_z(kb - 2) ? rqx2(sA, offA) : zero2;
  double2 ac = in_z(kb - 1) ? rqx2(sA + kFAPlane, offA) : zero2;
  double2 a2 = zero2;                          // A[t-2] x (own row)
  double2 c1 = zero2, c2 = zero2, c3 = zero2;  // C[t-1], C[t-2], C[t-3] (own row)
  double acc = 0.0;

#pragma unroll kC2Unroll
  for (int t = kb - 1; t <= ke + 1; ++t) {
    if (tid == 0 && t >= kb && t - 1 + kFD <= u_last) issue_unit(t - 1 + kFD);
    const bool s1 = t <= ke;
    double2 ap = zero2, cv = zero2, rt = zero2;
    if (s1) mbar_wait(&bars[bslot], bphase);
    // ---------------- stage 1: C[t] on the extended tile row
    if (s1) {
      const bool plane_in = t >= p.c_lo && t < p.c_hi, has_p = in_z(t + 1);
      ap = has_p && PCGX_C2F_EXP < 7 ? rq2(pAp, offA) : zero2;
      if (kIP && has_p) {
        // the own pair of plane t+1 in place; the halo warps take the two outer
        // columns on their side of rows 1..kFBY (their halo-column stencil reads them
        // in this iteration), warps 1..5 the outer rows 0 and kFAY-1 (first read in
        // the next iteration, behind the barrier). Measured: 317 -> 290 us per pass
        // at 320^3 against all the border on the halo warps; moving their outer
        // column to other warps as well was 2% slower.
        *reinterpret_cast<double2*>(const_cast<double*>(pAp) + offA) = ap;
        if (warp == 0 || warp == kFTY + 1) {
          for (int e = lane; e < 2 * kFBY; e += 32)
            combine_slot(const_cast<double*>(pAp), (1 + (e >> 1)) * kFW + (warp == 0 ? 0 : kFW - 2) + (e & 1));
          __syncwarp();
        } else if (tid - 32 < 2 * kFW) {
          const int e = tid - 32;
          combine_slot(const_cast<double*>(pAp), (e < kFW ? 0 : (kFAY - 1) * kFW - kFW) + e);
        }
      }
      if (kUpd && has_p && interior && do1 && t + 1 >= kb && t + 1 < ke && t + 1 >= p.c_lo && t + 1 < p.c_hi) {
        PCGX_DCHECK((long long)(t + 1) * p.nxy + (long long)gj * p.nx + gi + 2 <= g_hi);
        st2(p.rout + (long long)(t + 1) * p.nxy + (long long)gj * p.nx + gi, ap.x, ap.y);
        acc_rr = acc_rr + ap.x * ap.x;
        acc_rr = acc_rr + ap.y * ap.y;
      }
      double aw, ae;
      if (PCGX_C2F_EXP >= 2) {
        aw = ac.y;
        ae = ac.x;
      } else {
        aw = pAu[offA - 1];
        ae = pAu[offA + 2];
      }
      const double2 as = PCGX_C2F_EXP >= 1 ? ac : rqx2(pAu, offA - kFW);
      const double2 an = PCGX_C2F_EXP >= 1 ? ac : rqx2(pAu, offA + kFW);
      const double2 xc = ac;  // A[t] at the pair
      const double y0 = c2f_stencil(d, am.x, as.x, aw, ac.x, ac.y, an.x, ap.x);
      const double y1 = c2f_stencil(d, am.y, as.y, ac.x, ac.y, ae, an.y, ap.y);
      double2 c;
      if (kFirst) {
        const double2 yq = div2_rn(y0, y1, p.theta, inv_t);
        c.x = p.c1 * ((2.0 * xc.x) - yq.x);
        c.y = p.c1 * ((2.0 * xc.y) - yq.y);
      } else {
        const double2 bb = PCGX_C2F_EXP >= 7 ? zero2 : *reinterpret_cast<const double2*>(pBu + offB);
        const double2 rr = PCGX_C2F_EXP >= 7 ? zero2 : *reinterpret_cast<const double2*>(pRu + offB);
        rt = rr;
        if (PCGX_C2F_EXP >= 5) {
          c.x = (xc.x + bb.x) + (rr.x + y0);
          c.y = (xc.y + bb.y) + (rr.y + y1);
        } else {
        c.x = p.rk1 * (((p.c3 * xc.x) - (p.rk1m1 * bb.x)) + p.c2 * (rr.x - y0));
        c.y = p.rk1 * (((p.c3 * xc.y) - (p.rk1m1 * bb.y)) + p.c2 * (rr.y - y1));
        }
      }
      const bool live = plane_in && do1;
      if (live) cv = c;
      if (p.outC && live && interior && t >= kb && t < ke) {  // outC null: last pass
        PCGX_DCHECK(gCt - p.outC >= g_lo && gCt - p.outC + 2 <= g_hi);
        st2(gCt, cv.x, cv.y);
      }
      if (PCGX_C2F_EXP < 6) *reinterpret_cast<double2*>(pCu + offB) = cv;
      // i-halo columns of C[t] (read by stage 2 of plane t, two iterations on)
      if (PCGX_C2F_EXP < 3 && do_h) {
        double hx = 0.0;
        if (plane_in && h_in) {
          const double xc = rqx(pAu, offAh);
          const double y = stencil_point(d, in_z(t - 1) ? rqx(pAm, offAh) : 0.0, rqx(pAu, offAh - kFW),
                                         rqx(pAu, offAh - 1), xc, rqx(pAu, offAh + 1), rqx(pAu, offAh + kFW),
                                         has_p ? rqx(pAp, offAh) : 0.0);
          if (kFirst) hx = p.c1 * ((2.0 * xc) - div_rn(y, p.theta, inv_t));
          else hx = p.rk1 * (((p.c3 * xc) - (p.rk1m1 * pBu[offBh])) + p.c2 * (pRu[offBh] - y));
        }
        pCu[offBh] = hx;
      }
    }
    // ---------------- stage 2: E[t-2] on the own tile row (warps 1..8)
    if (interior && t - 2 >= kb) {
      double cw, ce;
      if (PCGX_C2F_EXP >= 2) {
        cw = c2.y;
        ce = c2.x;
      } else {
        cw = pC2[offB - 1];
        ce = pC2[offB + 2];
      }
      const double2 cs = PCGX_C2F_EXP >= 1 ? c2 : *reinterpret_cast<const double2*>(pC2 + offB - kFW);
      const double2 cn = PCGX_C2F_EXP >= 1 ? c2 : *reinterpret_cast<const double2*>(pC2 + offB + kFW);
      const double y0 = c2f_stencil(d, c3.x, cs.x, cw, c2.x, c2.y, cn.x, c1.x);
      const double y1 = c2f_stencil(d, c3.y, cs.y, c2.x, c2.y, ce, cn.y, c1.y);
      const double2 cc = c2;  // C[t-2] at the pair
      double2 rv, xo;
      if (kFirst) {
        rv = a2;  // A == R == r
        xo = div2_rn(a2.x, a2.y, p.theta, inv_t);
      } else {
        rv = r2;
        xo = a2;
      }
      const double e0 = PCGX_C2F_EXP >= 5 ? (cc.x + xo.x) + (rv.x + y0)
                                          : p.rk2 * (((p.c3 * cc.x) - (p.rk2m1 * xo.x)) + p.c2 * (rv.x - y0));
      const double e1 = PCGX_C2F_EXP >= 5 ? (cc.y + xo.y) + (rv.y + y1)
                                          : p.rk2 * (((p.c3 * cc.y) - (p.rk2m1 * xo.y)) + p.c2 * (rv.y - y1));
      if (do2) {
        PCGX_DCHECK(gEv - p.outE >= g_lo && gEv - p.outE + 2 <= g_hi);
        st2(gEv, e0, e1);
        if (kRed) acc = acc + (rv.x * e0 + rv.y * e1);
      }
    }
      __syncthreads();
    // rotate the register queues, rings and global pointers by one plane
    a2 = am;
    am = ac;
    ac = ap;
    c3 = c2;
    c2 = c1;
    c1 = cv;
    r2 = r1;
    r1 = rt;
    pAm = pAu;
    pAu = pAp;
    pAp = (pAp + kFAPlane == sAend) ? sA : pAp + kFAPlane;
    pBu = (pBu + kFEStride == sBend) ? sB : pBu + kFEStride;
    pRu = (pRu + kFEStride == sRend) ? sR : pRu + kFEStride;
    double* const pc = pC2;
    pC2 = pC1;
    pC1 = pCu;
    pCu = pc;
    if (++bslot == kFD) {
      bslot = 0;
      bphase ^= 1u;
    }
    gCt += p.nxy;
    gEv += p.nxy;
  }
  if (kRed) block_reduce_finish(acc, red);
  if (kUpd) block_reduce_finish(acc_rr, red_rr);
}

}  // namespace pcgx
