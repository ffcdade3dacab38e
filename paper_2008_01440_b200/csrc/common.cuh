// SPDX-License-Identifier: Apache-2.0
//
// Internal definitions shared by the pcgx kernels and host orchestration.
//
// Arithmetic contract: the whole
// library is compiled with --fmad=false and every elementwise expression is
// written in the reference's evaluation order, so each per-point result (SpMV,
// Chebyshev step, PCG vector update) is the same IEEE binary64 value the
// reference computes (proj/src/linop.cpp:246-254, polyprec.cpp:187-195,
// pcg.cpp:81-82,107). Only reductions differ: they use a fixed
// thread -> warp -> block -> grid tree (deterministic run to run).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "pcgx.h"

// Checked build (-DPCGX_CHECKED; tools/build_variant.py checked -DPCGX_CHECKED):
// device-side bounds checks on the hand-written TMA / shared-memory kernels --
// every shared-memory ring offset a thread uses, every global store index -- that
// trap on a violation. compute-sanitizer is not available on the GPU pool, so
// this is the memory-safety check the sanitizer run would have been
// (tools/sanitize_run.py drives it on ragged small grids). Compiled out by default.
#ifdef PCGX_CHECKED
#include <cstdio>
#define PCGX_DCHECK(cond)                                                                   \
  do {                                                                                      \
    if (!(cond)) {                                                                          \
      printf("pcgx check failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
             (int)blockIdx.x, (int)threadIdx.x);                                            \
      __trap();                                                                             \
    }                                                                                       \
  } while (0)
#else
#define PCGX_DCHECK(cond) \
  do {                   \
  } while (0)
#endif

namespace pcgx {

// ------------------------------------------------------------------ errors

struct Error : std::runtime_error {
  pcgx_status code;
  Error(pcgx_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(pcgx_status c, const std::string& m) { throw Error(c, m); }

#define PCGX_CUDA(call)                                                                  \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      ::pcgx::fail(PCGX_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));    \
  } while (0)

// ------------------------------------------------------------------ constants

// Stencil tile: one warp spans 32 consecutive i; kStencilBY rows in j per block;
// each block marches kz planes in k (register queue for k-1, k, k+1).
constexpr int kStencilBX = 32;
constexpr int kStencilBY = 8;
constexpr int kStencilThreads = kStencilBX * kStencilBY;
// CSR: kCsrRows row-threads per block, nnz staged through shared memory in
// chunks of kCsrChunk products.
constexpr int kCsrRows = 128;
constexpr int kCsrChunk = 2048;
// Vector kernels.
constexpr int kVecThreads = 256;
// Upper bound on blocks of any reducing launch (partials buffer size).
constexpr int kMaxBlocks = 1 << 17;

// Device scalar slots (double S[kSlots]). rr/rz of one parity are adjacent so
// a multi-GPU job all-reduces them with one 16-byte ncclAllReduce.
enum Slot : int {
  S_PQ0 = 0, S_PQ1 = 1,         // p'q of iteration parity 0/1
  S_RR0 = 2, S_RZ0 = 3,         // r'r, r'z of parity 0
  S_RR1 = 4, S_RZ1 = 5,         // r'r, r'z of parity 1
  S_BB = 6,                     // b'b
  S_EE = 7,                     // true residual e'e
  S_DOT = 8, S_DOT2 = 9,        // scratch reductions (Lanczos, tests)
  S_E0 = 10, S_E1 = 11, S_E2 = 12,  // eigen-estimator reductions (2-3 values at once)
  S_BNORM = 13, S_TOL = 14,     // ||b|| and tol of the running solve (device convergence test)
  kSlots = 16
};
__host__ __device__ inline int slot_pq(int par) { return par ? S_PQ1 : S_PQ0; }
__host__ __device__ inline int slot_rr(int par) { return par ? S_RR1 : S_RR0; }
__host__ __device__ inline int slot_rz(int par) { return par ? S_RZ1 : S_RZ0; }

// Reduction target of one launch: per-block partials, a ticket counter, the
// result slot and whether to add to (interior + boundary launches) or
// overwrite it.
struct Reduce {
  double* partials = nullptr;
  unsigned* counter = nullptr;
  double* result = nullptr;
  int accumulate = 0;
  double* mirror = nullptr;  // != nullptr: the result also goes to this host-mapped slot
  // != nullptr (a launch inside a conditional PCG segment): the result is r'r and
  // the reducing block also sets the segment's IF condition -- "not converged",
  // sqrt(r'r) / cond_bt[0] > cond_bt[1] (||b||, tol), the host's own test
  const double* cond_bt = nullptr;
  unsigned long long cond = 0;  // cudaGraphConditionalHandle
};

// Geometry of one (slab of a) 7-point stencil operator.
struct StencilGeom {
  int nx, ny;           // plane extent
  int nzl;              // planes owned by this rank
  long long nxy;        // nx * ny
  double d;             // inv_sqrt_diag (constant)
};

struct CsrGeom {
  int n;                 // rows owned
  const int* row_ptr;    // n+1
  const int* col_idx;    // nnz
  const double* values;  // nnz
  const double* dvec;    // inv_sqrt_diag (n)
};

}  // namespace pcgx
