// SPDX-License-Identifier: Apache-2.0
//
// Host orchestration of the B200 Chebyshev-PCG path and the C ABI (include/pcgx.h).
//
// One context = one GPU, one compute stream (+ one comm stream for halo
// overlap), device scalars S[] that the kernels read directly (alpha, beta never
// round-trip through the host), a pinned mirror of S read once per PCG
// iteration for the convergence test, and CUDA graphs for the per-iteration
// kernel chain. Multi-GPU: z-slab operator, NCCL send/recv of one halo plane
// per neighbour per SpMV overlapped with the interior planes, and two NCCL
// all-reduces (8 B and 16 B) per PCG iteration.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <dlfcn.h>
#include <fcntl.h>
#include <pthread.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <tuple>
#include <queue>
#include <memory>
#include <string>
#include <type_traits>
#include <vector>

#include "cheb2.cuh"
#include "cheb2f.cuh"
#include "cheb3.cuh"
#include "common.cuh"
#include "bsr3t.cuh"
#include "dia3t.cuh"
#include "dir_tma.cuh"
#include "host_math.hpp"
#include "kernels.cuh"
#include "pcgx.h"

using namespace pcgx;

// ============================================================================ types

// An instantiated CUDA graph of one speculative PCG segment and what one replay
// launches (kernels and all-reduces are counted per replay).
inline int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

// Library switches: A/B and test knobs whose defaults are the production path.
// Read from the environment ONCE, when an operator (or a context) is created, into
// this snapshot; kernels, launches and solves read the snapshot, never the
// environment. Names: PCGX_<FIELD> in upper case (see from_env).
struct Tuning {
  // operator storage / kernel choice (CSR detection, grid-tile and TMA kernels)
  int dia = 1, dia3 = 1, dia3_kz = 0, dia_bps = 0, bsr = 1, bsr_bps = 16, sell_bps = 8;
  int dia3t = 1, dia3t_dir = 1, dia3t_first = 1, dia3t_kz = 32;
  int bsr3t = 1, bsr3t_modes = 1, bsr3t_kz = 32;
  int csr_stencil = 0;
  // stencil kernels
  int kz = 0, kz2 = 32, pfd = 2, cheb2 = 1, cheb3 = 2, dir_tma = 1, fuse_upd_slab = 1;
  std::string c2plan;  // "" automatic chunk plan, "u" uniform kz2, "h1,h2,..." explicit
  // PCG schedule
  int fuse_upd = 1, no_graph = 0, graph_multi = 0, merged = 0, cond_graph = 10, no_fuse_p = 0, zdiv = 1,
      defer_x = 1, snap_memcpy = 0, step_reps = 20;
  // vector kernels
  int upd2 = 1, upd_bps = 8;
  static Tuning from_env() {
    Tuning t;
    auto g = [](const char* n, int& v) { v = env_int(n, v); };
    g("PCGX_DIA", t.dia);
    g("PCGX_DIA3", t.dia3);
    g("PCGX_DIA3_KZ", t.dia3_kz);
    g("PCGX_DIA_BPS", t.dia_bps);
    g("PCGX_BSR", t.bsr);
    g("PCGX_BSR_BPS", t.bsr_bps);
    g("PCGX_SELL_BPS", t.sell_bps);
    g("PCGX_DIA3T", t.dia3t);
    g("PCGX_DIA3T_DIR", t.dia3t_dir);
    g("PCGX_DIA3T_FIRST", t.dia3t_first);
    g("PCGX_DIA3T_KZ", t.dia3t_kz);
    g("PCGX_BSR3T", t.bsr3t);
    g("PCGX_BSR3T_MODES", t.bsr3t_modes);
    g("PCGX_BSR3T_KZ", t.bsr3t_kz);
    g("PCGX_CSR_STENCIL", t.csr_stencil);
    g("PCGX_KZ", t.kz);
    g("PCGX_KZ2", t.kz2);
    g("PCGX_PFD", t.pfd);
    g("PCGX_CHEB2", t.cheb2);
    g("PCGX_CHEB3", t.cheb3);
    g("PCGX_FUSE_UPD_SLAB", t.fuse_upd_slab);
    g("PCGX_DIR_TMA", t.dir_tma);
    if (const char* e = std::getenv("PCGX_C2PLAN")) t.c2plan = e;
    g("PCGX_FUSE_UPD", t.fuse_upd);
    g("PCGX_NO_GRAPH", t.no_graph);
    g("PCGX_GRAPH_MULTI", t.graph_multi);
    g("PCGX_MERGED", t.merged);
    g("PCGX_COND_GRAPH", t.cond_graph);
    g("PCGX_NO_FUSE_P", t.no_fuse_p);
    g("PCGX_ZDIV", t.zdiv);
    g("PCGX_DEFER_X", t.defer_x);
    g("PCGX_SNAP_MEMCPY", t.snap_memcpy);
    g("PCGX_STEP_REPS", t.step_reps);
    g("PCGX_UPD2", t.upd2);
    g("PCGX_UPD_BPS", t.upd_bps);
    return t;
  }
};

// NVTX ranges around the library's phases (header-only NVTX v3: free unless a
// profiler is attached) -- solve, setup, iterations, exit residual, applies,
// operator uploads -- so nsys / ncu timelines show where a solve's time goes.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

struct Graph {
  cudaGraphExec_t exec = nullptr;
  int64_t kernels = 0;
  int64_t allreduces = 0;
  int64_t body_kernels = 0;  // kernels inside the conditional (IF) node, if any
  ~Graph() {
    if (exec) cudaGraphExecDestroy(exec);
  }
};

std::atomic<uint64_t> g_op_uid{1};

struct pcgx_context_s {
  int device = 0;
  Tuning tune;  // environment snapshot at creation (vector-kernel knobs)
  int rank = 0, nranks = 1;
  int sms = 148;
  cudaStream_t s = nullptr;   // compute
  cudaStream_t cs = nullptr;  // halo exchange
  ncclComm_t comm = nullptr;
  struct CommBase* cm = nullptr;  // nullptr on a single-GPU context
  double* S = nullptr;        // device scalars
  double* hS = nullptr;       // pinned mirror (host-mapped)
  std::vector<double> hx;     // host copy of x for SolveOptions::on_iterate
  double* dS_map = nullptr;   // hS as seen from the device: single-rank reductions store there too
  double* partials = nullptr;
  unsigned* counter = nullptr;
  cudaEvent_t ev_t0 = nullptr, ev_t1 = nullptr, ev_sync = nullptr, ev_fork = nullptr,
              ev_join = nullptr;
  std::vector<cudaEvent_t> evpool;
  int64_t launches = 0;
  std::string err;
  // workspace (device), sized for the largest operator used
  long long ws_n = 0, ws_pad = 0;
  double *r = nullptr, *z = nullptr, *p = nullptr, *p2 = nullptr, *q = nullptr, *w0 = nullptr,
         *w1 = nullptr, *w2 = nullptr, *w3 = nullptr, *t0 = nullptr, *t1 = nullptr,
         *r2 = nullptr;  // r ping-pong partner when the update is fused into P r
  double* flush = nullptr;
  size_t flush_bytes = 0;
  // Newton-form level vectors L[0..nlev-1] (NewtonWorkspace, polyprec.hpp:69-71)
  std::vector<double*> nl;
  long long nl_n = 0;
  // instantiated PCG segment graphs, keyed by everything they bake in (operator,
  // preconditioner coefficients, schedule, workspace generation); reused across solves
  std::map<std::string, std::unique_ptr<Graph>> gcache;
  uint64_t ws_gen = 0;  // bumped whenever a workspace buffer is (re)allocated
  // solve-local bookkeeping
  int64_t cur_launches = 0;
  int64_t cur_allreduce = 0;
  int64_t cur_halo_bytes = 0;
  bool capturing = false;
  // conditional-graph capture (device-side convergence): the root graph, its IF
  // handle, and the launch count when the IF body's capture began
  cudaGraph_t cond_root = nullptr;
  cudaGraphConditionalHandle cond_h = 0;
  bool cond_split = false;
  int64_t cond_mark = 0;
};

struct pcgx_operator_s {
  pcgx_context ctx = nullptr;
  Tuning tune;  // environment snapshot at creation: every switch its launches and solves read
  uint64_t uid = g_op_uid.fetch_add(1);  // never reused (graph-cache key)
  int kind = 0;  // 0 stencil7, 1 csr
  long long n_global = 0, n_local = 0, nnz = 0;
  // stencil
  long long nx = 0, ny = 0, nz = 0, z0 = 0, nzl = 0;
  double d = 0.0;
  double *ghost_lo = nullptr, *ghost_hi = nullptr;    // ghost planes of the SpMV input
  double *ghost_lo2 = nullptr, *ghost_hi2 = nullptr;  // second set (fused p = z + beta p: p_old)
  int kz = 16;
  bool vec2 = false;  // even nx -> stencil7v2_kernel
  int pfd = 0;        // L2 prefetch distance (planes) of the v2 march
  bool cheb2 = false; // two Chebyshev steps per pass (stencil7_cheb2f_kernel, TMA)
  std::string c2plan;                     // PCGX_C2PLAN: "" auto, "u" uniform kz2, "h1,h2,..." explicit
  std::map<int, ChunkPlan> c2plans;       // chunk plan per launch span (planes)
  std::map<int, ChunkPlan> dirplans;      // the same for the direction step
  bool cheb3 = false;                     // three Chebyshev steps per pass (stencil7_cheb3_kernel)
  std::map<int, ChunkPlan> c3plans;       // chunk plans of the three-step pass
  int zpad = 0;       // ghost planes per side in the workspace vectors (z-slab + cheb2: 2)
  int kz2 = 32;       // z-chunk of the two-step kernel
  struct TmaPair { const double* ptr; CUtensorMap fa, fe; };
  std::vector<TmaPair> tmaps;  // per-buffer tensor maps: the two-step kernel's A box 68 x (kFTY+4)
                               // and B / R / direction-step box 68 x (kFTY+2)
  // csr
  // SELL-32 layout (sell_kernel, the default CSR path)
  long long* sell_ptr = nullptr;
  int* sell_len = nullptr;
  int* sell_col = nullptr;
  double* sell_val = nullptr;
  int nslices = 0;
  long long sell_padded = 0;
  // BSR-3 in SELL-32 over block rows (bsr3_kernel): replaces the SELL arrays when the
  // matrix is made of aligned 3x3 blocks (single rank)
  long long* bsr_ptr = nullptr;
  int* bsr_len = nullptr;
  int* bsr_col = nullptr;
  double* bsr_val = nullptr;
  int bsr_slices = 0;
  long long bsr_blocks = 0;     // stored (unpadded) blocks = nnz / 9
  long long bsr_padded = 0;     // blocks incl. slice padding
  // BSR-3 on a cubic node grid with the 27-point block box (bsr3t_kernel): grid copy
  // of the values gval[(s * 9 + e) * ldn + node] and a 27-bit presence mask per node
  double* b3g_val = nullptr;
  unsigned* b3g_mask = nullptr;
  long long b3g_ld = 0;
  int b3g_nx = 0;
  // offset (diagonal) storage (dia_kernel): K fixed column offsets, values by offset
  double* dia_val = nullptr;
  unsigned* dia_mask = nullptr;
  int dia_k = 0;
  int dia_off[32] = {0};
  long long dia_ld = 0;
  int dia3_pat = 0, dia3_nx = 0;  // structured pattern (27 / 7) on an nx^3 grid (dia3_kernel)
  int dia3_nzl = 0;                // z-slab rank: local planes of the grid (0: the whole grid)
  double *dia3_dlo = nullptr, *dia3_dhi = nullptr;  // Jacobi values of the neighbours' boundary planes
  struct GMap { const void* ptr; int kind; CUtensorMap m; };
  std::vector<GMap> gmaps;        // dia3t_kernel tensor maps per buffer
  // CSR block rows on a multi-rank context: this rank owns rows [row0, row0 + n_local);
  // columns >= n_local index the ghost array (values of other ranks' rows)
  long long row0 = 0, nghost = 0, nsend = 0;
  int* send_idx = nullptr;                 // concatenated per-neighbour send lists (local rows)
  double *sbuf_z = nullptr, *sbuf_p = nullptr, *ghost_z = nullptr, *ghost_p = nullptr;
  std::vector<int> nb_rank;                // neighbours with traffic
  std::vector<long long> send_off, send_cnt, recv_off, recv_cnt;
  int sl_b0 = 0, sl_b1 = 0;                // slices [sl_b0, sl_b1) read no ghost column
  int *rp = nullptr, *ci = nullptr;
  double *va = nullptr, *dvec = nullptr;
  std::atomic<uint64_t> matvecs{0};
};

namespace {

thread_local std::string g_thread_err;

// NCCL is resolved at run time (only dist contexts need it) so that loading
// libpcgx.so never drags a second libnccl.so.2 into a process that also uses
// torch's bundled one: an already-loaded libnccl.so.2 wins, then
// $PCGX_NCCL_LIB, then the system library.
struct Nccl {
  bool ok = false;
  std::string why;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
};

const Nccl& nccl() {
  static Nccl n = [] {
    Nccl t;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) {
      const char* env = std::getenv("PCGX_NCCL_LIB");
      if (env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      t.why = std::string("cannot load libnccl.so.2: ") + dlerror();
      return t;
    }
#define PCGX_SYM(f) t.f = reinterpret_cast<decltype(t.f)>(dlsym(h, "nccl" #f))
    PCGX_SYM(GetErrorString);
    PCGX_SYM(GetUniqueId);
    PCGX_SYM(CommInitRank);
    PCGX_SYM(CommDestroy);
    PCGX_SYM(AllReduce);
    PCGX_SYM(Send);
    PCGX_SYM(Recv);
    PCGX_SYM(GroupStart);
    PCGX_SYM(GroupEnd);
#undef PCGX_SYM
    t.ok = t.GetErrorString && t.GetUniqueId && t.CommInitRank && t.CommDestroy && t.AllReduce &&
           t.Send && t.Recv && t.GroupStart && t.GroupEnd;
    if (!t.ok) t.why = "libnccl.so.2 lacks a required symbol";
    return t;
  }();
  if (!n.ok) fail(PCGX_ERR_NCCL, n.why);
  return n;
}

#define PCGX_NCCL(call)                                                                   \
  do {                                                                                    \
    ncclResult_t r_ = (call);                                                             \
    if (r_ != ncclSuccess)                                                                \
      fail(PCGX_ERR_NCCL, std::string(#call) + ": " + nccl().GetErrorString(r_));         \
  } while (0)

template <class F>
pcgx_status guarded(pcgx_context ctx, F&& f) {
  try {
    f();
    return PCGX_OK;
  } catch (const Error& e) {
    (ctx ? ctx->err : g_thread_err) = e.what();
    g_thread_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    (ctx ? ctx->err : g_thread_err) = "host allocation failed";
    return PCGX_ERR_CUDA;
  } catch (const std::exception& e) {
    (ctx ? ctx->err : g_thread_err) = e.what();
    return PCGX_ERR_CUDA;
  }
}

void set_device(pcgx_context c) { PCGX_CUDA(cudaSetDevice(c->device)); }

// A reducing launch writes one partial per block (two for block_reduce_finish2)
// into c->partials (kMaxBlocks doubles): fail loudly instead of writing past it.
void check_red_grid(unsigned long long nblocks, int per_block = 1) {
  if (nblocks * (unsigned long long)per_block > (unsigned long long)kMaxBlocks)
    fail(PCGX_ERR_UNSUPPORTED, "reduction over " + std::to_string(nblocks) +
                                   " blocks exceeds the partials buffer (" + std::to_string(kMaxBlocks) + ")");
}
unsigned long long nblocks_of(const dim3& g) { return (unsigned long long)g.x * g.y * g.z; }

Reduce make_red(pcgx_context c, int slot, bool accumulate = false) {
  Reduce r;
  r.partials = c->partials;
  r.counter = c->counter;
  r.result = c->S + slot;
  r.accumulate = accumulate ? 1 : 0;
  // one rank: the reducing block also stores the scalar into the host-mapped slot
  // array, so a solve's per-iteration snapshot is an event, not a D2H copy
  r.mirror = (!c->cm && c->dS_map) ? c->dS_map + slot : nullptr;
  return r;
}

void count_launch(pcgx_context c) {
  c->launches++;
  c->cur_launches++;
}

void check_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fail(PCGX_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
}

long long ws_pad_of(pcgx_operator op) { return op->zpad * op->nx * op->ny; }

// Workspace vectors carry `pad` zeroed elements before and after (z-slab ranks:
// two ghost planes per side that the two-step kernel reads through TMA).
void ensure_workspace(pcgx_context c, long long n, long long pad = 0) {
  if (c->ws_n >= n && c->ws_pad == pad) return;
  double** bufs[] = {&c->r, &c->z, &c->p, &c->p2, &c->q, &c->w0, &c->w1, &c->w2, &c->w3, &c->t0, &c->t1,
                     &c->r2};
  for (double** b : bufs) {
    if (*b) cudaFree(*b - c->ws_pad);
    *b = nullptr;
  }
  c->ws_n = 0;
  for (double** b : bufs) {
    double* raw = nullptr;
    const size_t tot = (size_t)std::max(n, 1LL) + 2 * (size_t)pad;
    PCGX_CUDA(cudaMalloc(&raw, sizeof(double) * tot));
    // zeroed on the compute stream: a legacy-stream memset is unordered with the
    // (non-blocking) compute stream and could land after the first kernels
    if (pad) PCGX_CUDA(cudaMemsetAsync(raw, 0, sizeof(double) * tot, c->s));
    *b = raw + pad;
  }
  c->ws_n = n;
  c->ws_pad = pad;
  c->ws_gen++;
  c->gcache.clear();
}

int vec_grid(pcgx_context c, long long n) {
  const long long want = (n + kVecThreads - 1) / kVecThreads;
  return (int)std::max(1LL, std::min(want, (long long)c->sms * 8));
}

#include "host_comm.cuh"
// ---------------------------------------------------------------- operator launch

void NcclComm::halo_begin(pcgx_context c, pcgx_operator op, const double* const* xs, int nv) {
  const long long nxy = op->nx * op->ny;
  const long long nzl = op->nzl;
  PCGX_CUDA(cudaEventRecord(c->ev_fork, c->s));
  PCGX_CUDA(cudaStreamWaitEvent(c->cs, c->ev_fork, 0));
  PCGX_NCCL(nccl().GroupStart());
  for (int v = 0; v < nv; ++v) {
    const double* x = xs[v];
    double* glo = v ? op->ghost_lo2 : op->ghost_lo;
    double* ghi = v ? op->ghost_hi2 : op->ghost_hi;
    if (glo) {
      PCGX_NCCL(nccl().Send(x, (size_t)nxy, ncclDouble, c->rank - 1, c->comm, c->cs));
      PCGX_NCCL(nccl().Recv(glo, (size_t)nxy, ncclDouble, c->rank - 1, c->comm, c->cs));
    }
    if (ghi) {
      PCGX_NCCL(nccl().Send(x + (nzl - 1) * nxy, (size_t)nxy, ncclDouble, c->rank + 1, c->comm, c->cs));
      PCGX_NCCL(nccl().Recv(ghi, (size_t)nxy, ncclDouble, c->rank + 1, c->comm, c->cs));
    }
  }
  PCGX_NCCL(nccl().GroupEnd());
  PCGX_CUDA(cudaEventRecord(c->ev_join, c->cs));
}

void LocalComm::halo_begin(pcgx_context c, pcgx_operator op, const double* const* xs, int nv) {
  const long long nxy = op->nx * op->ny;
  const long long nzl = op->nzl;
  g->ghost_lo[rank] = op->ghost_lo;
  g->ghost_hi[rank] = op->ghost_hi;
  g->ghost_lo2[rank] = op->ghost_lo2;
  g->ghost_hi2[rank] = op->ghost_hi2;
  // ev_fork: my vectors are final AND my previous boundary kernels (ghost readers) are queued before it
  PCGX_CUDA(cudaEventRecord(c->ev_fork, c->s));
  g->bar.wait();
  PCGX_CUDA(cudaStreamWaitEvent(c->cs, c->ev_fork, 0));
  const size_t pb = sizeof(double) * (size_t)nxy;
  if (rank > 0) PCGX_CUDA(cudaStreamWaitEvent(c->cs, g->ctx[rank - 1]->ev_fork, 0));
  if (rank < g->nranks - 1) PCGX_CUDA(cudaStreamWaitEvent(c->cs, g->ctx[rank + 1]->ev_fork, 0));
  for (int v = 0; v < nv; ++v) {
    const double* x = xs[v];
    if (rank > 0)  // my first plane -> ghost_hi of rank-1, once rank-1 no longer reads it
      PCGX_CUDA(cudaMemcpyAsync(v ? g->ghost_hi2[rank - 1] : g->ghost_hi[rank - 1], x, pb,
                                cudaMemcpyDefault, c->cs));
    if (rank < g->nranks - 1)  // my last plane -> ghost_lo of rank+1
      PCGX_CUDA(cudaMemcpyAsync(v ? g->ghost_lo2[rank + 1] : g->ghost_lo[rank + 1],
                                x + (nzl - 1) * nxy, pb, cudaMemcpyDefault, c->cs));
  }
  PCGX_CUDA(cudaEventRecord(c->ev_join, c->cs));
  g->bar.wait();  // every rank's ev_join recorded before anyone waits on it
}

void NcclComm::xchg(pcgx_context c, pcgx_operator op, const PlaneX* items, int n) {
  const bool lo = op->ghost_lo != nullptr, hi = op->ghost_hi != nullptr;
  PCGX_CUDA(cudaEventRecord(c->ev_fork, c->s));
  PCGX_CUDA(cudaStreamWaitEvent(c->cs, c->ev_fork, 0));
  PCGX_NCCL(nccl().GroupStart());
  for (int i = 0; i < n; ++i) {
    const PlaneX& it = items[i];
    if (lo) {
      PCGX_NCCL(nccl().Send(it.send_lo, (size_t)it.count, ncclDouble, c->rank - 1, c->comm, c->cs));
      PCGX_NCCL(nccl().Recv(it.recv_lo, (size_t)it.count, ncclDouble, c->rank - 1, c->comm, c->cs));
    }
    if (hi) {
      PCGX_NCCL(nccl().Send(it.send_hi, (size_t)it.count, ncclDouble, c->rank + 1, c->comm, c->cs));
      PCGX_NCCL(nccl().Recv(it.recv_hi, (size_t)it.count, ncclDouble, c->rank + 1, c->comm, c->cs));
    }
  }
  PCGX_NCCL(nccl().GroupEnd());
  PCGX_CUDA(cudaEventRecord(c->ev_join, c->cs));
}

void LocalComm::xchg(pcgx_context c, pcgx_operator op, const PlaneX* items, int n) {
  (void)op;
  g->xrecv_lo[rank].assign((size_t)n, nullptr);
  g->xrecv_hi[rank].assign((size_t)n, nullptr);
  for (int i = 0; i < n; ++i) {
    g->xrecv_lo[rank][(size_t)i] = items[i].recv_lo;
    g->xrecv_hi[rank][(size_t)i] = items[i].recv_hi;
  }
  PCGX_CUDA(cudaEventRecord(c->ev_fork, c->s));
  g->bar.wait();
  PCGX_CUDA(cudaStreamWaitEvent(c->cs, c->ev_fork, 0));
  if (rank > 0) PCGX_CUDA(cudaStreamWaitEvent(c->cs, g->ctx[rank - 1]->ev_fork, 0));
  if (rank < g->nranks - 1) PCGX_CUDA(cudaStreamWaitEvent(c->cs, g->ctx[rank + 1]->ev_fork, 0));
  for (int i = 0; i < n; ++i) {
    const PlaneX& it = items[i];
    const size_t b = sizeof(double) * (size_t)it.count;
    if (rank > 0)
      PCGX_CUDA(cudaMemcpyAsync(g->xrecv_hi[rank - 1][(size_t)i], it.send_lo, b, cudaMemcpyDefault, c->cs));
    if (rank < g->nranks - 1)
      PCGX_CUDA(cudaMemcpyAsync(g->xrecv_lo[rank + 1][(size_t)i], it.send_hi, b, cudaMemcpyDefault, c->cs));
  }
  PCGX_CUDA(cudaEventRecord(c->ev_join, c->cs));
  g->bar.wait();
}

void NcclComm::sparse_xchg(pcgx_context c, pcgx_operator op, int nv, const double* const* sbuf,
                           double* const* gbuf) {
  PCGX_CUDA(cudaEventRecord(c->ev_fork, c->s));
  PCGX_CUDA(cudaStreamWaitEvent(c->cs, c->ev_fork, 0));
  PCGX_NCCL(nccl().GroupStart());
  for (int v = 0; v < nv; ++v)
    for (size_t i = 0; i < op->nb_rank.size(); ++i) {
      const int q = op->nb_rank[i];
      if (op->send_cnt[i])
        PCGX_NCCL(nccl().Send(sbuf[v] + op->send_off[i], (size_t)op->send_cnt[i], ncclDouble, q, c->comm, c->cs));
      if (op->recv_cnt[i])
        PCGX_NCCL(nccl().Recv(gbuf[v] + op->recv_off[i], (size_t)op->recv_cnt[i], ncclDouble, q, c->comm, c->cs));
    }
  PCGX_NCCL(nccl().GroupEnd());
  PCGX_CUDA(cudaEventRecord(c->ev_join, c->cs));
}

void LocalComm::sparse_xchg(pcgx_context c, pcgx_operator op, int nv, const double* const* sbuf,
                            double* const* gbuf) {
  const int P = g->nranks;
  auto& mine = g->srecv[rank];
  mine.assign((size_t)nv * P, nullptr);
  for (int v = 0; v < nv; ++v)
    for (size_t i = 0; i < op->nb_rank.size(); ++i)
      mine[(size_t)v * P + op->nb_rank[i]] = gbuf[v] + op->recv_off[i];
  PCGX_CUDA(cudaEventRecord(c->ev_fork, c->s));
  g->bar.wait();
  PCGX_CUDA(cudaStreamWaitEvent(c->cs, c->ev_fork, 0));
  for (size_t i = 0; i < op->nb_rank.size(); ++i)  // the receiver no longer reads its ghosts
    PCGX_CUDA(cudaStreamWaitEvent(c->cs, g->ctx[op->nb_rank[i]]->ev_fork, 0));
  for (int v = 0; v < nv; ++v)
    for (size_t i = 0; i < op->nb_rank.size(); ++i) {
      if (!op->send_cnt[i]) continue;
      const int q = op->nb_rank[i];
      PCGX_CUDA(cudaMemcpyAsync(g->srecv[q][(size_t)v * P + rank], sbuf[v] + op->send_off[i],
                                sizeof(double) * (size_t)op->send_cnt[i], cudaMemcpyDefault, c->cs));
    }
  PCGX_CUDA(cudaEventRecord(c->ev_join, c->cs));
  g->bar.wait();
}

StencilGeom geom_of(pcgx_operator op) {
  StencilGeom g;
  g.nx = (int)op->nx;
  g.ny = (int)op->ny;
  g.nzl = (int)op->nzl;
  g.nxy = op->nx * op->ny;
  g.d = op->d;
  return g;
}

template <class In, class Epi, bool kRed>
void stencil_launch(pcgx_context c, pcgx_operator op, const StencilGeom& g, const In& in,
                    const Epi& epi, int k_begin, int k_end, int slot, bool accumulate) {
  if (k_end <= k_begin) return;
  const unsigned gy = (unsigned)((g.ny + kStencilBY - 1) / kStencilBY);
  const unsigned gx = (unsigned)(op->vec2 ? (g.nx + 63) / 64 : (g.nx + kStencilBX - 1) / kStencilBX);
  // planes per block: op->kz, raised so a reducing grid fits the partials buffer
  const long long span = k_end - k_begin;
  const long long kz_min = kRed ? (span * gx * gy + kMaxBlocks - 1) / kMaxBlocks : 1;
  const int kz = (int)std::max(1LL, std::min((long long)span, std::max((long long)op->kz, kz_min)));
  dim3 block(kStencilBX, kStencilBY, 1);
  Reduce red = kRed ? make_red(c, slot, accumulate) : Reduce{};
  const unsigned gz = (unsigned)((span + kz - 1) / kz);
  if (kRed) check_red_grid((unsigned long long)gx * gy * gz);
  if (op->vec2) {  // even nx: two points per lane, 16-byte loads
    dim3 grid((unsigned)((g.nx + 63) / 64), gy, gz);
    stencil7v2_kernel<In, Epi, kRed><<<grid, block, 0, c->s>>>(g, in, epi, k_begin, k_end, kz, red,
                                                                op->pfd);
  } else {
    dim3 grid((unsigned)((g.nx + kStencilBX - 1) / kStencilBX), gy, gz);
    stencil7_kernel<In, Epi, kRed><<<grid, block, 0, c->s>>>(g, in, epi, k_begin, k_end, kz, red);
  }
  check_launch();
  count_launch(c);
}

// Input policies with the operator's ghost planes attached (or stripped for the
// interior planes of a slab, which need none).
InVec in_of(pcgx_operator op, const double* x, bool ghosts) {
  return InVec{x, ghosts ? op->ghost_lo : nullptr, ghosts ? op->ghost_hi : nullptr, op->ghost_z,
               op->n_local};
}
InComb in_of(pcgx_operator op, const double* z, const double* p, const double* S, int s_new,
             int s_old, int first, bool ghosts) {
  InComb in{};
  in.z = z;
  in.p = p;
  in.S = S;
  in.s_new = s_new;
  in.s_old = s_old;
  in.first = first;
  in.zlo = ghosts ? op->ghost_lo : nullptr;
  in.zhi = ghosts ? op->ghost_hi : nullptr;
  in.plo = ghosts ? op->ghost_lo2 : nullptr;
  in.phi = ghosts ? op->ghost_hi2 : nullptr;
  in.gz = op->ghost_z;
  in.gp = op->ghost_p;
  in.nloc = op->n_local;
  return in;
}
InVec strip(const InVec& in) {
  InVec o = in;
  o.glo = o.ghi = nullptr;
  return o;
}
InComb strip(const InComb& in) {
  InComb o = in;
  o.zlo = o.zhi = o.plo = o.phi = nullptr;
  return o;
}
int halo_vecs(const InVec& in, const double** xs) {
  xs[0] = in.x;
  return 1;
}
int halo_vecs(const InComb& in, const double** xs) {
  xs[0] = in.z;
  xs[1] = in.p;
  return in.first ? 1 : 2;
}

// Offset storage applied by grid tiles (dia3_kernel): the 27-point box by default
// (cfg3: 0.99 -> 0.83 ms per Chebyshev step at 256^3); the 7-point star only on
// request (PCGX_DIA3=2) — at cfg1's L2-resident 100^3 the row-thread kernel is 2x
// faster, its seven gathers hit L2.
bool dia3_on(pcgx_operator op) {
  const int e = op->tune.dia3;
  return (op->dia3_pat == 27 && e >= 1) || (op->dia3_pat == 7 && e >= 2);
}

template <bool kRed>
bool dia3t_launch(pcgx_context c, pcgx_operator op, const InVec& in, const EpiChebStep& epi, int slot);
template <bool kRed>
bool dia3t_launch(pcgx_context c, pcgx_operator op, const InVec& in, const EpiChebFirst& epi, int slot);
template <bool kRed>
bool dia3t_launch(pcgx_context c, pcgx_operator op, const InComb& in, const EpiStoreP& epi, int slot);
template <bool kRed>
bool bsr3t_launch(pcgx_context c, pcgx_operator op, const InVec& in, const EpiChebStep& epi, int slot);
template <bool kRed>
bool bsr3t_launch(pcgx_context c, pcgx_operator op, const InVec& in, const EpiChebFirst& epi, int slot);
template <bool kRed>
bool bsr3t_launch(pcgx_context c, pcgx_operator op, const InComb& in, const EpiStoreP& epi, int slot);

// Whether the operator's kernels accept the fused direction-update input.
bool fuses_dir_update(pcgx_operator op) {
  return op->kind == 0 || op->sell_ptr != nullptr || op->bsr_ptr != nullptr ||
         op->dia_val != nullptr;
}

// y-consuming launch of the scaled operator over the local rows, with the halo
// exchange of the input (multi-GPU) overlapped with the interior planes.
template <class In, class Epi, bool kRed>
void op_launch_in(pcgx_context c, pcgx_operator op, const In& in, const Epi& epi, int slot) {
  op->matvecs.fetch_add(1, std::memory_order_relaxed);
  if (op->kind == 1 && op->dia_val) {
    DiaGeom g{};
    g.n = (int)op->n_local;
    g.K = op->dia_k;
    g.ld = op->dia_ld;
    for (int k = 0; k < op->dia_k; ++k) g.off[k] = op->dia_off[k];
    g.val = op->dia_val;
    g.mask = op->dia_mask;
    g.dvec = op->dvec;
    // one full wave of resident blocks, grid-stride over the rows (a partial second
    // wave would leave SMs idle at the tail)
    const bool stream = (double)op->dia_k * (double)op->dia_ld * 8.0 > 64e6;  // values exceed ~half of L2
    if constexpr ((std::is_same<In, InVec>::value &&
                   (std::is_same<Epi, EpiChebStep>::value || std::is_same<Epi, EpiChebFirst>::value)) ||
                  (std::is_same<In, InComb>::value && std::is_same<Epi, EpiStoreP>::value)) {
      if (dia3t_launch<kRed>(c, op, in, epi, slot)) return;
    }
    if (dia3_on(op)) {
      const int nzl = op->dia3_nzl > 0 ? op->dia3_nzl : op->dia3_nx;
      auto launch3 = [&](int k0, int k1, bool accumulate) {
        if (k1 <= k0) return;
        Dia3Geom g3{op->dia3_nx, 0, op->dia_ld, op->dia_val, op->dia_mask, op->dvec};
        g3.nzl = nzl;
        g3.kb0 = k0;
        g3.ke0 = k1;
        g3.dlo = op->dia3_dlo;
        g3.dhi = op->dia3_dhi;
        const int tiles = ((g3.nx + kD3X - 1) / kD3X) * ((g3.nx + kD3Y - 1) / kD3Y);
        // z-chunks: about 8 waves of 3 resident CTAs per SM, at least 8 planes each
        const int want = std::max(1, (c->sms * 3 * 8 + tiles - 1) / tiles);
        g3.kz = std::max(op->tune.dia3_kz > 0 ? op->tune.dia3_kz : (nzl + want - 1) / want, std::min(8, nzl));
        const dim3 grid3(tiles, (k1 - k0 + g3.kz - 1) / g3.kz);
        if (kRed) check_red_grid(nblocks_of(grid3));
        Reduce red = kRed ? make_red(c, slot, accumulate) : Reduce{};
        if (op->dia3_pat == 27) {
          auto k3 = stream ? dia3_kernel<27, In, Epi, kRed, true> : dia3_kernel<27, In, Epi, kRed, false>;
          k3<<<grid3, kD3Threads, 0, c->s>>>(g3, in, epi, red);
        } else {
          auto k3 = stream ? dia3_kernel<7, In, Epi, kRed, true> : dia3_kernel<7, In, Epi, kRed, false>;
          k3<<<grid3, kD3Threads, 0, c->s>>>(g3, in, epi, red);
        }
        check_launch();
        count_launch(c);
      };
      const bool lo_nb = op->ghost_lo != nullptr, hi_nb = op->ghost_hi != nullptr;
      if (!lo_nb && !hi_nb) {
        launch3(0, nzl, false);
        return;
      }
      // z-slab rank of a grid-tile offset storage: my boundary planes to the
      // neighbours' ghost planes; the planes that read no ghost run meanwhile
      const double* xs[2];
      const int nv = halo_vecs(in, xs);
      c->cm->halo_begin(c, op, xs, nv);
      c->cur_halo_bytes += (long long)nv * ((lo_nb ? 1 : 0) + (hi_nb ? 1 : 0)) * op->nx * op->ny * 8;
      const int ib = lo_nb ? 1 : 0, ie = hi_nb ? nzl - 1 : nzl;
      bool wrote = false;
      if (ie > ib) {
        launch3(ib, ie, false);
        wrote = true;
      }
      c->cm->halo_wait(c);
      if (lo_nb) {
        launch3(0, std::min(1, nzl), wrote);
        wrote = true;
      }
      if (hi_nb && nzl - 1 >= ib) launch3(nzl - 1, nzl, wrote);
      return;
    }
    auto kern = stream ? dia_kernel<In, Epi, kRed, true> : dia_kernel<In, Epi, kRed, false>;
    // occupancy of this instantiation, queried once (atomic: local-group ranks drive
    // the library from several host threads)
    static std::atomic<int> occ_cache{0};
    int occ = occ_cache.load(std::memory_order_relaxed);
    if (!occ) {
      PCGX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, dia_kernel<In, Epi, kRed, true>, 256, 0));
      occ = std::max(occ, 1);
      occ_cache.store(occ, std::memory_order_relaxed);
    }
    const long long want = (op->n_local + 255) / 256;
    const int bps = op->tune.dia_bps;
    const int grid = (int)std::max(1LL, std::min(want, (long long)c->sms * (bps > 0 ? bps : occ)));
    Reduce red = kRed ? make_red(c, slot) : Reduce{};
    kern<<<grid, 256, 0, c->s>>>(g, in, epi, red);
    check_launch();
    count_launch(c);
    return;
  }
  if (op->kind == 1 && op->bsr_ptr) {
    if constexpr ((std::is_same<In, InVec>::value &&
                   (std::is_same<Epi, EpiChebStep>::value || std::is_same<Epi, EpiChebFirst>::value)) ||
                  (std::is_same<In, InComb>::value && std::is_same<Epi, EpiStoreP>::value)) {
      if (bsr3t_launch<kRed>(c, op, in, epi, slot)) return;
    }
    if (!op->nb_rank.empty()) {  // block-row rank: the ghost columns first (no overlap)
      const double* src[2];
      const int nv = halo_vecs(in, src);
      const double* sb[2] = {op->sbuf_z, op->sbuf_p};
      double* gb[2] = {op->ghost_z, op->ghost_p};
      for (int v = 0; v < nv && op->nsend; ++v) {
        pack_kernel<<<vec_grid(c, op->nsend), kVecThreads, 0, c->s>>>(op->nsend, op->send_idx, src[v],
                                                                       const_cast<double*>(sb[v]));
        check_launch();
        count_launch(c);
      }
      c->cm->sparse_xchg(c, op, nv, sb, gb);
      c->cur_halo_bytes += (long long)nv * op->nsend * 8;
      c->cm->halo_wait(c);
    }
    Bsr3Geom g{(int)(op->n_local / 3), 0, op->bsr_slices, op->bsr_ptr, op->bsr_len, op->bsr_col,
               op->bsr_val, op->dvec};
    const int wpb = 8;
    const int want = (op->bsr_slices + wpb - 1) / wpb;
    const int grid = std::max(1, std::min(want, c->sms * op->tune.bsr_bps));
    Reduce red = kRed ? make_red(c, slot) : Reduce{};
    bsr3_kernel<In, Epi, kRed><<<grid, 32 * wpb, 0, c->s>>>(g, in, epi, red);
    check_launch();
    count_launch(c);
    return;
  }
  if (op->kind == 1 && op->sell_ptr) {
    auto sell = [&](int s0, int s1, bool accumulate) {
      if (s1 <= s0) return;
      SellGeom g{(int)op->n_local, op->nslices, s0, s1, op->sell_ptr, op->sell_len, op->sell_col,
                 op->sell_val, op->dvec};
      const int wpb = 8;
      const int want = (s1 - s0 + wpb - 1) / wpb;
      const int grid = std::max(1, std::min(want, c->sms * op->tune.sell_bps));
      Reduce red = kRed ? make_red(c, slot, accumulate) : Reduce{};
      sell_kernel<In, Epi, kRed><<<grid, 32 * wpb, 0, c->s>>>(g, in, epi, red);
      check_launch();
      count_launch(c);
    };
    if (op->nb_rank.empty()) {
      sell(0, op->nslices, false);
      return;
    }
    // block-row halo: pack the rows other ranks reference, exchange, overlap the
    // ghost-free slices with the transfer, then the slices that read ghost columns
    const double* src[2];
    const int nv = halo_vecs(in, src);
    const double* sb[2] = {op->sbuf_z, op->sbuf_p};
    double* gb[2] = {op->ghost_z, op->ghost_p};
    for (int v = 0; v < nv; ++v) {
      if (!op->nsend) break;
      pack_kernel<<<vec_grid(c, op->nsend), kVecThreads, 0, c->s>>>(op->nsend, op->send_idx, src[v],
                                                                     const_cast<double*>(sb[v]));
      check_launch();
      count_launch(c);
    }
    c->cm->sparse_xchg(c, op, nv, sb, gb);
    c->cur_halo_bytes += (long long)nv * op->nsend * 8;
    sell(op->sl_b0, op->sl_b1, false);
    const bool wrote = op->sl_b1 > op->sl_b0;
    c->cm->halo_wait(c);
    sell(0, op->sl_b0, wrote);
    sell(op->sl_b1, op->nslices, wrote || op->sl_b0 > 0);
    return;
  }
  if constexpr (std::is_same_v<In, InVec>) {
    if (op->kind == 1) {
      CsrGeom g{(int)op->n_local, op->rp, op->ci, op->va, op->dvec};
      const int nrb = (int)((op->n_local + kCsrRows - 1) / kCsrRows);
      const int grid = std::max(1, std::min(nrb, c->sms * 12));
      Reduce red = kRed ? make_red(c, slot) : Reduce{};
      csr_kernel<Epi, kRed><<<grid, kCsrRows, 0, c->s>>>(g, in.x, epi, red);
      check_launch();
      count_launch(c);
      return;
    }
  } else {
    if (op->kind == 1) fail(PCGX_ERR_UNSUPPORTED, "fused direction update needs the SELL CSR kernel");
  }
  StencilGeom g = geom_of(op);
  const int nzl = (int)op->nzl;
  const bool lo_nb = op->ghost_lo != nullptr, hi_nb = op->ghost_hi != nullptr;
  if (!lo_nb && !hi_nb) {
    stencil_launch<In, Epi, kRed>(c, op, g, in, epi, 0, nzl, slot, false);
    return;
  }
  // halo: my first plane -> rank-1 (its ghosts), my last plane -> rank+1
  const double* xs[2];
  const int nv = halo_vecs(in, xs);
  c->cm->halo_begin(c, op, xs, nv);
  const long long nxy = op->nx * op->ny;
  c->cur_halo_bytes += (long long)nv * ((lo_nb ? 1 : 0) + (hi_nb ? 1 : 0)) * nxy * 8;
  // interior planes need no ghost: run them while the halo is in flight
  const int ib = lo_nb ? 1 : 0, ie = hi_nb ? nzl - 1 : nzl;
  bool wrote = false;
  if (ie > ib) {
    stencil_launch<In, Epi, kRed>(c, op, g, strip(in), epi, ib, ie, slot, false);
    wrote = true;
  }
  c->cm->halo_wait(c);
  if (lo_nb) {
    stencil_launch<In, Epi, kRed>(c, op, g, in, epi, 0, 1, slot, wrote);
    wrote = true;
  }
  if (hi_nb && (nzl - 1 >= (lo_nb ? 1 : 0))) {
    stencil_launch<In, Epi, kRed>(c, op, g, in, epi, nzl - 1, nzl, slot, wrote);
  }
}

template <class Epi, bool kRed>
void op_launch(pcgx_context c, pcgx_operator op, const double* x, const Epi& epi, int slot) {
  op_launch_in<InVec, Epi, kRed>(c, op, in_of(op, x, true), epi, slot);
}

// ---------------------------------------------------------------- vector launches

void launch_zr(pcgx_context c, long long n, double* z, const double* r, double theta, int divide,
               int slot) {
  zr_kernel<<<vec_grid(c, n), kVecThreads, 0, c->s>>>(n, z, r, theta, divide, make_red(c, slot));
  check_launch();
  count_launch(c);
}

// x += alpha p ; r -= alpha q (+ z = r / theta) with the r'r (, r'z) reduction:
// the 16-byte-pair kernel when every vector allows it.
// x == nullptr: the x update is deferred to the next direction step.
void launch_update(pcgx_context c, long long n, double* x, double* r, const double* p,
                   const double* q, int s_rho, int s_pq, int s_rr, int zm, double theta, double* z) {
  auto al16 = [](const void* v) { return ((uintptr_t)v & 15u) == 0; };
  const bool vec = (n % 2 == 0) && al16(x) && al16(r) && al16(p) && al16(q) && al16(z) &&
                   c->tune.upd2 != 0;
  const bool dox = x != nullptr;
  if (!vec) {
    update_kernel<<<vec_grid(c, n), kVecThreads, 0, c->s>>>(n, x, r, p, q, c->S, s_rho, s_pq,
                                                            make_red(c, s_rr), zm, theta, z);
    return;
  }
  const long long n2 = n / 2;
  const int bps = c->tune.upd_bps;
  const int grid = (int)std::max(1LL, std::min((n2 + kVecThreads - 1) / kVecThreads, (long long)c->sms * bps));
  auto d2 = [](const double* v) { return reinterpret_cast<double2*>(const_cast<double*>(v)); };
#define PCGX_UPD(ZM, X)                                                                          \
  update2_kernel<ZM, X><<<grid, kVecThreads, 0, c->s>>>(n2, d2(x), d2(r), d2(p), d2(q), c->S, s_rho, \
                                                        s_pq, make_red(c, s_rr), theta, d2(z))
  if (zm == 0) dox ? PCGX_UPD(0, true) : PCGX_UPD(0, false);
  else if (zm == 1) dox ? PCGX_UPD(1, true) : PCGX_UPD(1, false);
  else dox ? PCGX_UPD(2, true) : PCGX_UPD(2, false);
#undef PCGX_UPD
}

void launch_dot(pcgx_context c, long long n, const double* a, const double* b, int slot) {
  dot_kernel<<<vec_grid(c, n), kVecThreads, 0, c->s>>>(n, a, b, make_red(c, slot));
  check_launch();
  count_launch(c);
}

void launch_fill(pcgx_context c, long long n, double* v, double val) {
  fill_kernel<<<vec_grid(c, n), kVecThreads, 0, c->s>>>(n, v, val);
  check_launch();
  count_launch(c);
}

void copy_d2d(pcgx_context c, double* dst, const double* src, long long n) {
  if (dst != src)
    PCGX_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * (size_t)n, cudaMemcpyDeviceToDevice, c->s));
}

// S (device) -> hS (pinned) and wait.
void fetch_scalars(pcgx_context c) {
  PCGX_CUDA(cudaMemcpyAsync(c->hS, c->S, sizeof(double) * kSlots, cudaMemcpyDeviceToHost, c->s));
  PCGX_CUDA(cudaStreamSynchronize(c->s));
}

// ---------------------------------------------------------------- TMA tensor maps

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  if (!fn) fail(PCGX_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

CUtensorMap make_map(pcgx_operator op, const double* ptr, int bx, int by) {
  CUtensorMap m;
  // padded workspace (z-slab ranks): the map spans the zpad ghost planes on each side
  ptr -= (long long)op->zpad * op->nx * op->ny;
  const cuuint64_t dims[3] = {(cuuint64_t)op->nx, (cuuint64_t)op->ny,
                              (cuuint64_t)(op->nzl + 2 * op->zpad)};
  const cuuint64_t strides[2] = {(cuuint64_t)op->nx * 8, (cuuint64_t)(op->nx * op->ny) * 8};
  const cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode_tiled()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(ptr),
                                    dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(PCGX_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return m;
}

// The direction step's x tiles: a map over the rank's unpadded x, box 64 x kDTY.
const CUtensorMap& xtile_map(pcgx_operator op, const double* x) {
  for (auto& g : op->gmaps)
    if (g.ptr == x && g.kind == 10) return g.m;
  const cuuint64_t dims[3] = {(cuuint64_t)op->nx, (cuuint64_t)op->ny, (cuuint64_t)op->nzl};
  const cuuint64_t strides[2] = {(cuuint64_t)op->nx * 8, (cuuint64_t)(op->nx * op->ny) * 8};
  const cuuint32_t box[3] = {(cuuint32_t)kC2TX, (cuuint32_t)kDTY, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUtensorMap m;
  const CUresult r = encode_tiled()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(x), dims, strides,
                                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(PCGX_ERR_CUDA, "cuTensorMapEncodeTiled (x tiles) failed: " + std::to_string((int)r));
  op->gmaps.push_back({x, 10, m});
  return op->gmaps.back().m;
}

using TmaPair = pcgx_operator_s::TmaPair;
const TmaPair& tmaps_for(pcgx_operator op, const double* ptr) {
  for (auto& t : op->tmaps)
    if (t.ptr == ptr) return t;
  TmaPair t{ptr, make_map(op, ptr, kFW, kFAY), make_map(op, ptr, kFW, kFBY)};
  op->tmaps.push_back(t);
  return op->tmaps.back();
}

// dia3t_kernel (regular Chebyshev steps on 27-point grid-tile offset storage,
// every operand by TMA): tensor maps per buffer, cached on the operator.
// kind 0: fp64 (32, 8, 1) tiles; 1: fp64 (36, 10, 1) patches; 2: u32 mask tiles;
// 3: the 4D value array (nx, nx, nx, 27), box (32, 8, 1, 27).
const CUtensorMap& dia3t_map(pcgx_operator op, const void* ptr, int kind) {
  for (auto& g : op->gmaps)
    if (g.ptr == ptr && g.kind == kind) return g.m;
  const cuuint64_t nx = (cuuint64_t)op->dia3_nx;
  const cuuint64_t es = kind == 2 ? 4 : 8;
  const cuuint64_t dims[4] = {nx, nx, nx, (cuuint64_t)kT3K};
  const cuuint64_t strides[3] = {nx * es, nx * nx * es, (cuuint64_t)op->dia_ld * 8};
  const cuuint32_t box[4] = {(cuuint32_t)(kind == 1 ? kT3PX : kD3X), (cuuint32_t)(kind == 1 ? kT3PY : kD3Y), 1,
                             (cuuint32_t)kT3K};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUtensorMap m;
  const CUresult r = encode_tiled()(&m, kind == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                                    kind == 3 ? 4 : 3, const_cast<void*>(ptr), dims, strides, box, estr,
                                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(PCGX_ERR_CUDA, "cuTensorMapEncodeTiled (dia3t) failed: " + std::to_string((int)r));
  op->gmaps.push_back({ptr, kind, m});
  return op->gmaps.back().m;
}

template <bool kRed, class Epi, class In>
bool dia3t_launch_any(pcgx_context c, pcgx_operator op, const In& in, const Epi& epi, int slot) {
  constexpr bool kFirst = std::is_same<Epi, EpiChebFirst>::value;
  constexpr bool kDir = std::is_same<Epi, EpiStoreP>::value;
  const double* eout;
  const double* eout2 = nullptr;
  const double* er = nullptr;
  const double* exo = nullptr;
  const double* ex;
  const double* ep = nullptr;
  bool ghosts;
  if constexpr (kDir) {
    eout = epi.q;
    eout2 = epi.pout;
    ex = in.z;
    if (!in.first) ep = in.p;
    ghosts = in.gz || in.gp || in.zlo || in.zhi;
  } else {
    ex = in.x;
    ghosts = in.gx != nullptr;
    if constexpr (kFirst) {
      eout = epi.xout;
    } else {
      eout = epi.out;
      er = epi.r;
      if (!epi.xold_from_r) exo = epi.xold;
    }
  }
  const int nx = op->dia3_nx;
  auto al16 = [](const void* p) { return ((uintptr_t)p & 15u) == 0; };
  auto clash = [&](const double* o) { return o && (o == ex || o == ep || o == er); };
  if (!dia3_on(op) || op->dia3_pat != 27 || op->tune.dia3t == 0 || nx % 4 != 0 || nx < kT3PX ||
      op->dia3_nzl > 0 ||  // a z-slab rank: the grid-tile kernel with ghost planes (dia3_kernel)
      ghosts || !al16(ex) || (ep && !al16(ep)) || (er && !al16(er)) || !al16(eout) || (eout2 && !al16(eout2)) ||
      (exo && !al16(exo)) || clash(eout) || clash(eout2))
    return false;
  if (kDir && op->tune.dia3t_dir == 0) return false;
  if (kFirst && op->tune.dia3t_first == 0) return false;
  Dia3tMaps maps;
  maps.val = dia3t_map(op, op->dia_val, 3);
  maps.mask = dia3t_map(op, op->dia_mask, 2);
  maps.r = er ? dia3t_map(op, er, 0) : maps.mask;  // unused for the first / direction step
  maps.xo = exo ? dia3t_map(op, exo, 0) : maps.r;
  maps.x = dia3t_map(op, ex, 1);
  maps.d = dia3t_map(op, op->dvec, 1);
  maps.p = ep ? dia3t_map(op, ep, 1) : maps.x;
  const int kz = std::max(1, op->tune.dia3t_kz);  // 8: -3%, 16: -1.5% at 256^3
  const int tiles = ((nx + kD3X - 1) / kD3X) * ((nx + kD3Y - 1) / kD3Y);
  const dim3 grid(tiles, (nx + kz - 1) / kz);
  static std::atomic<uint64_t> attr{0};  // per device: the attribute is set per device
  const uint64_t bit = 1ull << (c->device & 63);
  if (!(attr.load() & bit)) {
    PCGX_CUDA(cudaFuncSetAttribute(dia3t_kernel<kRed, Epi, In>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)kDia3tSmem));
    attr.fetch_or(bit);
  }
  if (kRed) check_red_grid(nblocks_of(grid));
  Reduce red = kRed ? make_red(c, slot) : Reduce{};
  dia3t_kernel<kRed, Epi, In><<<grid, kD3Threads, kDia3tSmem, c->s>>>(maps, nx, kz, epi, red, in);
  check_launch();
  count_launch(c);
  return true;
}
template <bool kRed>
bool dia3t_launch(pcgx_context c, pcgx_operator op, const InVec& in, const EpiChebStep& epi, int slot) {
  return dia3t_launch_any<kRed>(c, op, in, epi, slot);
}
template <bool kRed>
bool dia3t_launch(pcgx_context c, pcgx_operator op, const InVec& in, const EpiChebFirst& epi, int slot) {
  return dia3t_launch_any<kRed>(c, op, in, epi, slot);
}
template <bool kRed>
bool dia3t_launch(pcgx_context c, pcgx_operator op, const InComb& in, const EpiStoreP& epi, int slot) {
  return dia3t_launch_any<kRed>(c, op, in, epi, slot);
}

// bsr3t_kernel tensor maps (cached per buffer): kind 20 value array (4D), 21 masks,
// 22 (3 nx, nx, nx) fp64 tiles of 96 x 4, 23 patches of 108 x 6.
const CUtensorMap& bsr3t_map(pcgx_operator op, const void* ptr, int kind) {
  for (auto& g : op->gmaps)
    if (g.ptr == ptr && g.kind == kind) return g.m;
  const cuuint64_t nx = (cuuint64_t)op->b3g_nx;
  CUtensorMap m;
  CUresult r;
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  if (kind == 20) {
    const cuuint64_t dims[4] = {nx, nx, nx, 243};
    const cuuint64_t strides[3] = {nx * 8, nx * nx * 8, (cuuint64_t)op->b3g_ld * 8};
    const cuuint32_t box[4] = {(cuuint32_t)kB3X, (cuuint32_t)kB3Y, 1, 27};
    r = encode_tiled()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<void*>(ptr), dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (kind == 21) {
    const cuuint64_t dims[3] = {nx, nx, nx};
    const cuuint64_t strides[2] = {nx * 4, nx * nx * 4};
    const cuuint32_t box[3] = {(cuuint32_t)kB3X, (cuuint32_t)kB3Y, 1};
    r = encode_tiled()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    const cuuint64_t dims[3] = {3 * nx, nx, nx};
    const cuuint64_t strides[2] = {3 * nx * 8, 3 * nx * nx * 8};
    const cuuint32_t box[3] = {(cuuint32_t)(kind == 22 ? 3 * kB3X : kB3PX), (cuuint32_t)(kind == 22 ? kB3Y : kB3PY),
                               1};
    r = encode_tiled()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) fail(PCGX_ERR_CUDA, "cuTensorMapEncodeTiled (bsr3t) failed: " + std::to_string((int)r));
  op->gmaps.push_back({ptr, kind, m});
  return op->gmaps.back().m;
}

template <bool kRed, class Epi, class In>
bool bsr3t_launch_any(pcgx_context c, pcgx_operator op, const In& in, const Epi& epi, int slot) {
  constexpr bool kFirst = std::is_same<Epi, EpiChebFirst>::value;
  constexpr bool kDir = std::is_same<Epi, EpiStoreP>::value;
  const double *eout, *eout2 = nullptr, *er = nullptr, *exo = nullptr, *ex, *ep = nullptr;
  bool ghosts;
  if constexpr (kDir) {
    eout = epi.q;
    eout2 = epi.pout;
    ex = in.z;
    if (!in.first) ep = in.p;
    ghosts = in.gz || in.gp || in.zlo || in.zhi;
  } else {
    ex = in.x;
    ghosts = in.gx != nullptr;
    if constexpr (kFirst) {
      eout = epi.xout;
    } else {
      eout = epi.out;
      er = epi.r;
      if (!epi.xold_from_r) exo = epi.xold;
    }
  }
  const int nx = op->b3g_nx;
  auto al16 = [](const void* p) { return ((uintptr_t)p & 15u) == 0; };
  auto clash = [&](const double* o) { return o && (o == ex || o == ep || o == er); };
  if (!op->b3g_val || op->tune.bsr3t == 0 || ghosts || !al16(ex) || (ep && !al16(ep)) ||
      (er && !al16(er)) || !al16(eout) || (eout2 && !al16(eout2)) || (exo && !al16(exo)) || clash(eout) ||
      clash(eout2))
    return false;
  if ((kDir || kFirst) && op->tune.bsr3t_modes == 0) return false;
  Bsr3tMaps maps;
  maps.val = bsr3t_map(op, op->b3g_val, 20);
  maps.mask = bsr3t_map(op, op->b3g_mask, 21);
  maps.r = er ? bsr3t_map(op, er, 22) : maps.mask;  // unused for the first / direction step
  maps.xo = exo ? bsr3t_map(op, exo, 22) : maps.r;
  maps.x = bsr3t_map(op, ex, 23);
  maps.d = bsr3t_map(op, op->dvec, 23);
  maps.p = ep ? bsr3t_map(op, ep, 23) : maps.x;
  const int kz = std::max(1, op->tune.bsr3t_kz);
  const int tiles = ((nx + kB3X - 1) / kB3X) * ((nx + kB3Y - 1) / kB3Y);
  const dim3 grid(tiles, (nx + kz - 1) / kz);
  static std::atomic<uint64_t> attr{0};  // per device: the attribute is set per device
  const uint64_t bit = 1ull << (c->device & 63);
  if (!(attr.load() & bit)) {
    PCGX_CUDA(cudaFuncSetAttribute(bsr3t_kernel<kRed, Epi, In>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)kBsr3tSmem));
    attr.fetch_or(bit);
  }
  if (kRed) check_red_grid(nblocks_of(grid));
  Reduce red = kRed ? make_red(c, slot) : Reduce{};
  bsr3t_kernel<kRed, Epi, In><<<grid, kB3Threads, kBsr3tSmem, c->s>>>(maps, nx, kz, epi, red, in);
  check_launch();
  count_launch(c);
  return true;
}
template <bool kRed>
bool bsr3t_launch(pcgx_context c, pcgx_operator op, const InVec& in, const EpiChebStep& epi, int slot) {
  return bsr3t_launch_any<kRed>(c, op, in, epi, slot);
}
template <bool kRed>
bool bsr3t_launch(pcgx_context c, pcgx_operator op, const InVec& in, const EpiChebFirst& epi, int slot) {
  return bsr3t_launch_any<kRed>(c, op, in, epi, slot);
}
template <bool kRed>
bool bsr3t_launch(pcgx_context c, pcgx_operator op, const InComb& in, const EpiStoreP& epi, int slot) {
  return bsr3t_launch_any<kRed>(c, op, in, epi, slot);
}


// Chunk heights of a two-step launch over `span` planes of `tiles` tiles with
// `slots` resident CTAs. The block scheduler dispatches chunk-major, greedily;
// uniform chunks leave a ragged last wave (4.5 waves at 320^3, 3 CTAs/SM). The
// plan is: uniform chunks of `big` planes, the last (up to three) chunks shrunk
// so the final wave ends evenly -- chosen by simulating the greedy dispatch (a
// chunk of h planes costs h + 2.5 plane-times: two halo planes plus the ring
// ramp). spec "u": uniform kz; "h1,h2,...": explicit heights summing to span.
ChunkPlan make_chunk_plan_search(const std::string& spec, int span, int kz, long long tiles, long long slots,
                                 double ovh, bool long_chunks);
// plans are pure functions of their arguments: searched once per process
ChunkPlan make_chunk_plan(const std::string& spec, int span, int kz, long long tiles, long long slots,
                          double ovh = 2.5, bool long_chunks = true) {
  static std::mutex mu;
  static std::map<std::tuple<std::string, int, int, long long, long long, double, bool>, ChunkPlan> cache;
  const auto key = std::make_tuple(spec, span, kz, tiles, slots, ovh, long_chunks);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  const ChunkPlan p = make_chunk_plan_search(spec, span, kz, tiles, slots, ovh, long_chunks);
  std::lock_guard<std::mutex> lk(mu);
  cache.emplace(key, p);
  return p;
}
ChunkPlan make_chunk_plan_search(const std::string& spec, int span, int kz, long long tiles, long long slots,
                                 double ovh, bool long_chunks) {
  auto pack = [&](const std::vector<int>& hs) {
    ChunkPlan p{};
    p.n = 0;
    p.start[0] = 0;
    for (int h : hs) {
      p.start[p.n + 1] = p.start[p.n] + h;
      ++p.n;
    }
    return p;
  };
  auto uniform = [&](int h) {
    std::vector<int> hs;
    for (int z = 0; z < span; z += h) hs.push_back(std::min(h, span - z));
    return hs;
  };
  std::vector<int> hs;
  if (spec == "u") {
    hs = uniform(std::max(kz, (span + ChunkPlan::kMax - 1) / ChunkPlan::kMax));
  } else if (!spec.empty()) {
    int sum = 0;
    for (size_t a = 0; a < spec.size();) {
      size_t b = spec.find(',', a);
      if (b == std::string::npos) b = spec.size();
      hs.push_back(std::max(1, std::atoi(spec.substr(a, b - a).c_str())));
      sum += hs.back();
      a = b + 1;
    }
    if (sum != span || (int)hs.size() > ChunkPlan::kMax) hs.clear();
  }
  if (hs.empty()) {
    double best = 0.0;
    std::vector<double> heap;
    // greedy in-order dispatch onto `slots` resident CTAs; gives up (returns a value
    // above `limit`) as soon as a chunk finishes after the best makespan so far
    auto makespan = [&](const std::vector<int>& h, double limit) {
      heap.assign((size_t)slots, 0.0);  // all-equal values: already a heap
      double end = 0.0;
      for (int c : h)
        for (long long t = 0; t < tiles; ++t) {
          std::pop_heap(heap.begin(), heap.end(), std::greater<double>());
          const double f = heap.back() + c + ovh;
          heap.back() = f;
          std::push_heap(heap.begin(), heap.end(), std::greater<double>());
          end = std::max(end, f);
          if (end > limit) return end;
        }
      return end;
    };
    std::vector<int> bigs = {16, 24, 32, 40, 48, 64, 80, 96};
    std::vector<int> tl = {0, 4, 8, 12, 16, 20, 24};
    // When every tile of a z-level runs at once (tiles <= resident CTAs: 80 tiles on
    // 148 SMs at 320^3) neighbouring tiles stay at the same z however long a chunk
    // is, so long chunks cost no L2 locality and save the per-chunk overhead: the
    // search then covers any first-chunk height and longer tails (320^3: 176, 88,
    // 28, 28 instead of 20, 80, 80, 80, 24, 24, 12: the two-step pass -3.7% live).
    // With more tiles than resident CTAs the tiles of a level run in turns and long
    // chunks let them drift out of the L2 window (measured at 640^3).
    // The long first chunk lies near the balanced makespan span * tiles / slots (the
    // other SMs share what is left), which keeps the search small. The direction
    // step keeps the short-chunk plans (long chunks measured 7% slower there).
    if (long_chunks && tiles <= slots && span > 96) {
      const int ideal = (int)((long long)span * tiles / slots);
      for (int b = std::max(100, (ideal - 16) / 4 * 4); b <= std::min(span, ideal + 32); b += 4) bigs.push_back(b);
      for (int t : {28, 32, 40, 48, 56, 64, 72, 80, 88, 96})
        if (t <= span / 2) tl.push_back(t);
    }
    for (int big : bigs)
      for (int t1 : tl)
        for (int t2 : tl)
          for (int t3 : tl) {
            if (t2 > t1 || t3 > t2) continue;
            const int tail = t1 + t2 + t3;
            if (tail > span) continue;
            const int rest = span - tail;
            std::vector<int> c;
            if (rest % big) c.push_back(rest % big);
            for (int k = 0; k < rest / big; ++k) c.push_back(big);
            for (int t : {t1, t2, t3})
              if (t) c.push_back(t);
            if (c.empty() || (int)c.size() > ChunkPlan::kMax) continue;
            const double m = makespan(c, hs.empty() ? 1e300 : best + 1e-9);
            if (hs.empty() || m < best - 1e-9 || (m < best + 1e-9 && c.size() < hs.size())) {
              best = m;
              hs = c;
            }
          }
    if (hs.empty()) hs = uniform((span + ChunkPlan::kMax - 1) / ChunkPlan::kMax);
  }
  // a reducing launch of `tiles` x chunks blocks must fit the partials buffer
  if ((long long)hs.size() * tiles > kMaxBlocks && tiles <= kMaxBlocks) {
    const long long maxn = std::max(1LL, (long long)kMaxBlocks / tiles);
    hs = uniform((int)((span + maxn - 1) / maxn));
  }
  return pack(hs);
}

// [0, ib) and [ie, nzl) as chunks 0 and 2 of one launch, the interior chunk masked
ChunkPlan strips_plan(int ib, int ie, int nzl) {
  ChunkPlan bp{};
  bp.n = 3;
  bp.start[0] = 0;
  bp.start[1] = ib;
  bp.start[2] = ie;
  bp.start[3] = nzl;
  bp.skip = 2ull;
  return bp;
}

template <bool kFirst, bool kRed>
void cheb2_launch(pcgx_context c, pcgx_operator op, const double* A, const double* B,
                  const double* R, const Cheb2Params& prm, int slot, int k_begin, int k_end, int kz,
                  bool accumulate, const ChunkPlan* forced = nullptr) {
  (void)kz;
  {
    if (k_end <= k_begin) return;
    auto kern = stencil7_cheb2f_kernel<kFirst, kRed>;
    PCGX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kC2FSmem));
    const CUtensorMap ma = tmaps_for(op, A).fa;
    const CUtensorMap mb = tmaps_for(op, B ? B : A).fe;
    const CUtensorMap mr = tmaps_for(op, R).fe;
    const long long tiles = ((op->nx + kC2TX - 1) / kC2TX) * ((op->ny + kFTY - 1) / kFTY);
    const int span = k_end - k_begin;
    auto it = op->c2plans.find(span);
    if (it == op->c2plans.end()) {
      int occ = 0;
      PCGX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kFThreads, kC2FSmem));
      it = op->c2plans.emplace(span, make_chunk_plan(op->c2plan, span, op->kz2, tiles,
                                                     (long long)std::max(occ, 1) * c->sms)).first;
    }
    const ChunkPlan& plan = forced ? *forced : it->second;
    if (kRed) check_red_grid((unsigned long long)tiles * plan.n);
    Reduce red = kRed ? make_red(c, slot, accumulate) : Reduce{};
    kern<<<dim3((unsigned)tiles, (unsigned)plan.n), kFThreads, kC2FSmem, c->s>>>(ma, mb, mr, prm, k_begin,
                                                                                  k_end, plan, red, Reduce{});
    check_launch();
    count_launch(c);
  }
}

// The direction step p_new = z + beta p_old, q = A p_new, p_new . q -> slot on a
// stencil operator (stencil7_dir_kernel, TMA-staged); on a z-slab rank the
// neighbours' boundary planes of z and p_old travel into the vectors' padding.
bool dir_tma_ok(pcgx_operator op) {
  const bool ghosts = op->ghost_lo || op->ghost_hi;
  return op->kind == 0 && op->vec2 && op->cheb2 && (!ghosts || op->zpad >= 1) &&
         op->tune.dir_tma != 0;
}

void dir_tma_launch(pcgx_context c, pcgx_operator op, const double* z, const double* pold,
                    double* pnew, double* q, int s_new, int s_old, int first, int slot,
                    double* x = nullptr, int s_pq = 0, double ztheta = 0.0) {
  op->matvecs.fetch_add(1, std::memory_order_relaxed);
  PCGX_CUDA(cudaFuncSetAttribute(stencil7_dir_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kDirSmem));
  static_assert(kDBY == kFBY, "direction-step box rows: no tensor map of that shape");
  const CUtensorMap mz = tmaps_for(op, z).fe;
  const CUtensorMap mx = (kDirXTma && x && !first) ? xtile_map(op, x) : mz;  // unused unless x is updated
  const CUtensorMap mp = tmaps_for(op, first ? z : pold).fe;
  const int nzl = (int)op->nzl;
  const bool lo = op->ghost_lo != nullptr, hi = op->ghost_hi != nullptr;
  DirParams prm{(int)op->nx, (int)op->ny, nzl, lo ? -1 : 0, hi ? nzl + 1 : nzl, op->zpad,
                op->nx * op->ny, op->d, c->S, s_new, s_old, first, x, s_pq, q, pnew, ztheta};
  auto launch = [&](int k_begin, int k_end, int kz, bool accumulate, const ChunkPlan* forced = nullptr) {
    if (k_end <= k_begin) return;
    const long long tiles = ((op->nx + kC2TX - 1) / kC2TX) * ((op->ny + kDTY - 1) / kDTY);
    const int span = k_end - k_begin;
    auto it = op->dirplans.find(span);
    if (it == op->dirplans.end()) {
      int occ = 0;
      PCGX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, stencil7_dir_kernel, kDirThreads,
                                                              kDirSmem));
      it = op->dirplans.emplace(span, make_chunk_plan(op->c2plan, span, kz, tiles,
                                                      (long long)std::max(occ, 1) * c->sms, 2.5, false)).first;
    }
    const ChunkPlan& plan = forced ? *forced : it->second;
    check_red_grid((unsigned long long)tiles * plan.n);
    stencil7_dir_kernel<<<dim3((unsigned)tiles, (unsigned)plan.n), kDirThreads, kDirSmem, c->s>>>(
        mz, mp, mx, prm, k_begin, k_end, plan, make_red(c, slot, accumulate));
    check_launch();
    count_launch(c);
  };
  if (!lo && !hi) {
    launch(0, nzl, op->kz2, false);
    return;
  }
  // my first / last plane of z (and p_old) -> the neighbours' padding; the planes
  // that do not read a ghost run while they travel
  const long long nxy = op->nx * op->ny;
  CommBase::PlaneX items[2];
  int ni = 0;
  items[ni++] = {z, const_cast<double*>(z) - nxy, z + (long long)(nzl - 1) * nxy,
                 const_cast<double*>(z) + (long long)nzl * nxy, nxy};
  if (!first)
    items[ni++] = {pold, const_cast<double*>(pold) - nxy, pold + (long long)(nzl - 1) * nxy,
                   const_cast<double*>(pold) + (long long)nzl * nxy, nxy};
  c->cm->xchg(c, op, items, ni);
  c->cur_halo_bytes += (long long)((lo ? 1 : 0) + (hi ? 1 : 0)) * ni * nxy * 8;
  const int ib = lo ? std::min(1, nzl) : 0, ie = hi ? std::max(ib, nzl - 1) : nzl;
  bool wrote = false;
  if (ie > ib) {
    launch(ib, ie, op->kz2, false);
    wrote = true;
  }
  c->cm->halo_wait(c);
  if (ib > 0 && ie < nzl && ie > ib) {
    const ChunkPlan bp = strips_plan(ib, ie, nzl);
    launch(0, nzl, 1, wrote, &bp);
    return;
  }
  if (ib > 0) {
    launch(0, ib, 1, wrote);
    wrote = true;
  }
  if (ie < nzl) launch(ie, nzl, 1, wrote);
}

// One two-step pass over the local slab. On a z-slab rank the neighbours' two
// A planes (one B plane) per side are first exchanged into the vectors'
// padding; the chunks that do not read them run while the planes travel.
template <bool kFirst, bool kRed>
void cheb2_pass(pcgx_context c, pcgx_operator op, const double* A, const double* B,
                const double* R, Cheb2Params prm, int slot, bool xchg_r = false) {
  op->matvecs.fetch_add(2, std::memory_order_relaxed);
  const int nzl = (int)op->nzl;
  const bool lo = op->ghost_lo != nullptr, hi = op->ghost_hi != nullptr;
  prm.zoff = op->zpad;
  prm.a_lo = lo ? -2 : 0;
  prm.a_hi = hi ? nzl + 2 : nzl;
  prm.c_lo = lo ? -1 : 0;
  prm.c_hi = hi ? nzl + 1 : nzl;
  if (!lo && !hi) {
    cheb2_launch<kFirst, kRed>(c, op, A, B, R, prm, slot, 0, nzl, op->kz2, false);
    return;
  }
  const long long nxy = op->nx * op->ny;
  CommBase::PlaneX items[3];
  int ni = 0;
  items[ni++] = {A, const_cast<double*>(A) - 2 * nxy, A + (long long)(nzl - 2) * nxy,
                 const_cast<double*>(A) + (long long)nzl * nxy, 2 * nxy};
  if (!kFirst)
    items[ni++] = {B, const_cast<double*>(B) - nxy, B + (long long)(nzl - 1) * nxy,
                   const_cast<double*>(B) + (long long)nzl * nxy, nxy};
  // r(it) came out of a fused first pass, which writes own planes only: its boundary
  // plane travels with this pass's operands (the passes read one ghost plane of r)
  if (xchg_r)
    items[ni++] = {R, const_cast<double*>(R) - nxy, R + (long long)(nzl - 1) * nxy,
                   const_cast<double*>(R) + (long long)nzl * nxy, nxy};
  c->cm->xchg(c, op, items, ni);
  c->cur_halo_bytes +=
      (long long)((lo ? 1 : 0) + (hi ? 1 : 0)) * (2 + (kFirst ? 0 : 1) + (xchg_r ? 1 : 0)) * nxy * 8;
  const int ib = lo ? std::min(2, nzl) : 0, ie = hi ? std::max(ib, nzl - 2) : nzl;
  bool wrote = false;
  if (ie > ib) {
    cheb2_launch<kFirst, kRed>(c, op, A, B, R, prm, slot, ib, ie, op->kz2, false);
    wrote = true;
  }
  c->cm->halo_wait(c);
  if (ib > 0 && ie < nzl && ie > ib) {
    // both boundary strips in ONE launch (chunks [0, ib), [ib, ie) masked, [ie, nzl)):
    // they run side by side instead of one after the other; a reducing pass adds
    // their shares to the interior's (the masked CTAs contribute zeros)
    const ChunkPlan bp = strips_plan(ib, ie, nzl);
    cheb2_launch<kFirst, kRed>(c, op, A, B, R, prm, slot, 0, nzl, 2, wrote, &bp);
    return;
  }
  if (ib > 0) {
    cheb2_launch<kFirst, kRed>(c, op, A, B, R, prm, slot, 0, ib, 2, wrote);
    wrote = true;
  }
  if (ie < nzl) cheb2_launch<kFirst, kRed>(c, op, A, B, R, prm, slot, ie, nzl, 2, wrote);
}

// The PCG update r(it) = r(it-1) - alpha q(it) and r'r fused into the first
// two-step pass of P r(it) (pipelined kernel; one GPU or a z-slab rank): the pass reads r(it-1)
// and q(it) through TMA, forms r(it) in shared memory (bitwise the update kernel's
// element operations), writes it to rnew and reduces r'r into s_rr. Saves the
// update launch and 8 B per unknown and iteration.
struct CgUpd {
  const double* rold;
  const double* q;
  double* rnew;
  int s_rho, s_pq, s_rr;
};

bool cheb_upd_ok(pcgx_context c, pcgx_operator op, int m) {
  if (!(m >= 3 && op->kind == 0 && op->cheb2 && op->tune.fuse_upd != 0)) return false;
  if (!c->cm) return op->zpad == 0;
  // z-slab rank: r(it-1) and q(it) travel as two ghost planes per side (round 2)
  return op->zpad >= 2 && op->nzl >= 4 && op->tune.fuse_upd_slab != 0;
}

void cheb2f_upd_launch(pcgx_context c, pcgx_operator op, const CgUpd& u, Cheb2Params prm) {
  op->matvecs.fetch_add(2, std::memory_order_relaxed);
  const int nzl = (int)op->nzl;
  const bool lo = op->ghost_lo != nullptr, hi = op->ghost_hi != nullptr;
  prm.zoff = op->zpad;
  prm.a_lo = lo ? -2 : 0;
  prm.a_hi = hi ? nzl + 2 : nzl;
  prm.c_lo = lo ? -1 : 0;
  prm.c_hi = hi ? nzl + 1 : nzl;
  prm.S = c->S;
  prm.s_rho = u.s_rho;
  prm.s_pq = u.s_pq;
  prm.rout = u.rnew;
  auto kern = stencil7_cheb2f_kernel<true, false, true>;
  PCGX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kC2FSmem));
  const CUtensorMap ma = tmaps_for(op, u.rold).fa;
  const CUtensorMap mq = tmaps_for(op, u.q).fa;
  const long long tiles = ((op->nx + kC2TX - 1) / kC2TX) * ((op->ny + kFTY - 1) / kFTY);
  auto launch = [&](int k_begin, int k_end, bool accumulate, const ChunkPlan* forced = nullptr) {
    if (k_end <= k_begin) return;
    const int span = k_end - k_begin;
    auto it = op->c2plans.find(span);
    if (it == op->c2plans.end()) {
      int occ = 0;
      PCGX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kFThreads, kC2FSmem));
      it = op->c2plans.emplace(span, make_chunk_plan(op->c2plan, span, op->kz2, tiles,
                                                     (long long)std::max(occ, 1) * c->sms)).first;
    }
    const ChunkPlan& plan = forced ? *forced : it->second;
    check_red_grid((unsigned long long)tiles * plan.n);
    Reduce rr = make_red(c, u.s_rr, accumulate);
    if (c->cond_root && !c->cond_split) {  // the head of a conditional segment: r'r closes it
      rr.cond_bt = c->S + S_BNORM;
      rr.cond = c->cond_h;
    }
    kern<<<dim3((unsigned)tiles, (unsigned)plan.n), kFThreads, kC2FSmem, c->s>>>(
        ma, mq, ma, prm, k_begin, k_end, plan, Reduce{}, rr);
    check_launch();
    count_launch(c);
  };
  if (!lo && !hi) {
    launch(0, nzl, false);
    return;
  }
  // z-slab rank: my two boundary planes of r(it-1) and of q(it) -> the neighbours'
  // padding; the chunks that read no ghost plane run while they travel, the boundary
  // strips after the join (their r'r contributions accumulate in that order)
  const long long nxy = op->nx * op->ny;
  double* ro = const_cast<double*>(u.rold);
  double* qo = const_cast<double*>(u.q);
  CommBase::PlaneX items[2] = {
      {ro, ro - 2 * nxy, ro + (long long)(nzl - 2) * nxy, ro + (long long)nzl * nxy, 2 * nxy},
      {qo, qo - 2 * nxy, qo + (long long)(nzl - 2) * nxy, qo + (long long)nzl * nxy, 2 * nxy}};
  c->cm->xchg(c, op, items, 2);
  c->cur_halo_bytes += (long long)((lo ? 1 : 0) + (hi ? 1 : 0)) * 4 * nxy * 8;
  const int ib = lo ? std::min(2, nzl) : 0, ie = hi ? std::max(ib, nzl - 2) : nzl;
  bool wrote = false;
  if (ie > ib) {
    launch(ib, ie, false);
    wrote = true;
  }
  c->cm->halo_wait(c);
  if (ib > 0 && ie < nzl && ie > ib) {
    const ChunkPlan bp = strips_plan(ib, ie, nzl);
    launch(0, nzl, wrote, &bp);
    return;
  }
  if (ib > 0) {
    launch(0, ib, wrote);
    wrote = true;
  }
  if (ie < nzl) launch(ie, nzl, wrote);
}

// Tensor maps of the three-step pass, cached per buffer: kind 20 the A box
// (72 x (k3TY+6)), kind 21 the B / R boxes (68 x (k3TY+4)).
CUtensorMap cheb3_map(pcgx_operator op, const double* ptr, int kind) {
  for (auto& g : op->gmaps)
    if (g.ptr == ptr && g.kind == kind) return g.m;
  const CUtensorMap m = kind == 20 ? make_map(op, ptr, k3AW, k3AR) : make_map(op, ptr, k3W, k3R);
  op->gmaps.push_back({ptr, kind, m});
  return m;
}

bool cheb3_ok(pcgx_context c, pcgx_operator op) {
  return op->kind == 0 && op->cheb3 && op->zpad == 0 && c->nranks == 1;
}

// One three-step pass (stencil7_cheb3_kernel) over the slab: reads A = x_{k-1},
// B = x_{k-2}, R = r; writes x_{k+1} (prm.outE, unless nullptr) and x_{k+2} (prm.outF).
template <bool kRed>
void cheb3_pass(pcgx_context c, pcgx_operator op, const double* A, const double* B, const double* R,
                Cheb3Params prm, int slot) {
  op->matvecs.fetch_add(3, std::memory_order_relaxed);
  const int nzl = (int)op->nzl;
  prm.nx = (int)op->nx;
  prm.ny = (int)op->ny;
  prm.nzl = nzl;
  prm.nxy = op->nx * op->ny;
  prm.d = op->d;
  prm.zoff = 0;
  prm.a_lo = 0;
  prm.a_hi = nzl;
  prm.c_lo = 0;
  prm.c_hi = nzl;
  auto kern = stencil7_cheb3_kernel<kRed>;
  PCGX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k3Smem));
  const CUtensorMap ma = cheb3_map(op, A, 20);
  const CUtensorMap mb = cheb3_map(op, B, 21);
  const CUtensorMap mr = cheb3_map(op, R, 21);
  const long long tiles = ((op->nx + kC2TX - 1) / kC2TX) * ((op->ny + k3TY - 1) / k3TY);
  auto it = op->c3plans.find(nzl);
  if (it == op->c3plans.end()) {
    int occ = 0;
    PCGX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, k3Threads, k3Smem));
    it = op->c3plans.emplace(nzl, make_chunk_plan(op->c2plan, nzl, op->kz2, tiles,
                                                  (long long)std::max(occ, 1) * c->sms, 4.5)).first;
  }
  if (kRed) check_red_grid((unsigned long long)tiles * it->second.n);
  Reduce red = kRed ? make_red(c, slot, false) : Reduce{};
  kern<<<dim3((unsigned)tiles, (unsigned)it->second.n), k3Threads, k3Smem, c->s>>>(ma, mb, mr, prm, 0, nzl,
                                                                                   it->second, red);
  check_launch();
  count_launch(c);
}

// ---------------------------------------------------------------- Chebyshev apply

struct Cheb {
  int m = 0;
  double theta = 0, delta = 0, sigma = 0;
  std::vector<double> rho;
};

Cheb cheb_from(const pcgx_cheb* p) {
  Cheb c;
  c.m = p->m;
  c.theta = p->theta;
  c.delta = p->delta;
  c.sigma = p->sigma;
  if (p->m < 0) fail(PCGX_ERR_INVALID, "cheb_apply: m must be >= 0");
  if (p->m > 0 && !p->rho) fail(PCGX_ERR_INVALID, "cheb_apply: rho must have m+1 entries");
  if (p->rho) c.rho.assign(p->rho, p->rho + p->m + 1);
  return c;
}

// out = p_m(A) r (polyprec.cpp:169-198); rz_slot >= 0 also reduces r . out there.
// Uses c->w0, c->w1 as the recurrence workspace. out must not alias r, w0, w1.
void enqueue_cheb(pcgx_context c, pcgx_operator op, const Cheb& P, const double* r, double* out,
                  int rz_slot, const CgUpd* upd = nullptr, const std::function<void()>& after_first = {}) {
  // upd: r is r(it) = upd->rnew, produced by the first pass itself (cheb_upd_ok)
  const long long n = op->n_local;
  if (P.m == 0) {  // out = r / theta
    launch_zr(c, n, out, r, P.theta, 1, rz_slot >= 0 ? rz_slot : S_DOT2);
    return;
  }
  const double c1 = 2.0 * P.rho[1] / P.delta;
  const double c2 = 2.0 / P.delta;
  const double c3 = 2.0 * P.sigma;
  if (P.m == 1) {
    EpiChebFirst e{out, P.theta, c1, 1.0 / P.theta};
    if (rz_slot >= 0) op_launch<EpiChebFirst, true>(c, op, r, e, rz_slot);
    else op_launch<EpiChebFirst, false>(c, op, r, e, -1);
    return;
  }
  if (op->kind == 0 && op->cheb2) {
    // two steps per pass: (1,2), (3,4), ...; an odd last step runs single-step
    Cheb2Params q{};
    q.nx = (int)op->nx;
    q.ny = (int)op->ny;
    q.nzl = (int)op->nzl;
    q.nxy = op->nx * op->ny;
    q.d = op->d;
    q.theta = P.theta;
    q.c1 = c1;
    q.c2 = c2;
    q.c3 = c3;
    double* bufs[4] = {c->w0, c->w1, c->w2, c->w3};
    const bool last12 = (P.m == 2);
    q.rk2 = P.rho[2];
    q.rk2m1 = P.rho[1];
    q.outC = last12 ? nullptr : bufs[0];  // x_1 is dead after a last pass
    q.outE = last12 ? out : bufs[1];
    if (upd) cheb2f_upd_launch(c, op, *upd, q);
    else if (last12 && rz_slot >= 0) cheb2_pass<true, true>(c, op, r, nullptr, r, q, rz_slot);
    else cheb2_pass<true, false>(c, op, r, nullptr, r, q, -1);
    if (after_first) after_first();
    if (last12) return;
    int iold = 0, icur = 1;  // x_{k-2}, x_{k-1} buffer indices
    auto free_pair = [&](int& fa, int& fb) {
      fa = fb = -1;
      for (int b = 0; b < 4; ++b)
        if (b != iold && b != icur) (fa < 0 ? fa : fb) = b;
    };
    int k = 3;
    // PCGX_CHEB3=2: two-step passes, and an odd m ends with ONE three-step pass
    // (steps m-2 .. m, 32 B per unknown) instead of a two-step pass + a single step
    const bool tail3 = cheb3_ok(c, op) && op->tune.cheb3 == 2 && (P.m % 2) == 1 && P.m >= 5;
    if (cheb3_ok(c, op) && op->tune.cheb3 != 2) {
      // three steps per pass (cheb3.cuh); the m - 2 remaining steps split into
      // three-step passes and at most two two-step passes (never a single step
      // unless m == 3)
      const int rest = P.m - 2;
      int n3 = rest / 3, n2 = 0;
      if (rest % 3 == 2) n2 = 1;
      if (rest % 3 == 1 && n3 >= 1) {
        n3 -= 1;
        n2 = 2;
      }
      for (int pass = 0; pass < n3; ++pass, k += 3) {
        const bool last = (k + 2 == P.m);
        int fe, ff;
        free_pair(fe, ff);
        Cheb3Params q3{};
        q3.c2 = c2;
        q3.c3 = c3;
        q3.rk1 = P.rho[k];
        q3.rk1m1 = P.rho[k - 1];
        q3.rk2 = P.rho[k + 1];
        q3.rk2m1 = P.rho[k];
        q3.rk3 = P.rho[k + 2];
        q3.rk3m1 = P.rho[k + 1];
        q3.outE = last ? nullptr : bufs[fe];
        q3.outF = last ? out : bufs[ff];
        if (last && rz_slot >= 0) cheb3_pass<true>(c, op, bufs[icur], bufs[iold], r, q3, rz_slot);
        else cheb3_pass<false>(c, op, bufs[icur], bufs[iold], r, q3, -1);
        iold = fe;
        icur = ff;
      }
      for (int pass = 0; pass < n2; ++pass, k += 2) {
        const bool last = (k + 1 == P.m);
        int fc, fe;
        free_pair(fc, fe);
        q.rk1 = P.rho[k];
        q.rk1m1 = P.rho[k - 1];
        q.rk2 = P.rho[k + 1];
        q.rk2m1 = P.rho[k];
        q.outC = last ? nullptr : bufs[fc];
        q.outE = last ? out : bufs[fe];
        if (last && rz_slot >= 0) cheb2_pass<false, true>(c, op, bufs[icur], bufs[iold], r, q, rz_slot);
        else cheb2_pass<false, false>(c, op, bufs[icur], bufs[iold], r, q, -1);
        iold = fc;
        icur = fe;
      }
    }
    // slab rank after a fused first pass: r(it)'s ghost planes ride in the next pass's exchange
    bool xr = upd != nullptr && c->cm != nullptr;
    for (; k + 1 <= P.m; k += 2) {
      if (tail3 && k + 2 == P.m) break;
      const bool last = (k + 1 == P.m);
      int fc, fe;
      free_pair(fc, fe);
      q.rk1 = P.rho[k];
      q.rk1m1 = P.rho[k - 1];
      q.rk2 = P.rho[k + 1];
      q.rk2m1 = P.rho[k];
      q.outC = last ? nullptr : bufs[fc];
      q.outE = last ? out : bufs[fe];
      if (last && rz_slot >= 0) cheb2_pass<false, true>(c, op, bufs[icur], bufs[iold], r, q, rz_slot, xr);
      else cheb2_pass<false, false>(c, op, bufs[icur], bufs[iold], r, q, -1, xr);
      xr = false;
      iold = fc;
      icur = fe;
    }
    if (tail3 && k + 2 == P.m) {
      Cheb3Params q3{};
      q3.c2 = c2;
      q3.c3 = c3;
      q3.rk1 = P.rho[k];
      q3.rk1m1 = P.rho[k - 1];
      q3.rk2 = P.rho[k + 1];
      q3.rk2m1 = P.rho[k];
      q3.rk3 = P.rho[k + 2];
      q3.rk3m1 = P.rho[k + 1];
      q3.outE = nullptr;
      q3.outF = out;
      if (rz_slot >= 0) cheb3_pass<true>(c, op, bufs[icur], bufs[iold], r, q3, rz_slot);
      else cheb3_pass<false>(c, op, bufs[icur], bufs[iold], r, q3, -1);
      k += 3;
    }
    if (k == P.m) {  // odd remainder: x_m = step(x_{m-1}, x_{m-2}) -> out
      EpiChebStep e{r, bufs[iold], out, P.rho[k], P.rho[k - 1], c2, c3, P.theta, 0, 1.0 / P.theta};
      if (rz_slot >= 0) op_launch<EpiChebStep, true>(c, op, bufs[icur], e, rz_slot);
      else op_launch<EpiChebStep, false>(c, op, bufs[icur], e, -1);
    }
    return;
  }
  EpiChebFirst e1{c->w1, P.theta, c1, 1.0 / P.theta};
  op_launch<EpiChebFirst, false>(c, op, r, e1, -1);
  double* cur = c->w1;  // x_{k-1}
  double* old = c->w0;  // x_{k-2} (not yet materialised at k == 2)
  for (int k = 2; k <= P.m; ++k) {
    const bool last = (k == P.m);
    double* dst = last ? out : old;
    EpiChebStep e{r, old, dst, P.rho[k], P.rho[k - 1], c2, c3, P.theta, k == 2 ? 1 : 0,
                  1.0 / P.theta};
    if (last && rz_slot >= 0) op_launch<EpiChebStep, true>(c, op, cur, e, rz_slot);
    else op_launch<EpiChebStep, false>(c, op, cur, e, -1);
    old = cur;
    cur = dst;
  }
}

// ---------------------------------------------------------------- Newton form

struct Newton {
  int nlev = 0;
  std::vector<double> zeta;
};

Newton newton_from(const pcgx_newton* p) {
  if (!p) fail(PCGX_ERR_INVALID, "apply_newton: null parameters");
  if (p->nlev < 0) fail(PCGX_ERR_INVALID, "apply_newton: nlev must be >= 0");
  if (p->nlev > kNewtonMaxLev)
    fail(PCGX_ERR_UNSUPPORTED, "apply_newton: nlev > " + std::to_string(kNewtonMaxLev));
  if (!p->zeta) fail(PCGX_ERR_INVALID, "apply_newton: zeta must have nlev+1 entries");
  Newton N;
  N.nlev = p->nlev;
  N.zeta.assign(p->zeta, p->zeta + p->nlev + 1);
  return N;
}

void ensure_newton_ws(pcgx_context c, long long n, int nlev) {
  if (c->nl_n < n) {
    for (double* b : c->nl) cudaFree(b);
    c->nl.clear();
    c->nl_n = n;
  }
  while ((int)c->nl.size() < nlev) {
    double* b = nullptr;
    PCGX_CUDA(cudaMalloc(&b, sizeof(double) * (size_t)std::max(n, 1LL)));
    c->nl.push_back(b);
    c->ws_gen++;
    c->gcache.clear();
  }
}

// The reference recursion (newton_rec, polyprec.cpp:135-147) unrolled into its
// element-wise op sequence. Vector ids: -1 = r, -2 = out, k >= 0 = L[k].
struct NOp {
  int kind;  // 0: out = zeta0 * in ; 1: out = A in ; 2: out = zeta_j ((2 L[j-1]) - out)
  int out, in, j;
};
void newton_ops(int j, int in, int out, std::vector<NOp>& v) {
  if (j == 0) {
    v.push_back({0, out, in, 0});
    return;
  }
  newton_ops(j - 1, in, j - 1, v);  // L[j-1] = P_{j-1} in
  v.push_back({1, out, j - 1, 0});  // out = A L[j-1]
  newton_ops(j - 1, out, out, v);   // out = P_{j-1} out
  v.push_back({2, out, j - 1, j});  // out = zeta_j (2 L[j-1] - out)
}

// out = P_nlev(A) r; rz_slot >= 0 also reduces r . out. Every SpMV is fused with
// the element-wise ops that follow it: the level-0 scale of its output (written
// straight to L[0] when the output itself is dead) and the chain of combine
// steps on it (up to three in the epilogue, the rest in one element-wise pass).
// Same ops in the same order per element: bitwise the reference's values.
void enqueue_newton(pcgx_context c, pcgx_operator op, const Newton& N, const double* r,
                    double* out, int rz_slot) {
  const long long n = op->n_local;
  ensure_newton_ws(c, n, N.nlev);
  std::vector<NOp> ops;
  newton_ops(N.nlev, -1, -2, ops);
  auto vec = [&](int id) -> double* {
    return id == -1 ? const_cast<double*>(r) : id == -2 ? out : c->nl[(size_t)id];
  };
  const double* z = N.zeta.data();
  const bool red = rz_slot >= 0;
  size_t i = 0;
  while (i < ops.size()) {
    const NOp& o = ops[i];
    if (o.kind == 0) {  // the first op (level-0 scale of r), or the whole apply at nlev 0
      const bool rd = red && i + 1 == ops.size();
      if (rd) nscale_kernel<true><<<vec_grid(c, n), kVecThreads, 0, c->s>>>(n, vec(o.out), vec(o.in), z[0], make_red(c, rz_slot));
      else nscale_kernel<false><<<vec_grid(c, n), kVecThreads, 0, c->s>>>(n, vec(o.out), vec(o.in), z[0], Reduce{});
      check_launch();
      count_launch(c);
      ++i;
      continue;
    }
    if (o.kind != 1 || i + 1 >= ops.size() || ops[i + 1].kind != 0 || ops[i + 1].in != o.out)
      fail(PCGX_ERR_INVALID, "apply_newton: unexpected op sequence");
    const NOp& sc = ops[i + 1];
    if (sc.out != o.out) {  // out dead after its level-0 scale: write zeta0 * (A x) to L[0]
      EpiNewton e{vec(sc.out), nullptr, nullptr, z[0], 0.0, 0.0, 0.0, 0};
      op_launch<EpiNewton, false>(c, op, vec(o.in), e, -1);
      i += 2;
      continue;
    }
    size_t k = i + 2;
    int J = 0;
    while (k < ops.size() && ops[k].kind == 2 && ops[k].out == o.out) {
      if (ops[k].j != J + 1 || ops[k].in != J) fail(PCGX_ERR_INVALID, "apply_newton: bad chain");
      ++J;
      ++k;
    }
    if (J < 1 || o.in != 0) fail(PCGX_ERR_INVALID, "apply_newton: bad chain head");
    const bool rd = red && k == ops.size();
    const int jf = std::min(J, rd ? 2 : 3);
    EpiNewton e{vec(o.out), nullptr, nullptr, z[0], z[1], jf >= 2 ? z[2] : 0.0, jf >= 3 ? z[3] : 0.0, jf};
    if (jf >= 2) e.u1 = c->nl[1];
    if (jf >= 3) e.u2 = c->nl[2];
    const bool rd_here = rd && jf == J;
    if (rd_here) (jf <= 1 ? e.u1 : e.u2) = r;
    if (rd_here) op_launch<EpiNewton, true>(c, op, vec(o.in), e, rz_slot);
    else op_launch<EpiNewton, false>(c, op, vec(o.in), e, -1);
    if (J > jf) {
      NewtonChain ch{};
      ch.j0 = jf + 1;
      ch.j1 = J;
      for (int j = 0; j <= J; ++j) ch.zeta[j] = z[j];
      for (int j = 1; j <= J; ++j) ch.L[j - 1] = c->nl[(size_t)(j - 1)];
      if (rd) nchain_kernel<true><<<vec_grid(c, n), kVecThreads, 0, c->s>>>(n, vec(o.out), ch, r, make_red(c, rz_slot));
      else nchain_kernel<false><<<vec_grid(c, n), kVecThreads, 0, c->s>>>(n, vec(o.out), ch, r, Reduce{});
      check_launch();
      count_launch(c);
    }
    i = k;
  }
}

double spmv_alg_bytes(pcgx_operator op);

// Algorithmic bytes of one Newton application (same plan as enqueue_newton).
double newton_bytes(pcgx_operator op, int nlev, bool red) {
  std::vector<NOp> ops;
  newton_ops(nlev, -1, -2, ops);
  const double N8 = 8.0 * (double)op->n_local;
  const double spmv = spmv_alg_bytes(op);
  double b = 0.0;
  size_t i = 0;
  while (i < ops.size()) {
    if (ops[i].kind == 0) {
      b += 2 * N8;
      ++i;
      continue;
    }
    if (ops[i + 1].out != ops[i].out) {
      b += spmv;
      i += 2;
      continue;
    }
    size_t k = i + 2;
    int J = 0;
    while (k < ops.size() && ops[k].kind == 2 && ops[k].out == ops[i].out) ++J, ++k;
    const bool rd = red && k == ops.size();
    const int jf = std::min(J, rd ? 2 : 3);
    b += spmv + (double)(jf - 1) * N8 + ((rd && jf == J) ? N8 : 0.0);
    if (J > jf) b += (double)(2 + (J - jf) + (rd ? 1 : 0)) * N8;
    i = k;
  }
  return b;
}

// The preconditioner of a solve: none (plain CG), Chebyshev or Newton form.
struct Prec {
  int kind = 0;  // 0 none, 1 Chebyshev, 2 Newton
  Cheb cheb;
  Newton newton;
  int degree() const { return kind == 1 ? cheb.m : kind == 2 ? (1 << newton.nlev) - 1 : 0; }
};

void enqueue_prec(pcgx_context c, pcgx_operator op, const Prec& P, const double* r, double* out,
                  int rz_slot) {
  if (P.kind == 1) enqueue_cheb(c, op, P.cheb, r, out, rz_slot);
  else enqueue_newton(c, op, P.newton, r, out, rz_slot);
}

#include "host_solve.cuh"
// ---------------------------------------------------------------- power method / DACG
// Device restatements of the reference's bound estimators (eigenest.cpp:35-167):
// same iteration, same elementwise rounding, deterministic tree reductions; the
// host reads the reduced scalars once or twice per iteration and runs the
// scalar logic (convergence, restart, the 2x2 pencil) exactly as the reference.

// start_vector (eigenest.cpp:35-46) into v (this rank's rows).
void start_vector_device(pcgx_context c, pcgx_operator op, uint64_t seed, const char* who, double* v) {
  const long long n = op->n_local;
  const unsigned long long off = (unsigned long long)pcgx_operator_row0(op);
  for (int attempt = 0; attempt < 2; ++attempt) {
    splitmix_kernel<<<vec_grid(c, n), kVecThreads, 0, c->s>>>(n, seed + (uint64_t)attempt, off, v);
    check_launch();
    count_launch(c);
    launch_dot(c, n, v, v, S_DOT);
    allreduce(c, S_DOT, 1);
    fetch_scalars(c);
    const double nrm = std::sqrt(c->hS[S_DOT]);
    if (nrm != 0.0) {
      scale_div_kernel<<<vec_grid(c, n), kVecThreads, 0, c->s>>>(n, v, nrm);
      check_launch();
      count_launch(c);
      return;
    }
  }
  fail(PCGX_ERR_NUMERICAL, std::string(who) + ": zero starting vector");
}

// out = {value, iters, matvecs, converged}
void power_method_device(pcgx_context c, pcgx_operator op, double tol, int maxit, uint64_t seed,
                         double* out) {
  if (!(tol > 0.0)) fail(PCGX_ERR_INVALID, "power_method: tol must be positive");
  const long long n = op->n_local;
  ensure_workspace(c, n, ws_pad_of(op));
  double* v = c->t0;
  double* w = c->t1;
  double value = 0.0, matvecs = 0.0;
  int iters = 0, conv = 0;
  start_vector_device(c, op, seed, "power_method", v);
  double beta_old = 0.0;
  for (int it = 1; it <= maxit; ++it) {
    op_launch<EpiStore, true>(c, op, v, EpiStore{w}, S_DOT);  // w = A v, beta = v'w
    allreduce(c, S_DOT, 1);
    launch_dot(c, n, w, w, S_DOT2);
    allreduce(c, S_DOT2, 1);
    fetch_scalars(c);
    matvecs += 1.0;
    const double beta = c->hS[S_DOT];
    value = beta;
    iters = it;
    if (it > 1 && std::abs(beta - beta_old) <= tol * std::abs(beta)) {
      conv = 1;
      break;
    }
    beta_old = beta;
    double wn = std::sqrt(c->hS[S_DOT2]);
    if (wn == 0.0) {  // A v = 0 exactly: restart from seed + 1 (eigenest.cpp:67-75)
      start_vector_device(c, op, seed + 1, "power_method", v);
      op_launch<EpiStore, false>(c, op, v, EpiStore{w}, -1);
      matvecs += 1.0;
      launch_dot(c, n, w, w, S_DOT2);
      allreduce(c, S_DOT2, 1);
      fetch_scalars(c);
      wn = std::sqrt(c->hS[S_DOT2]);
      if (wn == 0.0) fail(PCGX_ERR_NUMERICAL, "power_method: operator annihilates the start vector");
    }
    div_copy_kernel<<<vec_grid(c, n), kVecThreads, 0, c->s>>>(n, v, w, wn);
    check_launch();
    count_launch(c);
  }
  out[0] = value;
  out[1] = iters;
  out[2] = matvecs;
  out[3] = conv;
}

void dacg_device(pcgx_context c, pcgx_operator op, double tol, int maxit, uint64_t seed,
                 double* out) {
  if (!(tol > 0.0)) fail(PCGX_ERR_INVALID, "dacg_smallest: tol must be positive");
  constexpr int kRestart = 50;
  const long long n = op->n_local;
  ensure_workspace(c, n, ws_pad_of(op));
  double* x = c->t0;
  double* ax = c->t1;
  double* p = c->w0;
  double* ap = c->w1;
  double value = 0.0, matvecs = 0.0;
  int iters = 0, conv = 0;
  start_vector_device(c, op, seed, "dacg_smallest", x);
  op_launch<EpiStore, true>(c, op, x, EpiStore{ax}, S_DOT);  // ax = A x, q = x'ax
  allreduce(c, S_DOT, 1);
  fetch_scalars(c);
  matvecs += 1.0;
  double q = c->hS[S_DOT];
  if (!(q > 0.0)) fail(PCGX_ERR_NUMERICAL, "dacg_smallest: x'Ax <= 0, operator not positive definite");
  double g_old_sq = 0.0;
  bool have_p = false;
  const int grid = vec_grid(c, n);
  for (int it = 0; it <= maxit; ++it) {
    value = q;
    iters = it;
    dacg_g_kernel<<<grid, kVecThreads, 0, c->s>>>(n, x, ax, q, make_red(c, S_E0));
    check_launch();
    count_launch(c);
    allreduce(c, S_E0, 2);
    fetch_scalars(c);
    const double resid = std::sqrt(c->hS[S_E0]) / q;
    if (resid <= tol) {
      conv = 1;
      break;
    }
    if (it == maxit) break;
    const double gsq = c->hS[S_E1];
    const bool restart = !have_p || it % kRestart == 0;
    dacg_p_kernel<<<grid, kVecThreads, 0, c->s>>>(n, x, ax, q, p, restart ? 0.0 : gsq / g_old_sq,
                                                  restart ? 1 : 0);
    check_launch();
    count_launch(c);
    have_p = true;
    g_old_sq = gsq;
    op_launch<EpiStore, true>(c, op, p, EpiStore{ap}, S_DOT);  // ap = A p, hpp = p'ap
    allreduce(c, S_DOT, 1);
    dot3_kernel<<<grid, kVecThreads, 0, c->s>>>(n, x, p, ap, make_red(c, S_E0));
    check_launch();
    count_launch(c);
    allreduce(c, S_E0, 3);
    fetch_scalars(c);
    matvecs += 1.0;
    const double hxx = q, hxp = c->hS[S_E0], hpp = c->hS[S_DOT];
    const double mxx = 1.0, mxp = c->hS[S_E1], mpp = c->hS[S_E2];
    if (!(hpp > 0.0))
      fail(PCGX_ERR_NUMERICAL, "dacg_smallest: p'Ap <= 0, operator not positive definite");
    const double a2 = mxx * mpp - mxp * mxp;
    const double a1 = -(hxx * mpp + hpp * mxx - 2.0 * hxp * mxp);
    const double a0 = hxx * hpp - hxp * hxp;
    const double disc = std::sqrt(std::max(0.0, a1 * a1 - 4.0 * a2 * a0));
    const double lambda = (-a1 - disc) / (2.0 * a2);
    const double r11 = hxx - lambda * mxx, r12 = hxp - lambda * mxp;
    const double r22 = hpp - lambda * mpp;
    double cx, cp;
    if (std::abs(r12) + std::abs(r22) > std::abs(r11) + std::abs(r12)) {
      cx = -r22;
      cp = r12;
    } else {
      cx = -r12;
      cp = r11;
    }
    if (cx == 0.0 && cp == 0.0) {
      cx = 1.0;
      cp = 0.0;
    }
    dacg_x_kernel<<<grid, kVecThreads, 0, c->s>>>(n, x, ax, p, ap, cx, cp, make_red(c, S_DOT2));
    check_launch();
    count_launch(c);
    allreduce(c, S_DOT2, 1);
    fetch_scalars(c);
    const double xnorm = std::sqrt(c->hS[S_DOT2]);
    if (xnorm == 0.0) fail(PCGX_ERR_NUMERICAL, "dacg_smallest: line search collapsed");
    dacg_norm_kernel<<<grid, kVecThreads, 0, c->s>>>(n, x, ax, xnorm, make_red(c, S_DOT));
    check_launch();
    count_launch(c);
    allreduce(c, S_DOT, 1);
    fetch_scalars(c);
    const double q_prev = q;
    q = c->hS[S_DOT];
    if (!(q > 0.0))
      fail(PCGX_ERR_NUMERICAL, "dacg_smallest: x'Ax <= 0, operator not positive definite");
    if (q > q_prev * (1.0 + 1e-12)) fail(PCGX_ERR_NUMERICAL, "dacg_smallest: Rayleigh quotient increased");
  }
  out[0] = value;
  out[1] = iters;
  out[2] = matvecs;
  out[3] = conv;
}

// ---------------------------------------------------------------- Lanczos

void lanczos_device(pcgx_context c, pcgx_operator op, int steps_hi, int steps, uint64_t seed,
                    double* lo, double* hi) {
  if (steps < 1 || steps_hi < 1 || steps_hi > steps)
    fail(PCGX_ERR_INVALID, "lanczos: need 1 <= steps_hi <= steps");
  const long long n = op->n_local;
  ensure_workspace(c, n, ws_pad_of(op));
  double* v = c->t0;
  double* vprev = c->t1;
  double* w = c->w0;
  const unsigned long long offset = (unsigned long long)pcgx_operator_row0(op);
  splitmix_kernel<<<vec_grid(c, n), kVecThreads, 0, c->s>>>(n, seed, offset, v);
  check_launch();
  count_launch(c);
  launch_dot(c, n, v, v, S_DOT);
  allreduce(c, S_DOT, 1);
  fetch_scalars(c);
  const double nv = std::sqrt(c->hS[S_DOT]);
  if (nv == 0.0) fail(PCGX_ERR_NUMERICAL, "lanczos: zero starting vector");
  scale_div_kernel<<<vec_grid(c, n), kVecThreads, 0, c->s>>>(n, v, nv);
  check_launch();
  launch_fill(c, n, vprev, 0.0);
  std::vector<double> a, bb;
  double bprev = 0.0;
  for (int j = 0; j < steps; ++j) {
    op_launch<EpiStore, true>(c, op, v, EpiStore{w}, S_DOT);  // w = A v, a = v'w
    allreduce(c, S_DOT, 1);
    lanczos_w_kernel<<<vec_grid(c, n), kVecThreads, 0, c->s>>>(n, w, v, vprev, c->S, S_DOT, bprev,
                                                              make_red(c, S_DOT2));
    check_launch();
    count_launch(c);
    allreduce(c, S_DOT2, 1);
    fetch_scalars(c);
    const double aj = c->hS[S_DOT];
    const double bj = std::sqrt(c->hS[S_DOT2]);
    a.push_back(aj);
    bb.push_back(bj);
    if (bj == 0.0) break;
    lanczos_shift_kernel<<<vec_grid(c, n), kVecThreads, 0, c->s>>>(n, v, vprev, w, bj);
    check_launch();
    count_launch(c);
    bprev = bj;
  }
  double l1, h1, l2, h2;
  const int k = (int)a.size();
  tridiag_extremes(std::min(k, steps_hi), a.data(), bb.data(), &l1, &h1);
  tridiag_extremes(k, a.data(), bb.data(), &l2, &h2);
  *hi = h1;
  *lo = l2;
}

#include "host_create.cuh"
}  // namespace

// ============================================================================ C ABI

extern "C" {

int pcgx_abi_version(void) { return PCGX_ABI_VERSION; }

const char* pcgx_last_error(pcgx_context ctx) {
  return ctx ? ctx->err.c_str() : g_thread_err.c_str();
}

pcgx_status pcgx_context_create(int device, pcgx_context* out) {
  return guarded(nullptr, [&] {
    if (!out) fail(PCGX_ERR_INVALID, "context_create: null out");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
      fail(PCGX_ERR_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    if (device < 0 || device >= ndev) fail(PCGX_ERR_INVALID, "context_create: bad device index");
    auto c = std::make_unique<pcgx_context_s>();
    c->device = device;
    ctx_init(c.get());
    *out = c.release();
  });
}

pcgx_status pcgx_nccl_unique_id(void* id128) {
  return guarded(nullptr, [&] {
    ncclUniqueId id;
    PCGX_NCCL(nccl().GetUniqueId(&id));
    std::memcpy(id128, &id, sizeof id);
  });
}

pcgx_status pcgx_context_create_dist(int device, int nranks, int rank, const void* nccl_id,
                                     pcgx_context* out) {
  return guarded(nullptr, [&] {
    if (nranks < 1 || rank < 0 || rank >= nranks)
      fail(PCGX_ERR_INVALID, "context_create_dist: bad rank/nranks");
    auto c = std::make_unique<pcgx_context_s>();
    c->device = device;
    c->rank = rank;
    c->nranks = nranks;
    ctx_init(c.get());
    // a 1-rank job has nothing to communicate; PCGX_FORCE_NCCL=1 still routes its
    // all-reduces through a 1-rank NCCL communicator (exercises the NCCL path on one GPU)
    if (nranks > 1 || env_int("PCGX_FORCE_NCCL", 0)) {
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, sizeof id);
      PCGX_NCCL(nccl().CommInitRank(&c->comm, nranks, id, rank));
      c->cm = new NcclComm();
    }
    *out = c.release();
  });
}

pcgx_status pcgx_context_create_host(int device, int nranks, int rank, const char* name, size_t mailbox_bytes,
                                     pcgx_context* out) {
  return guarded(nullptr, [&] {
    if (nranks < 1 || rank < 0 || rank >= nranks || !name || !out)
      fail(PCGX_ERR_INVALID, "context_create_host: bad rank/nranks/name");
    auto c = std::make_unique<pcgx_context_s>();
    c->device = device;
    c->rank = rank;
    c->nranks = nranks;
    ctx_init(c.get());
    if (nranks > 1)
      c->cm = host_comm_open(nranks, rank, name[0] == '/' ? std::string(name) : "/" + std::string(name),
                             mailbox_bytes ? mailbox_bytes : ((size_t)64 << 20));
    *out = c.release();
  });
}

pcgx_status pcgx_context_create_loopback(int device, int nranks, int rank, pcgx_context* out) {
  return guarded(nullptr, [&] {
    if (nranks < 2 || rank < 0 || rank >= nranks || !out)
      fail(PCGX_ERR_INVALID, "context_create_loopback: bad rank/nranks");
    auto c = std::make_unique<pcgx_context_s>();
    c->device = device;
    c->rank = rank;
    c->nranks = nranks;
    ctx_init(c.get());
    c->cm = new LoopbackComm();
    *out = c.release();
  });
}

pcgx_status pcgx_context_create_ipc(int device, int nranks, int rank, const char* name, size_t mailbox_bytes,
                                    pcgx_context* out) {
  return guarded(nullptr, [&] {
    if (nranks < 1 || rank < 0 || rank >= nranks || !name || !out)
      fail(PCGX_ERR_INVALID, "context_create_ipc: bad rank/nranks/name");
    auto c = std::make_unique<pcgx_context_s>();
    c->device = device;
    c->rank = rank;
    c->nranks = nranks;
    ctx_init(c.get());
    if (nranks > 1)
      c->cm = ipc_comm_open(c.get(), name[0] == '/' ? std::string(name) : "/" + std::string(name),
                            mailbox_bytes ? mailbox_bytes : ((size_t)64 << 20));
    *out = c.release();
  });
}

pcgx_status pcgx_local_group_create(int nranks, const int* devices, pcgx_context* out) {
  return guarded(nullptr, [&] {
    if (nranks < 1 || !out) fail(PCGX_ERR_INVALID, "local_group_create: bad nranks");
    int ndev = 0;
    PCGX_CUDA(cudaGetDeviceCount(&ndev));
    if (devices)
      for (int r = 0; r < nranks; ++r)
        if (devices[r] < 0 || devices[r] >= ndev)
          fail(PCGX_ERR_INVALID, "local_group_create: device " + std::to_string(devices[r]) + " of rank " +
                                     std::to_string(r) + " does not exist (" + std::to_string(ndev) +
                                     " devices)");
    // the group's scalar contributions live on rank 0's device and every rank's
    // group_sum_kernel reads them: ranks on other devices need peer access to it
    // (and halo copies between devices use it too)
    if (devices)
      for (int r = 0; r < nranks; ++r)
        for (int q = 0; q < nranks; ++q) {
          if (devices[r] == devices[q]) continue;
          int can = 0;
          PCGX_CUDA(cudaDeviceCanAccessPeer(&can, devices[r], devices[q]));
          if (!can)
            fail(PCGX_ERR_UNSUPPORTED, "local_group_create: device " + std::to_string(devices[r]) +
                                           " cannot access device " + std::to_string(devices[q]) +
                                           " (peer access)");
          PCGX_CUDA(cudaSetDevice(devices[r]));
          const cudaError_t e = cudaDeviceEnablePeerAccess(devices[q], 0);
          if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
          else PCGX_CUDA(e);
        }
    auto grp = std::make_shared<LocalGroup>(nranks);
    std::vector<std::unique_ptr<pcgx_context_s>> made;
    for (int r = 0; r < nranks; ++r) {
      auto c = std::make_unique<pcgx_context_s>();
      c->device = devices ? devices[r] : 0;
      c->rank = r;
      c->nranks = nranks;
      ctx_init(c.get());
      PCGX_CUDA(cudaEventCreateWithFlags(&grp->ev_ar[r], cudaEventDisableTiming));
      PCGX_CUDA(cudaEventCreateWithFlags(&grp->ev_done[r], cudaEventDisableTiming));
      grp->ctx[r] = c.get();
      made.push_back(std::move(c));
    }
    PCGX_CUDA(cudaSetDevice(grp->ctx[0]->device));
    PCGX_CUDA(cudaMalloc(&grp->contrib, sizeof(double) * kSlots * nranks));
    PCGX_CUDA(cudaMemset(grp->contrib, 0, sizeof(double) * kSlots * nranks));
    for (int r = 0; r < nranks; ++r) {
      made[r]->cm = new LocalComm(grp, r);
      out[r] = made[r].release();
    }
  });
}

void pcgx_context_destroy(pcgx_context c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->s);
  if (c->comm) nccl().CommDestroy(c->comm);
  delete c->cm;
  double* ws[] = {c->r, c->z, c->p, c->p2, c->q, c->w0, c->w1, c->w2, c->w3, c->t0, c->t1, c->r2};
  for (double* b : ws)
    if (b) cudaFree(b - c->ws_pad);
  double* bufs[] = {c->flush, c->S, c->partials};
  for (double* b : bufs)
    if (b) cudaFree(b);
  for (double* b : c->nl) cudaFree(b);
  cudaFree(c->counter);
  cudaFreeHost(c->hS);
  cudaEvent_t evs[] = {c->ev_t0, c->ev_t1, c->ev_sync, c->ev_fork, c->ev_join};
  for (auto e : evs)
    if (e) cudaEventDestroy(e);
  cudaStreamDestroy(c->s);
  cudaStreamDestroy(c->cs);
  delete c;
}

int pcgx_context_rank(pcgx_context c) { return c ? c->rank : -1; }
int pcgx_context_nranks(pcgx_context c) { return c ? c->nranks : -1; }
int64_t pcgx_kernel_launches(pcgx_context c) { return c ? c->launches : 0; }

int pcgx_chunk_plan(int span, int64_t tiles, int64_t slots, int long_chunks, int* heights) {
  if (span < 1 || tiles < 1 || slots < 1 || !heights) return 0;
  try {
    const ChunkPlan p = make_chunk_plan("", span, 32, tiles, slots, 2.5, long_chunks != 0);
    for (int i = 0; i < p.n; ++i) heights[i] = p.start[i + 1] - p.start[i];
    return p.n;
  } catch (...) {
    return 0;
  }
}

pcgx_status pcgx_synchronize(pcgx_context c) {
  return guarded(c, [&] {
    set_device(c);
    PCGX_CUDA(cudaStreamSynchronize(c->s));
  });
}

pcgx_status pcgx_device_alloc(pcgx_context c, size_t bytes, void** dptr) {
  return guarded(c, [&] {
    set_device(c);
    PCGX_CUDA(cudaMalloc(dptr, std::max<size_t>(bytes, 8)));
  });
}
pcgx_status pcgx_device_free(pcgx_context c, void* dptr) {
  return guarded(c, [&] {
    set_device(c);
    PCGX_CUDA(cudaFree(dptr));
  });
}
pcgx_status pcgx_memcpy_h2d(pcgx_context c, void* dst, const void* src, size_t bytes) {
  return guarded(c, [&] {
    set_device(c);
    PCGX_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->s));
    PCGX_CUDA(cudaStreamSynchronize(c->s));
  });
}
pcgx_status pcgx_memcpy_d2h(pcgx_context c, void* dst, const void* src, size_t bytes) {
  return guarded(c, [&] {
    set_device(c);
    PCGX_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->s));
    PCGX_CUDA(cudaStreamSynchronize(c->s));
  });
}
pcgx_status pcgx_memcpy_d2d(pcgx_context c, void* dst, const void* src, size_t bytes) {
  return guarded(c, [&] {
    set_device(c);
    PCGX_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, c->s));
  });
}
pcgx_status pcgx_host_alloc(size_t bytes, void** hptr) {
  return guarded(nullptr, [&] { PCGX_CUDA(cudaMallocHost(hptr, std::max<size_t>(bytes, 8))); });
}
pcgx_status pcgx_host_free(void* hptr) {
  return guarded(nullptr, [&] { PCGX_CUDA(cudaFreeHost(hptr)); });
}

pcgx_status pcgx_timer_start(pcgx_context c) {
  return guarded(c, [&] { PCGX_CUDA(cudaEventRecord(c->ev_t0, c->s)); });
}
pcgx_status pcgx_timer_stop(pcgx_context c, double* ms) {
  return guarded(c, [&] {
    PCGX_CUDA(cudaEventRecord(c->ev_t1, c->s));
    PCGX_CUDA(cudaEventSynchronize(c->ev_t1));
    float f = 0.f;
    PCGX_CUDA(cudaEventElapsedTime(&f, c->ev_t0, c->ev_t1));
    *ms = f;
  });
}
pcgx_status pcgx_flush_l2(pcgx_context c, size_t bytes) {
  return guarded(c, [&] {
    set_device(c);
    if (c->flush_bytes < bytes) {
      if (c->flush) cudaFree(c->flush);
      c->flush = nullptr;
      PCGX_CUDA(cudaMalloc(&c->flush, bytes));
      c->flush_bytes = bytes;
    }
    const long long n = (long long)(bytes / 8);
    flush_kernel<<<c->sms * 4, 256, 0, c->s>>>(n, c->flush);
    check_launch();
    count_launch(c);
  });
}

// balanced z-slabs: the first (nz % P) ranks own one extra plane
void pcgx_slab_partition(int64_t nz, int nranks, int rank, int64_t* z0, int64_t* nz_local) {
  const int64_t base = nz / nranks, extra = nz % nranks;
  *nz_local = base + (rank < extra ? 1 : 0);
  *z0 = rank * base + std::min<int64_t>(rank, extra);
}

pcgx_status pcgx_stencil7_create(pcgx_context c, int64_t nx, int64_t ny, int64_t nz,
                                 double inv_sqrt_diag, pcgx_operator* out) {
  return guarded(c, [&] {
    NvtxRange nvtx_r("pcgx::operator_create");
    set_device(c);
    if (nx < 1 || ny < 1 || nz < 1) fail(PCGX_ERR_INVALID, "StencilOperator: nx must be >= 1");
    if (nx > (1 << 30) || ny > (1 << 30) || nx * ny > (1LL << 31))
      fail(PCGX_ERR_UNSUPPORTED, "stencil7_create: plane nx*ny too large");
    if (nz < c->nranks) fail(PCGX_ERR_INVALID, "stencil7_create: fewer planes than ranks");
    auto op = new pcgx_operator_s();
    op->ctx = c;
    op->tune = Tuning::from_env();
    stencil_setup(c, op, nx, ny, nz, inv_sqrt_diag);
    PCGX_CUDA(cudaDeviceSynchronize());  // legacy-stream uploads / memsets before any compute-stream work
    *out = op;
  });
}

pcgx_status pcgx_csr_create(pcgx_context c, int64_t n, const int64_t* row_ptr,
                            const int64_t* col_idx, const double* values,
                            const double* inv_sqrt_diag, pcgx_operator* out) {
  return guarded(c, [&] {
    NvtxRange nvtx_r("pcgx::operator_create");
    set_device(c);
    auto op = new pcgx_operator_s();
    op->ctx = c;
    op->tune = Tuning::from_env();
    csr_create_any(c, op, n, row_ptr, col_idx, values, inv_sqrt_diag);
    PCGX_CUDA(cudaDeviceSynchronize());  // legacy-stream uploads / memsets before any compute-stream work
    *out = op;
  });
}

pcgx_status pcgx_csr_create_local(pcgx_context c, int64_t n, int64_t row0, int64_t n_local,
                                  const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                                  const double* inv_sqrt_diag, pcgx_operator* out) {
  return guarded(c, [&] {
    NvtxRange nvtx_r("pcgx::operator_create");
    set_device(c);
    if (!c->cm && c->nranks == 1 && (row0 != 0 || n_local != n))
      fail(PCGX_ERR_INVALID, "csr_create_local: a single rank owns all rows");
    auto op = new pcgx_operator_s();
    op->ctx = c;
    op->tune = Tuning::from_env();
    try {
      if (c->nranks == 1) {
        if (row_ptr && row_ptr[0] != 0) fail(PCGX_ERR_INVALID, "csr_create_local: row_ptr must start at 0");
        csr_upload(c, op, n, row_ptr, col_idx, values, inv_sqrt_diag);
      } else {
        csr_upload_local(c, op, n, row0, n_local, row_ptr, col_idx, values, inv_sqrt_diag);
      }
    } catch (...) {
      free_op(op);
      throw;
    }
    PCGX_CUDA(cudaDeviceSynchronize());
    *out = op;
  });
}

pcgx_status pcgx_csr_create_i32(pcgx_context c, int64_t n, const int32_t* row_ptr,
                                const int32_t* col_idx, const double* values,
                                const double* inv_sqrt_diag, pcgx_operator* out) {
  return guarded(c, [&] {
    NvtxRange nvtx_r("pcgx::operator_create");
    set_device(c);
    auto op = new pcgx_operator_s();
    op->ctx = c;
    op->tune = Tuning::from_env();
    csr_create_any(c, op, n, row_ptr, col_idx, values, inv_sqrt_diag);
    PCGX_CUDA(cudaDeviceSynchronize());  // legacy-stream uploads / memsets before any compute-stream work
    *out = op;
  });
}

void pcgx_operator_destroy(pcgx_operator op) {
  if (!op) return;
  cudaSetDevice(op->ctx->device);
  cudaStreamSynchronize(op->ctx->s);
  free_op(op);
}

int64_t pcgx_operator_size(pcgx_operator op) { return op ? op->n_global : -1; }
int64_t pcgx_operator_local_size(pcgx_operator op) { return op ? op->n_local : -1; }
int64_t pcgx_operator_z0(pcgx_operator op) { return op ? op->z0 : -1; }
int64_t pcgx_operator_row0(pcgx_operator op) {
  if (!op) return -1;
  return op->kind == 0 ? op->z0 * op->nx * op->ny : op->row0;
}
int64_t pcgx_operator_nnz(pcgx_operator op) { return op ? op->nnz : -1; }
int pcgx_operator_storage(pcgx_operator op) {
  if (!op) return -1;
  if (op->kind == 0) return 0;
  if (op->bsr_ptr) return op->b3g_val && op->tune.bsr3t != 0 ? 7 : 2;
  if (op->dia_val) return dia3_on(op) ? 6 : 5;
  if (op->sell_ptr) return 1;
  return 4;  // the chunked CSR kernel: only an empty (n = 0) matrix has no other storage
}
uint64_t pcgx_operator_matvec_count(pcgx_operator op) { return op ? op->matvecs.load() : 0; }

pcgx_status pcgx_operator_apply_device(pcgx_context c, pcgx_operator op, const double* x,
                                       double* y) {
  return guarded(c, [&] {
    NvtxRange nvtx_r("pcgx::operator_apply");
    set_device(c);
    op_launch<EpiStore, false>(c, op, x, EpiStore{y}, -1);
  });
}

pcgx_status pcgx_operator_apply(pcgx_context c, pcgx_operator op, const double* x, double* y) {
  return guarded(c, [&] {
    NvtxRange nvtx_r("pcgx::operator_apply");
    set_device(c);
    const long long n = op->n_local;
    ensure_workspace(c, n, ws_pad_of(op));
    PCGX_CUDA(cudaMemcpyAsync(c->t0, x, sizeof(double) * (size_t)n, cudaMemcpyHostToDevice, c->s));
    op_launch<EpiStore, false>(c, op, c->t0, EpiStore{c->t1}, -1);
    PCGX_CUDA(cudaMemcpyAsync(y, c->t1, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost, c->s));
    PCGX_CUDA(cudaStreamSynchronize(c->s));
  });
}

pcgx_status pcgx_cheb_params(double alpha, double beta, int m, double scale, double* tds,
                             double* rho) {
  std::string msg;
  const int st = pcgx::cheb_params(alpha, beta, m, scale, tds, rho, &msg);
  if (st) g_thread_err = msg;
  return (pcgx_status)st;
}

double pcgx_cheb_eval(const pcgx_cheb* p, double lambda) {
  return cheb_eval(p->theta, p->delta, p->sigma, p->rho, p->m, lambda);
}

pcgx_status pcgx_cheb_apply_device(pcgx_context c, pcgx_operator op, const pcgx_cheb* p,
                                   const double* r, double* out) {
  return guarded(c, [&] {
    NvtxRange nvtx_r("pcgx::cheb_apply");
    set_device(c);
    if (r == out) fail(PCGX_ERR_INVALID, "apply_chebyshev: out must not alias r");
    ensure_workspace(c, op->n_local, ws_pad_of(op));
    Cheb P = cheb_from(p);
    if (op->zpad) {  // the two-step kernel reads r's neighbour planes from padding
      copy_d2d(c, c->t0, r, op->n_local);
      r = c->t0;
    }
    enqueue_cheb(c, op, P, r, out, -1);
  });
}

pcgx_status pcgx_cheb_apply(pcgx_context c, pcgx_operator op, const pcgx_cheb* p, const double* r,
                            double* out) {
  return guarded(c, [&] {
    NvtxRange nvtx_r("pcgx::cheb_apply");
    set_device(c);
    const long long n = op->n_local;
    ensure_workspace(c, n, ws_pad_of(op));
    Cheb P = cheb_from(p);
    PCGX_CUDA(cudaMemcpyAsync(c->t0, r, sizeof(double) * (size_t)n, cudaMemcpyHostToDevice, c->s));
    enqueue_cheb(c, op, P, c->t0, c->t1, -1);
    PCGX_CUDA(cudaMemcpyAsync(out, c->t1, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost, c->s));
    PCGX_CUDA(cudaStreamSynchronize(c->s));
  });
}

pcgx_status pcgx_cheb_apply_steps(pcgx_context c, pcgx_operator op, const pcgx_cheb* p,
                                  const double* r, double* steps) {
  return guarded(c, [&] {
    set_device(c);
    const long long n = op->n_local;
    ensure_workspace(c, n, ws_pad_of(op));
    const Cheb P = cheb_from(p);
    PCGX_CUDA(cudaMemcpyAsync(c->t0, r, sizeof(double) * (size_t)n, cudaMemcpyHostToDevice, c->s));
    for (int j = 1; j <= P.m; ++j) {
      Cheb Pj = P;
      Pj.m = j;
      Pj.rho.resize((size_t)j + 1);
      enqueue_cheb(c, op, Pj, c->t0, c->t1, -1);
      PCGX_CUDA(cudaMemcpyAsync(steps + (size_t)(j - 1) * (size_t)n, c->t1, sizeof(double) * (size_t)n,
                                cudaMemcpyDeviceToHost, c->s));
    }
    PCGX_CUDA(cudaStreamSynchronize(c->s));
  });
}

pcgx_status pcgx_newton_params(double alpha0, double beta0, int nlev, double scale,
                               double* zeta) {
  std::string msg;
  const int st = pcgx::newton_params(alpha0, beta0, nlev, scale, zeta, &msg);
  if (st) g_thread_err = msg;
  return (pcgx_status)st;
}

double pcgx_newton_eval(const pcgx_newton* p, double lambda) {
  return newton_eval(p->zeta, p->nlev, lambda);
}

pcgx_status pcgx_chi_sequence(double alpha, double beta, int nlev, double* chi) {
  std::string msg;
  const int st = pcgx::chi_sequence(alpha, beta, nlev, chi, &msg);
  if (st) g_thread_err = msg;
  return (pcgx_status)st;
}

pcgx_status pcgx_newton_apply_device(pcgx_context c, pcgx_operator op, const pcgx_newton* p,
                                     const double* r, double* out) {
  return guarded(c, [&] {
    NvtxRange nvtx_r("pcgx::newton_apply");
    set_device(c);
    if (r == out) fail(PCGX_ERR_INVALID, "apply_newton: out must not alias r");
    Newton N = newton_from(p);
    enqueue_newton(c, op, N, r, out, -1);
  });
}

pcgx_status pcgx_newton_apply(pcgx_context c, pcgx_operator op, const pcgx_newton* p,
                              const double* r, double* out) {
  return guarded(c, [&] {
    NvtxRange nvtx_r("pcgx::newton_apply");
    set_device(c);
    const long long n = op->n_local;
    ensure_workspace(c, n, ws_pad_of(op));
    Newton N = newton_from(p);
    PCGX_CUDA(cudaMemcpyAsync(c->t0, r, sizeof(double) * (size_t)n, cudaMemcpyHostToDevice, c->s));
    enqueue_newton(c, op, N, c->t0, c->t1, -1);
    PCGX_CUDA(cudaMemcpyAsync(out, c->t1, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost, c->s));
    PCGX_CUDA(cudaStreamSynchronize(c->s));
  });
}

pcgx_status pcgx_mm_load(const char* path, pcgx_csr_host* out) {
  if (!path || !out) {
    g_thread_err = "load_matrix_market: null argument";
    return PCGX_ERR_INVALID;
  }
  std::string msg;
  const int st = pcgx::mm_load(path, out, &msg);
  if (st) g_thread_err = msg;
  return (pcgx_status)st;
}

pcgx_status pcgx_mm_load_text(const char* text, size_t len, const char* name, pcgx_csr_host* out) {
  if ((!text && len) || !out) {
    g_thread_err = "load_matrix_market: null argument";
    return PCGX_ERR_INVALID;
  }
  std::string msg;
  const int st = pcgx::mm_load_text(text, len, name, out, &msg);
  if (st) g_thread_err = msg;
  return (pcgx_status)st;
}

void pcgx_csr_host_free(pcgx_csr_host* m) {
  if (!m) return;
  std::free(m->row_ptr);
  std::free(m->col_idx);
  std::free(m->values);
  m->row_ptr = m->col_idx = nullptr;
  m->values = nullptr;
  m->n = m->nnz = 0;
}

pcgx_status pcgx_mm_save_text(int64_t n, const int64_t* rp, const int64_t* ci, const double* va,
                              char** text, size_t* len) {
  if (n < 0 || !rp || !text || !len) {
    g_thread_err = "save_matrix_market: invalid argument";
    return PCGX_ERR_INVALID;
  }
  std::string s;
  pcgx::mm_save_text(n, rp, ci, va, &s);
  char* buf = (char*)std::malloc(s.size() + 1);
  if (!buf) {
    g_thread_err = "save_matrix_market: out of memory";
    return PCGX_ERR_INVALID;
  }
  std::memcpy(buf, s.data(), s.size());
  buf[s.size()] = '\0';
  *text = buf;
  *len = s.size();
  return PCGX_OK;
}

void pcgx_free_text(char* text) { std::free(text); }

pcgx_status pcgx_mm_save(const char* path, int64_t n, const int64_t* rp, const int64_t* ci,
                         const double* va) {
  if (!path || n < 0 || !rp) {
    g_thread_err = "save_matrix_market: invalid argument";
    return PCGX_ERR_INVALID;
  }
  std::string s;
  pcgx::mm_save_text(n, rp, ci, va, &s);
  FILE* f = std::fopen(path, "wb");
  if (!f) {
    g_thread_err = std::string(path) + ": cannot open file for writing";
    return PCGX_ERR_PARSE;
  }
  const size_t w = std::fwrite(s.data(), 1, s.size(), f);
  std::fclose(f);
  if (w != s.size()) {
    g_thread_err = std::string(path) + ": write failed";
    return PCGX_ERR_PARSE;
  }
  return PCGX_OK;
}

void pcgx_solve_opts_default(pcgx_solve_opts* o) {
  o->tol = 1e-8;
  o->maxit = 20000;
  o->x0 = nullptr;
  o->flags = 0;
  o->on_iterate = nullptr;
  o->on_iterate_user = nullptr;
}

namespace {
Prec prec_of_cheb(const pcgx_cheb* p) {
  Prec P;
  if (p) {
    P.kind = 1;
    P.cheb = cheb_from(p);
  }
  return P;
}
Prec prec_of_newton(const pcgx_newton* p) {
  Prec P;
  if (p) {
    P.kind = 2;
    P.newton = newton_from(p);
  }
  return P;
}

pcgx_status solve_device_entry(pcgx_context c, pcgx_operator op, const Prec& P, const double* b,
                               double* x, const pcgx_solve_opts* opts, pcgx_report* rep) {
  set_device(c);
  if (!rep) fail(PCGX_ERR_INVALID, "pcg_solve: null report");
  pcg_solve_device(c, op, P, b, x, opts, rep);
  return PCGX_OK;
}

// Host-buffer entry: b and x live in t0 / t1 for the call (the solver uses r z p q w0..w3).
void solve_host_entry(pcgx_context c, pcgx_operator op, const Prec& P, const double* b, double* x,
                      const pcgx_solve_opts* opts, pcgx_report* rep) {
  set_device(c);
  if (!rep) fail(PCGX_ERR_INVALID, "pcg_solve: null report");
  const long long n = op->n_local;
  ensure_workspace(c, n, ws_pad_of(op));
  PCGX_CUDA(cudaMemcpyAsync(c->t0, b, sizeof(double) * (size_t)n, cudaMemcpyHostToDevice, c->s));
  pcgx_solve_opts o;
  pcgx_solve_opts_default(&o);
  if (opts) o = *opts;
  if (o.x0) {
    PCGX_CUDA(cudaMemcpyAsync(c->t1, o.x0, sizeof(double) * (size_t)n, cudaMemcpyHostToDevice, c->s));
    o.x0 = c->t1;
  }
  pcg_solve_device(c, op, P, c->t0, c->t1, &o, rep);
  PCGX_CUDA(cudaMemcpyAsync(x, c->t1, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost, c->s));
  PCGX_CUDA(cudaStreamSynchronize(c->s));
}
}  // namespace

pcgx_status pcgx_pcg_solve_device(pcgx_context c, pcgx_operator op, const pcgx_cheb* prec,
                                  const double* b, double* x, const pcgx_solve_opts* opts,
                                  pcgx_report* rep) {
  return guarded(c, [&] { solve_device_entry(c, op, prec_of_cheb(prec), b, x, opts, rep); });
}

pcgx_status pcgx_pcg_solve_newton_device(pcgx_context c, pcgx_operator op,
                                         const pcgx_newton* prec, const double* b, double* x,
                                         const pcgx_solve_opts* opts, pcgx_report* rep) {
  return guarded(c, [&] { solve_device_entry(c, op, prec_of_newton(prec), b, x, opts, rep); });
}

pcgx_status pcgx_pcg_solve_newton(pcgx_context c, pcgx_operator op, const pcgx_newton* prec,
                                  const double* b, double* x, const pcgx_solve_opts* opts,
                                  pcgx_report* rep) {
  return guarded(c, [&] { solve_host_entry(c, op, prec_of_newton(prec), b, x, opts, rep); });
}

pcgx_status pcgx_pcg_solve(pcgx_context c, pcgx_operator op, const pcgx_cheb* prec,
                           const double* b, double* x, const pcgx_solve_opts* opts,
                           pcgx_report* rep) {
  return guarded(c, [&] { solve_host_entry(c, op, prec_of_cheb(prec), b, x, opts, rep); });
}

pcgx_status pcgx_random_uniform_device(pcgx_context c, int64_t n, uint64_t seed, uint64_t offset,
                                       double* out) {
  return guarded(c, [&] {
    set_device(c);
    splitmix_kernel<<<vec_grid(c, n), kVecThreads, 0, c->s>>>(n, seed, offset, out);
    check_launch();
    count_launch(c);
  });
}

void pcgx_random_uniform(int64_t n, uint64_t seed, uint64_t offset, double* out) {
  random_uniform_host(n, seed, offset, out);
}

void pcgx_analytic_extremes(int dim, int64_t nx, int scaled, double* lo, double* hi) {
  analytic_extremes(dim, nx, scaled, lo, hi);
}

void pcgx_analytic_extremes_box(int64_t nx, int64_t ny, int64_t nz, double* lo, double* hi) {
  analytic_extremes_box(nx, ny, nz, lo, hi);
}

pcgx_status pcgx_power_method(pcgx_context c, pcgx_operator op, double tol, int maxit,
                              uint64_t seed, double* out4) {
  return guarded(c, [&] {
    NvtxRange nvtx_r("pcgx::power_method");
    set_device(c);
    power_method_device(c, op, tol, maxit, seed, out4);
  });
}

pcgx_status pcgx_dacg_smallest(pcgx_context c, pcgx_operator op, double tol, int maxit,
                               uint64_t seed, double* out4) {
  return guarded(c, [&] {
    NvtxRange nvtx_r("pcgx::dacg");
    set_device(c);
    dacg_device(c, op, tol, maxit, seed, out4);
  });
}

pcgx_status pcgx_lanczos_bounds(pcgx_context c, pcgx_operator op, int steps_hi, int steps,
                                uint64_t seed, double* lo, double* hi) {
  return guarded(c, [&] {
    NvtxRange nvtx_r("pcgx::lanczos");
    set_device(c);
    lanczos_device(c, op, steps_hi, steps, seed, lo, hi);
  });
}

}  // extern "C"
