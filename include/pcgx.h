/* SPDX-License-Identifier: Apache-2.0
 *
 * pcgx — B200-native Chebyshev-polynomial-preconditioned CG (the hot path of
 * arxiv 2008.01440's reference library `polycg`), exported as a plain C ABI:
 * no exceptions, no C++ or torch types, plain pointers and sizes.
 *
 * Each entry point replaces one reference interface (paths under
 * /root/reference/proj):
 *
 *   pcgx_stencil7_create   StencilOperator(lap3d, nx) + jacobi_scale
 *                          (include/polycg/linop.hpp:94-108, 145-168; src/linop.cpp:200-259, 340-351)
 *   pcgx_csr_create        CsrMatrix(n, row_ptr, col_idx, values) + jacobi_scale
 *                          (include/polycg/linop.hpp:60-85; src/linop.cpp:67-197, 340-351)
 *   pcgx_operator_apply    LinearOperator::apply on the ScaledOperator
 *                          (include/polycg/linop.hpp:26-28; src/linop.cpp:41-49, 271-275)
 *   pcgx_cheb_params       cheb_params + check_positivity (include/polycg/polyprec.hpp:50-54;
 *                          src/polyprec.cpp:13-23, 56-79)
 *   pcgx_cheb_apply        apply_chebyshev / ChebyshevPreconditioner::apply
 *                          (include/polycg/polyprec.hpp:86-90, pcg.hpp:42-55; src/polyprec.cpp:169-198)
 *   pcgx_pcg_solve         pcg_solve (include/polycg/pcg.hpp:57-91; src/pcg.cpp:10-117)
 *   pcgx_random_uniform    random_uniform_vector (include/polycg/eigenest.hpp:58-60; src/eigenest.cpp:13-30)
 *   pcgx_analytic_extremes analytic_extremes (include/polycg/linop.hpp:160-162; src/linop.cpp:382-390)
 *
 * Builder-defined entry points the reference lacks (BASELINE.json configs 3-5):
 * pcgx_lanczos_bounds, pcgx_analytic_extremes_box, pcgx_gen_fe27_*,
 * pcgx_gen_elast27_*, and the multi-GPU z-slab context (pcgx_context_create_dist).
 *
 * Threading contract (mirrors include/polycg/linop.hpp:17-20 and pcg.hpp:16-19):
 * a context owns one CUDA device, its streams, workspace and (optionally) an
 * NCCL communicator, and runs one call at a time; operator handles are immutable
 * after creation and may be shared read-only by calls on their own context.
 *
 * Errors: every call returns a pcgx_status; pcgx_last_error(ctx) returns the
 * message, whose text follows the reference's (e.g. "pcg_solve: p'Ap = ...").
 * PCGX_ERR_INVALID  <-> std::invalid_argument, PCGX_ERR_NUMERICAL <-> polycg::NumericalError.
 */
#ifndef PCGX_H
#define PCGX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PCGX_ABI_VERSION 1

typedef enum {
  PCGX_OK = 0,
  PCGX_ERR_INVALID = 1,     /* std::invalid_argument in the reference */
  PCGX_ERR_NUMERICAL = 2,   /* polycg::NumericalError in the reference */
  PCGX_ERR_CUDA = 3,        /* CUDA runtime failure (no device, OOM, fault) */
  PCGX_ERR_NCCL = 4,        /* communicator failure */
  PCGX_ERR_OVERFLOW = 5,    /* index does not fit the int32 device CSR */
  PCGX_ERR_UNSUPPORTED = 6, /* valid reference input this build does not accelerate */
  PCGX_ERR_PARSE = 7,       /* polycg::ParseError (MatrixMarket input), message has file:line */
  PCGX_ERR_CALLBACK = 8     /* the on_iterate callback asked to stop (it holds the reason) */
} pcgx_status;

typedef struct pcgx_context_s* pcgx_context;
typedef struct pcgx_operator_s* pcgx_operator;

/* ------------------------------------------------------------------ context */

int pcgx_abi_version(void);
/* Last error message of a context (or of the calling thread when ctx is NULL). */
const char* pcgx_last_error(pcgx_context ctx);

/* Single-GPU context on `device`. */
pcgx_status pcgx_context_create(int device, pcgx_context* out);
/* One rank of an nranks-GPU z-slab job (one process per GPU). `nccl_id` is the
 * 128-byte ncclUniqueId produced by pcgx_nccl_unique_id on rank 0 and broadcast
 * by the caller (bench.py uses torch.distributed for that plumbing). */
pcgx_status pcgx_nccl_unique_id(void* id128);
pcgx_status pcgx_context_create_dist(int device, int nranks, int rank, const void* nccl_id,
                                     pcgx_context* out);
/* P ranks of a z-slab job inside ONE process (devices[r] per rank, NULL = all
 * on device 0): halo planes move by stream-ordered copies and scalars are
 * reduced in rank order; each context must be driven by its own host thread
 * (every rank calls the same sequence, as with NCCL). Used to exercise the
 * multi-rank slab path on a single GPU. */
pcgx_status pcgx_local_group_create(int nranks, const int* devices, pcgx_context* out);
/* One rank of an nranks-process job on ONE host whose ranks exchange through a
 * POSIX shared-memory segment `name` (host-staged, synchronous; all ranks pass the
 * same name, rank 0 creates it). Ranks may share a GPU: no kernel or stream waits
 * on another rank. mailbox_bytes (0 = 64 MiB) bounds one message per rank. For
 * running the multi-process slab / block-row algorithm where NCCL cannot (several
 * ranks on one device); scalars are summed in rank order. */
pcgx_status pcgx_context_create_host(int device, int nranks, int rank, const char* name,
                                     size_t mailbox_bytes, pcgx_context* out);
/* One rank of an nranks-process job on ONE node whose ranks exchange through
 * DEVICE memory: each rank exports a device mailbox and its events by CUDA IPC;
 * halo planes, block-row segments and scalars are copied stream-ordered into the
 * sender's mailbox and pulled by the receivers' streams (peer-to-peer over NVLink
 * between GPUs), ordered by IPC events; the host only meets the peers at one
 * shared-memory barrier (segment `name`) per exchange. Ranks may be on different
 * GPUs (peer access required) or share one: no kernel waits on another rank.
 * mailbox_bytes (0 = 64 MiB) bounds one message per rank; scalars are summed in
 * rank order (bitwise pcgx_context_create_host / pcgx_local_group_create). */
pcgx_status pcgx_context_create_ipc(int device, int nranks, int rank, const char* name,
                                    size_t mailbox_bytes, pcgx_context* out);
/* MEASUREMENT ONLY: one process standing in for rank `rank` of an nranks-rank z-slab
 * job on a single GPU. Operators own that rank's slab and run the whole slab code
 * path (ghost planes, exchange on the comm stream, interior / boundary launches,
 * all-reduce points), but the neighbours' planes are the rank's own opposite boundary
 * planes copied on the device and an all-reduce keeps the local value: the slab with
 * periodic ghosts in z. Times the slab path's own overhead without a link
 * (tools/slab_overhead.py); matrix-free stencil operators only. */
pcgx_status pcgx_context_create_loopback(int device, int nranks, int rank, pcgx_context* out);
void pcgx_context_destroy(pcgx_context ctx);
int pcgx_context_rank(pcgx_context ctx);
int pcgx_context_nranks(pcgx_context ctx);
pcgx_status pcgx_synchronize(pcgx_context ctx);
/* Number of pcgx kernels launched on this context so far (all kinds). */
int64_t pcgx_kernel_launches(pcgx_context ctx);

/* Device memory helpers so a C/ctypes host needs no other CUDA binding. */
pcgx_status pcgx_device_alloc(pcgx_context ctx, size_t bytes, void** dptr);
pcgx_status pcgx_device_free(pcgx_context ctx, void* dptr);
pcgx_status pcgx_memcpy_h2d(pcgx_context ctx, void* dst, const void* src, size_t bytes);
pcgx_status pcgx_memcpy_d2h(pcgx_context ctx, void* dst, const void* src, size_t bytes);
pcgx_status pcgx_memcpy_d2d(pcgx_context ctx, void* dst, const void* src, size_t bytes);
/* Pinned host memory (page-locked), for the end-to-end path. */
pcgx_status pcgx_host_alloc(size_t bytes, void** hptr);
pcgx_status pcgx_host_free(void* hptr);

/* Device-side timing on the context's compute stream (CUDA events). */
pcgx_status pcgx_timer_start(pcgx_context ctx);
pcgx_status pcgx_timer_stop(pcgx_context ctx, double* ms);
/* Writes `bytes` through a scratch buffer on the compute stream (L2 flush). */
pcgx_status pcgx_flush_l2(pcgx_context ctx, size_t bytes);

/* ---------------------------------------------------------------- operators */

/* D^{-1/2} A D^{-1/2} for the 3D 7-point FD Laplacian (diag 6, off-diagonal -1,
 * homogeneous Dirichlet) on an nx*ny*nz grid, i fastest (StencilOperator(lap3d, nx)
 * is nx = ny = nz; non-cubic boxes are the builder extension for config 5 weak
 * scaling). inv_sqrt_diag: the constant jacobi_scale produces, or <= 0 for the
 * default 1/sqrt(6). On a dist context the rank owns the z-slab
 * [pcgx_operator_z0, z0 + nz_local) and every vector is that slab. */
pcgx_status pcgx_stencil7_create(pcgx_context ctx, int64_t nx, int64_t ny, int64_t nz,
                                 double inv_sqrt_diag, pcgx_operator* out);
/* The z-slab partition every rank uses (host-only): rank r of P owns planes
 * [z0, z0 + nz_local), balanced, the first nz % P ranks one plane more. */
void pcgx_slab_partition(int64_t nz, int nranks, int rank, int64_t* z0, int64_t* nz_local);
/* The z-chunk plan of the temporally blocked stencil passes (inspection / tests; host
 * only, no device needed): the heights of the chunks a launch over `span` planes is
 * cut into for `tiles` column tiles on `slots` resident CTAs, in dispatch order.
 * long_chunks != 0: the Chebyshev passes' search (a long first chunk when tiles <=
 * slots); 0: the direction step's. heights must hold 48 entries; returns the count. */
int pcgx_chunk_plan(int span, int64_t tiles, int64_t slots, int long_chunks, int* heights);

/* CsrMatrix (symmetric, both triangles, int64 host arrays as in the reference)
 * Jacobi-scaled. Narrowed to int32 on upload (PCGX_ERR_OVERFLOW if nnz >= 2^31).
 * On a multi-rank context every rank passes the FULL matrix and keeps the block
 * of rows [pcgx_operator_row0, + local_size) (balanced; vectors are that block);
 * the columns other ranks own travel as a per-neighbour halo before each SpMV.
 * inv_sqrt_diag (n entries) may be NULL: it is then computed exactly as
 * jacobi_scale does (1/sqrt(diag), NumericalError naming the first diag <= 0).
 * Structural invariants are validated as CsrMatrix::validate does (symmetry of
 * values is the caller's CsrMatrix contract and is not re-checked). */
pcgx_status pcgx_csr_create(pcgx_context ctx, int64_t n, const int64_t* row_ptr,
                            const int64_t* col_idx, const double* values,
                            const double* inv_sqrt_diag, pcgx_operator* out);
/* Block-row CsrMatrix from THIS rank's rows only (no rank holds the full matrix;
 * the paper's distributed layout): rows [row0, row0 + n_local)
 * of a symmetric n x n matrix, row0 / n_local = pcgx_slab_partition(n, nranks,
 * rank) -- or, on every rank alike, the partitions pcgx_csr_create cuts a full
 * matrix by to keep its fast storages: whole 3 x 3 block rows (3 x
 * pcgx_slab_partition(n / 3, ...): BSR-3) or whole node planes of an nx^3 grid
 * (nx^2 x pcgx_slab_partition(nx, ...): the offset storage on z-slabs, for the
 * 27-point box). row_ptr has n_local+1 entries (any base), col_idx global,
 * ascending per row. The symmetric pattern gives every rank its send / receive lists without
 * communication; the ghost columns' Jacobi values (inv_sqrt_diag: this rank's
 * n_local entries, or NULL = computed from the local diagonal) are exchanged once.
 * Bitwise the same operator as pcgx_csr_create with the full matrix. A single-rank
 * context takes the whole matrix (row0 = 0, n_local = n). */
pcgx_status pcgx_csr_create_local(pcgx_context ctx, int64_t n, int64_t row0, int64_t n_local,
                                  const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                                  const double* inv_sqrt_diag, pcgx_operator* out);
/* Same, from int32 host arrays (the builder's generators produce these). */
pcgx_status pcgx_csr_create_i32(pcgx_context ctx, int64_t n, const int32_t* row_ptr,
                                const int32_t* col_idx, const double* values,
                                const double* inv_sqrt_diag, pcgx_operator* out);
void pcgx_operator_destroy(pcgx_operator op);

int64_t pcgx_operator_size(pcgx_operator op);        /* global n */
int64_t pcgx_operator_local_size(pcgx_operator op);  /* rows owned by this rank */
int64_t pcgx_operator_z0(pcgx_operator op);          /* first owned plane (stencil) */
int64_t pcgx_operator_row0(pcgx_operator op);        /* first owned global row (any kind) */
int64_t pcgx_operator_nnz(pcgx_operator op);         /* CSR nnz, or the assembled-equivalent for stencils */
/* Device storage chosen at creation: 0 matrix-free 7-point stencil, 1 SELL-32 CSR,
 * 2 BSR-3 (aligned 3x3 blocks, detected), 3 CSR row tiles (TMA), 4 chunked CSR,
 * 5 offset (diagonal) storage (at most 32 distinct column offsets, detected),
 * 6 offset storage on a cubic grid whose offsets are the 27-point box or the
 *   7-point star (detected; applied by grid tiles with t = d x staged on chip),
 * 7 BSR-3 whose nodes form a cubic grid with the 27-point block box: the BSR-3
 *   arrays plus a grid copy the regular Chebyshev steps stream by TMA. */
int pcgx_operator_storage(pcgx_operator op);
/* Number of matvecs applied so far (LinearOperator::matvec_count, linop.hpp:37). */
uint64_t pcgx_operator_matvec_count(pcgx_operator op);

/* y = A_scaled x. Host buffers (the parity entry) ... */
pcgx_status pcgx_operator_apply(pcgx_context ctx, pcgx_operator op, const double* x, double* y);
/* ... and device buffers (stream-ordered on the context stream). */
pcgx_status pcgx_operator_apply_device(pcgx_context ctx, pcgx_operator op, const double* x,
                                       double* y);

/* --------------------------------------------------------- the polynomial */

typedef struct {
  int m;          /* degree: number of SpMVs per application */
  double theta;   /* scale * (alpha + beta) / 2 */
  double delta;   /* (beta - alpha) / 2 */
  double sigma;   /* theta / delta */
  const double* rho; /* rho[0..m] */
} pcgx_cheb;

/* cheb_params verbatim (bit-exact): tds = {theta, delta, sigma}, rho[m+1].
 * Validates 0 < alpha < beta, m >= 0, scale >= 1 and positivity on a 1000-point grid. */
pcgx_status pcgx_cheb_params(double alpha, double beta, int m, double scale, double* tds,
                             double* rho);
/* eval_poly (Chebyshev form), host scalar. */
double pcgx_cheb_eval(const pcgx_cheb* p, double lambda);

/* out = p_m(A) r. out must not alias r (polyprec.hpp:86-87). */
pcgx_status pcgx_cheb_apply(pcgx_context ctx, pcgx_operator op, const pcgx_cheb* p,
                            const double* r, double* out);
pcgx_status pcgx_cheb_apply_device(pcgx_context ctx, pcgx_operator op, const pcgx_cheb* p,
                                   const double* r, double* out);

/* The per-degree-step intermediates of apply_chebyshev (the
 * parity entry): steps[(j-1)*n .. j*n) = x_j = p_j(A) r for j = 1..m (host
 * buffers, n = local size). x_j is the degree-j output (the rho prefix does not
 * depend on m), computed by the device path at every j. */
pcgx_status pcgx_cheb_apply_steps(pcgx_context ctx, pcgx_operator op, const pcgx_cheb* p,
                                  const double* r, double* steps);

/* Newton form (polyprec.hpp:22-31): degree 2^nlev - 1, zeta[0..nlev]. */
typedef struct {
  int nlev;
  const double* zeta; /* zeta[0..nlev] */
} pcgx_newton;

/* newton_params verbatim (polyprec.cpp:27-54, bit-exact): zeta[nlev+1].
 * Validates 0 < alpha0 <= beta0, nlev >= 0, scale >= 1 and positivity. */
pcgx_status pcgx_newton_params(double alpha0, double beta0, int nlev, double scale,
                               double* zeta);
/* eval_poly, Newton form (polyprec.cpp:81-87). */
double pcgx_newton_eval(const pcgx_newton* p, double lambda);
/* chi_sequence (polyprec.cpp:102-123): chi[nlev], 0 <= nlev <= 30. */
pcgx_status pcgx_chi_sequence(double alpha, double beta, int nlev, double* chi);
/* out = P_nlev(A) r by the reference's depth-nlev recursion (apply_newton,
 * polyprec.cpp:135-160): exactly 2^nlev - 1 matvecs, bitwise the reference's
 * per-element values. out must not alias r. */
pcgx_status pcgx_newton_apply(pcgx_context ctx, pcgx_operator op, const pcgx_newton* p,
                              const double* r, double* out);
pcgx_status pcgx_newton_apply_device(pcgx_context ctx, pcgx_operator op, const pcgx_newton* p,
                                     const double* r, double* out);

/* ------------------------------------------------------------------ solver */

#define PCGX_FLAG_TIME_KERNELS 1u /* time every Chebyshev-step launch with CUDA events */
#define PCGX_FLAG_NO_GRAPH 2u     /* launch kernels one by one instead of CUDA graphs */

/* SolveOptions::on_iterate (pcg.hpp:62-63, called at pcg.cpp:88): after every
 * iteration with (iteration, current x). x is a HOST copy of the rank's x (n
 * values), valid during the call. Return 0 to continue; nonzero aborts the solve
 * with PCGX_ERR_CALLBACK (the caller rethrows what its callback caught). */
typedef int (*pcgx_iterate_fn)(int64_t iter, const double* x, int64_t n, void* user);

typedef struct {
  double tol;         /* SolveOptions::tol (default 1e-8) */
  int maxit;          /* SolveOptions::maxit (default 20000) */
  const double* x0;   /* initial guess (same memory space as b), NULL = zero */
  uint32_t flags;
  pcgx_iterate_fn on_iterate; /* NULL = none; otherwise x is kept current every
                                 iteration (no deferred x / fused update) and
                                 copied to the host for the call */
  void* on_iterate_user;
} pcgx_solve_opts;

typedef struct {
  /* SolveReport (pcg.hpp:73-82), counted by the reference's rules */
  int64_t iters;
  int64_t ddot;
  int64_t matvec;
  int64_t prec_applies;
  double rel_res;
  double true_rel_res;
  double wall_time;    /* seconds, device events around the solve (pcg.cpp:20-30) */
  int64_t converged;
  /* builder extensions */
  int64_t kernel_launches;   /* pcgx kernels launched by this solve */
  int64_t wasted_matvec;     /* speculative P applications discarded at convergence */
  int64_t allreduces;        /* NCCL all-reduce calls (0 on one GPU) */
  int64_t halo_bytes;        /* bytes sent to z-neighbours */
  double alg_bytes;          /* algorithmic HBM bytes of the solve */
  double spmv_equiv_bytes;   /* matvec * SpMV-equivalent bytes (the BASELINE metric numerator) */
  double step_ms;            /* total device ms of timed Chebyshev-step launches */
  int64_t step_launches;     /* number of timed Chebyshev-step launches */
  double step_bytes;         /* algorithmic bytes per Chebyshev-step launch */
  int64_t step_steps;        /* Chebyshev degree steps per timed launch (1, 2 or 3) */
} pcgx_report;

void pcgx_solve_opts_default(pcgx_solve_opts* o);

/* pcg_solve. prec NULL = plain CG. Host buffers (end-to-end entry: b is copied
 * to the device, x back, inside the call). */
pcgx_status pcgx_pcg_solve(pcgx_context ctx, pcgx_operator op, const pcgx_cheb* prec,
                           const double* b, double* x, const pcgx_solve_opts* opts,
                           pcgx_report* rep);
/* Same with b, x (and opts->x0) already resident in device memory. */
pcgx_status pcgx_pcg_solve_device(pcgx_context ctx, pcgx_operator op, const pcgx_cheb* prec,
                                  const double* b, double* x, const pcgx_solve_opts* opts,
                                  pcgx_report* rep);

/* pcg_solve with a NewtonPreconditioner (pcg.hpp:27-40); counters as above with
 * degree 2^nlev - 1. */
pcgx_status pcgx_pcg_solve_newton(pcgx_context ctx, pcgx_operator op, const pcgx_newton* prec,
                                  const double* b, double* x, const pcgx_solve_opts* opts,
                                  pcgx_report* rep);
pcgx_status pcgx_pcg_solve_newton_device(pcgx_context ctx, pcgx_operator op,
                                         const pcgx_newton* prec, const double* b, double* x,
                                         const pcgx_solve_opts* opts, pcgx_report* rep);

/* ------------------------------------------------------- MatrixMarket files */

/* Host CSR arrays (int64, as CsrMatrix stores them, linop.hpp:72-74), owned by
 * the library: release with pcgx_csr_host_free. */
typedef struct {
  int64_t n, nnz;
  int64_t* row_ptr; /* n+1 */
  int64_t* col_idx; /* nnz */
  double* values;   /* nnz */
} pcgx_csr_host;

/* load_matrix_market(path) (matrix_market.cpp:55-59, 61-166): coordinate real,
 * symmetric (lower triangle) or general with symmetric content, 1-based; the
 * symmetrised CSR with both triangles. Errors: PCGX_ERR_PARSE with the
 * reference's "name:line: what" message. Multithreaded parse. */
pcgx_status pcgx_mm_load(const char* path, pcgx_csr_host* out);
/* load_matrix_market(istream, name): the same from an in-memory text. */
pcgx_status pcgx_mm_load_text(const char* text, size_t len, const char* name, pcgx_csr_host* out);
void pcgx_csr_host_free(pcgx_csr_host* m);
/* save_matrix_market (matrix_market.cpp:172-199): lower triangle, "%.16e" values,
 * byte-identical to the reference's output; load(save(m)) == m. */
pcgx_status pcgx_mm_save(const char* path, int64_t n, const int64_t* row_ptr,
                         const int64_t* col_idx, const double* values);
/* ... into a library-owned text buffer (release with pcgx_free_text). */
pcgx_status pcgx_mm_save_text(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                              const double* values, char** text, size_t* len);
void pcgx_free_text(char* text);

/* ------------------------------------------------------- inputs and bounds */

/* random_uniform_vector elements [offset, offset + n) into device memory. */
pcgx_status pcgx_random_uniform_device(pcgx_context ctx, int64_t n, uint64_t seed,
                                       uint64_t offset, double* out);
/* Host version (bit-identical). */
void pcgx_random_uniform(int64_t n, uint64_t seed, uint64_t offset, double* out);

/* analytic_extremes (dim 2 or 3, cubic). */
void pcgx_analytic_extremes(int dim, int64_t nx, int scaled, double* lo, double* hi);
/* Scaled 3D box nx*ny*nz: (2/3) sum_d sin^2(pi h_d/2), (2/3) sum_d cos^2(pi h_d/2). */
void pcgx_analytic_extremes_box(int64_t nx, int64_t ny, int64_t nz, double* lo, double* hi);

/* Lanczos bound estimate on the device: start vector = normalised
 * random_uniform_vector(n, seed); `steps` three-term steps without
 * reorthogonalisation; hi = largest Ritz value of the leading steps_hi x steps_hi
 * tridiagonal, lo = smallest Ritz value of the full steps x steps one. */
pcgx_status pcgx_lanczos_bounds(pcgx_context ctx, pcgx_operator op, int steps_hi, int steps,
                                uint64_t seed, double* lo, double* hi);

/* power_method and dacg_smallest (include/polycg/eigenest.hpp:29-45;
 * src/eigenest.cpp:48-167) on the device: same iteration and stopping rules,
 * the seeded start vector of random_uniform_vector; out4 = {value, iters,
 * matvecs, converged} (EigResult). Errors as the reference (NumericalError on
 * an indefinite operator). */
pcgx_status pcgx_power_method(pcgx_context ctx, pcgx_operator op, double tol, int maxit,
                              uint64_t seed, double* out4);
pcgx_status pcgx_dacg_smallest(pcgx_context ctx, pcgx_operator op, double tol, int maxit,
                               uint64_t seed, double* out4);

/* --------------------------------------------------- config generators */

/* Config 3: heterogeneous diffusion, Q1 (trilinear) finite elements on the
 * (nx+1)^3 cells of the unit cube, nx^3 interior nodes (Dirichlet boundary
 * eliminated) -> 27-point rows. Cell coefficient kappa_c = exp(sigma * N(0,1)),
 * N(0,1) by Box-Muller on splitmix64(seed). Values are assembled so that
 * a_ij == a_ji bitwise. Sizes first, then fill into caller arrays. */
pcgx_status pcgx_gen_fe27_size(int64_t nx, int64_t* n, int64_t* nnz);
pcgx_status pcgx_gen_fe27_fill(int64_t nx, double sigma, uint64_t seed, int32_t* row_ptr,
                               int32_t* col_idx, double* values);
/* Config 4: 3 dof per node, Q1 linear elasticity (Lame lambda, mu) on the same
 * mesh, element stiffness scaled per cell by (1 + eps * u_c), u_c uniform [0,1)
 * from seed (keeps every element PSD, the assembled matrix SPD). Rows are 3x3
 * blocks over the 27 neighbours: 81 entries per interior row. */
pcgx_status pcgx_gen_elast27_size(int64_t nx, int64_t* n, int64_t* nnz);
pcgx_status pcgx_gen_elast27_fill(int64_t nx, double lambda, double mu, double eps,
                                  uint64_t seed, int32_t* row_ptr, int32_t* col_idx,
                                  double* values);

#ifdef __cplusplus
}
#endif
#endif /* PCGX_H */
