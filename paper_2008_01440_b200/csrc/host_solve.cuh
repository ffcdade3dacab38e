// SPDX-License-Identifier: Apache-2.0
//
// Part of pcgx.cu (ONE translation unit): included in place, in the middle of that
// file's declarations; not a standalone header. pcg_solve_device: the PCG loop, its CUDA graphs and device-side convergence.
#pragma once

// ---------------------------------------------------------------- PCG

template <class F>
void capture(pcgx_context c, Graph& g, F&& body) {
  const int64_t before = c->cur_launches;
  const int64_t before_ar = c->cur_allreduce;
  PCGX_CUDA(cudaStreamBeginCapture(c->s, cudaStreamCaptureModeThreadLocal));
  c->capturing = true;
  try {
    body();
    c->capturing = false;
  } catch (...) {
    c->capturing = false;
    cudaGraph_t tmp;
    cudaStreamEndCapture(c->s, &tmp);
    if (tmp) cudaGraphDestroy(tmp);
    throw;
  }
  cudaGraph_t graph;
  PCGX_CUDA(cudaStreamEndCapture(c->s, &graph));
  PCGX_CUDA(cudaGraphInstantiate(&g.exec, graph, 0));
  cudaGraphDestroy(graph);
  g.kernels = c->cur_launches - before;
  c->cur_launches = before;  // counted per replay instead
  c->launches -= g.kernels;
  g.allreduces = c->cur_allreduce - before_ar;
  c->cur_allreduce = before_ar;
}

// Capture of a PCG segment whose tail runs only while the solve has not
// converged: body() enqueues the head, calls cond_split(c) once (after the kernel
// that writes the convergence flag), then the tail. The head is captured into the
// root graph, the tail into the body graph of an IF node that follows it, so at
// convergence the device skips the tail (the speculative P r and A p of the
// reference's stopping iteration, pcg.cpp:89-95) instead of computing and
// discarding it.
template <class F>
void capture_cond(pcgx_context c, Graph& g, F&& body) {
  const int64_t before = c->cur_launches;
  const int64_t before_ar = c->cur_allreduce;
  cudaGraph_t root = nullptr;
  PCGX_CUDA(cudaGraphCreate(&root, 0));
  c->cond_root = root;
  c->cond_split = false;
  c->cond_mark = 0;
  try {
    PCGX_CUDA(cudaGraphConditionalHandleCreate(&c->cond_h, root, 1u, cudaGraphCondAssignDefault));
    PCGX_CUDA(cudaStreamBeginCaptureToGraph(c->s, root, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    c->capturing = true;
    body();
    c->capturing = false;
    cudaGraph_t tmp = nullptr;
    PCGX_CUDA(cudaStreamEndCapture(c->s, &tmp));
    if (!c->cond_split) fail(PCGX_ERR_CUDA, "capture_cond: the segment never split");
    PCGX_CUDA(cudaGraphInstantiate(&g.exec, root, 0));
  } catch (...) {
    c->capturing = false;
    cudaStreamCaptureStatus st;
    if (cudaStreamIsCapturing(c->s, &st) == cudaSuccess && st != cudaStreamCaptureStatusNone) {
      cudaGraph_t tmp = nullptr;
      cudaStreamEndCapture(c->s, &tmp);
    }
    cudaGetLastError();
    cudaGraphDestroy(root);
    c->cond_root = nullptr;
    throw;
  }
  cudaGraphDestroy(root);
  c->cond_root = nullptr;
  g.kernels = c->cur_launches - before;
  g.body_kernels = c->cur_launches - c->cond_mark;
  c->cur_launches = before;
  c->launches -= g.kernels;
  g.allreduces = c->cur_allreduce - before_ar;
  c->cur_allreduce = before_ar;
}

__global__ void cond_kernel(cudaGraphConditionalHandle h, const double* S, int slot_rr, int slot_bnorm,
                            int slot_tol) {
  // the host's test, same operations: rel_res = sqrt(r'r) / ||b||; stop iff <= tol
  const double rel = sqrt(S[slot_rr]) / S[slot_bnorm];
  cudaGraphSetConditional(h, rel <= S[slot_tol] ? 0u : 1u);
}

// Inside capture_cond's body: the convergence flag from S[slot_rr], then the IF
// node; everything enqueued after this runs only if the solve goes on.
// with_kernel = false: the reducing block of the preceding launch already set the
// condition (Reduce::cond_bt, the fused first pass's r'r)
void cond_split(pcgx_context c, int slot_rr, bool with_kernel = true) {
  if (with_kernel) {
    cond_kernel<<<1, 1, 0, c->s>>>(c->cond_h, c->S, slot_rr, S_BNORM, S_TOL);
    check_launch();
    count_launch(c);
  }
  cudaStreamCaptureStatus st;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  PCGX_CUDA(cudaStreamGetCaptureInfo(c->s, &st, nullptr, nullptr, &deps, &nd));
  std::vector<cudaGraphNode_t> dv(deps, deps + nd);
  cudaGraphNodeParams cp{};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = c->cond_h;
  cp.conditional.type = cudaGraphCondTypeIf;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  PCGX_CUDA(cudaGraphAddNode(&node, c->cond_root, dv.data(), dv.size(), &cp));
  cudaGraph_t tmp = nullptr;
  PCGX_CUDA(cudaStreamEndCapture(c->s, &tmp));
  PCGX_CUDA(cudaStreamBeginCaptureToGraph(c->s, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                          cudaStreamCaptureModeThreadLocal));
  c->cond_split = true;
  c->cond_mark = c->cur_launches;
}

void replay(pcgx_context c, Graph& g) {
  PCGX_CUDA(cudaGraphLaunch(g.exec, c->s));
  c->cur_launches += g.kernels;
  c->launches += g.kernels;
  c->cur_allreduce += g.allreduces;
}

std::string fmt_double(double v) { return std::to_string(v); }

// Matrix bytes of one pass in the device storage: int32 CSR 12 nnz + 4 (n+1);
// BSR-3 8 nnz + 4 per block + 4 per block row; stencil none.
double matrix_bytes(pcgx_operator op) {
  if (op->kind == 0) return 0.0;
  // the grid copy the regular steps stream (bsr3t_kernel): every slot of every node
  // (absent blocks as zeros) + the masks; the other launches' SELL arrays are ~4% larger
  if (op->b3g_val && op->tune.bsr3t != 0)
    return 8.0 * 243.0 * (double)(op->n_local / 3) + 4.0 * (double)(op->n_local / 3);
  if (op->bsr_ptr)
    return 8.0 * (double)op->nnz + 4.0 * (double)op->bsr_blocks + 4.0 * (double)(op->n_local / 3 + 1);
  if (op->dia_val) return 8.0 * (double)op->dia_k * (double)op->n_local + 4.0 * (double)op->n_local;
  return 12.0 * (double)op->nnz + 4.0 * (double)(op->n_local + 1);
}
// SpMV-equivalent bytes, the BASELINE metric's numerator: stencil
// 16 B/unknown (read x, write y); CSR 12 nnz + 4 (n+1) + 16 n whatever the storage.
double spmv_equiv_bytes(pcgx_operator op) {
  if (op->kind == 0) return 16.0 * (double)op->n_local;
  return 12.0 * (double)op->nnz + 4.0 * (double)(op->n_local + 1) + 16.0 * (double)op->n_local;
}
// Algorithmic bytes of one SpMV pass in the actual storage (read x, write y).
double spmv_alg_bytes(pcgx_operator op) { return matrix_bytes(op) + 16.0 * (double)op->n_local; }
// Fused Chebyshev middle step: stencil 32 B/unknown; CSR / BSR matrix bytes + 32 n
// (+ 8 n for the inv_sqrt_diag vector read with the row).
double cheb_step_bytes(pcgx_operator op) {
  if (op->kind == 0) return 32.0 * (double)op->n_local;
  return matrix_bytes(op) + 40.0 * (double)op->n_local;
}

void pcg_solve_device(pcgx_context c, pcgx_operator op, const Prec& prec, const double* b,
                      double* x, const pcgx_solve_opts* o, pcgx_report* rep) {
  NvtxRange nvtx_solve("pcgx::pcg_solve");
  if (op->ctx != c) fail(PCGX_ERR_INVALID, "pcg_solve: operator belongs to another context");
  pcgx_solve_opts opts;
  pcgx_solve_opts_default(&opts);
  if (o) opts = *o;
  if (!(opts.tol > 0.0)) fail(PCGX_ERR_INVALID, "pcg_solve: tol must be positive");
  if (opts.maxit < 1) fail(PCGX_ERR_INVALID, "pcg_solve: maxit must be >= 1");
  const bool have_prec = prec.kind != 0;
  const Cheb& P = prec.cheb;
  const int m = prec.degree();
  const long long n = op->n_local;
  ensure_workspace(c, n, ws_pad_of(op));
  // CUDA graphs on one GPU; multi-rank solves launch directly by default (the
  // speculative schedule hides the launches either way; PCGX_GRAPH_MULTI=1 captures
  // the NCCL plane exchanges and all-reduces into the graphs too)
  const bool use_graph = !(opts.flags & PCGX_FLAG_NO_GRAPH) && op->tune.no_graph == 0 &&
                         (!c->cm || (c->cm->graph_capturable() && op->tune.graph_multi != 0));
  // one GPU: snapshot r'r right after the update and overlap the host check with
  // the speculative P r; multi-GPU: merge [r'r, r'z] into one all-reduce after P r
  // (PCGX_MERGED=1 forces the multi-GPU schedule on one GPU, for tests)
  const bool spec_after_update = !c->cm && op->tune.merged == 0;
  // one GPU with graphs: the speculative tail of each segment (P r and A p of the
  // next iteration) sits in a conditional IF node that a device-side convergence
  // test closes, so nothing is computed and discarded at convergence
  // (degree >= tune.cond_graph, default 10: below it the IF node's per-iteration
  // cost outweighs the one skipped tail per solve; m = 0 / plain CG never)
  const bool use_cond = use_graph && spec_after_update && op->tune.cond_graph > 0 && prec.kind != 0 &&
                        m >= op->tune.cond_graph;

  std::memset(rep, 0, sizeof *rep);
  c->cur_launches = 0;
  c->cur_allreduce = 0;
  c->cur_halo_bytes = 0;
  double* r = c->r;
  double* z = c->z;
  double* p = c->p;
  double* q = c->q;

  PCGX_CUDA(cudaEventRecord(c->ev_t0, c->s));
  auto finish = [&]() {
    PCGX_CUDA(cudaEventRecord(c->ev_t1, c->s));
    PCGX_CUDA(cudaEventSynchronize(c->ev_t1));
    float ms = 0.f;
    PCGX_CUDA(cudaEventElapsedTime(&ms, c->ev_t0, c->ev_t1));
    rep->wall_time = ms * 1e-3;
    rep->kernel_launches = c->cur_launches;
    rep->allreduces = c->cur_allreduce;
    rep->halo_bytes = c->cur_halo_bytes;
    rep->spmv_equiv_bytes = (double)rep->matvec * spmv_equiv_bytes(op);
  };
  double alg = 0.0;  // algorithmic bytes, accumulated per enqueued pass
  const double N8 = 8.0 * (double)n;
  auto cheb_bytes = [&]() -> double {  // one preconditioner application incl. r.z
    if (!have_prec) return 2 * N8;
    if (prec.kind == 2) return newton_bytes(op, prec.newton.nlev, true);
    if (m == 0) return 2 * N8;
    const double spmv_extra = matrix_bytes(op);
    if (m == 1) return spmv_extra + 2 * N8;
    if (op->kind == 0 && op->cheb2)  // (1,2): read r, write x1 x2; pairs: 3 reads 2 writes; odd tail: 4
      return 3 * N8 + (double)((m - 2) / 2) * 5 * N8 + ((m % 2) ? 4 * N8 : 0.0);
    return (spmv_extra + 2 * N8) + (spmv_extra + 3 * N8) + (double)(m - 2) * (spmv_extra + 4 * N8);
  };

  // ||b|| (pcg.cpp:32)
  auto nvtx_setup = std::make_unique<NvtxRange>("pcgx::pcg_solve setup");
  launch_dot(c, n, b, b, S_BB);
  allreduce(c, S_BB, 1);
  fetch_scalars(c);
  alg += N8;
  const double bnorm = std::sqrt(c->hS[S_BB]);
  rep->ddot++;
  if (use_cond) {  // ||b|| and tol for the device convergence test (cond_kernel)
    const double bt[2] = {bnorm, opts.tol};
    static_assert(S_TOL == S_BNORM + 1, "adjacent slots");
    PCGX_CUDA(cudaMemcpyAsync(c->S + S_BNORM, bt, sizeof bt, cudaMemcpyHostToDevice, c->s));
  }
  if (bnorm == 0.0) {
    launch_fill(c, n, x, 0.0);
    rep->converged = 1;
    finish();
    rep->alg_bytes = alg;
    return;
  }
  if (opts.x0) {
    copy_d2d(c, x, opts.x0, n);
    op_launch<EpiResid, true>(c, op, x, EpiResid{b, r}, S_RR0);  // r = b - A x0
    allreduce(c, S_RR0, 1);
    fetch_scalars(c);
    alg += spmv_alg_bytes(op) + 2 * N8;
    rep->matvec++;
    const double rnorm = std::sqrt(c->hS[S_RR0]);
    rep->ddot++;
    rep->rel_res = rnorm / bnorm;
    if (rep->rel_res <= opts.tol) {
      rep->converged = 1;
      rep->true_rel_res = rep->rel_res;
      finish();
      rep->alg_bytes = alg;
      return;
    }
  } else {
    copy_d2d(c, r, b, n);
    launch_fill(c, n, x, 0.0);
    alg += 3 * N8;
    rep->rel_res = 1.0;
  }

  // zmode: 0 = Chebyshev m >= 1 (z from the fused recurrence), 1 = m == 0 (z = r/theta
  // written by the update kernel), 2 = no preconditioner (z is r itself).
  const int zm = !have_prec ? 2 : (prec.kind == 1 && m == 0 ? 1 : 0);
  double* Pd[2] = {p, c->p2};  // direction ping-pong: p(it) lives in Pd[it & 1]
  const bool fuse = fuses_dir_update(op) && op->tune.no_fuse_p == 0;
  // m = 0 on the TMA direction step: z = r / theta is formed there from r, never
  // stored (the update kernel only reduces r'z): 8 B less per unknown and iteration
  const bool zdiv = zm == 1 && fuse && dir_tma_ok(op) && op->tune.zdiv != 0;
  const double* zvec = (zm == 2 || zdiv) ? r : z;
  // TMA direction step (stencil): x += alpha p moves from the update kernel into the next
  // direction step, which reads p_old anyway (8 B less per unknown and iteration)
  // (not with on_iterate: x must be current at every iteration's callback)
  const bool cb = opts.on_iterate != nullptr;
  const bool defer_x = fuse && dir_tma_ok(op) && op->tune.defer_x != 0 && !cb;
  // Chebyshev m >= 3 on the stencil (one GPU, or z-slab ranks with two ghost planes):
  // the update r -= alpha q, r'r rides in the first two-step pass of P r
  // (cheb2f_upd_launch); r(it) lives in Rb[it & 1]
  const bool fuse_upd = zm == 0 && prec.kind == 1 && (spec_after_update || c->cm != nullptr) && defer_x &&
                        cheb_upd_ok(c, op, m);
  double* Rb[2] = {r, fuse_upd ? c->r2 : r};

  // dir_spmv(it): p(it) = z + beta p(it-1) (p(1) = z), q = A p(it), p'q -> pq(par); the
  // direction update is fused into the SpMV's input (InComb) where the kernels allow it.
  auto enqueue_dir_spmv = [&](int it) {
    const int par = it & 1;
    double* pnew = Pd[par];
    const double* pold = Pd[par ^ 1];
    const int first = (it == 1) ? 1 : 0;
    if (fuse && dir_tma_ok(op)) {
      // the previous iteration's x += alpha p_old rides along (defer_x)
      dir_tma_launch(c, op, zvec, pold, pnew, q, slot_rz(par ^ 1), slot_rz(par), first, slot_pq(par),
                     defer_x ? x : nullptr, slot_pq(par ^ 1), zdiv ? P.theta : 0.0);
    } else if (fuse) {
      op_launch_in<InComb, EpiStoreP, true>(
          c, op, in_of(op, zvec, pold, c->S, slot_rz(par ^ 1), slot_rz(par), first, true),
          EpiStoreP{q, pnew}, slot_pq(par));
    } else {
      pupdate_kernel<<<vec_grid(c, n), kVecThreads, 0, c->s>>>(n, pnew, pold, zvec, c->S,
                                                                slot_rz(par ^ 1), slot_rz(par), first);
      check_launch();
      count_launch(c);
      op_launch<EpiStore, true>(c, op, pnew, EpiStore{q}, slot_pq(par));
    }
    allreduce(c, slot_pq(par), 1);
  };
  const double bytes_dir = fuse ? spmv_alg_bytes(op) + 2 * N8 : spmv_alg_bytes(op) + 3 * N8;
  // one rank: every scalar the host checks reached hS from its reducing kernel
  // (Reduce::mirror); several ranks: the all-reduced slots are copied
  const bool snap_copy = c->cm != nullptr || op->tune.snap_memcpy != 0;
  auto snapshot = [&]() {  // External: when captured, the graph records ev_sync on every replay
    if (snap_copy)
      PCGX_CUDA(cudaMemcpyAsync(c->hS, c->S, sizeof(double) * kSlots, cudaMemcpyDeviceToHost, c->s));
    if (c->capturing) PCGX_CUDA(cudaEventRecordWithFlags(c->ev_sync, c->s, cudaEventRecordExternal));
    else PCGX_CUDA(cudaEventRecord(c->ev_sync, c->s));
  };
  // snapshot right after the update when r'r (and r'z for zmode > 0) are final there
  const bool snap_after_update = spec_after_update || zm > 0;
  // B(it): [prec(it) -> z, r'z ; multi-GPU: all-reduce (r'r, r'z) + snapshot] ; dir_spmv(it+1)
  auto enqueue_B = [&](int it) {
    const int par = it & 1;
    if (fuse_upd) {
      // r(it) = r(it-1) - alpha(it) q(it) inside P r(it)'s first pass; the scalar
      // snapshot (r'r(it), p'q(it)) is taken right after that pass (and, with the
      // conditional graph, the convergence test: the rest runs only if not converged)
      const CgUpd u{Rb[par ^ 1], q, Rb[par], slot_rz(par ^ 1), slot_pq(par), slot_rr(par)};
      if (spec_after_update) {
        enqueue_cheb(c, op, P, Rb[par], z, slot_rz(par), &u, [&] {
          snapshot();
          if (use_cond) cond_split(c, slot_rr(par), false);  // the first pass set the condition
        });
      } else {
        // several ranks: the pass reduced this rank's share of r'r; [r'r, r'z] are
        // all-reduced together after P r, as without the fusion
        enqueue_cheb(c, op, P, Rb[par], z, slot_rz(par), &u);
        allreduce(c, slot_rr(par), 2);
        snapshot();
      }
    } else if (use_cond) {
      cond_split(c, slot_rr(par));  // r'r(it) came from the update kernel before this segment
      if (zm == 0) enqueue_prec(c, op, prec, r, z, slot_rz(par));
    } else if (zm == 0) {
      enqueue_prec(c, op, prec, r, z, slot_rz(par));
      if (!spec_after_update) {
        allreduce(c, slot_rr(par), 2);
        snapshot();
      }
    }
    enqueue_dir_spmv(it + 1);
  };
  // setup: z_0 = P r_0 and rho_0 = r'z -> rz(0) (pcg.cpp:57-64)
  if (zm == 0) enqueue_prec(c, op, prec, r, z, slot_rz(0));
  else if (zm == 1) launch_zr(c, n, z, r, P.theta, 1, slot_rz(0));
  else launch_dot(c, n, r, r, slot_rz(0));
  // the two segment graphs (iteration parity 1, 0): cached across solves; a new
  // one is captured here, on the host, while the device works on the setup P r
  Graph* gB[2] = {nullptr, nullptr};
  if (use_graph) {
    std::string key;
    auto add = [&](const void* v, size_t bytes) { key.append((const char*)v, bytes); };
    const uint64_t ids[3] = {op->uid, c->ws_gen, defer_x ? (uint64_t)(uintptr_t)x : 0};
    add(ids, sizeof ids);
    const int flags[8] = {prec.kind, m,        zm, fuse ? 1 : 0, spec_after_update ? 1 : 0, fuse_upd ? 1 : 0,
                          snap_copy ? 1 : 0, use_cond ? 1 : 0};
    add(flags, sizeof flags);
    if (prec.kind == 1) {
      const double t[3] = {P.theta, P.delta, P.sigma};
      add(t, sizeof t);
      add(P.rho.data(), sizeof(double) * P.rho.size());
    } else if (prec.kind == 2) {
      add(prec.newton.zeta.data(), sizeof(double) * prec.newton.zeta.size());
    }
    for (int par = 0; par < 2; ++par) {
      const std::string k = key + (par ? "1" : "0");
      auto hit = c->gcache.find(k);
      if (hit == c->gcache.end()) {
        if (c->gcache.size() >= 64) c->gcache.clear();
        auto g = std::make_unique<Graph>();
        if (use_cond) capture_cond(c, *g, [&] { enqueue_B(par ? 1 : 2); });
        else capture(c, *g, [&] { enqueue_B(par ? 1 : 2); });
        hit = c->gcache.emplace(k, std::move(g)).first;
      }
      gB[par] = hit->second.get();
    }
  }
  allreduce(c, slot_rz(0), 1);
  alg += cheb_bytes();
  if (have_prec) {
    rep->prec_applies++;
    rep->matvec += m;
  }
  rep->ddot++;
  fetch_scalars(c);
  {
    const double rho = c->hS[slot_rz(0)];
    if (!std::isfinite(rho) || rho <= 0.0)
      fail(PCGX_ERR_NUMERICAL,
           "pcg_solve: r'z = " + fmt_double(rho) + " at setup (preconditioner not SPD?)");
  }

  // fused: the first pass also reads q and writes r (+16 B), the update (24 B) is gone
  const double bytes_B = (zm == 0 ? cheb_bytes() : 0.0) + bytes_dir + (defer_x ? 2 * N8 : 0.0) +
                         (fuse_upd ? 2 * N8 : 0.0);
  const double bytes_update = (defer_x ? 3 : 6) * N8 + (zm == 1 && !zdiv ? N8 : 0.0);
  bool x_pending = false;  // a deferred x update no direction step has applied yet
  int x_par = 0;

  enqueue_dir_spmv(1);
  alg += bytes_dir;
  nvtx_setup.reset();
  auto nvtx_iter = std::make_unique<NvtxRange>("pcgx::pcg_solve iterations");
  for (int it = 1; it <= opts.maxit; ++it) {
    const int par = it & 1;
    const bool more = it < opts.maxit;
    const bool upd_in_B = fuse_upd && more;  // else a standalone update (in place)
    if (!upd_in_B) {
      launch_update(c, n, defer_x ? nullptr : x, Rb[par ^ 1], Pd[par], q, slot_rz(par ^ 1), slot_pq(par),
                    slot_rr(par), zm, zm == 1 ? P.theta : 1.0, zdiv ? nullptr : z);
      check_launch();
      count_launch(c);
      alg += bytes_update;
    }
    x_pending = defer_x;
    x_par = par;
    rep->matvec++;  // q = A p of this iteration
    if (!spec_after_update && (zm > 0 || !more)) allreduce(c, slot_rr(par), zm > 0 ? 2 : 1);
    if ((snap_after_update && !upd_in_B) || !more) snapshot();
    if (more) {
      if (use_graph) {
        replay(c, *gB[par]);
      } else {
        enqueue_B(it);
      }
      alg += bytes_B;
      x_pending = false;  // dir_spmv(it+1) applies it
    }
    PCGX_CUDA(cudaEventSynchronize(c->ev_sync));
    const double* hs = c->hS;
    // checks in the reference's order: r'z(it-1) [pcg.cpp:103-106], p'Ap [:76-79], ||r|| [:85]
    const bool rz_now = !spec_after_update || zm > 0;  // r'z(it) is in this snapshot
    if (it >= 2 && !rz_now) {
      const double rho_prev = hs[slot_rz(par ^ 1)];
      if (!std::isfinite(rho_prev) || rho_prev <= 0.0)
        fail(PCGX_ERR_NUMERICAL,
             "pcg_solve: r'z = " + fmt_double(rho_prev) + " (preconditioner not SPD?)");
    }
    const double pq = hs[slot_pq(par)];
    rep->ddot++;
    if (!std::isfinite(pq) || pq <= 0.0)
      fail(PCGX_ERR_NUMERICAL, "pcg_solve: p'Ap = " + fmt_double(pq) + " (operator not SPD?)");
    const double rnorm = std::sqrt(hs[slot_rr(par)]);
    rep->ddot++;
    if (!std::isfinite(rnorm)) fail(PCGX_ERR_NUMERICAL, "pcg_solve: residual norm is not finite");
    rep->iters = it;
    rep->rel_res = rnorm / bnorm;
    if (cb) {  // opts.on_iterate(it, x) (pcg.cpp:88): x(it) was final before the snapshot
      c->hx.resize((size_t)n);
      PCGX_CUDA(cudaMemcpyAsync(c->hx.data(), x, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost, c->s));
      PCGX_CUDA(cudaStreamSynchronize(c->s));
      if (opts.on_iterate(it, c->hx.data(), n, opts.on_iterate_user) != 0)
        fail(PCGX_ERR_CALLBACK, "pcg_solve: on_iterate stopped the solve at iteration " + std::to_string(it));
    }
    if (rep->rel_res <= opts.tol) {
      rep->converged = 1;
      if (more && use_cond) {
        // the device skipped the segment's tail (IF node): only a fused first pass
        // of P r ran; the direction step that would apply x += alpha p did not
        rep->wasted_matvec = fuse_upd ? 2 : 0;
        c->cur_launches -= gB[par]->body_kernels;
        c->launches -= gB[par]->body_kernels;
        alg -= bytes_B - (fuse_upd ? 5 * N8 : 0.0);
        x_pending = defer_x;
        x_par = par;
      } else if (more) {
        rep->wasted_matvec = (zm == 0 ? m : 0) + 1;  // speculative P r and A p
      }
      break;
    }
    if (!more) break;
    if (have_prec) {
      rep->prec_applies++;
      rep->matvec += m;
    }
    rep->ddot++;  // r'z
    if (rz_now) {
      const double rz = hs[slot_rz(par)];
      if (!std::isfinite(rz) || rz <= 0.0)
        fail(PCGX_ERR_NUMERICAL, "pcg_solve: r'z = " + fmt_double(rz) + " (preconditioner not SPD?)");
    }
  }
  if (x_pending) {  // the iteration limit ended the loop before the next direction step
    xupd_kernel<<<vec_grid(c, n), kVecThreads, 0, c->s>>>(n, x, Pd[x_par], c->S, slot_rz(x_par ^ 1),
                                                          slot_pq(x_par));
    check_launch();
    count_launch(c);
    alg += 3 * N8;
  }
  // true residual (pcg.cpp:112-115)
  nvtx_iter.reset();
  NvtxRange nvtx_exit("pcgx::pcg_solve true residual");
  op_launch<EpiResid, true>(c, op, x, EpiResid{b, nullptr}, S_EE);
  allreduce(c, S_EE, 1);
  fetch_scalars(c);
  alg += spmv_alg_bytes(op) + N8;
  rep->matvec++;
  rep->true_rel_res = std::sqrt(c->hS[S_EE]) / bnorm;
  rep->ddot++;
  finish();
  rep->alg_bytes = alg;
  rep->step_bytes = cheb_step_bytes(op);

  // Optional: time the dominant kernel with CUDA events on the compute stream, on
  // this solve's operator and buffers: the two-step pass (stencil, cheb2) or the
  // fused single middle step.
  if ((opts.flags & PCGX_FLAG_TIME_KERNELS) && prec.kind == 1 && m >= 4) {
    const int reps = std::max(3, op->tune.step_reps);
    const bool two = (op->kind == 0 && op->cheb2);
    Cheb2Params q{};
    if (two) {
      q.nx = (int)op->nx;
      q.ny = (int)op->ny;
      q.nzl = (int)op->nzl;
      q.nxy = op->nx * op->ny;
      q.d = op->d;
      q.theta = P.theta;
      q.c2 = 2.0 / P.delta;
      q.c3 = 2.0 * P.sigma;
      q.rk1 = P.rho[3];
      q.rk1m1 = P.rho[2];
      q.rk2 = P.rho[4];
      q.rk2m1 = P.rho[3];
      q.outC = c->w2;
      q.outE = c->w3;
    }
    EpiChebStep e{r, c->w0, c->w0, P.rho[3], P.rho[2], 2.0 / P.delta, 2.0 * P.sigma, P.theta, 0,
                  1.0 / P.theta};
    const bool three = two && cheb3_ok(c, op) && op->tune.cheb3 == 1 && m >= 5;
    Cheb3Params q3{};
    q3.c2 = 2.0 / P.delta;
    q3.c3 = 2.0 * P.sigma;
    q3.rk1 = P.rho[3];
    q3.rk1m1 = P.rho[2];
    q3.rk2 = P.rho[4];
    q3.rk2m1 = P.rho[3];
    q3.rk3 = P.rho[5];
    q3.rk3m1 = P.rho[4];
    q3.outE = c->w2;
    q3.outF = c->w3;
    auto launch = [&] {
      if (three) cheb3_pass<false>(c, op, c->w1, c->w0, r, q3, -1);
      else if (two) cheb2_pass<false, false>(c, op, c->w1, c->w0, r, q, -1);
      else op_launch<EpiChebStep, false>(c, op, c->w1, e, -1);
    };
    const uint64_t mv0 = op->matvecs.load();
    launch();  // warm
    PCGX_CUDA(cudaEventRecord(c->ev_t0, c->s));
    for (int i = 0; i < reps; ++i) launch();
    PCGX_CUDA(cudaEventRecord(c->ev_t1, c->s));
    PCGX_CUDA(cudaEventSynchronize(c->ev_t1));
    op->matvecs.store(mv0);
    float ms = 0.f;
    PCGX_CUDA(cudaEventElapsedTime(&ms, c->ev_t0, c->ev_t1));
    rep->step_ms = ms;
    rep->step_launches = reps;
    rep->step_bytes = two ? 40.0 * (double)op->n_local : cheb_step_bytes(op);
    rep->step_steps = three ? 3 : (two ? 2 : 1);
  }
}

