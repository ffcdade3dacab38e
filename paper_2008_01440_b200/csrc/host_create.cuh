// SPDX-License-Identifier: Apache-2.0
//
// Part of pcgx.cu (ONE translation unit): included in place, in the middle of that
// file's declarations; not a standalone header. Operator creation: stencil operators, CSR upload and storage detection, block rows / slabs.
#pragma once

// ---------------------------------------------------------------- operator creation

void init_stencil_ghosts(pcgx_context c, pcgx_operator op) {
  const size_t pb = sizeof(double) * (size_t)(op->nx * op->ny);
  if (c->nranks > 1) {
    if (c->rank > 0) {
      PCGX_CUDA(cudaMalloc(&op->ghost_lo, pb));
      PCGX_CUDA(cudaMalloc(&op->ghost_lo2, pb));
    }
    if (c->rank < c->nranks - 1) {
      PCGX_CUDA(cudaMalloc(&op->ghost_hi, pb));
      PCGX_CUDA(cudaMalloc(&op->ghost_hi2, pb));
    }
  }
}

int default_kz(pcgx_context c, long long nx, long long ny, long long nzl) {
  (void)0;
  (void)c;
  (void)nx;
  (void)ny;
  (void)nzl;
  return 16;
}

void build_sell(pcgx_operator op, long long n, const std::vector<int>& rp32,
                const std::vector<int>& ci32, const double* va);
void build_bsr3(pcgx_operator op, long long n, const std::vector<int>& rp32,
                const std::vector<int>& ci32, const double* va);
bool is_bsr3(long long n, const std::vector<int>& rp, const std::vector<int>& ci);
bool dia_offsets(long long n, const std::vector<int>& rp, const std::vector<int>& ci, std::vector<int>& off,
                 long long row_base = 0);
template <int P>
bool dia3_match(long long n, int nx, const std::vector<int>& rp, const std::vector<int>& ci,
                const std::vector<int>& off, long long row_base = 0);

// Offset storage of one plane-aligned z-slab of a 27-point-box matrix on an nx^3
// grid (multi-rank cfg3): the rank owns node planes [z0, z0 + nzl) (pcgx_slab_partition
// of the nx planes), its rows' values by offset as build_dia lays them out, the
// Jacobi values of its rows and of the neighbours' boundary planes (from the full
// matrix: no exchange), and x-ghost planes the stencil slab machinery fills before
// each SpMV (dia3_kernel reads them as planes -1 and nzl).
// local: rp32 / va / dv hold this rank's rows only (rp32 from 0, ci32 global); the
// neighbours' boundary-plane Jacobi values then come through the plane exchange.
void dia_slab_upload(pcgx_context c, pcgx_operator op, long long n, int nx, const std::vector<int>& rp32,
                     const std::vector<int>& ci32, const double* va, const std::vector<double>& dv,
                     const std::vector<int>& off, bool local = false) {
  const int P = c->nranks, me = c->rank;
  int64_t z0 = 0, nzl = 0;
  pcgx_slab_partition(nx, P, me, &z0, &nzl);
  const long long nxy = (long long)nx * nx, r0 = z0 * nxy, nloc = nzl * nxy;
  const long long rb = local ? r0 : 0;  // rp32 / dv index of global row g: g - rb
  const int K = (int)off.size();
  const long long ld = (nloc + 31) / 32 * 32;
  std::vector<double> val((size_t)(ld * K), 0.0);
  std::vector<unsigned> mask((size_t)nloc, 0u);
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < nloc; ++i) {
    const long long g = r0 + i;
    int q = 0;
    for (int k = rp32[(size_t)(g - rb)]; k < rp32[(size_t)(g - rb) + 1]; ++k) {
      const int o = (int)((long long)ci32[(size_t)k] - g);
      while (off[(size_t)q] != o) ++q;  // both ascending
      val[(size_t)(q * ld + i)] = va[k];
      mask[(size_t)i] |= 1u << q;
    }
  }
  op->kind = 1;
  op->n_global = n;
  op->nnz = (long long)rp32[(size_t)(r0 - rb + nloc)] - rp32[(size_t)(r0 - rb)];
  op->row0 = r0;
  op->n_local = nloc;
  op->dia_k = K;
  op->dia_ld = ld;
  for (int k = 0; k < K; ++k) op->dia_off[k] = off[(size_t)k];
  op->dia3_pat = 27;
  op->dia3_nx = nx;
  op->dia3_nzl = (int)nzl;
  op->nx = op->ny = nx;
  op->nz = nx;
  op->z0 = z0;
  op->nzl = nzl;
  PCGX_CUDA(cudaMalloc(&op->dia_val, sizeof(double) * val.size()));
  PCGX_CUDA(cudaMalloc(&op->dia_mask, sizeof(unsigned) * std::max<size_t>(mask.size(), 1)));
  PCGX_CUDA(cudaMemcpy(op->dia_val, val.data(), sizeof(double) * val.size(), cudaMemcpyHostToDevice));
  PCGX_CUDA(cudaMemcpy(op->dia_mask, mask.data(), sizeof(unsigned) * mask.size(), cudaMemcpyHostToDevice));
  PCGX_CUDA(cudaMalloc(&op->dvec, sizeof(double) * (size_t)std::max(nloc, 1LL)));
  PCGX_CUDA(cudaMemcpy(op->dvec, dv.data() + (r0 - rb), sizeof(double) * (size_t)nloc, cudaMemcpyHostToDevice));
  if (me > 0) PCGX_CUDA(cudaMalloc(&op->dia3_dlo, sizeof(double) * (size_t)nxy));
  if (me < P - 1) PCGX_CUDA(cudaMalloc(&op->dia3_dhi, sizeof(double) * (size_t)nxy));
  init_stencil_ghosts(c, op);  // x / p ghost planes (nx * nx) for the plane exchange
  if (!local) {
    if (me > 0)
      PCGX_CUDA(cudaMemcpy(op->dia3_dlo, dv.data() + r0 - nxy, sizeof(double) * (size_t)nxy, cudaMemcpyHostToDevice));
    if (me < P - 1)
      PCGX_CUDA(cudaMemcpy(op->dia3_dhi, dv.data() + r0 + nloc, sizeof(double) * (size_t)nxy, cudaMemcpyHostToDevice));
    return;
  }
  // the neighbours' boundary planes of d, once, through the operator's own plane exchange
  PCGX_CUDA(cudaDeviceSynchronize());  // legacy-stream uploads before the compute / comm streams
  const double* xs[1] = {op->dvec};
  c->cm->halo_begin(c, op, xs, 1);
  c->cm->halo_wait(c);
  if (me > 0)
    PCGX_CUDA(cudaMemcpyAsync(op->dia3_dlo, op->ghost_lo, sizeof(double) * (size_t)nxy, cudaMemcpyDeviceToDevice, c->s));
  if (me < P - 1)
    PCGX_CUDA(cudaMemcpyAsync(op->dia3_dhi, op->ghost_hi, sizeof(double) * (size_t)nxy, cudaMemcpyDeviceToDevice, c->s));
  PCGX_CUDA(cudaStreamSynchronize(c->s));
}

// CSR block rows (the paper's MPI block-row SpMV): this rank
// keeps rows [row0, row0 + nloc) with columns remapped to the local space:
// owned columns -> [0, nloc), others -> nloc + (position in the ascending list
// of ghost columns). Entries keep their order (the reference's summation order).
// Each rank holds the full matrix on the host, so the send lists (the rows of
// mine other ranks' rows reference) are computed without communication.
void csr_upload_block(pcgx_context c, pcgx_operator op, long long n, const std::vector<int>& rp32,
                      const std::vector<int>& ci32, const double* va, const std::vector<double>& dv) {
  const int P = c->nranks, me = c->rank;
  // a matrix of aligned 3 x 3 blocks keeps BSR-3 on every rank: rows split in whole
  // block rows (the balanced partition of the n/3 block rows), the local columns
  // remapped to [local | ghost] stay aligned triples, and bsr3_kernel reads the
  // ghost columns through the same exchange as SELL
  const bool bsr = op->tune.bsr != 0 && n % 3 == 0 && n >= 3LL * P && is_bsr3(n, rp32, ci32);
  // offset storage on a cubic grid with the 27-point box (cfg3): plane-aligned
  // z-slabs and the grid-tile kernel with the neighbours' boundary planes as ghosts
  if (!bsr && op->tune.dia != 0 && op->tune.dia3 != 0) {
    std::vector<int> doff;
    const long long nnz_all = rp32[(size_t)n];
    int nx = (int)std::llround(std::cbrt((double)n));
    while ((long long)nx * nx * nx > n) --nx;
    while ((long long)(nx + 1) * (nx + 1) * (nx + 1) <= n) ++nx;
    if ((long long)nx * nx * nx == n && nx >= 3 && nx >= P && dia_offsets(n, rp32, ci32, doff) &&
        (double)doff.size() * (double)n <= 1.5 * (double)nnz_all && dia3_match<27>(n, nx, rp32, ci32, doff)) {
      dia_slab_upload(c, op, n, nx, rp32, ci32, va, dv, doff);
      return;
    }
  }
  std::vector<long long> start(P + 1);
  for (int q = 0; q < P; ++q) {
    int64_t z0, nl;
    if (bsr) {
      pcgx_slab_partition(n / 3, P, q, &z0, &nl);
      z0 *= 3;
    } else {
      pcgx_slab_partition(n, P, q, &z0, &nl);
    }
    start[(size_t)q] = z0;
  }
  start[(size_t)P] = n;
  const long long r0 = start[(size_t)me], r1 = start[(size_t)me + 1], nloc = r1 - r0;
  if (nloc < 1) fail(PCGX_ERR_INVALID, "csr_create: fewer rows than ranks");
  // ghost columns of my rows, ascending (hence grouped by owner)
  std::vector<int> ghosts;
  for (long long i = r0; i < r1; ++i)
    for (int k = rp32[(size_t)i]; k < rp32[(size_t)i + 1]; ++k) {
      const int col = ci32[(size_t)k];
      if (col < r0 || col >= r1) ghosts.push_back(col);
    }
  std::sort(ghosts.begin(), ghosts.end());
  ghosts.erase(std::unique(ghosts.begin(), ghosts.end()), ghosts.end());
  // local CSR
  const long long k0 = rp32[(size_t)r0];
  std::vector<int> lrp((size_t)nloc + 1), lci((size_t)(rp32[(size_t)r1] - k0));
  for (long long i = r0; i <= r1; ++i) lrp[(size_t)(i - r0)] = (int)(rp32[(size_t)i] - k0);
  for (long long k = k0; k < rp32[(size_t)r1]; ++k) {
    const int col = ci32[(size_t)k];
    lci[(size_t)(k - k0)] = (col >= r0 && col < r1)
                                ? (int)(col - r0)
                                : (int)(nloc + (std::lower_bound(ghosts.begin(), ghosts.end(), col) -
                                                ghosts.begin()));
  }
  // per-neighbour traffic: recv = my ghosts owned by q; send = my rows q's rows reference
  op->nb_rank.clear();
  op->send_off.clear();
  op->send_cnt.clear();
  op->recv_off.clear();
  op->recv_cnt.clear();
  std::vector<int> send_idx;
  for (int q = 0; q < P; ++q) {
    if (q == me) continue;
    const long long lo = std::lower_bound(ghosts.begin(), ghosts.end(), (int)start[(size_t)q]) - ghosts.begin();
    const long long hi = std::lower_bound(ghosts.begin(), ghosts.end(), (int)start[(size_t)q + 1]) - ghosts.begin();
    std::vector<int> need;  // rows of mine referenced by q's rows, ascending
    for (long long i = start[(size_t)q]; i < start[(size_t)q + 1]; ++i)
      for (int k = rp32[(size_t)i]; k < rp32[(size_t)i + 1]; ++k) {
        const int col = ci32[(size_t)k];
        if (col >= r0 && col < r1) need.push_back(col);
      }
    std::sort(need.begin(), need.end());
    need.erase(std::unique(need.begin(), need.end()), need.end());
    if (hi == lo && need.empty()) continue;
    op->nb_rank.push_back(q);
    op->recv_off.push_back(lo);
    op->recv_cnt.push_back(hi - lo);
    op->send_off.push_back((long long)send_idx.size());
    op->send_cnt.push_back((long long)need.size());
    for (int col : need) send_idx.push_back((int)(col - r0));
  }
  op->row0 = r0;
  op->n_local = nloc;
  op->nghost = (long long)ghosts.size();
  op->nsend = (long long)send_idx.size();
  std::vector<double> dext((size_t)(nloc + op->nghost));
  for (long long i = 0; i < nloc; ++i) dext[(size_t)i] = dv[(size_t)(r0 + i)];
  for (long long g = 0; g < op->nghost; ++g) dext[(size_t)(nloc + g)] = dv[(size_t)ghosts[(size_t)g]];
  PCGX_CUDA(cudaMalloc(&op->dvec, sizeof(double) * dext.size()));
  PCGX_CUDA(cudaMemcpy(op->dvec, dext.data(), sizeof(double) * dext.size(), cudaMemcpyHostToDevice));
  PCGX_CUDA(cudaMalloc(&op->rp, sizeof(int) * lrp.size()));
  PCGX_CUDA(cudaMemcpy(op->rp, lrp.data(), sizeof(int) * lrp.size(), cudaMemcpyHostToDevice));
  const size_t ng = (size_t)std::max(op->nghost, 1LL), nsd = (size_t)std::max(op->nsend, 1LL);
  PCGX_CUDA(cudaMalloc(&op->send_idx, sizeof(int) * nsd));
  if (op->nsend)
    PCGX_CUDA(cudaMemcpy(op->send_idx, send_idx.data(), sizeof(int) * send_idx.size(), cudaMemcpyHostToDevice));
  PCGX_CUDA(cudaMalloc(&op->sbuf_z, sizeof(double) * nsd));
  PCGX_CUDA(cudaMalloc(&op->sbuf_p, sizeof(double) * nsd));
  PCGX_CUDA(cudaMalloc(&op->ghost_z, sizeof(double) * ng));
  PCGX_CUDA(cudaMalloc(&op->ghost_p, sizeof(double) * ng));
  if (bsr && is_bsr3(nloc, lrp, lci)) build_bsr3(op, nloc, lrp, lci, va + k0);
  else build_sell(op, nloc, lrp, lci, va + k0);
}

// Block-row CSR from THIS rank's rows only (the paper's distributed matrix,
// PAPER.md:683-685): rows [row0, row0 + nloc) of a symmetric n x n matrix with
// global column indices, the balanced row partition pcgx_slab_partition gives.
// No rank holds the full matrix. The halo lists need no communication because the
// pattern is symmetric (a_ic != 0 <=> a_ci != 0): rank q needs my x_c exactly when
// my row c has a column in q's rows, and I receive my ghost columns from their
// owners -- both sides list them in ascending column order. The Jacobi values of
// the ghost columns (other ranks' diagonals) travel once through the operator's own
// block-row exchange. Values are uploaded as given: bitwise the rows the full-matrix
// path uploads, so every SpMV / Chebyshev step equals the single-domain result.
template <class I>
void csr_upload_local(pcgx_context c, pcgx_operator op, long long n, long long r0, long long nloc, const I* rp,
                      const I* ci, const double* va, const double* isd) {
  const int P = c->nranks, me = c->rank;
  if (!rp || !ci || !va) fail(PCGX_ERR_INVALID, "CsrMatrix: null array");
  // The rows may follow one of three balanced partitions (the ones pcgx_csr_create
  // cuts a full matrix by): plain rows; whole 3 x 3 block rows (n % 3 == 0: keeps
  // BSR-3); whole node planes of an nx^3 grid (keeps the offset storage on z-slabs).
  // Every rank reports which ones its [row0, row0 + n_local) matches and the job
  // takes the first that all ranks match -- rows, block rows, planes.
  int nxg = (int)std::llround(std::cbrt((double)n));
  while ((long long)nxg * nxg * nxg > n) --nxg;
  while ((long long)(nxg + 1) * (nxg + 1) * (nxg + 1) <= n) ++nxg;
  const bool cube = (long long)nxg * nxg * nxg == n && nxg >= 3 && nxg >= P;
  auto part_start = [&](int kind, int q) -> long long {  // first row of rank q (q == P: n)
    if (q == P) return n;
    int64_t z0, nl;
    if (kind == 1) {
      pcgx_slab_partition(n / 3, P, q, &z0, &nl);
      return 3 * z0;
    }
    if (kind == 2) {
      pcgx_slab_partition(nxg, P, q, &z0, &nl);
      return z0 * (long long)nxg * nxg;
    }
    pcgx_slab_partition(n, P, q, &z0, &nl);
    return z0;
  };
  auto matches = [&](int kind) {
    if (kind == 1 && (n % 3 != 0 || n < 3LL * P)) return false;
    if (kind == 2 && !cube) return false;
    return r0 == part_start(kind, me) && r0 + nloc == part_start(kind, me + 1);
  };
  // local int32 arrays (rp from 0, global columns) for the pattern checks of the
  // plane partition; validated below like every other path
  int kind = -1;
  bool slab = false;
  std::vector<int> doff;
  {
    double f[4] = {matches(0) ? 1.0 : 0.0, matches(1) ? 1.0 : 0.0, matches(2) ? 1.0 : 0.0, 0.0};
    std::vector<int> grp, gci;
    if (f[2] > 0.0 && op->tune.dia != 0 && op->tune.dia3 != 0 && nloc >= 1 && n < (1LL << 31) &&
        (long long)rp[nloc] - (long long)rp[0] < (1LL << 31)) {
      const long long base0 = (long long)rp[0], nz = (long long)rp[nloc] - base0;
      grp.resize((size_t)nloc + 1);
      gci.resize((size_t)nz);
      bool sane = true;
      for (long long i = 0; i <= nloc; ++i) {
        grp[(size_t)i] = (int)((long long)rp[i] - base0);
        if (i && grp[(size_t)i] < grp[(size_t)i - 1]) sane = false;
      }
      for (long long k = 0; k < nz && sane; ++k) {
        gci[(size_t)k] = (int)ci[k];
        if ((long long)ci[k] < 0 || (long long)ci[k] >= n) sane = false;
      }
      if (sane && dia_offsets(nloc, grp, gci, doff, r0) && dia3_match<27>(nloc, nxg, grp, gci, doff, r0)) f[3] = 1.0;
    }
    double g[4];
    allreduce_host(c, f, g, 4);
    if (g[2] == (double)P && g[3] == (double)P) {
      kind = 2;
      slab = true;
    } else if (g[0] == (double)P) {
      kind = 0;
    } else if (g[1] == (double)P) {
      kind = 1;
    } else if (g[2] == (double)P) {
      kind = 2;
    } else {
      fail(PCGX_ERR_INVALID, "csr_create_local: rank " + std::to_string(me) + " must own rows [" +
                                 std::to_string(part_start(0, me)) + ", " + std::to_string(part_start(0, me + 1)) +
                                 ") (pcgx_slab_partition of the rows; or, on every rank, of the 3 x 3 block rows "
                                 "or of the node planes of a cubic grid)");
    }
  }
  std::vector<long long> start(P + 1);
  for (int q = 0; q <= P; ++q) start[(size_t)q] = part_start(kind, q);
  if (nloc < 1) fail(PCGX_ERR_INVALID, "csr_create: fewer rows than ranks");
  const long long base = (long long)rp[0], nnz = (long long)rp[nloc] - base;
  if (nnz >= (1LL << 31) || n >= (1LL << 31))
    fail(PCGX_ERR_OVERFLOW, "csr_create: nnz " + std::to_string(nnz) + " does not fit the int32 device CSR");
  const long long r1 = r0 + nloc;
  std::vector<int> ghosts;
  std::vector<double> dv((size_t)nloc);
  long long bad = -1;
  for (long long i = 0; i < nloc; ++i) {
    if (rp[i + 1] < rp[i]) fail(PCGX_ERR_INVALID, "CsrMatrix: row_ptr not nondecreasing");
    double diag = 0.0;
    for (long long k = (long long)rp[i] - base; k < (long long)rp[i + 1] - base; ++k) {
      const long long col = (long long)ci[k];
      if (col < 0 || col >= n)
        fail(PCGX_ERR_INVALID, "CsrMatrix: column index out of range in row " + std::to_string(r0 + i));
      if (k > (long long)rp[i] - base && col <= (long long)ci[k - 1])
        fail(PCGX_ERR_INVALID, "CsrMatrix: columns not strictly increasing in row " + std::to_string(r0 + i));
      if (col == r0 + i) diag = va[k];
      if (col < r0 || col >= r1) ghosts.push_back((int)col);
    }
    if (isd) dv[(size_t)i] = isd[i];
    else if (!(diag > 0.0)) {
      if (bad < 0) bad = r0 + i;
    } else {
      dv[(size_t)i] = 1.0 / std::sqrt(diag);  // jacobi_scale (linop.cpp:340-351)
    }
  }
  // every rank learns whether any rank's diagonal is nonpositive (no rank may be
  // left waiting in the exchange below)
  {
    const double flag = bad >= 0 ? 1.0 : 0.0;
    double any = 0.0;
    allreduce_host(c, &flag, &any, 1);
    if (bad >= 0) fail(PCGX_ERR_NUMERICAL, "jacobi_scale: nonpositive diagonal entry at index " + std::to_string(bad));
    if (any > 0.0) fail(PCGX_ERR_NUMERICAL, "jacobi_scale: nonpositive diagonal entry on another rank");
  }
  if (slab) {
    // 27-point box on plane-aligned slabs: the offset storage, ghost planes through
    // the stencil's plane exchange (as pcgx_csr_create keeps it for a full matrix)
    std::vector<int> grp((size_t)nloc + 1), gci((size_t)nnz);
    for (long long i = 0; i <= nloc; ++i) grp[(size_t)i] = (int)((long long)rp[i] - base);
    for (long long k = 0; k < nnz; ++k) gci[(size_t)k] = (int)ci[k];
    dia_slab_upload(c, op, n, nxg, grp, gci, va, dv, doff, true);
    return;
  }
  std::sort(ghosts.begin(), ghosts.end());
  ghosts.erase(std::unique(ghosts.begin(), ghosts.end()), ghosts.end());
  std::vector<int> lrp((size_t)nloc + 1), lci((size_t)nnz);
  for (long long i = 0; i <= nloc; ++i) lrp[(size_t)i] = (int)((long long)rp[i] - base);
  for (long long k = 0; k < nnz; ++k) {
    const long long col = (long long)ci[k];
    lci[(size_t)k] = (col >= r0 && col < r1)
                         ? (int)(col - r0)
                         : (int)(nloc + (std::lower_bound(ghosts.begin(), ghosts.end(), (int)col) - ghosts.begin()));
  }
  op->nb_rank.clear();
  op->send_off.clear();
  op->send_cnt.clear();
  op->recv_off.clear();
  op->recv_cnt.clear();
  std::vector<int> send_idx;
  for (int q = 0; q < P; ++q) {
    if (q == me) continue;
    const long long lo = std::lower_bound(ghosts.begin(), ghosts.end(), (int)start[(size_t)q]) - ghosts.begin();
    const long long hi = std::lower_bound(ghosts.begin(), ghosts.end(), (int)start[(size_t)q + 1]) - ghosts.begin();
    std::vector<int> need;  // my rows with a column in q's rows (= the rows of mine q's rows reference)
    for (long long i = 0; i < nloc; ++i)
      for (long long k = lrp[(size_t)i]; k < lrp[(size_t)i + 1]; ++k) {
        const long long col = (long long)ci[k];
        if (col >= start[(size_t)q] && col < start[(size_t)q + 1]) {
          need.push_back((int)i);
          break;
        }
      }
    if (hi == lo && need.empty()) continue;
    op->nb_rank.push_back(q);
    op->recv_off.push_back(lo);
    op->recv_cnt.push_back(hi - lo);
    op->send_off.push_back((long long)send_idx.size());
    op->send_cnt.push_back((long long)need.size());
    for (int r : need) send_idx.push_back(r);
  }
  // The lists are consistent only if the pattern is symmetric across ranks: check
  // it before any point-to-point exchange (a mismatch would hang NCCL). Every rank
  // contributes its row of the P x P "receive from" and "send to" count matrices;
  // after the all-reduce recv[a][b] must equal send[b][a] everywhere.
  {
    std::vector<double> cnt(2 * (size_t)P * P, 0.0);
    for (size_t i = 0; i < op->nb_rank.size(); ++i) {
      cnt[(size_t)me * P + op->nb_rank[i]] = (double)op->recv_cnt[i];
      cnt[(size_t)P * P + (size_t)me * P + op->nb_rank[i]] = (double)op->send_cnt[i];
    }
    const int chunk = S_E2 - S_DOT + 1;  // scratch slots S_DOT .. S_E2
    for (size_t b0 = 0; b0 < cnt.size(); b0 += (size_t)chunk) {
      const int k = (int)std::min<size_t>((size_t)chunk, cnt.size() - b0);
      allreduce_host(c, cnt.data() + b0, cnt.data() + b0, k);
    }
    for (int a = 0; a < P; ++a)
      for (int q = 0; q < P; ++q)
        if (cnt[(size_t)a * P + q] != cnt[(size_t)P * P + (size_t)q * P + a])
          fail(PCGX_ERR_INVALID, "CsrMatrix: block rows are not symmetric: rank " + std::to_string(a) +
                                     " needs " + std::to_string((long long)cnt[(size_t)a * P + q]) +
                                     " values of rank " + std::to_string(q) + ", which would send " +
                                     std::to_string((long long)cnt[(size_t)P * P + (size_t)q * P + a]));
  }
  op->kind = 1;
  op->n_global = n;
  op->nnz = nnz;  // this rank's rows
  op->row0 = r0;
  op->n_local = nloc;
  op->nghost = (long long)ghosts.size();
  op->nsend = (long long)send_idx.size();
  PCGX_CUDA(cudaMalloc(&op->dvec, sizeof(double) * (size_t)(nloc + std::max(op->nghost, 1LL))));
  PCGX_CUDA(cudaMemcpy(op->dvec, dv.data(), sizeof(double) * (size_t)nloc, cudaMemcpyHostToDevice));
  PCGX_CUDA(cudaMalloc(&op->rp, sizeof(int) * lrp.size()));
  PCGX_CUDA(cudaMemcpy(op->rp, lrp.data(), sizeof(int) * lrp.size(), cudaMemcpyHostToDevice));
  const size_t ng = (size_t)std::max(op->nghost, 1LL), nsd = (size_t)std::max(op->nsend, 1LL);
  PCGX_CUDA(cudaMalloc(&op->send_idx, sizeof(int) * nsd));
  if (op->nsend)
    PCGX_CUDA(cudaMemcpy(op->send_idx, send_idx.data(), sizeof(int) * send_idx.size(), cudaMemcpyHostToDevice));
  PCGX_CUDA(cudaMalloc(&op->sbuf_z, sizeof(double) * nsd));
  PCGX_CUDA(cudaMalloc(&op->sbuf_p, sizeof(double) * nsd));
  PCGX_CUDA(cudaMalloc(&op->ghost_z, sizeof(double) * ng));
  PCGX_CUDA(cudaMalloc(&op->ghost_p, sizeof(double) * ng));
  PCGX_CUDA(cudaDeviceSynchronize());  // legacy-stream uploads before the compute stream
  // the ghost columns' Jacobi values from their owners, through the block-row exchange
  if (op->nsend)
    pack_kernel<<<vec_grid(c, op->nsend), kVecThreads, 0, c->s>>>(op->nsend, op->send_idx, op->dvec,
                                                                   op->sbuf_z);
  check_launch();
  const double* sb[1] = {op->sbuf_z};
  double* gb[1] = {op->ghost_z};
  c->cm->sparse_xchg(c, op, 1, sb, gb);
  c->cm->halo_wait(c);
  if (op->nghost)
    PCGX_CUDA(cudaMemcpyAsync(op->dvec + nloc, op->ghost_z, sizeof(double) * (size_t)op->nghost,
                              cudaMemcpyDeviceToDevice, c->s));
  PCGX_CUDA(cudaStreamSynchronize(c->s));
  // whole 3 x 3 block rows with block-aligned ghost columns keep BSR-3 (a per-rank
  // choice: the exchange lists do not depend on the storage)
  if (op->tune.bsr != 0 && r0 % 3 == 0 && is_bsr3(nloc, lrp, lci)) build_bsr3(op, nloc, lrp, lci, va);
  else build_sell(op, nloc, lrp, lci, va);
}

// SELL-32 arrays of an int32 CSR (n rows, local column space) -> op (see sell_kernel).
void build_sell(pcgx_operator op, long long n, const std::vector<int>& rp32,
                const std::vector<int>& ci32, const double* va) {
  const long long ns = (n + 31) / 32;
  std::vector<long long> sp((size_t)ns + 1, 0);
  std::vector<int> rl((size_t)std::max(n, 1LL));
  for (long long sI = 0; sI < ns; ++sI) {
    int L = 0;
    for (long long r = sI * 32; r < std::min(n, sI * 32 + 32); ++r) {
      rl[(size_t)r] = rp32[(size_t)r + 1] - rp32[(size_t)r];
      L = std::max(L, rl[(size_t)r]);
    }
    sp[(size_t)sI + 1] = sp[(size_t)sI] + 32LL * L;
  }
  const long long tot = sp[(size_t)ns];
  std::vector<int> scol((size_t)std::max(tot, 1LL), 0);
  std::vector<double> sval((size_t)std::max(tot, 1LL), 0.0);
#pragma omp parallel for schedule(static)
  for (long long sI = 0; sI < ns; ++sI)
    for (long long r = sI * 32; r < std::min(n, sI * 32 + 32); ++r) {
      const long long lane = r - sI * 32;
      for (int k = 0; k < rl[(size_t)r]; ++k) {
        const long long src = rp32[(size_t)r] + k;
        const long long dst = sp[(size_t)sI] + 32LL * k + lane;
        scol[(size_t)dst] = ci32[(size_t)src];
        sval[(size_t)dst] = va[src];
      }
    }
  op->nslices = (int)ns;
  PCGX_CUDA(cudaMalloc(&op->sell_ptr, sizeof(long long) * sp.size()));
  PCGX_CUDA(cudaMalloc(&op->sell_len, sizeof(int) * rl.size()));
  PCGX_CUDA(cudaMalloc(&op->sell_col, sizeof(int) * scol.size()));
  PCGX_CUDA(cudaMalloc(&op->sell_val, sizeof(double) * sval.size()));
  PCGX_CUDA(cudaMemcpy(op->sell_ptr, sp.data(), sizeof(long long) * sp.size(), cudaMemcpyHostToDevice));
  PCGX_CUDA(cudaMemcpy(op->sell_len, rl.data(), sizeof(int) * rl.size(), cudaMemcpyHostToDevice));
  PCGX_CUDA(cudaMemcpy(op->sell_col, scol.data(), sizeof(int) * scol.size(), cudaMemcpyHostToDevice));
  PCGX_CUDA(cudaMemcpy(op->sell_val, sval.data(), sizeof(double) * sval.size(), cudaMemcpyHostToDevice));
  op->sell_padded = tot;
  // slices that touch no ghost column (local columns are < n): run while the halo travels
  int b0 = (int)ns, b1 = 0;
  for (long long sI = 0; sI < ns; ++sI) {
    bool ghost = false;
    for (long long r = sI * 32; r < std::min(n, sI * 32 + 32) && !ghost; ++r)
      for (int k = rp32[(size_t)r]; k < rp32[(size_t)r + 1]; ++k)
        if (ci32[(size_t)k] >= n) {
          ghost = true;
          break;
        }
    if (ghost) {
      b0 = std::min(b0, (int)sI);
      b1 = std::max(b1, (int)sI + 1);
    }
  }
  if (b0 >= b1) {  // no ghost anywhere
    op->sl_b0 = 0;
    op->sl_b1 = (int)ns;
  } else {  // ghost slices are a prefix and a suffix for block rows: interior in between
    int lead = 0;
    while (lead < (int)ns) {
      bool ghost = false;
      for (long long r = (long long)lead * 32; r < std::min(n, (long long)lead * 32 + 32) && !ghost; ++r)
        for (int k = rp32[(size_t)r]; k < rp32[(size_t)r + 1]; ++k)
          if (ci32[(size_t)k] >= n) {
            ghost = true;
            break;
          }
      if (!ghost) break;
      ++lead;
    }
    int trail = (int)ns;
    while (trail > lead) {
      bool ghost = false;
      const long long sI = trail - 1;
      for (long long r = sI * 32; r < std::min(n, sI * 32 + 32) && !ghost; ++r)
        for (int k = rp32[(size_t)r]; k < rp32[(size_t)r + 1]; ++k)
          if (ci32[(size_t)k] >= n) {
            ghost = true;
            break;
          }
      if (!ghost) break;
      --trail;
    }
    // any ghost slice strictly inside [lead, trail) forces the whole range after the halo
    bool inner_ghost = false;
    for (long long sI = lead; sI < trail && !inner_ghost; ++sI)
      for (long long r = sI * 32; r < std::min(n, sI * 32 + 32) && !inner_ghost; ++r)
        for (int k = rp32[(size_t)r]; k < rp32[(size_t)r + 1]; ++k)
          if (ci32[(size_t)k] >= n) {
            inner_ghost = true;
            break;
          }
    op->sl_b0 = inner_ghost ? 0 : lead;
    op->sl_b1 = inner_ghost ? 0 : trail;
  }
}

// Rows in aligned triples (3I, 3I+1, 3I+2) sharing one pattern of full 3x3 blocks
// (columns 3J, 3J+1, 3J+2 consecutive): the 3-dof-per-node block structure.
bool is_bsr3(long long n, const std::vector<int>& rp, const std::vector<int>& ci) {
  if (n <= 0 || n % 3) return false;
  const long long nb = n / 3;
  int ok = 1;
#pragma omp parallel for schedule(static) reduction(&& : ok)
  for (long long I = 0; I < nb; ++I) {
    if (!ok) continue;
    const long long a = 3 * I;
    const int len = rp[(size_t)a + 1] - rp[(size_t)a];
    bool good = len % 3 == 0;
    for (int c = 1; c < 3 && good; ++c) good = rp[(size_t)a + c + 1] - rp[(size_t)a + c] == len;
    for (int k = 0; k < len && good; k += 3) {
      const int c0 = ci[(size_t)rp[(size_t)a] + k];
      good = c0 % 3 == 0;
      for (int c = 0; c < 3 && good; ++c)
        for (int d = 0; d < 3 && good; ++d) good = ci[(size_t)rp[(size_t)a + c] + k + d] == c0 + d;
    }
    ok = ok && good;
  }
  return ok != 0;
}

// The sorted set of column offsets (col - row) if it has at most kDiaMax members.
// (rows [row_base, row_base + n) of a larger matrix: rp is local, ci global)
bool dia_offsets(long long n, const std::vector<int>& rp, const std::vector<int>& ci,
                 std::vector<int>& off, long long row_base) {
  off.clear();
  // rows mostly repeat their neighbour's offset pattern: only new patterns are merged
  int pa = 0, pb = 0;  // previous row's entries [pa, pb) and its row index
  long long prow = -1;
  for (long long i = 0; i < n; ++i) {
    const int a = rp[(size_t)i], b = rp[(size_t)i + 1];
    bool same = prow >= 0 && b - a == pb - pa;
    for (int k = 0; k < b - a && same; ++k)
      same = (long long)ci[(size_t)(a + k)] - i == (long long)ci[(size_t)(pa + k)] - prow;
    if (!same)
      for (int k = a; k < b; ++k) {
        const long long o = (long long)ci[(size_t)k] - (i + row_base);
        if (std::find(off.begin(), off.end(), (int)o) == off.end()) {
          if ((int)off.size() == kDiaMax) return false;
          off.push_back((int)o);
        }
      }
    pa = a;
    pb = b;
    prow = i;
  }
  std::sort(off.begin(), off.end());
  return !off.empty();
}

// dia3_kernel applies when the matrix lives on a cubic nx^3 grid in the
// reference's index order, its column offsets are exactly DiaPat<P>'s (slot s =
// grid neighbour s) and no coupling wraps across a grid face.
template <int P>
bool dia3_match(long long n, int nx, const std::vector<int>& rp, const std::vector<int>& ci,
                const std::vector<int>& off, long long row_base) {
  using Pat = DiaPat<P>;
  if ((int)off.size() != Pat::K) return false;
  const long long nxy = (long long)nx * nx;
  for (int s = 0; s < Pat::K; ++s)
    if ((long long)off[(size_t)s] != Pat::dz(s) * nxy + Pat::dy(s) * (long long)nx + Pat::dx(s)) return false;
  int ok = 1;
#pragma omp parallel for schedule(static) reduction(&& : ok)
  for (long long rl = 0; rl < n; ++rl) {
    const long long r = rl + row_base;
    const int a = (int)(r % nx), b = (int)((r / nx) % nx), c = (int)(r / nxy);
    for (int k = rp[(size_t)rl]; k < rp[(size_t)rl + 1]; ++k) {
      const long long o = (long long)ci[(size_t)k] - r;
      int s = 0;
      while (s < Pat::K && off[(size_t)s] != o) ++s;
      const int aa = a + Pat::dx(s), bb = b + Pat::dy(s), cc = c + Pat::dz(s);
      if (aa < 0 || aa >= nx || bb < 0 || bb >= nx || cc < 0 || cc >= nx) ok = 0;
    }
  }
  return ok != 0;
}

void dia3_detect(pcgx_operator op, long long n, const std::vector<int>& rp, const std::vector<int>& ci,
                 const std::vector<int>& off) {
  op->dia3_pat = 0;
  int nx = (int)std::llround(std::cbrt((double)n));
  while ((long long)nx * nx * nx > n) --nx;
  while ((long long)(nx + 1) * (nx + 1) * (nx + 1) <= n) ++nx;
  if (nx < 3 || (long long)nx * nx * nx != n) return;
  if (dia3_match<27>(n, nx, rp, ci, off)) op->dia3_pat = 27;
  else if (dia3_match<7>(n, nx, rp, ci, off)) op->dia3_pat = 7;
  op->dia3_nx = nx;
}

// Offset-storage arrays (see dia_kernel).
void build_dia(pcgx_operator op, long long n, const std::vector<int>& rp32,
               const std::vector<int>& ci32, const double* va, const std::vector<int>& off) {
  const int K = (int)off.size();
  const long long ld = (n + 31) / 32 * 32;  // rows incl. the last slice's padding
  std::vector<double> val((size_t)(ld * K), 0.0);
  std::vector<unsigned> mask((size_t)n, 0u);
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < n; ++i) {
    int q = 0;
    for (int k = rp32[(size_t)i]; k < rp32[(size_t)i + 1]; ++k) {
      const int o = (int)((long long)ci32[(size_t)k] - i);
      while (off[(size_t)q] != o) ++q;  // both ascending
      val[(size_t)(q * ld + i)] = va[k];
      mask[(size_t)i] |= 1u << q;
    }
  }
  op->dia_k = K;
  op->dia_ld = ld;
  dia3_detect(op, n, rp32, ci32, off);
  for (int k = 0; k < K; ++k) op->dia_off[k] = off[(size_t)k];
  PCGX_CUDA(cudaMalloc(&op->dia_val, sizeof(double) * val.size()));
  PCGX_CUDA(cudaMalloc(&op->dia_mask, sizeof(unsigned) * mask.size()));
  PCGX_CUDA(cudaMemcpy(op->dia_val, val.data(), sizeof(double) * val.size(), cudaMemcpyHostToDevice));
  PCGX_CUDA(cudaMemcpy(op->dia_mask, mask.data(), sizeof(unsigned) * mask.size(), cudaMemcpyHostToDevice));
}

// The bsr3t_kernel's grid copy of a BSR-3 matrix whose nodes form a cubic nx^3
// grid (nx % 4 == 0, nx >= 36: TMA strides and boxes) and whose blocks lie in the
// 27-point box without wrapping across a face; built slot by slot (one 9 ldn
// host buffer at a time) so the host never holds a second full copy.
void bsr3_grid_build(pcgx_operator op, long long n, const std::vector<int>& rp32,
                     const std::vector<int>& ci32, const double* va) {
  if (op->tune.bsr3t == 0) return;
  const long long nb = n / 3;
  long long nx = (long long)std::llround(std::cbrt((double)nb));
  while (nx * nx * nx > nb) --nx;
  while ((nx + 1) * (nx + 1) * (nx + 1) <= nb) ++nx;
  if (nx * nx * nx != nb || nx % 4 != 0 || nx < kB3PX / 3) return;
  const long long nxy = nx * nx;
  std::vector<signed char> pos((size_t)nb * 27, (signed char)-1);  // block index of slot s
  int ok = 1;
#pragma omp parallel for schedule(static) reduction(&& : ok)
  for (long long b = 0; b < nb; ++b) {
    const int a = (int)(b % nx), bb = (int)((b / nx) % nx), cc = (int)(b / nxy);
    const int len = (rp32[(size_t)(3 * b + 1)] - rp32[(size_t)(3 * b)]) / 3;
    for (int k = 0; k < len && ok; ++k) {
      const long long o = (long long)(ci32[(size_t)rp32[(size_t)(3 * b)] + 3 * k] / 3) - b;
      int s = -1;
      for (int q = 0; q < 27; ++q)
        if (o == (q / 9 - 1) * nxy + ((q / 3) % 3 - 1) * nx + (q % 3 - 1)) s = q;
      if (s < 0) { ok = 0; break; }
      const int x2 = a + s % 3 - 1, y2 = bb + (s / 3) % 3 - 1, z2 = cc + s / 9 - 1;
      if (x2 < 0 || x2 >= nx || y2 < 0 || y2 >= nx || z2 < 0 || z2 >= nx) { ok = 0; break; }
      pos[(size_t)(b * 27 + s)] = (signed char)k;
    }
  }
  if (!ok) return;
  const long long ldn = (nb + 31) / 32 * 32;
  std::vector<unsigned> mask((size_t)nb, 0u);
#pragma omp parallel for schedule(static)
  for (long long b = 0; b < nb; ++b)
    for (int s = 0; s < 27; ++s)
      if (pos[(size_t)(b * 27 + s)] >= 0) mask[(size_t)b] |= 1u << s;
  PCGX_CUDA(cudaMalloc(&op->b3g_val, sizeof(double) * (size_t)(243 * ldn)));
  PCGX_CUDA(cudaMalloc(&op->b3g_mask, sizeof(unsigned) * (size_t)nb));
  PCGX_CUDA(cudaMemcpy(op->b3g_mask, mask.data(), sizeof(unsigned) * (size_t)nb, cudaMemcpyHostToDevice));
  std::vector<double> buf((size_t)(9 * ldn));
  for (int s = 0; s < 27; ++s) {
#pragma omp parallel for schedule(static)
    for (long long b = 0; b < ldn; ++b) {
      const int k = b < nb ? pos[(size_t)(b * 27 + s)] : -1;
      for (int c = 0; c < 3; ++c)
        for (int d = 0; d < 3; ++d)
          buf[(size_t)((3 * c + d) * ldn + b)] = k >= 0 ? va[(size_t)rp32[(size_t)(3 * b + c)] + 3 * k + d] : 0.0;
    }
    PCGX_CUDA(cudaMemcpy(op->b3g_val + (size_t)(9 * s * ldn), buf.data(), sizeof(double) * buf.size(),
                         cudaMemcpyHostToDevice));
  }
  op->b3g_ld = ldn;
  op->b3g_nx = (int)nx;
}

// BSR-3 / SELL-32 arrays (see bsr3_kernel) of an int32 CSR with is_bsr3 structure.
void build_bsr3(pcgx_operator op, long long n, const std::vector<int>& rp32,
                const std::vector<int>& ci32, const double* va) {
  const long long nb = n / 3;
  const long long ns = (nb + 31) / 32;
  std::vector<long long> sp((size_t)ns + 1, 0);
  std::vector<int> bl((size_t)nb);
  for (long long sI = 0; sI < ns; ++sI) {
    int L = 0;
    for (long long b = sI * 32; b < std::min(nb, sI * 32 + 32); ++b) {
      bl[(size_t)b] = (rp32[(size_t)(3 * b + 1)] - rp32[(size_t)(3 * b)]) / 3;
      L = std::max(L, bl[(size_t)b]);
    }
    sp[(size_t)sI + 1] = sp[(size_t)sI] + 32LL * L;
  }
  const long long tot = sp[(size_t)ns];
  std::vector<int> bcol((size_t)std::max(tot, 1LL), 0);
  std::vector<double> bval((size_t)std::max(tot, 1LL) * 9, 0.0);
#pragma omp parallel for schedule(static)
  for (long long sI = 0; sI < ns; ++sI)
    for (long long b = sI * 32; b < std::min(nb, sI * 32 + 32); ++b) {
      const long long lane = b - sI * 32;
      for (int k = 0; k < bl[(size_t)b]; ++k) {
        const long long slot = sp[(size_t)sI] + 32LL * k;
        bcol[(size_t)(slot + lane)] = ci32[(size_t)rp32[(size_t)(3 * b)] + 3 * k] / 3;
        for (int c = 0; c < 3; ++c)
          for (int d = 0; d < 3; ++d)
            bval[(size_t)(slot * 9 + 32 * (3 * c + d) + lane)] =
                va[(size_t)rp32[(size_t)(3 * b + c)] + 3 * k + d];
      }
    }
  op->bsr_slices = (int)ns;
  op->bsr_blocks = (long long)rp32[(size_t)n] / 9;
  op->bsr_padded = tot;
  PCGX_CUDA(cudaMalloc(&op->bsr_ptr, sizeof(long long) * sp.size()));
  PCGX_CUDA(cudaMalloc(&op->bsr_len, sizeof(int) * bl.size()));
  PCGX_CUDA(cudaMalloc(&op->bsr_col, sizeof(int) * bcol.size()));
  PCGX_CUDA(cudaMalloc(&op->bsr_val, sizeof(double) * bval.size()));
  PCGX_CUDA(cudaMemcpy(op->bsr_ptr, sp.data(), sizeof(long long) * sp.size(), cudaMemcpyHostToDevice));
  PCGX_CUDA(cudaMemcpy(op->bsr_len, bl.data(), sizeof(int) * bl.size(), cudaMemcpyHostToDevice));
  PCGX_CUDA(cudaMemcpy(op->bsr_col, bcol.data(), sizeof(int) * bcol.size(), cudaMemcpyHostToDevice));
  PCGX_CUDA(cudaMemcpy(op->bsr_val, bval.data(), sizeof(double) * bval.size(), cudaMemcpyHostToDevice));
  bsr3_grid_build(op, n, rp32, ci32, va);
}

template <class IdxT>
void csr_upload(pcgx_context c, pcgx_operator op, long long n, const IdxT* rp, const IdxT* ci,
                const double* va, const double* inv_sqrt) {
  if (n < 0) fail(PCGX_ERR_INVALID, "LinearOperator: negative dimension");
  if (!rp || (n > 0 && (!ci || !va)) ) fail(PCGX_ERR_INVALID, "CsrMatrix: null array");
  if (rp[0] != 0) fail(PCGX_ERR_INVALID, "CsrMatrix: row_ptr must have length n+1 and start at 0");
  const long long nnz = (long long)rp[n];
  if (nnz >= (1LL << 31) || n >= (1LL << 31))
    fail(PCGX_ERR_OVERFLOW, "csr_create: nnz " + std::to_string(nnz) +
                                " does not fit the int32 device CSR");
  std::vector<int> rp32((size_t)n + 1);
  std::vector<int> ci32((size_t)nnz);
  std::vector<double> dv((size_t)std::max(n, 1LL));
  for (long long i = 0; i < n; ++i) {
    if (rp[i + 1] < rp[i]) fail(PCGX_ERR_INVALID, "CsrMatrix: row_ptr not nondecreasing");
    double diag = 0.0;
    for (long long k = rp[i]; k < rp[i + 1]; ++k) {
      const long long col = (long long)ci[k];
      if (col < 0 || col >= n)
        fail(PCGX_ERR_INVALID, "CsrMatrix: column index out of range in row " + std::to_string(i));
      if (k > rp[i] && col <= (long long)ci[k - 1])
        fail(PCGX_ERR_INVALID, "CsrMatrix: columns not strictly increasing in row " + std::to_string(i));
      if (col == i) diag = va[k];
      ci32[(size_t)k] = (int)col;
    }
    rp32[(size_t)i + 1] = (int)rp[i + 1];
    if (inv_sqrt) {
      dv[(size_t)i] = inv_sqrt[i];
    } else {  // jacobi_scale (linop.cpp:340-351)
      if (!(diag > 0.0))
        fail(PCGX_ERR_NUMERICAL, "jacobi_scale: nonpositive diagonal entry at index " +
                                     std::to_string(i) + " (" + std::to_string(diag) + ")");
      dv[(size_t)i] = 1.0 / std::sqrt(diag);
    }
  }
  op->kind = 1;
  op->n_global = n;
  op->nnz = nnz;
  if (c->nranks > 1) {
    csr_upload_block(c, op, n, rp32, ci32, va, dv);
    return;
  }
  op->n_local = n;
  PCGX_CUDA(cudaMalloc(&op->rp, sizeof(int) * (size_t)(n + 1)));
  // +8 entries of padding: the TMA tile copies round their length up to 4 entries
  PCGX_CUDA(cudaMalloc(&op->ci, sizeof(int) * (size_t)(nnz + 8)));
  PCGX_CUDA(cudaMalloc(&op->va, sizeof(double) * (size_t)(nnz + 8)));
  PCGX_CUDA(cudaMemset(op->ci, 0, sizeof(int) * (size_t)(nnz + 8)));
  PCGX_CUDA(cudaMemset(op->va, 0, sizeof(double) * (size_t)(nnz + 8)));
  PCGX_CUDA(cudaMalloc(&op->dvec, sizeof(double) * (size_t)std::max(n, 1LL)));
  PCGX_CUDA(cudaMemcpy(op->rp, rp32.data(), sizeof(int) * (size_t)(n + 1), cudaMemcpyHostToDevice));
  if (nnz) {
    PCGX_CUDA(cudaMemcpy(op->ci, ci32.data(), sizeof(int) * (size_t)nnz, cudaMemcpyHostToDevice));
    PCGX_CUDA(cudaMemcpy(op->va, va, sizeof(double) * (size_t)nnz, cudaMemcpyHostToDevice));
  }
  if (n) PCGX_CUDA(cudaMemcpy(op->dvec, dv.data(), sizeof(double) * (size_t)n, cudaMemcpyHostToDevice));
  std::vector<int> doff;
  // offset storage moves fewer bytes than int32 CSR while 8 K n + 4 n < 12 nnz + 4 n
  const bool dia = n > 0 && op->tune.dia != 0 && dia_offsets(n, rp32, ci32, doff) &&
                   (double)doff.size() * (double)n <= 1.5 * (double)nnz;
  if (dia) {
    build_dia(op, n, rp32, ci32, va, doff);
    cudaFree(op->ci);
    cudaFree(op->va);
    op->ci = nullptr;
    op->va = nullptr;
  } else if (n > 0 && op->tune.bsr != 0 && is_bsr3(n, rp32, ci32)) {
    build_bsr3(op, n, rp32, ci32, va);
    cudaFree(op->ci);
    cudaFree(op->va);
    op->ci = nullptr;
    op->va = nullptr;
  } else if (n > 0) {
    build_sell(op, n, rp32, ci32, va);
    // the SELL copy replaces the CSR value/index arrays on the device
    cudaFree(op->ci);
    cudaFree(op->va);
    op->ci = nullptr;
    op->va = nullptr;
  }
}

void free_op(pcgx_operator op) {
  if (!op) return;
  cudaFree(op->ghost_lo);
  cudaFree(op->ghost_hi);
  cudaFree(op->ghost_lo2);
  cudaFree(op->ghost_hi2);
  cudaFree(op->rp);
  cudaFree(op->ci);
  cudaFree(op->va);
  cudaFree(op->dvec);
  cudaFree(op->sell_ptr);
  cudaFree(op->sell_len);
  cudaFree(op->sell_col);
  cudaFree(op->sell_val);
  cudaFree(op->bsr_ptr);
  cudaFree(op->bsr_len);
  cudaFree(op->bsr_col);
  cudaFree(op->bsr_val);
  cudaFree(op->b3g_val);
  cudaFree(op->b3g_mask);
  cudaFree(op->dia_val);
  cudaFree(op->dia_mask);
  cudaFree(op->dia3_dlo);
  cudaFree(op->dia3_dhi);
  cudaFree(op->send_idx);
  cudaFree(op->sbuf_z);
  cudaFree(op->sbuf_p);
  cudaFree(op->ghost_z);
  cudaFree(op->ghost_p);
  delete op;
}

void ctx_init(pcgx_context c) {
  c->tune = Tuning::from_env();
  PCGX_CUDA(cudaSetDevice(c->device));
  PCGX_CUDA(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, c->device));
  PCGX_CUDA(cudaStreamCreateWithFlags(&c->s, cudaStreamNonBlocking));
  PCGX_CUDA(cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking));
  PCGX_CUDA(cudaMalloc(&c->S, sizeof(double) * kSlots));
  PCGX_CUDA(cudaMemset(c->S, 0, sizeof(double) * kSlots));
  PCGX_CUDA(cudaHostAlloc(&c->hS, sizeof(double) * kSlots, cudaHostAllocMapped));
  PCGX_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->dS_map), c->hS, 0));
  PCGX_CUDA(cudaMalloc(&c->partials, sizeof(double) * kMaxBlocks));
  PCGX_CUDA(cudaMalloc(&c->counter, sizeof(unsigned) * 4));
  PCGX_CUDA(cudaMemset(c->counter, 0, sizeof(unsigned) * 4));
  PCGX_CUDA(cudaEventCreate(&c->ev_t0));
  PCGX_CUDA(cudaEventCreate(&c->ev_t1));
  PCGX_CUDA(cudaEventCreateWithFlags(&c->ev_sync, cudaEventDisableTiming));
  PCGX_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  PCGX_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  // the legacy-stream memsets above are unordered with the non-blocking streams
  PCGX_CUDA(cudaDeviceSynchronize());
}

// The matrix-free 7-point operator's fields (frees op on failure).
void stencil_setup(pcgx_context c, pcgx_operator op, int64_t nx, int64_t ny, int64_t nz, double inv_sqrt_diag) {
  {
    op->kind = 0;
    op->nx = nx;
    op->ny = ny;
    op->nz = nz;
    int64_t z0 = 0, nzl = 0;
    pcgx_slab_partition(nz, c->nranks, c->rank, &z0, &nzl);
    op->nzl = nzl;
    op->z0 = z0;
    op->n_global = nx * ny * nz;
    op->n_local = nx * ny * op->nzl;
    op->nnz = 7 * op->n_global - 2 * (ny * nz + nx * nz + nx * ny);
    op->d = inv_sqrt_diag > 0.0 ? inv_sqrt_diag : 1.0 / std::sqrt(6.0);
    op->kz = default_kz(c, nx, ny, op->nzl);
    op->vec2 = (nx % 2 == 0);
    op->pfd = op->tune.pfd;
    op->cheb2 = op->vec2 && op->tune.cheb2 != 0;
    op->kz2 = op->tune.kz2;
    op->c2plan = op->tune.c2plan;
    try {
      init_stencil_ghosts(c, op);
      if (c->nranks > 1 && op->nzl < 2) op->cheb2 = false;  // 2-plane halos need >= 2 planes
      op->zpad = (op->cheb2 && c->nranks > 1) ? 2 : 0;
      op->cheb3 = op->cheb2 && c->nranks == 1 && op->tune.cheb3 != 0;
    } catch (...) {
      free_op(op);
      throw;
    }
  }
}

// Whether a CSR matrix is exactly assemble_laplacian(lap3d, nx) (linop.cpp:299-331):
// cubic n = nx^3, every row the 7-point star in ascending columns with the
// Dirichlet neighbours omitted, diagonal 6 and off-diagonals -1, and (if given) the
// Jacobi vector 1/sqrt(6). Its scaled apply is then bitwise the StencilOperator's
// (test_linop.cpp:67-79), so the matrix-free kernels can serve it. Opt-in
// (PCGX_CSR_STENCIL=1): a CsrMatrix input is benchmarked as CSR (config 1 keeps its
// offset storage and reads its values), this is a user-side shortcut.
template <class I>
bool csr_is_lap3d(int64_t n, const I* rp, const I* ci, const double* va, const double* isd, int64_t* nx_out) {
  if (n < 8) return false;
  int64_t nx = (int64_t)std::llround(std::cbrt((double)n));
  while (nx * nx * nx > n) --nx;
  while ((nx + 1) * (nx + 1) * (nx + 1) <= n) ++nx;
  if (nx * nx * nx != n || nx < 2) return false;
  const int64_t nxy = nx * nx;
  const double d6 = 1.0 / std::sqrt(6.0);
  int ok = 1;
#pragma omp parallel for schedule(static) reduction(&& : ok)
  for (int64_t r = 0; r < n; ++r) {
    if (!ok) continue;
    const int64_t i = r % nx, j = (r / nx) % nx, k = r / nxy;
    const int64_t off[7] = {-nxy, -nx, -1, 0, 1, nx, nxy};
    const bool on[7] = {k > 0, j > 0, i > 0, true, i < nx - 1, j < nx - 1, k < nx - 1};
    int64_t p = (int64_t)rp[r];
    for (int s = 0; s < 7 && ok; ++s) {
      if (!on[s]) continue;
      if (p >= (int64_t)rp[r + 1] || (int64_t)ci[p] != r + off[s] || va[p] != (s == 3 ? 6.0 : -1.0)) ok = 0;
      ++p;
    }
    if (p != (int64_t)rp[r + 1]) ok = 0;
    if (isd && isd[r] != d6) ok = 0;
  }
  if (ok) *nx_out = nx;
  return ok != 0;
}

template <class I>
void csr_create_any(pcgx_context c, pcgx_operator op, int64_t n, const I* rp, const I* ci, const double* va,
                    const double* isd) {
  int64_t nx = 0;
  if (c->nranks == 1 && rp && ci && va && op->tune.csr_stencil != 0 &&
      csr_is_lap3d(n, rp, ci, va, isd, &nx)) {
    stencil_setup(c, op, nx, nx, nx, 1.0 / std::sqrt(6.0));
    op->nnz = (int64_t)rp[n];
    return;
  }
  try {
    csr_upload(c, op, n, rp, ci, va, isd);
  } catch (...) {
    free_op(op);
    throw;
  }
}

