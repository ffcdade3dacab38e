// SPDX-License-Identifier: Apache-2.0
//
// Part of pcgx.cu (ONE translation unit): included in place, in the middle of that
// file's declarations; not a standalone header. The communicators (CommBase: NCCL, in-process group, host shared memory, CUDA-IPC mailboxes, loopback).
#pragma once

// ---------------------------------------------------------------- communication
//
// CommBase is the only place ranks meet. NcclComm: one process per GPU, NCCL
// over NVLink/NVSwitch (the production path). LocalGroup: P ranks as P
// contexts in ONE process (one host thread each, any devices), exchanging halo
// planes with stream-ordered cudaMemcpyAsync and reducing scalars in rank
// order; no kernel ever waits on another kernel (dependencies are CUDA events
// plus a host barrier), so the multi-rank slab logic can be exercised on a
// single GPU. Both are collective: every rank calls them at the same point.

}  // namespace
struct CommBase {
  virtual ~CommBase() = default;
  virtual void allreduce(pcgx_context c, int slot, int count) = 0;
  // Start exchanging the first/last owned plane of each of the nv vectors into
  // the neighbours' ghost set v (v = 0: ghost_lo/hi, v = 1: ghost_lo2/hi2).
  virtual void halo_begin(pcgx_context c, pcgx_operator op, const double* const* xs, int nv) = 0;
  // Make c->s wait until this rank's ghost planes hold the neighbours' planes.
  virtual void halo_wait(pcgx_context c) = 0;
  // Generic plane exchange (two-step kernel): for each item my bottom `count`
  // elements go to rank-1's recv_hi and my top ones to rank+1's recv_lo; I
  // receive into my recv_lo / recv_hi. Completes like halo_begin (halo_wait).
  struct PlaneX {
    const double* send_lo;
    double* recv_lo;
    const double* send_hi;
    double* recv_hi;
    long long count;
  };
  virtual void xchg(pcgx_context c, pcgx_operator op, const PlaneX* items, int n) = 0;
  // CSR block rows: send nv packed buffers' per-neighbour segments, receive the
  // neighbours' segments into the ghost arrays (op->nb_rank / send_* / recv_*).
  virtual void sparse_xchg(pcgx_context c, pcgx_operator op, int nv, const double* const* sbuf,
                           double* const* gbuf) = 0;
  virtual bool graph_capturable() const = 0;
};
namespace {

struct NcclComm : CommBase {
  void allreduce(pcgx_context c, int slot, int count) override {
    PCGX_NCCL(nccl().AllReduce(c->S + slot, c->S + slot, count, ncclDouble, ncclSum, c->comm, c->s));
  }
  void halo_begin(pcgx_context c, pcgx_operator op, const double* const* xs, int nv) override;
  void halo_wait(pcgx_context c) override { PCGX_CUDA(cudaStreamWaitEvent(c->s, c->ev_join, 0)); }
  void xchg(pcgx_context c, pcgx_operator op, const PlaneX* items, int n) override;
  void sparse_xchg(pcgx_context c, pcgx_operator op, int nv, const double* const* sbuf,
                   double* const* gbuf) override;
  bool graph_capturable() const override { return true; }
};

// LoopbackComm (measurement only): ONE process standing in for a rank of a P-rank
// z-slab job on a single GPU. It owns its slab of the global grid and runs the whole
// slab code path -- ghost planes, the exchange forked onto the comm stream, interior
// launches meanwhile, boundary launches after the join, per-iteration all-reduce
// points -- but its neighbours' planes are its OWN opposite boundary planes, copied
// device-to-device with the real exchange's sizes, and an all-reduce keeps the local
// value. What it solves is the slab with periodic ghosts in z (still SPD: Dirichlet in
// x and y), so a PCG solve converges and its per-iteration time is that of a rank with
// two neighbours minus the link: the slab path's own overhead, measurable on one GPU
// (tools/slab_overhead.py). Not a product communicator.
struct LoopbackComm : CommBase {
  void allreduce(pcgx_context, int, int) override {}
  void halo_begin(pcgx_context c, pcgx_operator op, const double* const* xs, int nv) override {
    const long long nxy = op->nx * op->ny, nzl = op->nzl;
    const size_t pb = sizeof(double) * (size_t)nxy;
    PCGX_CUDA(cudaEventRecord(c->ev_fork, c->s));
    PCGX_CUDA(cudaStreamWaitEvent(c->cs, c->ev_fork, 0));
    for (int v = 0; v < nv; ++v) {
      double* glo = v ? op->ghost_lo2 : op->ghost_lo;
      double* ghi = v ? op->ghost_hi2 : op->ghost_hi;
      if (glo) PCGX_CUDA(cudaMemcpyAsync(glo, xs[v] + (nzl - 1) * nxy, pb, cudaMemcpyDeviceToDevice, c->cs));
      if (ghi) PCGX_CUDA(cudaMemcpyAsync(ghi, xs[v], pb, cudaMemcpyDeviceToDevice, c->cs));
    }
    PCGX_CUDA(cudaEventRecord(c->ev_join, c->cs));
  }
  void halo_wait(pcgx_context c) override { PCGX_CUDA(cudaStreamWaitEvent(c->s, c->ev_join, 0)); }
  void xchg(pcgx_context c, pcgx_operator op, const PlaneX* items, int n) override {
    const bool lo = op->ghost_lo != nullptr, hi = op->ghost_hi != nullptr;
    PCGX_CUDA(cudaEventRecord(c->ev_fork, c->s));
    PCGX_CUDA(cudaStreamWaitEvent(c->cs, c->ev_fork, 0));
    for (int i = 0; i < n; ++i) {
      const PlaneX& it = items[i];
      const size_t bytes = sizeof(double) * (size_t)it.count;
      if (lo) PCGX_CUDA(cudaMemcpyAsync(it.recv_lo, it.send_hi, bytes, cudaMemcpyDeviceToDevice, c->cs));
      if (hi) PCGX_CUDA(cudaMemcpyAsync(it.recv_hi, it.send_lo, bytes, cudaMemcpyDeviceToDevice, c->cs));
    }
    PCGX_CUDA(cudaEventRecord(c->ev_join, c->cs));
  }
  void sparse_xchg(pcgx_context, pcgx_operator, int, const double* const*, double* const*) override {
    fail(PCGX_ERR_UNSUPPORTED, "loopback context: matrix-free stencil operators only");
  }
  bool graph_capturable() const override { return false; }
};

class HostBarrier {
 public:
  explicit HostBarrier(int n) : n_(n) {}
  void wait() {
    std::unique_lock<std::mutex> lk(m_);
    const long gen = gen_;
    if (++count_ == n_) {
      count_ = 0;
      ++gen_;
      cv_.notify_all();
    } else {
      cv_.wait(lk, [&] { return gen != gen_; });
    }
  }

 private:
  std::mutex m_;
  std::condition_variable cv_;
  int n_, count_ = 0;
  long gen_ = 0;
};

// rank-ordered sum of the group's contributions into every rank's slots
__global__ void group_sum_kernel(const double* contrib, int nranks, int slot, int count, double* S) {
  const int i = threadIdx.x;
  if (i < count) {
    double s = 0.0;
    for (int q = 0; q < nranks; ++q) s += contrib[q * kSlots + slot + i];
    S[slot + i] = s;
  }
}

struct LocalGroup {
  int nranks;
  HostBarrier bar;
  std::vector<pcgx_context> ctx;
  std::vector<double*> ghost_lo, ghost_hi, ghost_lo2, ghost_hi2;
  std::vector<std::vector<double*>> xrecv_lo, xrecv_hi;  // per rank, per xchg item
  std::vector<std::vector<double*>> srecv;               // [rank][v * nranks + src] ghost destination
  std::vector<cudaEvent_t> ev_ar;   // rank's contribution copied
  std::vector<cudaEvent_t> ev_done; // rank finished reading contributions
  double* contrib = nullptr;        // nranks * kSlots doubles on the first rank's device
  std::atomic<int> refs{0};
  explicit LocalGroup(int n)
      : nranks(n), bar(n), ctx(n), ghost_lo(n), ghost_hi(n), ghost_lo2(n), ghost_hi2(n),
        xrecv_lo(n), xrecv_hi(n), srecv(n), ev_ar(n), ev_done(n) {}
};

struct LocalComm : CommBase {
  std::shared_ptr<LocalGroup> g;
  int rank;
  LocalComm(std::shared_ptr<LocalGroup> grp, int r) : g(std::move(grp)), rank(r) {}
  void allreduce(pcgx_context c, int slot, int count) override {
    // previous allreduce fully consumed by every rank before contrib is reused
    for (int q = 0; q < g->nranks; ++q) PCGX_CUDA(cudaStreamWaitEvent(c->s, g->ev_done[q], 0));
    PCGX_CUDA(cudaMemcpyAsync(g->contrib + rank * kSlots + slot, c->S + slot, sizeof(double) * count,
                              cudaMemcpyDefault, c->s));
    PCGX_CUDA(cudaEventRecord(g->ev_ar[rank], c->s));
    g->bar.wait();
    for (int q = 0; q < g->nranks; ++q) PCGX_CUDA(cudaStreamWaitEvent(c->s, g->ev_ar[q], 0));
    group_sum_kernel<<<1, 32, 0, c->s>>>(g->contrib, g->nranks, slot, count, c->S);
    check_launch();
    PCGX_CUDA(cudaEventRecord(g->ev_done[rank], c->s));
    g->bar.wait();
  }
  void halo_begin(pcgx_context c, pcgx_operator op, const double* const* xs, int nv) override;
  void halo_wait(pcgx_context c) override {  // my ghosts are written by the other ranks' copies
    for (int q = 0; q < g->nranks; ++q)
      if (q != rank) PCGX_CUDA(cudaStreamWaitEvent(c->s, g->ctx[q]->ev_join, 0));
  }
  void xchg(pcgx_context c, pcgx_operator op, const PlaneX* items, int n) override;
  void sparse_xchg(pcgx_context c, pcgx_operator op, int nv, const double* const* sbuf,
                   double* const* gbuf) override;
  bool graph_capturable() const override { return false; }
};

// ---------------------------------------------------------------- host-staged comm
// HostComm: P ranks in P processes on one host (any devices, also all on ONE GPU)
// exchanging through a POSIX shared-memory segment: every plane / segment / scalar
// is copied device -> shared memory -> device by the host, synchronously, with a
// process-shared barrier between the write and read phases. No kernel and no
// stream ever waits on another rank, so ranks that share a GPU cannot deadlock
// it. It exists to run the multi-process slab / block-row algorithm (the same
// CommBase calls NCCL serves) where there is one GPU: bitwise the LocalGroup
// results (scalars are summed in rank order, like group_sum_kernel).
struct ShmHeader {
  std::atomic<uint64_t> magic;
  std::atomic<int> count;  // barrier arrivals of the current generation
  std::atomic<int> gen;    // barrier generation
  std::atomic<int> abort;  // a rank gave up (timeout): the others fail instead of waiting
  int nranks;
  size_t cap;
};
static_assert(std::atomic<int>::is_always_lock_free && std::atomic<uint64_t>::is_always_lock_free,
              "host comm: atomics in shared memory must be address-free (lock-free)");
constexpr uint64_t kShmMagic = 0x70636778686f7374ull;  // "pcgxhost"
constexpr size_t kShmHdr = 4096;

struct HostComm : CommBase {
  int rank = 0, nranks = 1;
  std::string name;
  unsigned char* base = nullptr;
  size_t total = 0, cap = 0;
  ShmHeader* hdr() const { return reinterpret_cast<ShmHeader*>(base); }
  double* box(int r) const { return reinterpret_cast<double*>(base + kShmHdr + (size_t)r * cap); }
  // Counter barrier on lock-free atomics in the shared segment (release / acquire
  // orders each rank's outbox writes before the peers' reads). A rank that waits
  // longer than PCGX_HOSTCOMM_TIMEOUT seconds (default 600) marks the job aborted
  // and fails; every waiting rank then fails too instead of hanging.
  void barrier() const {
    ShmHeader* h = hdr();
    if (h->abort.load(std::memory_order_acquire)) fail(PCGX_ERR_NCCL, "host comm: a peer rank gave up");
    const int g = h->gen.load(std::memory_order_acquire);
    if (h->count.fetch_add(1, std::memory_order_acq_rel) + 1 == nranks) {
      h->count.store(0, std::memory_order_relaxed);
      h->gen.store(g + 1, std::memory_order_release);
      return;
    }
    const double limit = (double)std::max(1, env_int("PCGX_HOSTCOMM_TIMEOUT", 600));
    const auto t0 = std::chrono::steady_clock::now();
    for (long spins = 0; h->gen.load(std::memory_order_acquire) == g; ++spins) {
      if (h->abort.load(std::memory_order_acquire)) fail(PCGX_ERR_NCCL, "host comm: a peer rank gave up");
      if (spins > 2000) {
        usleep(20);
        if ((spins & 1023) == 0 &&
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit) {
          h->abort.store(1, std::memory_order_release);
          fail(PCGX_ERR_NCCL, "host comm: barrier timed out (a peer rank is gone)");
        }
      }
    }
  }
  // A rank that cannot continue marks the job aborted first, so the peers fail at
  // their next barrier instead of waiting out the timeout.
  void give_up() const { hdr()->abort.store(1, std::memory_order_release); }
  void need(size_t bytes) const {
    if (bytes > cap) {
      give_up();
      fail(PCGX_ERR_UNSUPPORTED, "host comm: message of " + std::to_string(bytes) + " bytes exceeds the " +
                                     std::to_string(cap) + "-byte mailbox");
    }
  }
  ~HostComm() override {
    if (!base) return;
    try {
      barrier();
    } catch (...) {
    }
    munmap(base, total);
    if (rank == 0) shm_unlink(name.c_str());
  }
  void allreduce(pcgx_context c, int slot, int count) override {
    PCGX_CUDA(cudaStreamSynchronize(c->s));
    PCGX_CUDA(cudaMemcpy(box(rank), c->S + slot, sizeof(double) * count, cudaMemcpyDeviceToHost));
    barrier();
    double sum[kSlots];
    for (int i = 0; i < count; ++i) {
      double v = 0.0;
      for (int q = 0; q < nranks; ++q) v += box(q)[i];
      sum[i] = v;
    }
    barrier();
    PCGX_CUDA(cudaMemcpyAsync(c->S + slot, sum, sizeof(double) * count, cudaMemcpyHostToDevice, c->s));
    PCGX_CUDA(cudaStreamSynchronize(c->s));
  }
  void xchg(pcgx_context c, pcgx_operator op, const PlaneX* items, int n) override {
    (void)op;
    PCGX_CUDA(cudaStreamSynchronize(c->s));
    size_t off = 0;
    for (int i = 0; i < n; ++i) off += 2 * (size_t)items[i].count;
    need(sizeof(double) * off);
    off = 0;
    for (int i = 0; i < n; ++i) {  // my outbox: [lo part | hi part] per item
      const size_t b = sizeof(double) * (size_t)items[i].count;
      if (rank > 0) PCGX_CUDA(cudaMemcpy(box(rank) + off, items[i].send_lo, b, cudaMemcpyDeviceToHost));
      if (rank < nranks - 1)
        PCGX_CUDA(cudaMemcpy(box(rank) + off + items[i].count, items[i].send_hi, b, cudaMemcpyDeviceToHost));
      off += 2 * (size_t)items[i].count;
    }
    barrier();
    off = 0;
    for (int i = 0; i < n; ++i) {  // rank-1's top -> my recv_lo, rank+1's bottom -> my recv_hi
      const size_t b = sizeof(double) * (size_t)items[i].count;
      if (rank > 0 && items[i].recv_lo)
        PCGX_CUDA(cudaMemcpyAsync(items[i].recv_lo, box(rank - 1) + off + items[i].count, b,
                                  cudaMemcpyHostToDevice, c->s));
      if (rank < nranks - 1 && items[i].recv_hi)
        PCGX_CUDA(cudaMemcpyAsync(items[i].recv_hi, box(rank + 1) + off, b, cudaMemcpyHostToDevice, c->s));
      off += 2 * (size_t)items[i].count;
    }
    PCGX_CUDA(cudaStreamSynchronize(c->s));  // the peers may refill their outboxes after the barrier
    barrier();
  }
  void halo_begin(pcgx_context c, pcgx_operator op, const double* const* xs, int nv) override {
    const long long nxy = op->nx * op->ny, nzl = op->nzl;
    PlaneX items[2];
    for (int v = 0; v < nv && v < 2; ++v)
      items[v] = {xs[v], v ? op->ghost_lo2 : op->ghost_lo, xs[v] + (nzl - 1) * nxy,
                  v ? op->ghost_hi2 : op->ghost_hi, nxy};
    xchg(c, op, items, std::min(nv, 2));
  }
  void halo_wait(pcgx_context c) override { (void)c; }  // the exchange completed synchronously
  void sparse_xchg(pcgx_context c, pcgx_operator op, int nv, const double* const* sbuf,
                   double* const* gbuf) override {
    PCGX_CUDA(cudaStreamSynchronize(c->s));
    const int P = nranks;
    // my outbox: a directory (offset, count) per destination rank, then the data
    int64_t* dir = reinterpret_cast<int64_t*>(box(rank));
    for (int q = 0; q < 2 * P; ++q) dir[q] = 0;
    size_t off = 2 * (size_t)P;  // in doubles (int64 and double are both 8 bytes)
    for (size_t i = 0; i < op->nb_rank.size(); ++i) {
      const int q = op->nb_rank[i];
      dir[q] = (int64_t)off;
      dir[P + q] = op->send_cnt[i];
      need(sizeof(double) * (off + (size_t)nv * op->send_cnt[i]));
      for (int v = 0; v < nv; ++v) {
        if (op->send_cnt[i])
          PCGX_CUDA(cudaMemcpy(box(rank) + off, sbuf[v] + op->send_off[i], sizeof(double) * op->send_cnt[i],
                               cudaMemcpyDeviceToHost));
        off += (size_t)op->send_cnt[i];
      }
    }
    barrier();
    for (size_t i = 0; i < op->nb_rank.size(); ++i) {
      const int q = op->nb_rank[i];
      const int64_t* qd = reinterpret_cast<const int64_t*>(box(q));
      const int64_t qoff = qd[rank], qcnt = qd[P + rank];
      if (qcnt != op->recv_cnt[i]) fail(PCGX_ERR_NCCL, "host comm: block-row segment size mismatch");
      for (int v = 0; v < nv; ++v)
        if (qcnt)
          PCGX_CUDA(cudaMemcpyAsync(gbuf[v] + op->recv_off[i], box(q) + qoff + (size_t)v * qcnt,
                                    sizeof(double) * qcnt, cudaMemcpyHostToDevice, c->s));
    }
    PCGX_CUDA(cudaStreamSynchronize(c->s));
    barrier();
  }
  bool graph_capturable() const override { return false; }
};

HostComm* host_comm_open(int nranks, int rank, const std::string& name, size_t cap) {
  auto hc = std::make_unique<HostComm>();
  hc->rank = rank;
  hc->nranks = nranks;
  hc->name = name;
  hc->cap = (cap + 4095) / 4096 * 4096;
  hc->total = kShmHdr + (size_t)nranks * hc->cap;
  int fd = -1;
  if (rank == 0) {
    shm_unlink(name.c_str());  // a stale segment of a crashed job
    fd = shm_open(name.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
    if (fd < 0) fail(PCGX_ERR_NCCL, "host comm: shm_open(" + name + ") failed");
    if (ftruncate(fd, (off_t)hc->total) != 0) {
      close(fd);
      fail(PCGX_ERR_NCCL, "host comm: ftruncate failed");
    }
  } else {
    for (int tries = 0; fd < 0; ++tries) {  // rank 0 creates it; up to 120 s
      fd = shm_open(name.c_str(), O_RDWR, 0600);
      struct stat st;
      if (fd >= 0 && (fstat(fd, &st) != 0 || (size_t)st.st_size < hc->total)) {
        close(fd);
        fd = -1;
      }
      if (fd < 0) {
        if (tries > 120000) fail(PCGX_ERR_NCCL, "host comm: segment " + name + " never appeared");
        usleep(1000);
      }
    }
  }
  void* m = mmap(nullptr, hc->total, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (m == MAP_FAILED) fail(PCGX_ERR_NCCL, "host comm: mmap failed");
  hc->base = static_cast<unsigned char*>(m);
  ShmHeader* h = hc->hdr();
  if (rank == 0) {
    h->count.store(0, std::memory_order_relaxed);
    h->gen.store(0, std::memory_order_relaxed);
    h->abort.store(0, std::memory_order_relaxed);
    h->nranks = nranks;
    h->cap = hc->cap;
    h->magic.store(kShmMagic, std::memory_order_release);
  } else {
    for (int tries = 0; h->magic.load(std::memory_order_acquire) != kShmMagic; ++tries) {
      if (tries > 120000) fail(PCGX_ERR_NCCL, "host comm: segment " + name + " never initialised");
      usleep(1000);
    }
    if (h->nranks != nranks || h->cap != hc->cap) fail(PCGX_ERR_INVALID, "host comm: ranks disagree on the job shape");
  }
  hc->barrier();  // everyone attached
  return hc.release();
}

// ---------------------------------------------------------------- peer-memory comm
// IpcComm: P ranks in P processes on one node (one GPU each over NVLink / NVSwitch,
// or sharing a GPU) exchanging through DEVICE memory: each rank exports a device
// mailbox (two parity areas) and four events by CUDA IPC; every exchange is
// stream-ordered -- the sender's stream copies its planes / segments / scalars
// into its own mailbox and records `ready`, the receivers' streams wait on that
// event and pull straight from the peer's mailbox into their ghost buffers (a
// peer-to-peer copy over NVLink between GPUs), then record `done`. The host only
// meets the peers at one shared-memory barrier per exchange (so each wait is
// issued after the record it waits for); no host-side stream synchronisation, no
// host staging, and the halo copies overlap the interior kernels like NCCL's.
// No kernel ever waits on another rank (only streams wait on recorded events),
// so ranks that share a GPU cannot deadlock it. Parity areas: an exchange reuses
// the area of two exchanges ago only after every peer's `done` of that exchange
// (the barrier in between orders the host calls). Scalars are summed in rank
// order by peer_sum_kernel (bitwise the LocalGroup / HostComm sums).
__global__ void peer_sum_kernel(const double* const* boxes, long long area_off, int nranks, int slot, int count,
                                double* S) {
  const int i = threadIdx.x;
  if (i < count) {
    double s = 0.0;
    for (int q = 0; q < nranks; ++q) s += boxes[q][area_off + i];
    S[slot + i] = s;
  }
}

struct IpcExport {
  cudaIpcMemHandle_t box;
  cudaIpcEventHandle_t ready[2], done[2];
  int device;
  long long cap;
};

struct IpcComm : CommBase {
  std::unique_ptr<HostComm> hc;  // barrier + setup exchange + block-row directories
  int rank = 0, nranks = 1, device = 0;
  long long capd = 0;                    // doubles per parity area (kSlots scalars + data)
  double* box = nullptr;                 // my mailbox: 2 parity areas
  std::vector<double*> peer;             // every rank's mailbox as mapped here (peer[rank] = box)
  const double** d_peer = nullptr;       // the same table on the device (peer_sum_kernel)
  cudaEvent_t ready[2] = {}, done[2] = {};
  std::vector<std::array<cudaEvent_t, 2>> pready, pdone;  // the peers' events, opened here
  uint64_t seq = 0;

  double* area(int q, int par) const { return peer[(size_t)q] + (size_t)par * capd; }
  // host-side block-row directory of rank q for parity par (offset, count per rank)
  int64_t* dir(int q, int par) const { return reinterpret_cast<int64_t*>(hc->box(q)) + (size_t)par * 2 * nranks; }
  void need(long long doubles) const {
    if (doubles > capd - kSlots) {
      hc->give_up();
      fail(PCGX_ERR_UNSUPPORTED, "ipc comm: message of " + std::to_string(8 * doubles) + " bytes exceeds the " +
                                     std::to_string(8 * (capd - kSlots)) + "-byte mailbox");
    }
  }
  // Start exchange `seq` on stream st: the parity area is free once every peer has
  // finished reading it (their `done` of two exchanges ago).
  int begin(cudaStream_t st) {
    const int par = (int)(seq++ & 1);
    for (int q = 0; q < nranks; ++q)
      if (q != rank) PCGX_CUDA(cudaStreamWaitEvent(st, pdone[(size_t)q][par], 0));
    return par;
  }
  void publish(cudaStream_t st, int par) {
    PCGX_CUDA(cudaEventRecord(ready[par], st));
    hc->barrier();  // every rank's `ready` recorded before anyone waits on it
  }
  void finish(pcgx_context c, cudaStream_t st, int par, bool join) {
    PCGX_CUDA(cudaEventRecord(done[par], st));
    if (join) PCGX_CUDA(cudaEventRecord(c->ev_join, st));
  }
  void copy(double* dst, const double* src, long long count, cudaStream_t st) {
    if (count > 0) PCGX_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * (size_t)count, cudaMemcpyDefault, st));
  }

  ~IpcComm() override {
    if (!hc) return;
    cudaSetDevice(device);
    cudaDeviceSynchronize();  // my streams no longer touch the peers' mailboxes
    try {
      hc->barrier();
    } catch (...) {
    }
    for (int q = 0; q < nranks; ++q) {
      if (q == rank) continue;
      if (peer[(size_t)q]) cudaIpcCloseMemHandle(peer[(size_t)q]);
      for (int par = 0; par < 2; ++par) {
        if (pready[(size_t)q][par]) cudaEventDestroy(pready[(size_t)q][par]);
        if (pdone[(size_t)q][par]) cudaEventDestroy(pdone[(size_t)q][par]);
      }
    }
    try {
      hc->barrier();  // nobody maps my mailbox any more
    } catch (...) {
    }
    for (int par = 0; par < 2; ++par) {
      if (ready[par]) cudaEventDestroy(ready[par]);
      if (done[par]) cudaEventDestroy(done[par]);
    }
    if (d_peer) cudaFree(d_peer);
    if (box) cudaFree(box);
  }

  void allreduce(pcgx_context c, int slot, int count) override {
    cudaStream_t st = c->s;
    const int par = begin(st);
    copy(area(rank, par), c->S + slot, count, st);
    publish(st, par);
    for (int q = 0; q < nranks; ++q)
      if (q != rank) PCGX_CUDA(cudaStreamWaitEvent(st, pready[(size_t)q][par], 0));
    peer_sum_kernel<<<1, 32, 0, st>>>(d_peer, (long long)par * capd, nranks, slot, count, c->S);
    check_launch();
    finish(c, st, par, false);
  }
  void xchg(pcgx_context c, pcgx_operator op, const PlaneX* items, int n) override {
    (void)op;
    long long tot = 0;
    for (int i = 0; i < n; ++i) tot += 2 * items[i].count;
    need(tot);
    PCGX_CUDA(cudaEventRecord(c->ev_fork, c->s));
    PCGX_CUDA(cudaStreamWaitEvent(c->cs, c->ev_fork, 0));
    cudaStream_t st = c->cs;
    const int par = begin(st);
    double* mine = area(rank, par) + kSlots;
    long long off = 0;
    for (int i = 0; i < n; ++i) {  // my area: [bottom planes | top planes] per item
      if (rank > 0) copy(mine + off, items[i].send_lo, items[i].count, st);
      if (rank < nranks - 1) copy(mine + off + items[i].count, items[i].send_hi, items[i].count, st);
      off += 2 * items[i].count;
    }
    publish(st, par);
    if (rank > 0) PCGX_CUDA(cudaStreamWaitEvent(st, pready[(size_t)rank - 1][par], 0));
    if (rank < nranks - 1) PCGX_CUDA(cudaStreamWaitEvent(st, pready[(size_t)rank + 1][par], 0));
    off = 0;
    for (int i = 0; i < n; ++i) {  // rank-1's top -> my recv_lo, rank+1's bottom -> my recv_hi
      if (rank > 0 && items[i].recv_lo)
        copy(items[i].recv_lo, area(rank - 1, par) + kSlots + off + items[i].count, items[i].count, st);
      if (rank < nranks - 1 && items[i].recv_hi)
        copy(items[i].recv_hi, area(rank + 1, par) + kSlots + off, items[i].count, st);
      off += 2 * items[i].count;
    }
    finish(c, st, par, true);
  }
  void halo_begin(pcgx_context c, pcgx_operator op, const double* const* xs, int nv) override {
    const long long nxy = op->nx * op->ny, nzl = op->nzl;
    PlaneX items[2];
    for (int v = 0; v < nv && v < 2; ++v)
      items[v] = {xs[v], v ? op->ghost_lo2 : op->ghost_lo, xs[v] + (nzl - 1) * nxy,
                  v ? op->ghost_hi2 : op->ghost_hi, nxy};
    xchg(c, op, items, std::min(nv, 2));
  }
  void halo_wait(pcgx_context c) override { PCGX_CUDA(cudaStreamWaitEvent(c->s, c->ev_join, 0)); }
  void sparse_xchg(pcgx_context c, pcgx_operator op, int nv, const double* const* sbuf,
                   double* const* gbuf) override {
    const int P = nranks;
    long long tot = 0;
    for (size_t i = 0; i < op->nb_rank.size(); ++i) tot += (long long)nv * op->send_cnt[i];
    need(tot);
    PCGX_CUDA(cudaEventRecord(c->ev_fork, c->s));
    PCGX_CUDA(cudaStreamWaitEvent(c->cs, c->ev_fork, 0));
    cudaStream_t st = c->cs;
    const int par = begin(st);
    int64_t* d = dir(rank, par);  // host directory: where my segment for rank q starts, its length
    for (int q = 0; q < 2 * P; ++q) d[q] = 0;
    double* mine = area(rank, par) + kSlots;
    long long off = 0;
    for (size_t i = 0; i < op->nb_rank.size(); ++i) {
      const int q = op->nb_rank[i];
      d[q] = off;
      d[P + q] = op->send_cnt[i];
      for (int v = 0; v < nv; ++v) {
        copy(mine + off, sbuf[v] + op->send_off[i], op->send_cnt[i], st);
        off += op->send_cnt[i];
      }
    }
    publish(st, par);
    for (size_t i = 0; i < op->nb_rank.size(); ++i) {
      const int q = op->nb_rank[i];
      const int64_t* qd = dir(q, par);
      const int64_t qoff = qd[rank], qcnt = qd[P + rank];
      if (qcnt != op->recv_cnt[i]) fail(PCGX_ERR_NCCL, "ipc comm: block-row segment size mismatch");
      if (!qcnt) continue;
      PCGX_CUDA(cudaStreamWaitEvent(st, pready[(size_t)q][par], 0));
      for (int v = 0; v < nv; ++v)
        copy(gbuf[v] + op->recv_off[i], area(q, par) + kSlots + qoff + (long long)v * qcnt, qcnt, st);
    }
    finish(c, st, par, true);
  }
  bool graph_capturable() const override { return false; }
};

IpcComm* ipc_comm_open(pcgx_context c, const std::string& name, size_t mailbox_bytes) {
  auto ic = std::make_unique<IpcComm>();
  const int P = c->nranks;
  ic->rank = c->rank;
  ic->nranks = P;
  ic->device = c->device;
  // the shared-memory segment holds the setup exports and two block-row directories
  const size_t hbox = std::max(sizeof(IpcExport), (size_t)4 * P * sizeof(int64_t));
  ic->hc.reset(host_comm_open(P, c->rank, name, hbox));
  ic->capd = (long long)((mailbox_bytes + 127) / 128 * 16) + kSlots;  // 128-byte aligned areas
  PCGX_CUDA(cudaMalloc(&ic->box, sizeof(double) * 2 * (size_t)ic->capd));
  IpcExport ex{};
  PCGX_CUDA(cudaIpcGetMemHandle(&ex.box, ic->box));
  for (int par = 0; par < 2; ++par) {
    PCGX_CUDA(cudaEventCreateWithFlags(&ic->ready[par], cudaEventDisableTiming | cudaEventInterprocess));
    PCGX_CUDA(cudaEventCreateWithFlags(&ic->done[par], cudaEventDisableTiming | cudaEventInterprocess));
    PCGX_CUDA(cudaIpcGetEventHandle(&ex.ready[par], ic->ready[par]));
    PCGX_CUDA(cudaIpcGetEventHandle(&ex.done[par], ic->done[par]));
  }
  ex.device = c->device;
  ex.cap = ic->capd;
  std::memcpy(ic->hc->box(c->rank), &ex, sizeof ex);
  ic->hc->barrier();
  ic->peer.assign((size_t)P, nullptr);
  ic->pready.assign((size_t)P, {nullptr, nullptr});
  ic->pdone.assign((size_t)P, {nullptr, nullptr});
  ic->peer[(size_t)c->rank] = ic->box;
  for (int q = 0; q < P; ++q) {
    if (q == c->rank) continue;
    IpcExport qe;
    std::memcpy(&qe, ic->hc->box(q), sizeof qe);
    if (qe.cap != ic->capd) fail(PCGX_ERR_INVALID, "ipc comm: ranks disagree on the mailbox size");
    if (qe.device != c->device) {
      int can = 0;
      PCGX_CUDA(cudaDeviceCanAccessPeer(&can, c->device, qe.device));
      if (!can)
        fail(PCGX_ERR_UNSUPPORTED, "ipc comm: device " + std::to_string(c->device) + " cannot access device " +
                                       std::to_string(qe.device) + " (peer access)");
    }
    void* m = nullptr;
    PCGX_CUDA(cudaIpcOpenMemHandle(&m, qe.box, cudaIpcMemLazyEnablePeerAccess));
    ic->peer[(size_t)q] = static_cast<double*>(m);
    for (int par = 0; par < 2; ++par) {
      PCGX_CUDA(cudaIpcOpenEventHandle(&ic->pready[(size_t)q][par], qe.ready[par]));
      PCGX_CUDA(cudaIpcOpenEventHandle(&ic->pdone[(size_t)q][par], qe.done[par]));
    }
  }
  PCGX_CUDA(cudaMalloc(&ic->d_peer, sizeof(double*) * (size_t)P));
  PCGX_CUDA(cudaMemcpy(ic->d_peer, ic->peer.data(), sizeof(double*) * (size_t)P, cudaMemcpyHostToDevice));
  ic->hc->barrier();  // every rank has read the exports: the segment's boxes become directories
  return ic.release();
}

void allreduce(pcgx_context c, int slot, int count) {
  if (!c->cm) return;
  c->cm->allreduce(c, slot, count);
  c->cur_allreduce++;
}

// Sum k <= 5 host doubles over the ranks through the scratch slots S_DOT..S_E2 (setup
// checks), stream-ordered on c->s: the comms' all-reduces are asynchronous there.
void allreduce_host(pcgx_context c, const double* in, double* out, int k) {
  PCGX_CUDA(cudaMemcpyAsync(c->S + S_DOT, in, sizeof(double) * k, cudaMemcpyHostToDevice, c->s));
  allreduce(c, S_DOT, k);
  PCGX_CUDA(cudaMemcpyAsync(out, c->S + S_DOT, sizeof(double) * k, cudaMemcpyDeviceToHost, c->s));
  PCGX_CUDA(cudaStreamSynchronize(c->s));
}

