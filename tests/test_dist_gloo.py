# SPDX-License-Identifier: Apache-2.0
"""The N>1 path on CPU: world_size-2 gloo processes.

1. bench.py's Dist plumbing (unique-id broadcast, barrier, max/sum over ranks).
2. The z-slab decomposition the GPU ranks use — partition from libpcgx
   (pcgx_slab_partition), per-rank slab of the seeded x_true (counter RNG with
   offset z0*nx*ny), one halo plane per neighbour per SpMV (send/recv), and the
   two all-reduces per PCG iteration ([p'q], [r'r, r'z]) — replayed in numpy on
   each rank's slab and checked against the single-domain oracle: the SpMV and
   every Chebyshev step bitwise, the solve within the PCG parity bar.
"""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SEED = 20240801


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _stencil_slab(x, ghost_lo, ghost_hi, nx, ny, d):
    """Scaled 7-pt on a slab (nzl, ny, nx) with ghost planes (zeros = Dirichlet),
    the reference's term order (proj/src/linop.cpp:246-254)."""
    nzl = x.shape[0]
    xp = np.zeros((nzl + 2, ny + 2, nx + 2))
    xp[1:-1, 1:-1, 1:-1] = x
    xp[0, 1:-1, 1:-1] = ghost_lo
    xp[-1, 1:-1, 1:-1] = ghost_hi
    c = xp[1:-1, 1:-1, 1:-1]
    s = np.zeros_like(x)
    for nb in (xp[:-2, 1:-1, 1:-1], xp[1:-1, :-2, 1:-1], xp[1:-1, 1:-1, :-2]):
        s = s + (-(d * nb))
    s = s + (6.0 * (d * c))
    for nb in (xp[1:-1, 1:-1, 2:], xp[1:-1, 2:, 1:-1], xp[2:, 1:-1, 1:-1]):
        s = s + (-(d * nb))
    return s * d


def _worker(rank, ws, port, nx, ny, nz, m, out_q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import bench
    import paper_2008_01440_b200 as P
    D = bench.Dist(ws, rank, 0, backend="gloo")
    dist = D.dist
    res = {}
    # 1. plumbing
    uid = D.bcast_bytes(b"unique-id-from-rank-0" if rank == 0 else None)
    res["uid"] = uid
    res["max"] = D.max(float(rank + 1))
    res["sum"] = D.sum(1.0)
    D.barrier()
    # 2. slab decomposition
    z0, nzl = P.slab_partition(nz, ws, rank)
    nxy = nx * ny
    d = 1.0 / np.sqrt(6.0)

    def halo(v):
        v3 = v.reshape(nzl, ny, nx)
        lo = torch.zeros(nxy, dtype=torch.float64)
        hi = torch.zeros(nxy, dtype=torch.float64)
        reqs = []
        if rank > 0:
            reqs.append(dist.isend(torch.from_numpy(v3[0].ravel().copy()), rank - 1))
            reqs.append(dist.irecv(lo, rank - 1))
        if rank < ws - 1:
            reqs.append(dist.isend(torch.from_numpy(v3[-1].ravel().copy()), rank + 1))
            reqs.append(dist.irecv(hi, rank + 1))
        for r_ in reqs:
            r_.wait()
        return lo.numpy().reshape(ny, nx), hi.numpy().reshape(ny, nx)

    def A(v):
        lo, hi = halo(v)
        return _stencil_slab(v.reshape(nzl, ny, nx), lo, hi, nx, ny, d).ravel()

    def allreduce(vals):
        t = torch.tensor(vals, dtype=torch.float64)
        dist.all_reduce(t)
        return t.numpy()

    xt = P.random_uniform_vector(nzl * nxy, SEED, offset=z0 * nxy)
    b = A(xt)
    res["b"] = (z0 * nxy, b)
    a0, b0 = P.analytic_extremes_box(nx, ny, nz)
    prm = P.cheb_params(a0, b0, m, 1.001)

    def cheb(r):  # polyprec.cpp:169-198 on the slab
        if m == 0:
            return r / prm.theta
        xo = r / prm.theta
        x = (2.0 * prm.rho[1] / prm.delta) * (2.0 * r - A(r) / prm.theta)
        for k in range(2, m + 1):
            z = (2.0 / prm.delta) * (r - A(x))
            xn = prm.rho[k] * ((2.0 * prm.sigma) * x - prm.rho[k - 1] * xo + z)
            xo, x = x, xn
        return x

    res["z"] = cheb(P.random_uniform_vector(nzl * nxy, 77, offset=z0 * nxy))
    # PCG with two all-reduces per iteration (pcg.cpp:10-117 order)
    bnorm = np.sqrt(allreduce([b @ b])[0])
    x = np.zeros_like(b)
    r = b.copy()
    z = cheb(r)
    p = z.copy()
    rho = allreduce([r @ z])[0]
    it = 0
    n_ar = 2
    for it in range(1, 20001):
        q = A(p)
        pq = allreduce([p @ q])[0]
        alpha = rho / pq
        x = x + alpha * p
        r = r - alpha * q
        z = cheb(r)                                   # speculative, as the GPU
        rr, rz = allreduce([r @ r, r @ z])            # one 16-byte all-reduce
        n_ar += 2
        if np.sqrt(rr) / bnorm <= 1e-8:
            break
        p = z + (rz / rho) * p
        rho = rz
    res["x"] = x
    res["iters"] = it
    res["n_allreduce"] = n_ar
    out_q.put((rank, res))
    D.barrier()
    D.close()


@pytest.mark.parametrize("dims,m", [((12, 10, 14), 5), ((16, 16, 9), 10)])
def test_gloo_world2_slab_pcg(pcgx, oracle, dims, m):
    import torch.multiprocessing as mp
    from oracle.oracle import OracleOp
    nx, ny, nz = dims
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, nx, ny, nz, m, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res[0]["uid"] == res[1]["uid"] == b"unique-id-from-rank-0"
    assert res[0]["max"] == res[1]["max"] == 2.0 and res[0]["sum"] == 2.0
    opo = OracleOp("lap3d", nx=nx, ny=ny, nz=nz)
    n = nx * ny * nz
    b_full = oracle.apply(opo, oracle.random_uniform(n, SEED))
    b_g = np.concatenate([res[0]["b"][1], res[1]["b"][1]])
    assert np.array_equal(b_g, b_full)                       # halo-exchanged SpMV: bitwise
    a0, b0 = oracle.analytic_extremes_box(nx, ny, nz)
    prm = oracle.cheb_params(a0, b0, m, 1.001)
    z_full = oracle.apply_chebyshev(opo, prm, oracle.random_uniform(n, 77))
    assert np.array_equal(np.concatenate([res[0]["z"], res[1]["z"]]), z_full)
    x_full, rep = oracle.pcg_solve(opo, prm, b_full)
    assert res[0]["iters"] == res[1]["iters"]
    assert abs(res[0]["iters"] - rep["iters"]) <= 1
    x_g = np.concatenate([res[0]["x"], res[1]["x"]])
    assert np.linalg.norm(x_g - x_full) / np.linalg.norm(x_full) <= 1e-10
    assert res[0]["n_allreduce"] == 2 * res[0]["iters"] + 2
