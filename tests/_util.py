# SPDX-License-Identifier: Apache-2.0
import hashlib

import numpy as np


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def fh(s) -> float:
    return float.fromhex(s)


def fhs(lst):
    return np.array([float.fromhex(s) for s in lst])


def rel_norm(a, b) -> float:
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb else 1.0))


def lap3d_csr(nx):
    """assemble_laplacian(lap3d, nx) (proj/src/linop.cpp:299-331) as int64 CSR."""
    n = nx ** 3
    nxy = nx * nx
    r = np.arange(n)
    i, j, k = r % nx, (r // nx) % nx, r // nxy
    cols, vals, counts = [], [], np.zeros(n, dtype=np.int64)
    entries = [(k > 0, -nxy, -1.0), (j > 0, -nx, -1.0), (i > 0, -1, -1.0), (np.ones(n, bool), 0, 6.0),
               (i < nx - 1, 1, -1.0), (j < nx - 1, nx, -1.0), (k < nx - 1, nxy, -1.0)]
    mask = np.stack([e[0] for e in entries], axis=1)  # n x 7, column order ascending
    offs = np.array([e[1] for e in entries])
    vv = np.array([e[2] for e in entries])
    counts = mask.sum(1)
    rp = np.zeros(n + 1, dtype=np.int64)
    rp[1:] = np.cumsum(counts)
    ci = (r[:, None] + offs[None, :])[mask].astype(np.int64)
    va = np.broadcast_to(vv, (n, 7))[mask].astype(np.float64)
    return rp, ci, va


def csr_to_dense(rp, ci, va, n):
    A = np.zeros((n, n))
    for i in range(n):
        A[i, ci[rp[i]:rp[i + 1]]] = va[rp[i]:rp[i + 1]]
    return A


def lap2d_csr(nx):
    """assemble_laplacian(lap2d, nx) (proj/src/linop.cpp:299-331) as int64 CSR:
    diagonal 4, off-diagonal -1, the 5-point star in ascending columns."""
    n = nx * nx
    rp, ci, va = [0], [], []
    for r in range(n):
        i, j = r % nx, r // nx
        for off, ok in ((-nx, j > 0), (-1, i > 0), (0, True), (1, i < nx - 1), (nx, j < nx - 1)):
            if ok:
                ci.append(r + off)
                va.append(4.0 if off == 0 else -1.0)
        rp.append(len(ci))
    return np.array(rp, dtype=np.int64), np.array(ci, dtype=np.int64), np.array(va)
