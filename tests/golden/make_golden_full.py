# SPDX-License-Identifier: Apache-2.0
"""Full-size known answers for every BASELINE config, from the REFERENCE ITSELF.

Runs in the build container only (oracle/_ref/libpolycg_ref.so is the reference
library compiled from /root/reference/proj/src by oracle/Makefile). Each job runs
`polycg::pcg_solve` (proj/src/pcg.cpp:10-117) on one BASELINE configuration at
its full size and writes tests/golden/full/<tag>.json plus <tag>_xs.npy (the
reference's solution x at 8192 seeded sample indices), which the GPU suite
(tests/test_gpu_fullsize.py) checks the device solve against:

  * b = A x_true: SHA-256 of the reference's b (bitwise: the scaled SpMV at full size);
  * iterations / ddot / matvec / prec_applies: the reference's counters;
  * rel_res, true_rel_res, ||x - x_true|| / ||x_true||: hex floats;
  * x at sampled indices (the x-vector parity reading of SURVEY §8c).

Inputs are the bench's: x_true = random_uniform_vector(n, 20240801), s = 1.001,
tol 1e-8, analytic bounds (cfg2 / cfg5s / cfg5w P=1, proj/src/linop.cpp:382-390)
or Lanczos bounds (cfg3 / cfg4; 20 steps -> lambda_max, 30 -> lambda_min, from the
C oracle's or_lanczos; the reference has no Lanczos) recorded as hex and fed
bit-identically to both sides. cfg3 / cfg4 matrices come from the repo's
generators (csrc/gen.cpp, host C++), the same arrays the GPU uploads.

    python tests/golden/make_golden_full.py --all            # schedules every job
    python tests/golden/make_golden_full.py --job cfg2_k20   # one job
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import subprocess
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
OUT = os.path.join(HERE, "full")
sys.path.insert(0, ROOT)

SEED = 20240801
SCALE = 1.001
NSAMPLE = 8192
SAMPLE_SEED = 4711

# tag -> (kind, nx, m, est. peak GB)
JOBS = {
    "cfg5s_k40": ("lap3d", 640, 40, 27),
    "cfg5w_p1_k40": ("lap3d", 512, 40, 14),
    "cfg4_k30": ("elast27", 160, 30, 34),
    "cfg3_k40": ("fe27", 256, 40, 22),
    "cfg2_k80": ("lap3d", 320, 80, 4),
    "cfg2_k40": ("lap3d", 320, 40, 4),
    "cfg2_k20": ("lap3d", 320, 20, 4),
    "cfg2_k10": ("lap3d", 320, 10, 4),
    "cfg2_k5": ("lap3d", 320, 5, 4),
    "cfg2_k0": ("lap3d", 320, 0, 4),
}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def sample_indices(n):
    """The sampled indices the GPU test reads x at (sorted, without repeats)."""
    rng = np.random.default_rng(SAMPLE_SEED)
    return np.unique(rng.integers(0, n, size=NSAMPLE, dtype=np.int64))


def run_job(tag, threads):
    from oracle.oracle import Oracle, OracleOp, RefLib
    kind, nx, m, _ = JOBS[tag]
    R = RefLib()
    R.set_threads(threads)
    t0 = time.time()
    rec = {"tag": tag, "kind": kind, "nx": nx, "m": m, "scale": SCALE.hex(), "tol": 1e-8,
           "seed": SEED, "threads": threads}
    csr = None
    if kind == "lap3d":
        a, b = R.analytic_extremes(3, nx)
        rkind = "lap3d"
        rec["bounds"] = "analytic_extremes (linop.cpp:382-390)"
    else:
        from paper_2008_01440_b200 import pcgx as P
        A = P.gen_fe27(nx, 1.0, SEED) if kind == "fe27" else P.gen_elast27(nx, 1.0, 0.5, 0.1, SEED)
        rec["nnz"] = int(A.nnz())
        rp = A.row_ptr.astype(np.int64)
        ci = A.col_idx.astype(np.int64)
        va = A.values
        del A
        rec["csr_sha256"] = {"row_ptr": hashlib.sha256(rp.astype("<i8").tobytes()).hexdigest(),
                             "col_idx": hashlib.sha256(ci.astype("<i8").tobytes()).hexdigest(),
                             "values": sha(va)}
        O = Oracle()
        op = OracleOp("csr", row_ptr=rp, col_idx=ci, values=va)
        lo30, _, al, be = O.lanczos(op, 30, SEED)
        _, hi20 = O.tridiag_extremes(al[:20], be[:20])
        a, b = lo30, hi20
        del op, O
        rec["bounds"] = "oracle or_lanczos: 20 steps -> lambda_max, 30 steps -> lambda_min"
        rec["lanczos_alpha"] = [float(v).hex() for v in al]
        rec["lanczos_beta"] = [float(v).hex() for v in be]
        csr = (rp, ci, va)
        rkind = "csr"
        print(tag, "lanczos", a, b, f"{time.time() - t0:.0f}s", file=sys.stderr, flush=True)
    rec["alpha"], rec["beta"] = float(a).hex(), float(b).hex()
    prm = R.cheb_params(a, b, m, SCALE)
    rec["theta"] = float(prm["theta"]).hex()
    t1 = time.time()
    x, bvec, rep = R.pcg_solve(rkind, a, b, m, SCALE, nx=nx, csr=csr, seed=SEED, tol=1e-8,
                               maxit=100000)
    rec["solve_wall_s"] = time.time() - t1
    del csr
    n = len(x)
    xt = R.random_uniform(n, SEED)
    err = float(np.linalg.norm(x - xt) / np.linalg.norm(xt))
    rec["n"] = n
    rec["report"] = {k: (float(v).hex() if isinstance(v, float) else int(v))
                     for k, v in rep.items() if k != "wall_time"}
    rec["report_wall_time_s"] = rep["wall_time"]
    rec["err"] = err.hex()
    rec["x_norm"] = float(np.linalg.norm(x)).hex()
    rec["b_sha256"] = sha(bvec)
    rec["x_sha256"] = sha(x)
    idx = sample_indices(n)
    rec["sample"] = {"seed": SAMPLE_SEED, "requested": NSAMPLE, "count": int(len(idx))}
    np.save(os.path.join(OUT, f"{tag}_xs.npy"), x[idx])
    rec["total_wall_s"] = time.time() - t0
    with open(os.path.join(OUT, f"{tag}.json"), "w") as f:
        json.dump(rec, f, indent=1)
    print(tag, rep["iters"], rep["ddot"], rep["matvec"], rep["rel_res"], err,
          f"{rec['total_wall_s']:.0f}s", file=sys.stderr, flush=True)


def run_all(budget_gb, max_jobs, threads, only):
    todo = [t for t in JOBS if (not only or t in only)
            and not os.path.exists(os.path.join(OUT, f"{t}.json"))]
    running = {}
    while todo or running:
        for t, p in list(running.items()):
            if p.poll() is not None:
                print(f"[done] {t} rc={p.returncode}", flush=True)
                del running[t]
        used = sum(JOBS[t][3] for t in running)
        for t in list(todo):
            if len(running) < max_jobs and used + JOBS[t][3] <= budget_gb:
                log = open(os.path.join(OUT, f"{t}.log"), "w")
                running[t] = subprocess.Popen(
                    [sys.executable, __file__, "--job", t, "--threads", str(threads)],
                    stdout=log, stderr=subprocess.STDOUT, cwd=ROOT)
                used += JOBS[t][3]
                todo.remove(t)
                print(f"[start] {t}", flush=True)
        time.sleep(5)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--job")
    ap.add_argument("--all", action="store_true")
    ap.add_argument("--only", nargs="*")
    ap.add_argument("--threads", type=int, default=2)
    ap.add_argument("--budget-gb", type=float, default=54)
    ap.add_argument("--max-jobs", type=int, default=6)
    a = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    if a.job:
        run_job(a.job, a.threads)
    else:
        run_all(a.budget_gb, a.max_jobs, a.threads, a.only)


if __name__ == "__main__":
    main()
