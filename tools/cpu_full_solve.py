# SPDX-License-Identifier: Apache-2.0
"""The reference's own time-to-1e-8 on this host: one full polycg::pcg_solve
(oracle/_ref, the reference library compiled from its sources) on BASELINE cfg2
(320^3 matrix-free, Jacobi-scaled, k = 20, s = 1.001, x_true seed 20240801),
all host threads for its OpenMP apply_impl (its Eigen vector ops single-threaded,
as shipped). Prints one JSON line; bench.py reports it beside the GPU solve.

    python tools/cpu_full_solve.py [k] [nx] > profiles/r02_cpu_full_k20.json
"""
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.oracle import RefLib  # noqa: E402


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def main():
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    nx = int(sys.argv[2]) if len(sys.argv) > 2 else 320
    R = RefLib()
    threads = os.cpu_count() or 1
    R.set_threads(threads)
    a, b = R.analytic_extremes(3, nx)
    t0 = time.time()
    _, _, rep = R.pcg_solve("lap3d", a, b, k, 1.001, nx=nx, seed=20240801, tol=1e-8, maxit=100000,
                            want_x=False)
    print(json.dumps({"what": "reference pcg_solve time-to-1e-8 (oracle/_ref = /root/reference/proj/src)",
                      "config": {"workload": "cfg2", "nx": nx, "k": k, "theta_scale": 1.001, "tol": 1e-8},
                      "iters": rep["iters"], "ddot": rep["ddot"], "matvec": rep["matvec"],
                      "rel_res": rep["rel_res"], "time_to_1e8_s": round(rep["wall_time"], 3),
                      "wall_incl_setup_s": round(time.time() - t0, 3),
                      "spmv_equiv_GBps": round(rep["matvec"] * 16.0 * nx ** 3 / rep["wall_time"] / 1e9, 3),
                      "threads": threads, "cpu": cpu_model(), "host": platform.node()}), flush=True)


if __name__ == "__main__":
    main()
