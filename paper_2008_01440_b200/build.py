# SPDX-License-Identifier: Apache-2.0
"""Build recipe for the in-tree native library ``libpcgx.so`` (sm_100a).

    python -m paper_2008_01440_b200.build

One nvcc invocation compiles the CUDA kernels + host orchestration
(csrc/pcgx.cu) and the host C++ (csrc/host_math.cpp, csrc/gen.cpp) into
paper_2008_01440_b200/libpcgx.so, linked against NCCL. Flags:

* ``-gencode arch=compute_100a,code=sm_100a`` — B200 only, no PTX fallback;
* ``--fmad=false`` and ``-ffp-contract=off`` — no FMA contraction anywhere, so
  per-point results are the reference's IEEE values (parity);
* ``-lineinfo`` — ncu source-page mapping.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libpcgx.so")
SOURCES = ["pcgx.cu", "host_math.cpp", "gen.cpp", "mm.cpp"]
HEADERS = sorted(f for f in os.listdir(os.path.join(os.path.dirname(os.path.abspath(__file__)), "csrc"))
                 if f.endswith((".cuh", ".hpp", ".h")))


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _host_cxx():
    for cand in ("/usr/bin/g++", shutil.which("g++")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("g++ not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "pcgx.h"))
    deps.append(__file__)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


CHECKED_LIB = os.path.join(PKG, "libpcgx_checked.so")


def _stale_lib(lib: str) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "pcgx.h"))
    deps.append(__file__)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build_checked(force: bool = False) -> str:
    """The checked build (-DPCGX_CHECKED: device-side bounds asserts in the TMA /
    shared-memory kernels, common.cuh PCGX_DCHECK) as libpcgx_checked.so beside
    the production library. compute-sanitizer is not available on the GPU pool;
    tests/test_gpu_checked.py runs a ragged small-grid workload on this build."""
    if not (force or _stale_lib(CHECKED_LIB)):
        return CHECKED_LIB
    cmd = command(["-DPCGX_CHECKED"])
    tmp = CHECKED_LIB + f".tmp{os.getpid()}"
    cmd[cmd.index("-o") + 1] = tmp
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("libpcgx_checked build failed:\n" + res.stdout + res.stderr)
    os.replace(tmp, CHECKED_LIB)
    return CHECKED_LIB


def command(extra=()):
    return [
        _nvcc(), "-ccbin", _host_cxx(), "-O3", "-std=c++17",
        "-gencode", "arch=compute_100a,code=sm_100a",
        "-lineinfo", "--fmad=false",
        "-Xcompiler", "-fPIC,-ffp-contract=off,-fopenmp,-O3",
        "-Xptxas", "-v" if os.environ.get("PCGX_PTXAS_V") else "-O3",
        "-I", os.path.join(ROOT, "include"), "-I", CSRC,
        "-shared", "-o", LIB,
        *[os.path.join(CSRC, f) for f in SOURCES],
        "-ldl", "-lgomp", *extra,
    ]


def build(force: bool = False, verbose: bool = False) -> str:
    if not (force or _stale()):
        return LIB
    # one builder at a time (torchrun ranks, pytest workers): the others wait on the
    # lock and then find the library fresh
    import fcntl
    with open(os.path.join(PKG, ".build.lock"), "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        try:
            if force or _stale():
                cmd = command()
                if verbose:
                    print(" ".join(cmd), file=sys.stderr)
                tmp = LIB + f".tmp{os.getpid()}"
                cmd[cmd.index("-o") + 1] = tmp
                res = subprocess.run(cmd, capture_output=True, text=True)
                if res.returncode != 0:
                    raise RuntimeError("libpcgx build failed:\n" + res.stdout + res.stderr)
                os.replace(tmp, LIB)  # atomic: a concurrent loader sees the old or the new file
                if verbose and res.stderr:
                    print(res.stderr, file=sys.stderr)
        finally:
            fcntl.flock(lk, fcntl.LOCK_UN)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
    if "--checked" in sys.argv:
        print(build_checked(force="--force" in sys.argv))
