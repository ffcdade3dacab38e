# SPDX-License-Identifier: Apache-2.0
"""A/B micro-benchmark of the two-step Chebyshev pass at 320^3: each variant is
an env setting (read at operator creation) and optionally a library build
(`lib=tools/bin/libpcgx_NAME.so` runs that variant in a subprocess). Variants
are interleaved over several rounds so thermal / power-cap drift hits all of
them alike; the SM clock is sampled (NVML) while each variant runs.

    python tools/kbench_cheb2.py [--rounds 3] [--nx 320] VARIANT ...
    VARIANT = "PCGX_CHEB3=1" | "lib=tools/bin/libpcgx_d3.so+PCGX_KZ2=16" (settings joined by +)

--same: env-only variants as operators of ONE context, alternated on the same
device buffers (run-to-run allocation effects cancel).
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one(nx, m, reps):
    sys.path.insert(0, ROOT)
    import paper_2008_01440_b200 as P
    from paper_2008_01440_b200 import pcgx
    import ctypes as C
    clocks = []
    stop = threading.Event()

    def sample():
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(0)
            while not stop.is_set():
                clocks.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                time.sleep(0.01)
        except Exception:
            pass

    with P.Context(0) as ctx:
        op, _ = P.jacobi_scale(P.StencilOperator(nx), ctx)
        n = op.local_size()
        a, b = P.analytic_extremes(3, nx)
        cp = P.cheb_params(a, b, m, 1.001)._c()
        r = P.random_uniform_vector(n, 1, ctx=ctx)
        out = P.DeviceVector(ctx, n)
        L = pcgx.lib()
        for _ in range(3):
            pcgx._check(L.pcgx_cheb_apply_device(ctx.h, op.h, C.byref(cp), r.ptr, out.ptr), ctx.h)
        ctx.synchronize()
        th = threading.Thread(target=sample)
        th.start()
        ctx.timer_start()
        for _ in range(reps):
            pcgx._check(L.pcgx_cheb_apply_device(ctx.h, op.h, C.byref(cp), r.ptr, out.ptr), ctx.h)
        ms = ctx.timer_stop() / reps
        stop.set()
        th.join()
        op.close()
    passes = m // 2
    clocks.sort()
    return {"apply_ms": round(ms, 4), "pass_ms": round(ms / passes, 5),
            "pass_GBps": round(40 * n / (ms / passes) / 1e6, 1),
            "sm_mhz": clocks[len(clocks) // 2] if clocks else None}


def same(nx, m, reps, rounds, variants):
    sys.path.insert(0, ROOT)
    import ctypes as C
    import paper_2008_01440_b200 as P
    from paper_2008_01440_b200 import pcgx
    L = pcgx.lib()
    with P.Context(0) as ctx:
        ops = []
        for v in variants:
            env = dict(kv.split("=", 1) for kv in v.split("+"))
            os.environ.update(env)
            ops.append(P.jacobi_scale(P.StencilOperator(nx), ctx)[0])
            for k in env:
                del os.environ[k]
        n = ops[0].local_size()
        a, b = P.analytic_extremes(3, nx)
        cp = P.cheb_params(a, b, m, 1.001)._c()
        r = P.random_uniform_vector(n, 1, ctx=ctx)
        out = P.DeviceVector(ctx, n)
        res = {v: [] for v in variants}
        clk = {v: [] for v in variants}
        try:
            import pynvml
            pynvml.nvmlInit()
            hdl = pynvml.nvmlDeviceGetHandleByIndex(0)
        except Exception:
            hdl = None
        for op in ops:
            for _ in range(3):
                pcgx._check(L.pcgx_cheb_apply_device(ctx.h, op.h, C.byref(cp), r.ptr, out.ptr), ctx.h)
        for rnd in range(rounds):
            for v, op in zip(variants, ops):
                ctx.synchronize()
                ctx.timer_start()
                for i in range(reps):
                    pcgx._check(L.pcgx_cheb_apply_device(ctx.h, op.h, C.byref(cp), r.ptr, out.ptr), ctx.h)
                    if hdl is not None and i == reps // 2:
                        clk[v].append(pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_SM))
                res[v].append(ctx.timer_stop() / reps / (m // 2))
        for v in variants:
            t = sorted(res[v])
            print(json.dumps({"variant": v, "pass_ms_min": round(t[0], 5), "pass_ms_med": round(t[len(t) // 2], 5),
                              "pass_GBps_med": round(40 * n / t[len(t) // 2] / 1e6, 1),
                              "sm_mhz": sorted(clk[v])[len(clk[v]) // 2] if clk[v] else None,
                              "all": [round(x, 4) for x in res[v]]}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--nx", type=int, default=320)
    ap.add_argument("--m", type=int, default=40)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--child", default=None)
    ap.add_argument("--same", action="store_true")
    ap.add_argument("variants", nargs="*")
    a = ap.parse_args()
    if a.child is not None:
        print(json.dumps(one(a.nx, a.m, a.reps)))
        return
    if a.same:
        same(a.nx, a.m, a.reps, a.rounds, a.variants)
        return
    for rnd in range(a.rounds):
        for v in a.variants:
            env = dict(os.environ)
            for kv in v.split("+"):
                k, val = kv.split("=", 1)
                env["PCGX_LIB" if k == "lib" else k] = val
            r = subprocess.run([sys.executable, __file__, "--child", "1", "--nx", str(a.nx), "--m",
                                str(a.m), "--reps", str(a.reps)], env=env, capture_output=True, text=True)
            line = r.stdout.strip().splitlines()[-1] if r.returncode == 0 else r.stderr[-400:]
            print(json.dumps({"round": rnd, "variant": v, "result": line}), flush=True)


if __name__ == "__main__":
    main()
