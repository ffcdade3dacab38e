# SPDX-License-Identifier: Apache-2.0
"""Sustained-load probe: runs one workload back to back for a few seconds and
samples NVML power, SM / memory clocks and throttle reasons meanwhile, to tell a
power-capped kernel from a bandwidth- or latency-bound one.

    python tools/power_probe.py [copy|step|cheb2|cheb3] [seconds]
"""
import ctypes as C
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "cheb2"
    secs = float(sys.argv[2]) if len(sys.argv) > 2 else 4.0
    import pynvml
    import torch
    import paper_2008_01440_b200 as P
    from paper_2008_01440_b200 import pcgx
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    nx = 320
    if what == "cheb3":
        os.environ["PCGX_CHEB3"] = "1"
    with P.Context(0) as ctx:
        op, _ = P.jacobi_scale(P.StencilOperator(nx), ctx)
        n = op.local_size()
        a, b = P.analytic_extremes(3, nx)
        r = P.random_uniform_vector(n, 1, ctx=ctx)
        out = P.DeviceVector(ctx, n)
        L = pcgx.lib()
        if what == "copy":
            src = torch.empty(n * 4, dtype=torch.float64, device="cuda")
            dst = torch.empty_like(src)
            run = lambda: dst.copy_(src)  # noqa: E731
            nbytes = 2 * src.numel() * 8
            sync = torch.cuda.synchronize
        else:
            m = 40 if what.startswith("cheb") else 1
            cp = P.cheb_params(a, b, m, 1.001)._c()
            if what == "step":  # single fused step kernel: m = 1 apply = one first step
                cp = P.cheb_params(a, b, 1, 1.001)._c()
            run = lambda: pcgx._check(L.pcgx_cheb_apply_device(ctx.h, op.h, C.byref(cp), r.ptr, out.ptr), ctx.h)  # noqa: E731
            nbytes = (40 * n * (m // 2)) if m > 1 else 16 * n
            sync = ctx.synchronize
        samples = []
        stop = threading.Event()

        def sample():
            while not stop.is_set():
                samples.append((pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                                pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
                                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)))
                time.sleep(0.02)

        for _ in range(3):
            run()
        sync()
        th = threading.Thread(target=sample)
        th.start()
        t0 = time.perf_counter()
        iters = 0
        while time.perf_counter() - t0 < secs:
            for _ in range(5):
                run()
            sync()
            iters += 5
        dt = time.perf_counter() - t0
        stop.set()
        th.join()
        half = samples[len(samples) // 2:]
        med = lambda i: sorted(s[i] for s in half)[len(half) // 2]  # noqa: E731
        reasons = 0
        for s in half:
            reasons |= s[3]
        print(json.dumps({"what": what, "GBps": round(nbytes * iters / dt / 1e9, 1),
                          "power_w": med(0), "sm_mhz": med(1), "mem_mhz": med(2),
                          "limit_w": pynvml.nvmlDeviceGetEnforcedPowerLimit(h) / 1000.0,
                          "reasons_mask": hex(reasons)}))


if __name__ == "__main__":
    main()
