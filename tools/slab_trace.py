# SPDX-License-Identifier: Apache-2.0
"""Device timeline (CUPTI via torch.profiler) of a few PCG iterations on a loopback
middle rank (tools/slab_overhead.py) against the single domain: per-kernel totals,
memcpy totals and idle gaps.   python tools/slab_trace.py [NX NY NZL K ITERS]"""
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def trace(loop, nx, ny, nzl, k, iters):
    import torch
    from torch.profiler import ProfilerActivity, profile
    import paper_2008_01440_b200 as P
    torch.cuda.init()
    ctx = P.Context(0, nranks=3, rank=1, loopback=True) if loop else P.Context(0)
    with ctx:
        op, _ = P.jacobi_scale(P.StencilOperator(nx, ny, 3 * nzl if loop else nzl), ctx)
        nl = op.local_size()
        a, b = P.analytic_extremes_box(nx, ny, 3 * nzl if loop else nzl)
        rhs = op.apply(P.random_uniform_vector(nl, 20240801, ctx=ctx, offset=op.row0()))
        prec = P.ChebyshevPreconditioner(P.cheb_params(a, b, k, 1.001))
        x = P.DeviceVector(ctx, nl)
        opts = P.SolveOptions(tol=1e-30, maxit=iters)
        for _ in range(2):
            P.pcg_solve(op, rhs, opts, prec, x_out=x)
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            _, rep = P.pcg_solve(op, rhs, opts, prec, x_out=x)
        path = os.path.join(tempfile.mkdtemp(), "t.json")
        prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    iv = sorted((e["ts"], e["ts"] + e["dur"], e.get("name", ""), e["cat"]) for e in ev
                if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e)
    kinds, busy, last, gap = {}, 0.0, None, 0.0
    for s, t, name, cat in iv:
        key = name.split("(")[0].replace("void ", "").replace("pcgx::", "")[:44] if cat == "kernel" else cat
        kinds.setdefault(key, [0, 0.0])
        kinds[key][0] += 1
        kinds[key][1] += t - s
        if last is not None and s > last:
            gap += s - last
        last = t if last is None else max(last, t)
    span = iv[-1][1] - iv[0][0]
    print(json.dumps({"loopback": loop, "solve_ms": round(rep.wall_time * 1e3, 3), "span_ms": round(span / 1e3, 3),
                      "gap_ms": round(gap / 1e3, 3),
                      "by_kind": {k2: [v[0], round(v[1] / 1e3, 3)] for k2, v in
                                  sorted(kinds.items(), key=lambda kv: -kv[1][1])}}))


if __name__ == "__main__":
    a = [int(v) for v in sys.argv[1:]]
    nx, ny, nzl, k, iters = a if len(a) == 5 else (320, 320, 320, 20, 10)
    trace(False, nx, ny, nzl, k, iters)
    trace(True, nx, ny, nzl, k, iters)
