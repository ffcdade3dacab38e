# SPDX-License-Identifier: Apache-2.0
"""Device timeline of one solve through CUPTI (torch.profiler): kernel and memcpy
intervals on the GPU, the summed idle gaps between them, and the largest gaps —
tells launch / host-sync bubbles from kernel time.

    python tools/gap_trace.py [NX] [K]
"""
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    nx = int(sys.argv[1]) if len(sys.argv) > 1 else 320
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    import torch
    from torch.profiler import ProfilerActivity, profile
    import paper_2008_01440_b200 as P
    torch.cuda.init()
    with P.Context(0) as ctx:
        op, _ = P.jacobi_scale(P.StencilOperator(nx), ctx)
        a, b = P.analytic_extremes(3, nx)
        rhs = op.apply(P.random_uniform_vector(nx ** 3, 20240801, ctx=ctx))
        prec = P.ChebyshevPreconditioner(P.cheb_params(a, b, k, 1.001))
        x = P.DeviceVector(ctx, nx ** 3)
        for _ in range(2):
            P.pcg_solve(op, rhs, None, prec, x_out=x)
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            _, rep = P.pcg_solve(op, rhs, None, prec, x_out=x)
        path = os.path.join(tempfile.mkdtemp(), "trace.json")
        prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    iv = sorted((e["ts"], e["ts"] + e.get("dur", 0), e.get("name", ""), e.get("cat", ""))
                for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e)
    busy, gaps, last_end = 0.0, [], None
    for s, t, name, cat in iv:
        if last_end is not None and s > last_end:
            gaps.append((s - last_end, name))
        busy += t - s
        last_end = t if last_end is None else max(last_end, t)
    span = iv[-1][1] - iv[0][0]
    gaps.sort(reverse=True)
    kinds = {}
    for s, t, name, cat in iv:
        key = name.split("(")[0].replace("void ", "").replace("pcgx::", "")[:48] if cat == "kernel" else cat
        kinds.setdefault(key, [0, 0.0])
        kinds[key][0] += 1
        kinds[key][1] += t - s
    print(json.dumps({"nx": nx, "k": k, "iters": rep.iters, "solve_ms": round(rep.wall_time * 1e3, 3),
                      "span_ms": round(span / 1e3, 3), "busy_ms": round(busy / 1e3, 3),
                      "gap_ms": round(sum(g for g, _ in gaps) / 1e3, 3), "n_gaps": len(gaps),
                      "largest_gaps_us": [(round(g, 1), n[:40]) for g, n in gaps[:8]],
                      "by_kind_ms": {k2: [v[0], round(v[1] / 1e3, 3)] for k2, v in kinds.items()}}))


if __name__ == "__main__":
    main()
