# SPDX-License-Identifier: Apache-2.0
"""A/B of whole solves (device wall_time of pcg_solve) between library builds,
interleaved over rounds: python tools/solve_ab.py NX M ROUNDS VARIANT ...
VARIANT = LIB[+NAME=VALUE...] (library path, then environment settings).
Each (round, lib) runs in a subprocess: build the operator, one warm-up solve,
then three timed solves; prints the median."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(nx, m):
    sys.path.insert(0, ROOT)
    import paper_2008_01440_b200 as P
    with P.Context(0) as ctx:
        op, _ = P.jacobi_scale(P.StencilOperator(nx), ctx)
        a, b = P.analytic_extremes(3, nx)
        rhs = op.apply(P.random_uniform_vector(nx ** 3, 20240801, ctx=ctx))
        prec = P.ChebyshevPreconditioner(P.cheb_params(a, b, m, 1.001)) if m >= 0 else None
        ts = []
        for i in range(4):
            x, rep = P.pcg_solve(op, rhs, None, prec)
            if i:
                ts.append(rep.wall_time)
        print(json.dumps({"iters": rep.iters, "t": sorted(ts)[1]}))


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(int(sys.argv[2]), int(sys.argv[3]))
        sys.exit(0)
    nx, m, rounds, libs = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4:]
    res = {l: [] for l in libs}
    for r in range(rounds):
        for l in libs:
            parts = l.split("+")
            env = dict(os.environ, PCGX_LIB=parts[0])
            env.update(kv.split("=", 1) for kv in parts[1:])
            out = subprocess.run([sys.executable, __file__, "--child", str(nx), str(m)], env=env,
                                 capture_output=True, text=True).stdout.strip().splitlines()[-1]
            res[l].append(json.loads(out)["t"])
    for l in libs:
        t = sorted(res[l])
        print(json.dumps({"lib": l, "median_s": t[len(t) // 2], "all": t}))
