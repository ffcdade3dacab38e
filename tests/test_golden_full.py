# SPDX-License-Identifier: Apache-2.0
"""CPU checks of the full-size reference fixtures (tests/golden/full/, written by
tests/golden/make_golden_full.py from the reference library itself): complete,
self-consistent under the reference's counting rules (include/polycg/pcg.hpp:66-82:
ddot = 3 iters + 2, matvec = iters (m + 1) + 1 on a converged zero-x0 solve), and
the inputs the GPU suite re-creates (bounds, theta) are the reference's own."""
import glob
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
FULL = os.path.join(HERE, "golden", "full")
CASES = sorted(os.path.basename(p)[:-5] for p in glob.glob(os.path.join(FULL, "*.json")))

EXPECTED = {"cfg2_k0", "cfg2_k5", "cfg2_k10", "cfg2_k20", "cfg2_k40", "cfg2_k80", "cfg3_k40", "cfg4_k30",
            "cfg5s_k40", "cfg5w_p1_k40"}


def test_all_baseline_configs_pinned():
    missing = EXPECTED - set(CASES)
    # the long CPU jobs (cfg3/4/5) may still be running when the suite is run mid-build
    assert {"cfg2_k0", "cfg2_k5", "cfg2_k10", "cfg2_k20", "cfg2_k40", "cfg2_k80"} <= set(CASES)
    if missing:
        pytest.skip(f"fixtures not generated yet: {sorted(missing)}")


@pytest.mark.parametrize("tag", CASES)
def test_fixture_consistent(tag):
    with open(os.path.join(FULL, tag + ".json")) as f:
        g = json.load(f)
    r = g["report"]
    m = g["m"]
    assert r["converged"] == 1
    assert r["ddot"] == 3 * r["iters"] + 2
    assert r["matvec"] == r["iters"] * (m + 1) + 1
    assert r["prec_applies"] == r["iters"]
    assert float.fromhex(r["rel_res"]) <= g["tol"]
    assert 0 < float.fromhex(g["err"]) < 1e-4
    xs = np.load(os.path.join(FULL, tag + "_xs.npy"))
    assert xs.shape == (g["sample"]["count"],) and np.all(np.isfinite(xs))
    if g["kind"] == "lap3d":
        from paper_2008_01440_b200 import pcgx as P
        a, b = P.analytic_extremes(3, g["nx"])
        assert (a.hex(), b.hex()) == (g["alpha"], g["beta"])
        assert g["n"] == g["nx"] ** 3
    else:
        assert len(g["lanczos_alpha"]) == 30 and len(g["lanczos_beta"]) == 30


def test_cfg2_sweep_matches_survey_known_answer():
    """SURVEY Appendix A measured cfg2 k = 20 by running the reference: 39
    iterations, 119 ddot, 820 matvec, rel_res 7.515e-9, error 1.513e-6."""
    with open(os.path.join(FULL, "cfg2_k20.json")) as f:
        g = json.load(f)
    r = g["report"]
    assert (r["iters"], r["ddot"], r["matvec"]) == (39, 119, 820)
    assert float.fromhex(r["rel_res"]) == pytest.approx(7.515e-9, rel=1e-3)
    assert float.fromhex(g["err"]) == pytest.approx(1.513e-6, rel=1e-3)
