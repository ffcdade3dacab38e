# SPDX-License-Identifier: Apache-2.0
"""The reference-side C++ binding (include/polycg_gpu/adapter.hpp): compiled
against the reference's own headers and objects (oracle/_ref) and linked to
libpcgx.so; on a GPU it must reproduce polycg::pcg_solve through the same call."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "adapter_test")


def test_adapter_builds_against_reference_headers():
    if not os.path.exists("/root/reference/proj/include/polycg/pcg.hpp") and not os.path.exists(BIN):
        pytest.skip("reference sources absent and no prebuilt adapter_test")
    if os.path.exists("/root/reference/proj/include/polycg/pcg.hpp"):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "adapter_test"], check=True,
                       stdout=subprocess.DEVNULL)
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_adapter_matches_reference_pcg_solve():
    assert os.path.exists(BIN), "oracle/_ref/adapter_test must be prebuilt (make -C oracle)"
    res = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    lines = [json.loads(l) for l in res.stdout.splitlines() if l.startswith("{")]
    assert res.returncode == 0, res.stdout + res.stderr
    assert {l["case"] for l in lines} >= {"stencil40_m10", "csr30_m20", "stencil40_newton3", "on_iterate_stencil24_m6",
                                         "reject_custom_prec"}
    for l in lines:
        assert l["ok"], l
        if "iters" in l:
            assert l["iters"][0] == l["iters"][1]
            assert l.get("cheb7_bitwise", True) and l.get("newton4_bitwise", True)
