# SPDX-License-Identifier: Apache-2.0
"""Memory safety of the hand-written TMA / shared-memory kernels: compute-sanitizer
is closed on this GPU pool (profiles/r02_compute_sanitizer_unavailable.log), so
the library is also built with device-side bounds asserts (-DPCGX_CHECKED,
libpcgx_checked.so: every shared-ring offset a thread uses and every global store
index of the two- / three-step passes, the direction step and the grid-tile CSR
kernels trap when out of range) and tools/sanitize_run.py drives every such
kernel on ragged small grids through it, checking the results against the oracle."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_checked_build_runs_clean(pcgx):
    from paper_2008_01440_b200 import build as B
    lib = B.build_checked()
    env = dict(os.environ, PCGX_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py")], env=env,
                       capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0 and "sanitize workload ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
    assert "check failed" not in r.stdout + r.stderr
