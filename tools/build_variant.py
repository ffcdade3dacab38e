"""Build libpcgx.so variants with extra nvcc defines into tools/bin/ (kernel tuning).

    python tools/build_variant.py NAME [-DMACRO=V ...]   -> tools/bin/libpcgx_NAME.so
Use with PCGX_LIB=tools/bin/libpcgx_NAME.so python tools/kbench.py ...
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_01440_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "bin", f"libpcgx_{name}.so")
os.makedirs(os.path.dirname(out), exist_ok=True)
cmd = B.command(defs)
cmd[cmd.index("-o") + 1] = out
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stdout + r.stderr)
print(out)
