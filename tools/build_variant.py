#!/usr/bin/env python
"""Build a tuning variant of libstokes_er.so with extra -D macros (for sweeps on the GPU box).

    python tools/build_variant.py NAME -DSER_NEAR_TAIL_PCT=0 [...]
    -> build/variants/libstokes_er_NAME.so   (select with STOKES_ER_LIB=...)
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_00156_b200 import build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(ROOT, "build", "variants")
os.makedirs(out_dir, exist_ok=True)
out = os.path.join(out_dir, f"libstokes_er_{name}.so")
cmd = [b.NVCC, *b.FLAGS, *defs, "-I" + os.path.join(ROOT, "include"), "-o", out, *b.cu_sources()]
res = subprocess.run(cmd, capture_output=True, text=True)
if res.returncode:
    sys.exit(res.stderr)
for line in res.stderr.splitlines():
    if "fused_kernelILi3ELi2ELb0" in line:
        i = res.stderr.splitlines().index(line)
        print(name, " | ".join(l.strip() for l in res.stderr.splitlines()[i + 1:i + 3]))
        break
print(out)
