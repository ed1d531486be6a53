#!/usr/bin/env python
"""Build an experiment variant of libspo_b200.so with extra nvcc defines, e.g.
    python scripts/micro/build_variant.py bpl128 -DSPO_LINE_BPL=128 -DSPO_LINE_R32=22
-> paper_1611_02665_b200/libspo_b200_bpl128.so; load it with SPO_LIB=<path>."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1611_02665_b200 import build as b  # noqa: E402

tag, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(b.PKG, f"libspo_b200_{tag}.so")
cmd = [b.nvcc(), *[f for f in b.NVCC_FLAGS if f != "-v" and f != "-Xptxas"], *defs, "-shared", "-o", out, *b.SOURCES]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.stderr.write(r.stderr)
    sys.exit(1)
print(out)
