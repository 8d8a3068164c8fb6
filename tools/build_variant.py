#!/usr/bin/env python
"""Build an experiment variant of libcd with extra -D flags: python tools/build_variant.py NAME -DX=1 ...
-> paper_1911_05063_b200/lib/libcd_NAME.so (loaded with CD_LIB_VARIANT=NAME)."""
import os
import subprocess
import sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1911_05063_b200"))
import build  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(build.LIBDIR, f"libcd_{name}.so")
cmd = [build.nvcc(), *build.NVCC_FLAGS, *defs, "-I", os.path.join(build.ROOT, "include"), "-o", out, *build.sources()]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr[-2000:])
print(out)
