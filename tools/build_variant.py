#!/usr/bin/env python
"""Build an experimental variant of libtcx.so with extra nvcc flags (A/B experiments only; loaded
with TCX_LIB_PATH, never by default): python tools/build_variant.py NAME -DFLAG=1 ...
-> paper_2206_02874_b200/variants/libtcx_NAME.so"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2206_02874_b200 import build as b  # noqa: E402


def main():
    name, flags = sys.argv[1], sys.argv[2:]
    bdir = os.path.join(b.HERE, "build", "variant_" + name)
    os.makedirs(bdir, exist_ok=True)
    objs = [b._compile(s, flags, bdir, force=True) for s in b.sources()]
    out = os.path.join(b.HERE, "variants", f"libtcx_{name}.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    subprocess.check_call([b.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out] + objs +
                          ["-cudart", "static"])
    print(out)


if __name__ == "__main__":
    main()
