#!/usr/bin/env python
"""Dump the C2 SUBNORMAL class (inputs + mma.sync d00) for offline model fitting:
python tools/subnormal_dump.py -> $TCX_REPORT_DIR/subnormal_<fmt>.npz (fmt = bf16, tf32, f16)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import tcxgen  # noqa: E402
import paper_2206_02874_b200 as tcx  # noqa: E402
from parity import host_bits  # noqa: E402

out = os.environ.get("TCX_REPORT_DIR", "gpurun_out")
torch.cuda.set_device(0)
for fmt in ("bf16", "tf32", "f16"):
    d = tcxgen.probe_classes(fmt, 8192, seed=0)
    sel = d["cls"] == tcxgen.CLASSES.index("SUBNORMAL")
    A, B, C = d["A"][sel].cuda(), d["B"][sel].cuda(), d["C"][sel].cuda()
    D = tcx.mma_tiles(A, B, C, tf32=(fmt == "tf32"))
    D5 = tcx.mma_tiles_tc05(A, B, C, tf32=(fmt == "tf32"))
    torch.cuda.synchronize()
    np.savez(os.path.join(out, f"subnormal_{fmt}.npz"), a=host_bits(A[:, 0, :]), b=host_bits(B[:, 0, :]),
             c=host_bits(C[:, 0, 0]), d=host_bits(D)[:, 0, 0], d5=host_bits(D5)[:, 0, 0])
    print(fmt, int(sel.sum()))
