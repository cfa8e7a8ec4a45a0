#!/usr/bin/env python
"""run one C3 variant a few times (for ncu): python tools/exp_one.py <variant> [reps]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import bench  # noqa: E402

v = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
torch.cuda.set_device(0)
w = bench.Work("c3", 0, 1, torch.device("cuda", 0))
D16 = torch.empty(8192, 8192, dtype=torch.bfloat16, device="cuda")
fns = {"cublas": lambda: torch.matmul(w.A, w.B.t(), out=D16),
       "narrow_noC": lambda: w.tcx.gemm(w.A, w.B, None, w.D, tile_n=256),
       "wide_noC": lambda: w.tcx.gemm(w.A, w.B, None, w.D, tile_n=512),
       "narrow": lambda: w.tcx.gemm(w.A, w.B, w.C, w.D, tile_n=256),
       "wide": lambda: w.tcx.gemm(w.A, w.B, w.C, w.D, tile_n=512),
       "mc12": lambda: w.tcx.gemm(w.A, w.B, w.C, w.D, pairs=(1, 2)),
       "mc21": lambda: w.tcx.gemm(w.A, w.B, w.C, w.D, pairs=(2, 1)),
       "mc22": lambda: w.tcx.gemm(w.A, w.B, w.C, w.D, pairs=(2, 2))}
for _ in range(reps):
    fns[v]()
torch.cuda.synchronize()
print("ok", v)
