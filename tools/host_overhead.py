#!/usr/bin/env python
"""Host-side cost per call of the Python binding + C ABI (tiny problems, GPU time negligible):
python tools/host_overhead.py"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import tcxgen as g  # noqa: E402
import paper_2206_02874_b200 as tcx  # noqa: E402


def per_call(fn, n=2000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    return round((t1 - t0) / n * 1e6, 2), round((t2 - t0) / n * 1e6, 2)


torch.cuda.set_device(0)
dev = "cuda"
A = g.normal_matrix((256, 64), "bf16", 0, g.STREAM_A, dev)
B = g.normal_matrix((256, 64), "bf16", 0, g.STREAM_B, dev)
C = torch.zeros(256, 256, device=dev)
D = torch.empty_like(C)
L = tcx.lib()
At = g.uniform_matrix((64, 16, 16), "f16", 0, 1, device=dev)
Bt = g.uniform_matrix((64, 8, 16), "f16", 0, 2, device=dev)
Dt = torch.empty(64, 16, 8, device=dev)
res = {}
res["ctypes_tcx_version"] = per_call(lambda: L.tcx_version())
res["tcx.gemm_256x256x64"] = per_call(lambda: tcx.gemm(A, B, C, D))
res["tcx.mma_tiles_64"] = per_call(lambda: tcx.mma_tiles(At, Bt, None, Dt))
Bt_ = B.t()
res["torch.matmul_256x256x64"] = per_call(lambda: torch.matmul(A, Bt_))
res["raw_ctypes_tcx_gemm"] = per_call(lambda: L.tcx_gemm(tcx.BF16, tcx.F32, 256, 256, 64, A.data_ptr(), 64, B.data_ptr(), 64,
                                                        C.data_ptr(), 256, D.data_ptr(), 256, None))
print(json.dumps({k: {"host_us_per_call": v[0], "wall_us_per_call_incl_gpu": v[1]} for k, v in res.items()}, indent=1))
