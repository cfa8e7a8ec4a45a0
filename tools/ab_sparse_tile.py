#!/usr/bin/env python
"""A/B the sparse tile height (256 x 240 vs 512 x 240) on a bench config or a shape, interleaved, in the
bench's burst conditions (1 s idle, 5 warm-ups, `steps` event-timed steps):
python tools/ab_sparse_tile.py c3sptf32|c5|f16:M:N:K|tf32:M:N:K [steps] [rounds]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3sptf32"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 4
torch.cuda.set_device(0)
if cfg.startswith(("f16:", "tf32:")):          # f16:M:N:K / tf32:M:N:K — a 2:4 FP16 (1:2 TF32) problem
    import types
    import tcxgen as g
    import paper_2206_02874_b200 as tcx
    fmt = cfg.split(":")[0]
    M, N, K = (int(x) for x in cfg.split(":")[1:])
    vals, meta = g.sp12_problem_tf32(M, K, 0, "cuda") if fmt == "tf32" else g.sp24_problem(M, K, 0, fmt, "cuda")
    w = types.SimpleNamespace(tcx=tcx, vals=vals, meta_hw=tcx.sp24_pack_meta(meta, M, K, ab=tcx.TF32 if fmt == "tf32" else tcx.F16),
                              B=g.normal_matrix((N, K), fmt, 0, g.STREAM_B, "cuda"),
                              C=torch.zeros(M, N, device="cuda"), D=torch.empty(M, N, device="cuda"), flops=2.0 * M * N * K)
else:
    w = bench.Work(cfg, 0, 1, torch.device("cuda", 0))
tf = cfg == "c3sptf32" or cfg.startswith("tf32:")
for r in range(rounds):
    for tm in ((256, 512) if r % 2 == 0 else (512, 256)):
        step = lambda: w.tcx.gemm_sp24(w.vals, w.meta_hw, w.B, w.C, w.D, tf32=tf, tile_m=tm)
        torch.cuda.synchronize()
        time.sleep(1.0)
        for _ in range(5):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        print(json.dumps({"cfg": cfg, "round": r, "tile_m": tm, "ms": round(ms, 4),
                          "tflops": round(w.flops / (ms * 1e-3) / 1e12, 1)}), flush=True)
