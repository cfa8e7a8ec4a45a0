#!/usr/bin/env python
"""A/B tcx_gemm_sp24 options on a 2:4 FP16 / 1:2 TF32 shape in the bench's burst conditions:
python tools/ab_sparse_opts.py f16|tf32 M N K "tile_m=256;pairs=1x2" [steps] [rounds]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import torch  # noqa: E402

import tcxgen as g  # noqa: E402
import paper_2206_02874_b200 as tcx  # noqa: E402
from ab_burst import parse  # noqa: E402


def main():
    fmt, M, N, K = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    variants = sys.argv[5].split(";")
    steps = int(sys.argv[6]) if len(sys.argv) > 6 else 20
    rounds = int(sys.argv[7]) if len(sys.argv) > 7 else 3
    torch.cuda.set_device(0)
    vals, meta = g.sp12_problem_tf32(M, K, 0, "cuda") if fmt == "tf32" else g.sp24_problem(M, K, 0, fmt, "cuda")
    hw = tcx.sp24_pack_meta(meta, M, K, ab=tcx.TF32 if fmt == "tf32" else tcx.F16)
    B = g.normal_matrix((N, K), fmt, 0, g.STREAM_B, "cuda")
    C, D = torch.zeros(M, N, device="cuda"), torch.empty(M, N, device="cuda")
    for r in range(rounds):
        for v in (variants if r % 2 == 0 else variants[::-1]):
            kw = parse(v)
            step = lambda: tcx.gemm_sp24(vals, hw, B, C, D, tf32=(fmt == "tf32"), **kw)
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
            print(json.dumps({"cfg": f"{fmt}:{M}:{N}:{K}", "round": r, "variant": v, "ms": round(ms, 4),
                              "tflops": round(2.0 * M * N * K / (ms * 1e-3) / 1e12, 1), "sm_mhz_in_run": 0}), flush=True)


if __name__ == "__main__":
    main()
