#!/usr/bin/env python
"""A/B dense tcx_gemm options on an arbitrary shape in the bench's burst conditions (1 s idle, 5
warm-ups, `steps` event-timed steps), interleaved rounds:
python tools/ab_dense_shape.py bf16|tf32|s8 M N K "tile_n=256;tile_n=512" [steps] [rounds]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import tcxgen as g  # noqa: E402
import paper_2206_02874_b200 as tcx  # noqa: E402
from ab_burst import parse  # noqa: E402


def main():
    fmt, M, N, K = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    variants = sys.argv[5].split(";")
    steps = int(sys.argv[6]) if len(sys.argv) > 6 else 20
    rounds = int(sys.argv[7]) if len(sys.argv) > 7 else 4
    torch.cuda.set_device(0)
    dev = "cuda"
    if fmt == "s8":
        A, B = g.int8_matrix((M, K), 0, g.STREAM_A, dev), g.int8_matrix((N, K), 0, g.STREAM_B, dev)
        C = g.int32_matrix((M, N), 0, g.STREAM_C, device=dev)
        D = torch.empty(M, N, dtype=torch.int32, device=dev)
    else:
        A, B = g.normal_matrix((M, K), fmt, 0, g.STREAM_A, dev), g.normal_matrix((N, K), fmt, 0, g.STREAM_B, dev)
        C, D = torch.zeros(M, N, device=dev), torch.empty(M, N, device=dev)
    for r in range(rounds):
        for v in (variants if r % 2 == 0 else variants[::-1]):
            kw = parse(v)
            step = lambda: tcx.gemm(A, B, C, D, tf32=(fmt == "tf32"), **kw)
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
