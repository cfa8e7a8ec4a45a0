#!/usr/bin/env python
"""Wave quantisation study: event-timed tcx_gemm on row-sharded-rank shapes (C3 / C4 split over
2, 4, 8 GPUs) with the 256-wide tile vs the library's wave-aware width (tile_n = 0) and forced
widths; interleaved rounds.  python tools/wave_study.py [rounds]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import tcxgen  # noqa: E402
import paper_2206_02874_b200 as tcx  # noqa: E402


def timed(fn, steps=20, warmup=5):
    for _ in range(warmup):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(steps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / steps


def main():
    rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    dev = "cuda"
    shapes = [("c3/8", "bf16", 1024, 8192, 8192), ("c3/4", "bf16", 2048, 8192, 8192), ("c3/2", "bf16", 4096, 8192, 8192),
              ("c3/1", "bf16", 8192, 8192, 8192), ("c4/8", "s8", 2048, 16384, 16384), ("c4/4", "s8", 4096, 16384, 16384)]
    if len(sys.argv) > 2 and sys.argv[2] == "small":    # latency-bound calls: the tile count decides
        shapes = [("512^3", "bf16", 512, 512, 512), ("1024^3", "bf16", 1024, 1024, 1024),
                  ("2048^3", "bf16", 2048, 2048, 2048), ("256x4096x4096", "bf16", 256, 4096, 4096),
                  ("1024x1280x1024", "bf16", 1024, 1280, 1024)]
    variants = {"w256": dict(tile_n=256), "w256_plain": dict(tile_n=256, pairs=(1, 1)), "auto": {},
                "w224": dict(tile_n=224), "w192": dict(tile_n=192), "w160": dict(tile_n=160), "w128": dict(tile_n=128)}
    for name, fmt, M, N, K in shapes:
        if fmt == "s8":
            A = tcxgen.int8_matrix((M, K), 0, tcxgen.STREAM_A, dev)
            B = tcxgen.int8_matrix((N, K), 0, tcxgen.STREAM_B, dev)
            C = tcxgen.int32_matrix((M, N), 0, tcxgen.STREAM_C, device=dev)
            D = torch.empty(M, N, dtype=torch.int32, device=dev)
        else:
            A = tcxgen.normal_matrix((M, K), fmt, 0, tcxgen.STREAM_A, dev)
            B = tcxgen.normal_matrix((N, K), fmt, 0, tcxgen.STREAM_B, dev)
            C = torch.zeros(M, N, dtype=torch.float32, device=dev)
            D = torch.empty(M, N, dtype=torch.float32, device=dev)
        for r in range(rounds):
            for v, kw in (list(variants.items()) if r % 2 == 0 else list(variants.items())[::-1]):
                time.sleep(0.3)
                ms = timed(lambda: tcx.gemm(A, B, C, D, **kw))
                print(json.dumps({"shape": name, "M": M, "N": N, "K": K, "variant": v, "round": r, "ms": round(ms, 5),
                                  "tflops": round(2 * M * N * K / ms / 1e9, 1)}), flush=True)
        del A, B, C, D


if __name__ == "__main__":
    main()
