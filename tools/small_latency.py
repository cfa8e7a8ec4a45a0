#!/usr/bin/env python
"""Per-call time of small dense GEMMs: eager back-to-back Python calls vs the same calls replayed
from a CUDA graph (no host cost), beside cuBLAS (torch.matmul BF16 out, no C) — separates the
host-side cost of a call from the kernel's own latency.  python tools/small_latency.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import tcxgen as g  # noqa: E402
import paper_2206_02874_b200 as tcx  # noqa: E402


def per_call_us(fn, n=50, graph=False):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        run = fn
        if graph:
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=s):
                for _ in range(n):
                    fn()
            run = gr.replay
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        if graph:
            run()
        else:
            for _ in range(n):
                run()
        e1.record(s)
        torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) * 1e3 / n, 2)


def main():
    torch.cuda.set_device(0)
    dev = "cuda"
    out = []
    for M, N, K in [(256, 256, 256), (512, 512, 512), (1024, 1024, 1024), (2048, 2048, 2048), (4096, 4096, 4096)]:
        A = g.normal_matrix((M, K), "bf16", 0, g.STREAM_A, dev)
        B = g.normal_matrix((N, K), "bf16", 0, g.STREAM_B, dev)
        C = torch.zeros(M, N, device=dev)
        D = torch.empty_like(C)
        Bt = B.t()
        r = {"shape": [M, N, K]}
        for name, fn in [("tcx", lambda: tcx.gemm(A, B, C, D)), ("tcx_noC", lambda: tcx.gemm(A, B, None, D)),
                         ("cublas_bf16_noC", lambda: torch.matmul(A, Bt))]:
            r[name + "_eager_us"] = per_call_us(fn)
            r[name + "_graph_us"] = per_call_us(fn, graph=True)
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
