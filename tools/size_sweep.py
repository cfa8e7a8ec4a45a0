#!/usr/bin/env python
"""TFLOP/s vs problem size on one B200: dense BF16 (FP32 C/D) square GEMMs 512..16384 through tcx_gemm,
beside cuBLAS torch.matmul (bf16 out, no C) at the same sizes as context, and 2:4 FP16 GEMMs.
CUDA events over back-to-back launches after warm-up; python tools/size_sweep.py > out.jsonl"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import tcxgen as g  # noqa: E402
import paper_2206_02874_b200 as tcx  # noqa: E402


def timeit(fn, flops, min_ms=200.0):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    n = 1
    while True:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if ms >= min_ms or n >= 4096:
            return round(flops * n / (ms * 1e-3) / 1e12, 1), round(ms / n * 1e3, 2)
        n *= 2


def main():
    torch.cuda.set_device(0)
    dev = "cuda"
    for S in (512, 1024, 2048, 4096, 6144, 8192, 12288, 16384):
        A = g.normal_matrix((S, S), "bf16", 0, g.STREAM_A, dev)
        B = g.normal_matrix((S, S), "bf16", 0, g.STREAM_B, dev)
        C = torch.zeros(S, S, dtype=torch.float32, device=dev)
        D = torch.empty_like(C)
        f = 2.0 * S ** 3
        t, us = timeit(lambda: tcx.gemm(A, B, C, D), f)
        Bt = B.t()
        c, cus = timeit(lambda: torch.matmul(A, Bt), f)
        print(json.dumps({"kind": "dense_bf16", "M=N=K": S, "tcx_tflops": t, "tcx_us": us,
                          "cublas_bf16out_tflops": c, "cublas_us": cus}), flush=True)
        del A, B, C, D
        torch.cuda.empty_cache()
    for M, N, K in ((2048, 2048, 2048), (4096, 4096, 4096), (8192, 8192, 8192), (16384, 16384, 16384),
                    (65536, 16384, 16384)):
        vals, meta = g.sp24_problem(M, K, 0, "f16", dev)
        hw = tcx.sp24_pack_meta(meta, M, K)
        del meta
        B = g.normal_matrix((N, K), "f16", 0, g.STREAM_B, dev)
        C = torch.zeros(M, N, dtype=torch.float32, device=dev)
        D = torch.empty_like(C)
        t, us = timeit(lambda: tcx.gemm_sp24(vals, hw, B, C, D), 2.0 * M * N * K)
        print(json.dumps({"kind": "sp24_f16", "M": M, "N": N, "K": K, "tcx_tflops_dense_eq": t, "tcx_us": us}), flush=True)
        del vals, hw, B, C, D
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
