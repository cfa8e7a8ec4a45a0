#!/usr/bin/env python
"""C3 variants vs same-run cuBLAS (context): python tools/exp_anchor.py [steps]"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import bench  # noqa: E402


def timeit(fn, steps, flops):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    return round(flops / ms / 1e9, 1), round(ms, 4)


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    w = bench.Work("c3", 0, 1, dev)
    tcx = w.tcx
    Bt = w.B.t()
    D16 = torch.empty(8192, 8192, dtype=torch.bfloat16, device=dev)
    variants = {
        "cublas_bf16_out": lambda: torch.matmul(w.A, Bt, out=D16),
        "tcx_default": lambda: tcx.gemm(w.A, w.B, w.C, w.D),
        "tcx_noC": lambda: tcx.gemm(w.A, w.B, None, w.D),
        "tcx_narrow_noC": lambda: tcx.gemm(w.A, w.B, None, w.D, tile_n=256),
        "tcx_narrow": lambda: tcx.gemm(w.A, w.B, w.C, w.D, tile_n=256),
        "tcx_wide": lambda: tcx.gemm(w.A, w.B, w.C, w.D, tile_n=512),
        "tcx_wide_g16": lambda: tcx.gemm(w.A, w.B, w.C, w.D, tile_n=512, group_m=16),
        "tcx_cg1": lambda: tcx.gemm(w.A, w.B, w.C, w.D, cta_group=1),
    }
    for rnd in range(2):
        for name, fn in variants.items():
            tf, ms = timeit(fn, steps, w.flops)
            print(json.dumps({"round": rnd, "variant": name, "tflops": tf, "ms": ms}), flush=True)
            time.sleep(1.0)


if __name__ == "__main__":
    main()
