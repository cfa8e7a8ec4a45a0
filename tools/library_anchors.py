#!/usr/bin/env python
"""Same-work library anchors (context for the bench's denominators; nothing here is on the tcx path):
  * C3: cuBLAS through torch.addmm(C, A, B^T, out_dtype=float32) — BF16 inputs, FP32 C read and FP32 D
    written, the same work as tcx_gemm on configs[2] (torch.matmul's BF16-out line does less);
  * C5: cuSPARSELt through torch._cslt_sparse_mm on the same 2:4 operand (if available).
Burst = best of 10 single launches; sustained = median of 20-launch chunks over ~3 s.
python tools/library_anchors.py OUT.jsonl"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def timeit(fn, flops, seconds=3.0):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    vals = []
    t0 = time.time()
    while time.time() - t0 < seconds:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            fn()
        e1.record(); e1.synchronize()
        vals.append(e0.elapsed_time(e1) / 20)
    vals.sort()
    return {"burst_tflops": round(flops / (best * 1e-3) / 1e12, 1),
            "sustained_tflops": round(flops / (vals[len(vals) // 2] * 1e-3) / 1e12, 1)}


def main():
    out = open(sys.argv[1], "w") if len(sys.argv) > 1 else None
    torch.cuda.set_device(0)
    res = {}
    w = bench.Work("c3", 0, 1, torch.device("cuda", 0))
    Bt = w.B.t()
    D = torch.empty_like(w.D)
    res["c3_tcx"] = timeit(lambda: w.step(), w.flops)
    try:
        res["c3_cublas_addmm_fp32_out"] = timeit(lambda: torch.addmm(w.C, w.A, Bt, out_dtype=torch.float32, out=D), w.flops)
        ref = torch.addmm(w.C, w.A, Bt, out_dtype=torch.float32)
        res["c3_cublas_addmm_fp32_out"]["max_abs_diff_vs_tcx"] = float((ref - w.D).abs().max())
    except Exception as e:
        res["c3_cublas_addmm_fp32_out"] = {"error": f"{type(e).__name__}: {e}"[:200]}
    res["c3_cublas_matmul_bf16_out"] = timeit(lambda: torch.matmul(w.A, Bt), w.flops)
    del w, Bt, D
    torch.cuda.empty_cache()
    res["cusparselt_available"] = bool(getattr(torch.backends, "cusparselt", None) and torch.backends.cusparselt.is_available())
    w5 = bench.Work("c5", 0, 1, torch.device("cuda", 0))
    res["c5_tcx"] = timeit(lambda: w5.step(), w5.flops)
    if res["cusparselt_available"]:
        try:
            import tcxgen as g
            M, N, K = w5.shape
            # the same 2:4 operand, dense (M x K) f16 -> cuSPARSELt's compressed form
            meta = None
            vals, meta = g.sp24_problem(M, K, 0, "f16", "cuda")
            dense = torch.zeros(M, K, dtype=torch.float16, device="cuda")
            pairs = g.sp24_pairs(M, K, 0, g.STREAM_POS, "cuda").long()
            P = torch.tensor(g.PAIRS, device="cuda")
            cols = (torch.arange(K // 4, device="cuda") * 4).view(1, -1)
            i0 = cols + P[pairs][..., 0]
            i1 = cols + P[pairs][..., 1]
            dense.scatter_(1, i0, vals[:, 0::2])
            dense.scatter_(1, i1, vals[:, 1::2])
            del vals, meta, pairs, i0, i1
            comp = torch._cslt_compress(dense)
            del dense
            torch.cuda.empty_cache()
            Bd = w5.B.t()                                   # K x N (column-major view of B)
            fn = lambda: torch._cslt_sparse_mm(comp, Bd, out_dtype=torch.float32)
            try:
                fn()
                res["c5_cusparselt_fp32_out"] = timeit(fn, w5.flops)
            except Exception as e:
                res["c5_cusparselt_fp32_out"] = {"error": f"{type(e).__name__}: {e}"[:200]}
                fn = lambda: torch._cslt_sparse_mm(comp, Bd)
                res["c5_cusparselt_f16_out"] = timeit(fn, w5.flops)
        except Exception as e:
            res["c5_cusparselt"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    print(json.dumps(res, indent=1))
    if out:
        out.write(json.dumps(res) + "\n")


if __name__ == "__main__":
    main()
