#!/usr/bin/env python
"""The paper's §V/§VI microbenchmark sweep re-measured on B200 through tcx_probe.

For every instruction shape of Table A100-mma and Table A100-mmasp
(PAPER.md:608-624): completion latency (1 warp, ILP 1) and the
(#warps in {1,2,4,6,8,12,16}) x (ILP 1..6) grid; plus the tcgen05 analogue (one issuing thread,
ILP MMAs in flight per commit, cta_group 1/2).  Writes JSON (+ a markdown summary) to argv[1].
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2206_02874_b200 as tcx  # noqa: E402

F16, BF16, TF32, F32, S8, S32 = tcx.F16, tcx.BF16, tcx.TF32, tcx.F32, tcx.S8, tcx.S32
NAMES = {F16: "FP16", BF16: "BF16", TF32: "TF32", F32: "FP32", S8: "INT8", S32: "INT32"}

DENSE = [(F16, F32, 16, 8, 16), (F16, F32, 16, 8, 8), (F16, F16, 16, 8, 16), (F16, F16, 16, 8, 8),
         (BF16, F32, 16, 8, 16), (BF16, F32, 16, 8, 8), (TF32, F32, 16, 8, 8), (TF32, F32, 16, 8, 4),
         (S8, S32, 8, 8, 16), (S8, S32, 16, 8, 32), (S8, S32, 16, 8, 16)]
SPARSE = [(F16, F32, 16, 8, 32), (F16, F32, 16, 8, 16), (BF16, F32, 16, 8, 32), (BF16, F32, 16, 8, 16),
          (TF32, F32, 16, 8, 16), (TF32, F32, 16, 8, 8), (S8, S32, 16, 8, 64), (S8, S32, 16, 8, 32)]
WARPS = [1, 2, 4, 6, 8, 12, 16]
ILPS = [1, 2, 3, 4, 5, 6]
# paper's A100 peaks for context: (completion, best thr, (w, ilp))
PAPER_A100 = {"FP16->FP32 m16n8k16": (24.7, 1004.2), "FP16->FP32 m16n8k8": (17.7, 974.1),
              "FP16->FP16 m16n8k16": (24.4, 996.6), "FP16->FP16 m16n8k8": (17.7, 1002.6),
              "TF32->FP32 m16n8k8": (25.0, 492.4), "TF32->FP32 m16n8k4": (18.1, 477.5),
              "INT8->INT32 m8n8k16": (15.9, 998.3), "INT8->INT32 m16n8k32": (24.7, 1986.5),
              "INT8->INT32 m16n8k16": (17.6, 1965.1), "sp FP16->FP32 m16n8k32": (24.7, 1979.1),
              "sp FP16->FP32 m16n8k16": (17.9, 1290.5), "sp INT8->INT32 m16n8k64": (None, 3961.5)}


def label(ab, cd, m, n, k, sp=False):
    return ("sp " if sp else "") + f"{NAMES[ab]}->{NAMES[cd]} m{m}n{n}k{k}"


def sweep_sync(kind, shapes, iters):
    out = []
    for ab, cd, m, n, k in shapes:
        sp = kind == "mma_sp_sync"
        comp = tcx.probe(kind, ab, cd, m, n, k, warps=1, ilp=1, iters=iters, repeats=5)
        grid = []
        for w in WARPS:
            for ilp in ILPS:
                r = tcx.probe(kind, ab, cd, m, n, k, warps=w, ilp=ilp, iters=iters, repeats=3)
                grid.append({"warps": w, "ilp": ilp, "latency": round(r["latency_cycles"], 2),
                             "fma_clk_sm": round(r["fma_per_clk_per_sm"], 1)})
        best = max(grid, key=lambda g: g["fma_clk_sm"])
        lab = label(ab, cd, m, n, k, sp)
        out.append({"instr": lab, "completion_latency": round(comp["latency_cycles"], 2), "sm_mhz": round(comp["sm_mhz"]),
                    "best": best, "grid": grid, "a100_paper": PAPER_A100.get(lab)})
        print(f"{lab:28s} completion {comp['latency_cycles']:6.1f} cyc  best {best['fma_clk_sm']:8.1f} FMA/clk/SM at "
              f"({best['warps']},{best['ilp']})", flush=True)
    return out


def sweep_tc05(iters):
    out = []
    cases = [("tc05", BF16, F32, 16, 1, 128), ("tc05", BF16, F32, 16, 2, 256), ("tc05", F16, F32, 16, 1, 64),
             ("tc05", TF32, F32, 8, 1, 128), ("tc05", TF32, F32, 8, 2, 256), ("tc05", S8, S32, 32, 1, 128),
             ("tc05", S8, S32, 32, 2, 256), ("tc05_sp", F16, F32, 32, 1, 128), ("tc05_sp", F16, F32, 32, 2, 256),
             ("tc05_sp", BF16, F32, 32, 2, 256), ("tc05_sp", TF32, F32, 16, 2, 256), ("tc05_sp", S8, S32, 64, 2, 256)]
    for kind, ab, cd, k, cg, m in cases:
        for n in (64, 128, 256):
            row = {"kind": kind, "instr": label(ab, cd, m, n, k, kind == "tc05_sp") + f" cta_group::{cg}", "points": []}
            for ilp in (1, 2, 4, 8, 16, 32):
                try:
                    r = tcx.probe(kind, ab, cd, m, n, k, cta_group=cg, ilp=ilp, iters=iters, repeats=3)
                except tcx.TcxError as e:
                    row["error"] = str(e)
                    break
                row["points"].append({"ilp": ilp, "latency": round(r["latency_cycles"], 1),
                                      "fma_clk_sm": round(r["fma_per_clk_per_sm"], 1), "sm_mhz": round(r["sm_mhz"])})
            if row["points"]:
                b = max(row["points"], key=lambda p: p["fma_clk_sm"])
                print(f"{row['instr']:44s} ILP1 {row['points'][0]['latency']:7.1f} cyc   best {b['fma_clk_sm']:8.1f} "
                      f"FMA/clk/SM (ILP {b['ilp']})", flush=True)
            out.append(row)
    return out


def main():
    path = sys.argv[1] if len(sys.argv) > 1 else "probe_sweep.json"
    torch.cuda.set_device(0)
    res = {"device": torch.cuda.get_device_name(0),
           "mma_sync": sweep_sync("mma_sync", DENSE, 1024),
           "mma_sp_sync": sweep_sync("mma_sp_sync", SPARSE, 1024),
           "tcgen05": sweep_tc05(256)}
    json.dump(res, open(path, "w"), indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
