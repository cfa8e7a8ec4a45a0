#!/usr/bin/env python
"""A/B a dense or sparse GEMM option under the bench's own burst conditions: per round and variant,
idle ~1 s (the board leaves its power cap), then W warm-ups and K event-timed steps, exactly as
bench.time_steps; interleaved rounds.  python tools/ab_burst.py c3 "tile_n=256;tile_n=512" [rounds]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def parse(v):
    kw = {}
    for part in v.split(","):
        if part.startswith("env:"):          # env:NAME=VALUE (library A/B knobs read per call)
            k, x = part[4:].split("=")
            os.environ[k] = x
        elif part:
            k, x = part.split("=")
            kw[k] = tuple(int(t) for t in x.split("x")) if "x" in x else int(x)
    return kw


def main():
    cfg, variants = sys.argv[1], sys.argv[2].split(";")
    rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 6
    torch.cuda.set_device(0)
    w = bench.Work(cfg, 0, 1, torch.device("cuda", 0))
    sparse = hasattr(w, "vals")
    base = w.step
    for r in range(rounds):
        for v in (variants if r % 2 == 0 else variants[::-1]):
            kw = parse(v)
            if cfg == "c1":                              # the tile batch has no kernel options
                w.step = base
            elif sparse:
                w.step = lambda: w.tcx.gemm_sp24(w.vals, w.meta_hw, w.B, w.C, w.D, tf32=cfg == "c3sptf32", **kw)
            else:
                w.step = lambda: w.tcx.gemm(w.A, w.B, w.C, w.D, tf32=getattr(w, "tf32", False),
                                            f16_acc=cfg == "c3f16acc", **kw)
            torch.cuda.synchronize()
            time.sleep(1.0)
            ms, _, _, _ = bench.time_steps(w, 20, 5, False)
            print(json.dumps({"cfg": cfg, "round": r, "variant": v, "ms": round(ms, 5),
                              "tflops": round(w.flops / (ms * 1e-3) / 1e12, 1),
                              "sm_mhz_in_run": round(w.sm_mhz_eff or 0, 1)}), flush=True)
    w.step = base


if __name__ == "__main__":
    main()
