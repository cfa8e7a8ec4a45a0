#!/usr/bin/env python
"""Kernel-configuration sweep for the GEMM paths (raster group, CTA mode).

usage: python tools/exp_gemm.py c5|c3|c4|c3tf32|c4sp|c3sptf32 [steps] [variant ...]
variant = "g<group_m>c<cta_group>[w][p<pm><pn>]" e.g. g8c2, g16c2, g8c1, g8c2w (w = the 512-wide tile),
g8c2p12 (multicast cluster of 1 x 2 CTA pairs).  Prints one JSON line per variant
with device time (CUDA events), TFLOP/s, NVML SM clock / power during the run, and whether D is
bit-identical to the first variant's D (the knobs change no arithmetic)."""
import json
import os
import re
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def parse(v):
    m = re.fullmatch(r"g(-?\d+)c(\d)(w?)(?:p(\d)(\d))?", v)
    kw = dict(group_m=int(m.group(1)), cta_group=int(m.group(2)))
    if m.group(3):
        kw["wide"] = True
    if m.group(4):
        kw["pairs"] = (int(m.group(4)), int(m.group(5)))
    return kw


def main():
    cfg = sys.argv[1]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    variants = sys.argv[3:] or ["g8c2"]
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    w = bench.Work(cfg, 0, 1, dev)
    tcx = w.tcx
    sampler = bench.ClockSampler(0)
    try:
        import pynvml
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
    except Exception:
        h = None
    ref = None
    for v in variants:
        kw = parse(v)
        wide = kw.pop("wide", False)
        if hasattr(w, "vals"):                          # sparse configs (c5, c4sp, c3sptf32)
            tf = cfg == "c3sptf32"
            step = lambda: tcx.gemm_sp24(w.vals, w.meta_hw, w.B, w.C, w.D, tf32=tf,
                                         tile_m=512 if wide else 256, **kw)
        else:
            step = lambda: tcx.gemm(w.A, w.B, w.C, w.D, tf32=getattr(w, "tf32", False), tile_n=512 if wide else 0, **kw)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        pw = []
        sampler.samples = []
        sampler.start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.time()
        e0.record()
        for _ in range(steps):
            step()
        e1.record()
        if h is not None:
            while not e1.query():
                try:
                    pw.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0)
                except Exception:
                    pass
                time.sleep(0.01)
        torch.cuda.synchronize()
        t1 = time.time()
        sampler.stop()
        ms = e0.elapsed_time(e1) / steps
        clk = sampler.summary(t0, t1)
        same = None
        if ref is None:
            ref = w.D.clone()
        else:
            same = bool(torch.equal(ref.view(torch.int32), w.D.view(torch.int32)))
        print(json.dumps({"cfg": cfg, "variant": v, "ms": round(ms, 4), "tflops": round(w.flops / ms / 1e9, 1),
                          "sm_mhz": clk.get("sm_mhz"), "reasons": clk.get("reasons"),
                          "power_w": round(sorted(pw)[len(pw) // 2], 1) if pw else None, "bit_identical": same}),
              flush=True)


if __name__ == "__main__":
    main()
