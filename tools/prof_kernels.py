#!/usr/bin/env python
"""Run a few launches of one hot-path kernel for ncu (`ncu -k regex:<kernel> ...`).
Usage: python tools/prof_kernels.py c3|c3tf32|c4|c5|c5s|c1 [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    w = bench.Work(cfg, 0, 1, dev)
    for _ in range(reps):
        w.step()
    torch.cuda.synchronize()
    print("ok", cfg, reps)


if __name__ == "__main__":
    main()
