#!/usr/bin/env python
"""Run a few launches of one energy-study variant (tools/energy_study.py names) for ncu:
python tools/prof_variant.py c5_mwpn2 [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402

import energy_study as es  # noqa: E402


def main():
    name = sys.argv[1]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    torch.cuda.set_device(0)
    step, _ = es.variant(name)
    for _ in range(reps):
        step()
    torch.cuda.synchronize()
    print("ok", name, reps)


if __name__ == "__main__":
    main()
