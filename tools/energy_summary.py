#!/usr/bin/env python
"""Median over rounds of tools/energy_study.py lines, per variant: python tools/energy_summary.py a.jsonl [b.jsonl ...]"""
import json
import statistics
import sys
from collections import defaultdict


def main():
    rows = defaultdict(list)
    for p in sys.argv[1:]:
        for ln in open(p):
            if ln.strip():
                d = json.loads(ln)
                rows[(p.split("/")[-1], d["variant"])].append(d)
    print(f"{'file':16s} {'variant':28s} {'n':>2s} {'ms':>8s} {'J/launch':>9s} {'W':>7s} {'TFLOP/s':>8s} {'pJ/FLOP':>8s} {'MHz':>6s}")
    for (f, v), ds in rows.items():
        med = lambda k: statistics.median([d[k] for d in ds if d.get(k) is not None]) if any(d.get(k) is not None for d in ds) else float("nan")
        print(f"{f:16s} {v:28s} {len(ds):2d} {med('ms'):8.3f} {med('J_per_launch'):9.4f} {med('W'):7.1f} "
              f"{med('tflops'):8.1f} {med('pJ_per_flop'):8.4f} {med('sm_mhz_median'):6.0f}")


if __name__ == "__main__":
    main()
