#!/usr/bin/env python
"""Median / min / max per variant (and lib) of tools/ab_burst.py lines: python tools/ab_summary.py f.jsonl ..."""
import collections
import json
import statistics
import sys

for p in sys.argv[1:]:
    d = collections.defaultdict(list)
    for ln in open(p):
        if ln.startswith("{"):
            r = json.loads(ln)
            d[(r.get("lib", ""), r["cfg"], r["variant"])].append((r["tflops"], r["sm_mhz_in_run"]))
    for (lib, cfg, v), xs in d.items():
        t = [x[0] for x in xs]
        print(f"{p.split('/')[-1]:28s} {lib:8s} {cfg:9s} {v:28s} n={len(xs)} median {statistics.median(t):8.1f} "
              f"min {min(t):8.1f} max {max(t):8.1f} MHz {statistics.median([x[1] for x in xs]):.0f}")
