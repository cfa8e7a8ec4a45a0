#!/usr/bin/env python
"""grep an ncu report's raw page: python tools/ncu_grep.py rep.ncu-rep pattern [pattern...]"""
import csv, io, re, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u = rows[0], rows[1]
pats = [re.compile(p) for p in sys.argv[2:]]
for n, v in enumerate(rows[2:]):
    for i, k in enumerate(h):
        if any(p.search(k) for p in pats):
            print(n, k, v[i], u[i])
