#!/usr/bin/env python
"""From a round's full ncu captures (profiles/<tag>_<cfg>.ncu-rep) write profiles/<tag>_ncu_summary.txt
and profiles/traffic.json (dram read + write bytes per launch, the bench's roofline.traffic).
usage: python tools/ncu_traffic.py <tag> [cfg ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import summary  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def nbytes(s):
    v, u = s.split()
    return float(v.replace(",", "")) * UNITS[u]


def main():
    tag = sys.argv[1]
    cfgs = sys.argv[2:] or ["c3", "c3tf32", "c4", "c5", "c1"]
    traffic = {}
    lines = []
    for cfg in cfgs:
        rep = os.path.join(ROOT, "profiles", f"{tag}_{cfg}.ncu-rep")
        if not os.path.exists(rep):
            continue
        d = summary(rep)[0]
        traffic[cfg] = int(nbytes(d["dram__bytes_read.sum"]) + nbytes(d["dram__bytes_write.sum"]))
        lines.append(f"== {cfg}")
        lines += [f"{k} {v}" for k, v in sorted(d.items())]
    traffic["_source"] = (f"ncu --set full --clock-control none, one launch per config (profiles/{tag}_<cfg>.ncu-rep): "
                          "dram__bytes_read.sum + dram__bytes_write.sum per launch")
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(os.path.join(ROOT, "profiles", "traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main()
