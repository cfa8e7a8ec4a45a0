#!/usr/bin/env python
"""Offline fit of the truncation point on the C2 SUBNORMAL class (tools/subnormal_dump.py output):
for every tile, the set of truncation exponents L for which
    RZ_fp32( sum_k trunc_L(a_k b_k) + trunc_L(c) ) == GPU d00
is found by exact integer arithmetic, and reported relative to the block's nominal leading exponent
(esum2: product e_a + e_b + 1, c: lead + 1).  python tools/subnormal_fit.py gpurun_out/subnormal_bf16.npz"""
import sys
from collections import Counter

import numpy as np

S = 400                       # values are integers in units of 2^-S


def dec(fmt, bits):
    """-> (sign, mant, exp) with value = (-1)^sign mant 2^exp, plus the unbiased exponent eu."""
    bits = int(bits)
    if fmt == "f16":
        s, e, f, fb, bias = bits >> 15 & 1, bits >> 10 & 0x1F, bits & 0x3FF, 10, 15
    elif fmt == "bf16":
        s, e, f, fb, bias = bits >> 15 & 1, bits >> 7 & 0xFF, bits & 0x7F, 7, 127
    else:
        s, e, f, fb, bias = bits >> 31 & 1, bits >> 23 & 0xFF, bits & 0x7FFFFF, 23, 127
    eu = (1 - bias) if e == 0 else e - bias
    if e == 0 and f == 0:
        return 0, 0, 0, eu
    m = f if e == 0 else f | (1 << fb)
    return s, m, eu - fb, eu


def to_int(s, m, x):
    v = m << (x + S)
    return -v if s else v


def trunc(v, L):
    q = 1 << (L + S)
    return -((-v) // q * q) if v < 0 else v // q * q


def rz32(v):
    """round toward zero into FP32 (subnormals kept), returned in the same integer units"""
    if v == 0:
        return 0
    a = abs(v)
    E = a.bit_length() - 1 - S           # leading exponent
    qexp = max(E - 23, -149)
    q = 1 << (qexp + S)
    r = a // q * q
    return -r if v < 0 else r


def f32_int(bits):
    s, m, x, _ = dec("f32", bits)
    return to_int(s, m, x) if m else 0


def main():
    path = sys.argv[1]
    fmt = path.rsplit("_", 1)[1].split(".")[0]
    z = np.load(path)
    a, b, c, d = z["a"], z["b"], z["c"], z["d"]
    rel = Counter()
    exact_ok = 0
    n = len(d)
    rows = []
    for t in range(n):
        terms, noms = [], []
        for k in range(a.shape[1]):
            sa, ma, xa, ea = dec(fmt, a[t, k])
            sb, mb, xb, eb = dec(fmt, b[t, k])
            if ma == 0 or mb == 0:
                continue
            terms.append(to_int(sa ^ sb, ma * mb, xa + xb))
            noms.append(ea + eb + 1)
        cv = f32_int(c[t])
        if cv:
            terms.append(cv)
            noms.append(abs(cv).bit_length() - 1 - S + 1)
        if not terms:
            continue
        emax = max(noms)
        g = f32_int(d[t])
        if rz32(sum(terms)) == g:
            exact_ok += 1
        ok = [L for L in range(emax - 60, emax - 10) if rz32(sum(trunc(v, L) for v in terms)) == g]
        lo, hi = (min(ok) - emax, max(ok) - emax) if ok else (None, None)
        rows.append((emax, lo, hi))
        rel[(lo, hi)] += 1
    print(f"{fmt}: {n} tiles, GPU == RZ32(exact) on {exact_ok}")
    print("feasible (L - emax) intervals (lo, hi) -> count:")
    for k, v in sorted(rel.items(), key=lambda kv: -kv[1])[:25]:
        print("  ", k, v)
    # does a fixed offset work for all tiles?  and an offset depending on emax?
    for off in range(-40, -18):
        good = sum(1 for e, lo, hi in rows if lo is not None and lo <= off <= hi)
        if good == len(rows):
            print("fixed offset fits all:", off)
    by_e = {}
    for e, lo, hi in rows:
        by_e.setdefault(e, []).append((lo, hi))
    print("per emax: (emax, n, intersection of feasible offsets)")
    for e in sorted(by_e):
        iv = by_e[e]
        if any(lo is None for lo, _ in iv):
            print("  ", e, len(iv), "infeasible for some")
            continue
        lo = max(l for l, _ in iv); hi = min(h for _, h in iv)
        print("  ", e, len(iv), (lo, hi), "abs L:", (e + lo, e + hi))


if __name__ == "__main__":
    main()
