"""Independent brute-force helpers for pinning the oracle (tests only).

Nothing here shares code with oracle/ or the product: exact rational arithmetic with
fractions.Fraction, numpy's own float conversions, and nearest-neighbour searches.
"""
from fractions import Fraction

import numpy as np

F32_MAX = Fraction((2 ** 24 - 1) * 2 ** 104)
F32_OVF = Fraction(2 ** 128 - 2 ** 103)        # >= this rounds to inf under RNE


def f32_bits_of(x: float) -> int:
    return int(np.array([x], dtype=np.float32).view(np.uint32)[0])


def f32_from_bits(b: int) -> np.float32:
    return np.array([b & 0xFFFFFFFF], dtype=np.uint32).view(np.float32)[0]


def rne_f32_bits(x: Fraction) -> int:
    """RNE of an exact rational into binary32, by nearest-neighbour search with exact
    comparisons (ties to the even significand)."""
    if x == 0:
        return 0
    sign = 1 if x < 0 else 0
    ax = -x if x < 0 else x
    if ax >= F32_OVF:
        return (sign << 31) | 0x7F800000
    guess = np.float32(float(ax))                     # within an ulp or two
    cands = set()
    g = guess
    for _ in range(3):
        g = np.nextafter(g, np.float32(0))
    for _ in range(7):
        if np.isfinite(g):
            cands.add(f32_bits_of(float(g)))
        g = np.nextafter(g, np.float32(np.inf))
    best = None
    for b in sorted(cands):
        v = Fraction(float(f32_from_bits(b)))
        d = abs(v - ax)
        key = (d, b & 1)                               # prefer smaller distance, then even
        if best is None or key < best[0]:
            best = (key, b)
    return best[1] | (sign << 31)


def rne_bits_generic(x: Fraction, P: int, emin: int, emax: int):
    """RNE of x into a binary format with P significand bits: returns (sign, kept, qexp) or
    'inf' / 'zero'.  Brute force with Fractions (independent of the oracle's bigint code)."""
    if x == 0:
        return "zero"
    sign = 1 if x < 0 else 0
    ax = abs(x)
    E = 0
    while Fraction(2) ** E > ax:
        E -= 1
    while Fraction(2) ** (E + 1) <= ax:
        E += 1
    qexp = max(E - (P - 1), emin - (P - 1))
    scaled = ax / Fraction(2) ** qexp
    fl = scaled.numerator // scaled.denominator
    rem = scaled - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    if fl == 2 ** P:
        fl //= 2
        qexp += 1
    if fl == 0:
        return "zero"
    if fl >= 2 ** (P - 1) and qexp + P - 1 > emax:
        return "inf"
    return sign, fl, qexp


F16_OVF = Fraction(65504 + 16)                 # >= this rounds to inf under RNE (65504 has an odd significand)


def f16_bits_of(x: float) -> int:
    return int(np.array([x], dtype=np.float16).view(np.uint16)[0])


def f16_from_bits(b: int) -> np.float16:
    return np.array([b & 0xFFFF], dtype=np.uint16).view(np.float16)[0]


def rne_f16_bits(x: Fraction, rz: bool = False) -> int:
    """RNE (or round-toward-zero) of an exact rational into binary16 by nearest-neighbour search
    over numpy float16 candidates, with exact Fraction comparisons."""
    if x == 0:
        return 0
    sign = 1 if x < 0 else 0
    ax = -x if x < 0 else x
    if not rz and ax >= F16_OVF:
        return (sign << 15) | 0x7C00
    if rz and ax >= Fraction(65504):
        return (sign << 15) | 0x7BFF
    g = np.float16(min(float(ax), 65504.0))
    for _ in range(3):
        g = np.nextafter(g, np.float16(0))
    cands = []
    for _ in range(7):
        if np.isfinite(g):
            cands.append(f16_bits_of(float(g)))
        g = np.nextafter(g, np.float16(np.inf))
    best = None
    for b in sorted(set(cands)):
        v = Fraction(float(f16_from_bits(b)))
        if rz:
            if v <= ax and (best is None or v > best[0]):
                best = (v, b)
        else:
            key = (abs(v - ax), b & 1)
            if best is None or key < best[0]:
                best = (key, b)
    return best[1] | (sign << 15)
