"""Pins for the oracle's format codec (quantize / decode), -m "not gpu".

Pinned against: SPEC worked examples and SURVEY closed forms (tests/golden/quantize_pins.txt),
numpy's own IEEE conversions (float16 / float32: correctly rounded library routines),
exhaustive 2^16 round trips, and brute-force Fraction rounding for BF16/TF32.
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
from fp_ref import rne_bits_generic

GOLD = os.path.join(os.path.dirname(__file__), "golden")
FMT = {"f16": O.F16, "bf16": O.BF16, "tf32": O.TF32, "f32": O.F32}


def _rows(name):
    with open(os.path.join(GOLD, name)) as f:
        for ln in f:
            ln = ln.strip()
            if ln and not ln.startswith("#"):
                yield ln.split()


def test_quantize_golden_pins():
    n = 0
    for fmt, x, exp, *cite in _rows("quantize_pins.txt"):
        xv = eval(x)  # exact python expressions from the fixture
        got = O.decode(FMT[fmt], O.quantize(float(xv), FMT[fmt]))
        if exp == "inf":
            assert math.isinf(got) and got > 0, (fmt, x, got, cite)
        else:
            assert got == float(eval(exp)), (fmt, x, got, exp, cite)
        n += 1
    assert n >= 14


def test_f16_exhaustive_roundtrip_and_numpy_decode():
    bits = np.arange(1 << 16, dtype=np.uint32)
    ref = bits.astype(np.uint16).view(np.float16).astype(np.float64)
    L = O.lib()
    for b, r in zip(bits.tolist(), ref.tolist()):
        d = L.tcxref_decode(O.F16, b)
        if math.isnan(r):
            assert math.isnan(d)
            continue
        assert d == r and math.copysign(1, d) == math.copysign(1, r), hex(b)
        assert L.tcxref_quantize(d, O.F16, 0) == b, hex(b)


def test_bf16_exhaustive_roundtrip_and_bitshift_decode():
    bits = np.arange(1 << 16, dtype=np.uint32)
    ref = (bits << 16).view(np.float32).astype(np.float64)   # BF16 = top half of FP32
    L = O.lib()
    for b, r in zip(bits.tolist(), ref.tolist()):
        d = L.tcxref_decode(O.BF16, b)
        if math.isnan(r):
            assert math.isnan(d)
            continue
        assert d == r and math.copysign(1, d) == math.copysign(1, r), hex(b)
        assert L.tcxref_quantize(d, O.BF16, 0) == b, hex(b)


def _random_doubles(rng, n, lo_exp, hi_exp):
    m = rng.random(n) + 1.0
    e = rng.integers(lo_exp, hi_exp, n)
    s = rng.choice([-1.0, 1.0], n)
    return s * np.ldexp(m, e)


def test_quantize_f16_f32_vs_numpy():
    rng = np.random.default_rng(1)
    L = O.lib()
    xs = np.concatenate([_random_doubles(rng, 20000, -30, 18),
                         # exact ties at FP16 precision
                         np.ldexp(rng.integers(1 << 11, 1 << 12, 2000) * 2 + 1, -12).astype(np.float64)])
    ref16 = xs.astype(np.float16).view(np.uint16)
    for x, r in zip(xs.tolist(), ref16.tolist()):
        assert L.tcxref_quantize(x, O.F16, 0) == r, x
    xs32 = _random_doubles(rng, 20000, -160, 130)
    ref32 = xs32.astype(np.float32).view(np.uint32)
    for x, r in zip(xs32.tolist(), ref32.tolist()):
        assert L.tcxref_quantize(x, O.F32, 0) == r, x


@pytest.mark.parametrize("fmt,P,emin,emax", [(O.BF16, 8, -126, 127), (O.TF32, 11, -126, 127)])
def test_quantize_bf16_tf32_vs_fraction(fmt, P, emin, emax):
    rng = np.random.default_rng(2 + fmt)
    xs = np.concatenate([_random_doubles(rng, 3000, -140, 129),
                         # ties at target precision
                         np.ldexp((rng.integers(1 << (P - 1), 1 << P, 500) * 2 + 1).astype(np.float64), -P)])
    for x in xs.tolist():
        got = O.decode(fmt, O.quantize(x, fmt))
        r = rne_bits_generic(Fraction(x), P, emin, emax)
        if r == "inf":
            assert math.isinf(got)
        elif r == "zero":
            assert got == 0
        else:
            s, kept, q = r
            assert Fraction(got) == (-1 if s else 1) * kept * Fraction(2) ** q, x


def test_tf32_bits_low13_zero():
    rng = np.random.default_rng(3)
    for x in rng.standard_normal(1000).tolist():
        assert O.quantize(x, O.TF32) & 0x1FFF == 0


def test_round_toward_zero_bound():
    """|decode(quantize(x, RZ))| <= |x|"""
    rng = np.random.default_rng(4)
    for x in _random_doubles(rng, 3000, -20, 20).tolist():
        for fmt in (O.F16, O.BF16, O.TF32, O.F32):
            assert abs(O.decode(fmt, O.quantize(x, fmt, rz=True))) <= abs(x)


def test_tf32_convert_modes_closed_form():
    """TF32 input conversions (reading C1): ulp(1) in TF32 = 2^-10; 1 + 2^-11 is a tie."""
    import struct
    def b(x):
        return np.array([struct.unpack("<I", struct.pack("<f", x))[0]], np.uint32)
    def f(u):
        return struct.unpack("<f", struct.pack("<I", int(u[0])))[0]
    tie, above, below = 1 + 2.0 ** -11, 1 + 2.0 ** -11 + 2.0 ** -20, 1 + 2.0 ** -11 - 2.0 ** -20
    odd_tie = 1 + 2.0 ** -10 + 2.0 ** -11
    assert f(O.tf32_convert(b(tie), "rz")) == 1.0
    assert f(O.tf32_convert(b(tie), "rne")) == 1.0
    assert f(O.tf32_convert(b(tie), "rna")) == 1 + 2.0 ** -10
    assert f(O.tf32_convert(b(odd_tie), "rne")) == 1 + 2.0 ** -9
    assert f(O.tf32_convert(b(above), "rz")) == 1.0 and f(O.tf32_convert(b(above), "rne")) == 1 + 2.0 ** -10
    assert f(O.tf32_convert(b(below), "rna")) == 1.0
    assert f(O.tf32_convert(b(-tie), "rna")) == -(1 + 2.0 ** -10)
    assert f(O.tf32_convert(b(0.7), "fp32")) == np.float32(0.7)
