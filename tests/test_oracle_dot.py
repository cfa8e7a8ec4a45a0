"""Pins for the oracle's exact dot product / GEMM / tiles (-m "not gpu").

Pinned against:
  * brute-force rational arithmetic (fractions.Fraction) on >= 10^4 tiny tiles with extreme
    exponent spread, rounded by an independent nearest-neighbour search (tests/fp_ref.py);
  * closed-form tie cases (tests/golden/rounding_cases.txt);
  * the closed form that FP16/BF16/TF32 pairwise products are exact in FP64;
  * numpy float64 dot within 1 FP32 ulp for normal-range data (library special case);
  * the paper's zero-error cells: with init_low inputs, the multiplication and inner-product
    probes equal the CPU FP32 result exactly;
  * textbook integer matmul (int64) + two's-complement wrap for INT8 (north_star).
"""
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
from fp_ref import rne_f32_bits, f32_from_bits

GOLD = os.path.join(os.path.dirname(__file__), "golden")
NP = {O.F16: np.uint16, O.BF16: np.uint16, O.TF32: np.uint32}


def _rand_bits(rng, fmt, n, lo_exp, hi_exp):
    """random finite values of fmt with exponents spread over [lo_exp, hi_exp)"""
    m = rng.random(n) + 1.0
    e = rng.integers(lo_exp, hi_exp, n)
    s = rng.choice([-1.0, 1.0], n)
    x = s * np.ldexp(m, e)
    z = rng.random(n) < 0.1
    x[z] = 0.0
    return np.array([O.quantize(v, fmt) for v in x.tolist()], dtype=NP[fmt])


def _frac(fmt, b):
    return Fraction(O.decode(fmt, int(b)))


@pytest.mark.parametrize("fmt,lo,hi", [(O.F16, -26, 16), (O.BF16, -130, 126), (O.TF32, -130, 126)])
def test_dot_vs_fraction_bruteforce(fmt, lo, hi):
    rng = np.random.default_rng(10 + fmt)
    ntile = 3400
    for t in range(ntile):
        K = int(rng.integers(1, 9))
        a = _rand_bits(rng, fmt, K, lo, hi)
        b = _rand_bits(rng, fmt, K, lo, hi)
        c = float(np.float32(rng.standard_normal() * 2.0 ** int(rng.integers(-140, 120))))
        if rng.random() < 0.1:
            c = 0.0
        cb = int(np.array([c], dtype=np.float32).view(np.uint32)[0])
        exact = Fraction(c) + sum(_frac(fmt, x) * _frac(fmt, y) for x, y in zip(a, b))
        got, absv = O.dot_fp(fmt, a, b, cb)
        want = rne_f32_bits(exact)
        if exact == 0:
            assert float(f32_from_bits(got)) == 0.0
        else:
            assert got == want, (t, K, hex(got), hex(want))
        abs_exact = abs(Fraction(c)) + sum(abs(_frac(fmt, x) * _frac(fmt, y)) for x, y in zip(a, b))
        assert Fraction(absv) <= abs_exact and (abs_exact == 0 or Fraction(absv) >= abs_exact * (1 - Fraction(1, 2 ** 50)))


def _rows(name):
    with open(os.path.join(GOLD, name)) as f:
        for ln in f:
            ln = ln.strip()
            if ln and not ln.startswith("#"):
                yield ln.split()


def _fp16_factor(p):
    """write an exact product p as a*b with a, b FP16 (p = m*2^e: a = m*2^(e//2), b = 2^(e-e//2))"""
    f = Fraction(p)
    sgn = -1 if f < 0 else 1
    f = abs(f)
    e = 0
    while f.denominator != 1:
        f *= 2
        e -= 1
    m = f.numerator
    while m % 2 == 0 and m > 1:
        m //= 2
        e += 1
    ea = e // 2
    return sgn * m * 2.0 ** ea, 2.0 ** (e - ea)


def test_closed_form_tie_table():
    """SURVEY §8(c) rounding cases, paper probe placement."""
    for name, c, prods, rne, rz, *cite in _rows("rounding_cases.txt"):
        plist = [eval(p) for p in prods.split(",")]
        a, b = zip(*[_fp16_factor(p) for p in plist])
        abits = np.array([O.quantize(x, O.F16) for x in a], dtype=np.uint16)
        bbits = np.array([O.quantize(x, O.F16) for x in b], dtype=np.uint16)
        for x, y, p in zip(abits, bbits, plist):
            assert O.decode(O.F16, int(x)) * O.decode(O.F16, int(y)) == p
        cb = int(np.array([float(eval(c))], dtype=np.float32).view(np.uint32)[0])
        got, _ = O.dot_fp(O.F16, abits, bbits, cb)
        assert float(f32_from_bits(got)) == float(eval(rne)), (name, cite)
        # RZ column is the exact+RZ model: M(Ki, inf, RZ, ., c-in-block)
        gz = O.model_dot(O.F16, abits, bbits, cb, Ki=16, g=16, p=-1, rz=True)
        assert float(f32_from_bits(gz)) == float(eval(rz)), (name, cite)


def test_fp32_overflow_and_subnormal_results():
    # sum rounding to inf: c = max-finite, product = 2^103 (exact tie, max-finite has odd last bit)
    cmax = int(np.array([np.finfo(np.float32).max], dtype=np.float32).view(np.uint32)[0])
    a = np.array([O.quantize(2.0 ** 52, O.BF16)], dtype=np.uint16)
    b = np.array([O.quantize(2.0 ** 51, O.BF16)], dtype=np.uint16)
    got, _ = O.dot_fp(O.BF16, a, b, cmax)
    assert got == 0x7F800000
    # FP32-subnormal exact result from normal BF16 operands: 2^-120 * 2^-30 = 2^-150 -> tie -> 0
    a = np.array([O.quantize(2.0 ** -120, O.BF16)], dtype=np.uint16)
    b = np.array([O.quantize(2.0 ** -30, O.BF16)], dtype=np.uint16)
    got, _ = O.dot_fp(O.BF16, a, b, 0)
    assert got == 0
    b3 = np.array([O.quantize(3 * 2.0 ** -30, O.BF16)], dtype=np.uint16)
    got, _ = O.dot_fp(O.BF16, a, b3, 0)          # 3*2^-150 -> 2^-148 (tie to even)
    assert got == 2


def test_products_exact_in_fp64_closed_form():
    """FP16/BF16/TF32 products have <= 22-bit significands: exact in FP64 (north_star)."""
    rng = np.random.default_rng(5)
    for fmt, lo, hi in [(O.F16, -24, 16), (O.BF16, -62, 62), (O.TF32, -62, 62)]:
        a = _rand_bits(rng, fmt, 4000, lo, hi)
        b = _rand_bits(rng, fmt, 4000, lo, hi)
        for x, y in zip(a.tolist(), b.tolist()):
            da, db = O.decode(fmt, x), O.decode(fmt, y)
            p = da * db
            assert Fraction(p) == Fraction(da) * Fraction(db)
            got, _ = O.dot_fp(fmt, np.array([x], NP[fmt]), np.array([y], NP[fmt]), 0)
            assert Fraction(float(f32_from_bits(got))) == Fraction(np.float32(p).item()) or p == 0


def test_vs_numpy_float64_within_one_ulp():
    rng = np.random.default_rng(6)
    M, N, K = 24, 20, 300
    A = rng.standard_normal((M, K)).astype(np.float16)
    B = rng.standard_normal((N, K)).astype(np.float16)
    C = rng.standard_normal((M, N)).astype(np.float32)
    out, absv = O.gemm_full(O.F16, A.view(np.uint16), B.view(np.uint16), C.view(np.uint32))
    D = out.view(np.float32).astype(np.float64)
    ref = A.astype(np.float64) @ B.astype(np.float64).T + C.astype(np.float64)
    ulp = np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)
    assert np.all(np.abs(D - ref) <= ulp + 1e-30)
    refabs = np.abs(A.astype(np.float64)) @ np.abs(B.astype(np.float64)).T + np.abs(C)
    assert np.allclose(absv, refabs, rtol=1e-12)


@pytest.mark.parametrize("fmt", [O.F16, O.BF16, O.TF32])
def test_paper_zero_error_cells(fmt):
    """init_low: multiplication and inner-product probes are exact w.r.t. CPU FP32
    (PAPER.md:923-924 BF16, 955-956 FP16, 996-997 TF32)."""
    rng = np.random.default_rng(7)
    for _ in range(500):
        x = rng.standard_normal(4)
        q = [O.decode(fmt, O.quantize(v, fmt)) for v in x]
        a0, b0, a1, b1 = q
        bits = lambda v: O.quantize(v, fmt)
        # multiplication probe d0 = a0*b0 (Fig. mul)
        got, _ = O.dot_fp(fmt, np.array([bits(a0)] + [0] * 15, NP[fmt]), np.array([bits(b0)] + [0] * 15, NP[fmt]), 0)
        assert float(f32_from_bits(got)) == float(np.float32(a0) * np.float32(b0))
        # inner-product probe d0 = a0*b0 + a1*b1: CPU FP32 result computed in binary32
        got, _ = O.dot_fp(fmt, np.array([bits(a0), bits(a1)] + [0] * 14, NP[fmt]),
                          np.array([bits(b0), bits(b1)] + [0] * 14, NP[fmt]), 0)
        cpu = np.float32(np.float32(a0) * np.float32(b0)) + np.float32(np.float32(a1) * np.float32(b1))
        # equal unless the binary32 add itself rounds (then within 1/2 ulp, paper reports 0.0 mean)
        assert abs(float(f32_from_bits(got)) - float(cpu)) <= float(np.spacing(np.float32(abs(cpu)))) / 2


def test_int8_textbook_and_wrap():
    rng = np.random.default_rng(8)
    M, N, K = 16, 12, 200
    A = rng.integers(-128, 128, (M, K)).astype(np.int8)
    B = rng.integers(-128, 128, (N, K)).astype(np.int8)
    C = rng.integers(-(1 << 31), 1 << 31, (M, N)).astype(np.int64).astype(np.int32)
    out, _ = O.gemm_full(O.S8, A, B, C)
    ref = (A.astype(np.int64) @ B.astype(np.int64).T + C.astype(np.int64))
    ref = ((ref + (1 << 31)) % (1 << 32) - (1 << 31)).astype(np.int32)
    assert np.array_equal(out.view(np.int32), ref)
    # crafted wrap cases
    assert O.dot_s8(np.array([1], np.int8), np.array([1], np.int8), (1 << 31) - 1) == -(1 << 31)
    K2 = 1 << 17
    a = np.full(K2, -128, np.int8)
    assert O.dot_s8(a, a, 0) == -(1 << 31)


def test_tiles_match_gemm_samples():
    rng = np.random.default_rng(9)
    count = 7
    A = rng.standard_normal((count, 16, 16)).astype(np.float16)
    B = rng.standard_normal((count, 8, 16)).astype(np.float16)
    C = rng.standard_normal((count, 16, 8)).astype(np.float32)
    D, _ = O.tiles(O.F16, 16, 8, 16, A.view(np.uint16), B.view(np.uint16), C.view(np.uint32))
    for t in range(count):
        out, _ = O.gemm_full(O.F16, A[t].view(np.uint16), B[t].view(np.uint16), C[t].view(np.uint32))
        assert np.array_equal(D[t], out)


def test_signed_zero():
    z = np.array([0x8000], np.uint16)   # -0 in FP16
    one = np.array([0x3C00], np.uint16)
    got, _ = O.dot_fp(O.F16, z, one, 0x80000000)   # (-0)(1) + (-0) = -0
    assert got == 0x80000000
    got, _ = O.dot_fp(O.F16, z, one, 0)            # (-0) + (+0) = +0
    assert got == 0
