"""Pins for the oracle's FP16-accumulate path (C and D in FP16; the mma f16.f16.f16.f16 variant of
PAPER.md:428-429, whose numerics PAPER.md:962-982 profiles) — -m "not gpu".

The oracle's reading (DESIGN.md R-F16): D = RNE_fp16(c + sum_k a_k b_k), every product and the
whole sum exact, ONE rounding into FP16 ("the hardware conducts the computation in
high-precision and only converts the final result to low-precision FP16 in the end").

Pinned against (none of it the oracle retyped):
  * brute-force rational arithmetic (fractions.Fraction) on thousands of tiny tiles, rounded into
    FP16 by an independent nearest-neighbour search over numpy float16 values (tests/fp_ref.py);
  * closed-form FP16 tie / overflow cases (ulp(2048) = 2; max-finite 65504 has an odd significand);
  * the paper's zero-error cells of Table FP16-FP16-numeric-profiling: with FP16
    init, d0 = a0*b0 equals the CPU FP32 result converted to FP16 (numpy float32 -> float16), and so
    do the inner-product / accumulation probes whenever the CPU FP32 sum is itself exact.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
from fp_ref import rne_f16_bits


def _f16(x):
    return np.array(x, dtype=np.float16).view(np.uint16)


def _fr(b):
    return Fraction(float(np.array([b], dtype=np.uint16).view(np.float16)[0]))


def _rand_f16(rng, n, lo, hi):
    m = rng.random(n) + 1.0
    e = rng.integers(lo, hi, n)
    s = rng.choice([-1.0, 1.0], n)
    x = (s * np.ldexp(m, e)).astype(np.float16)          # numpy RNE into FP16 (the generator's job)
    x[rng.random(n) < 0.1] = 0
    return x.view(np.uint16)


@pytest.mark.parametrize("rz", [False, True])
def test_fp16_out_vs_fraction_bruteforce(rz):
    rng = np.random.default_rng(77 + rz)
    for t in range(3000):
        K = int(rng.integers(1, 17))
        a = _rand_f16(rng, K, -14, 6)
        b = _rand_f16(rng, K, -14, 6)
        c = _rand_f16(rng, 1, -20, 14)[0]
        exact = _fr(c) + sum(_fr(x) * _fr(y) for x, y in zip(a, b))
        got, absv = O.dot_fp(O.F16, a, b, int(c), c_fmt=O.F16, out_fmt=O.F16, rz=rz)
        if exact == 0:
            assert got & 0x7FFF == 0
            continue
        assert got == rne_f16_bits(exact, rz=rz), (t, K, hex(got))
        abs_exact = abs(_fr(c)) + sum(abs(_fr(x) * _fr(y)) for x, y in zip(a, b))
        assert abs(Fraction(absv) - abs_exact) <= abs_exact * Fraction(1, 2 ** 50)


@pytest.mark.parametrize("c,prods,rne,rz", [
    (2048.0, [1.0], 2048.0, 2048.0),        # tie at ulp 2 -> even
    (2050.0, [1.0], 2052.0, 2050.0),        # tie, odd neighbour -> up (RNE), down (RZ)
    (2048.0, [1.5], 2050.0, 2048.0),        # above half ulp
    (-2048.0, [-1.0], -2048.0, -2048.0),    # negative tie
    (65504.0, [8.0, 8.0], float("inf"), 65504.0),   # exactly half an ulp above max-finite
    (65504.0, [8.0, 7.5], 65504.0, 65504.0),        # just below the overflow threshold
    (1.0, [2.0 ** -11], 1.0, 1.0),          # tie at 1: ulp(1) = 2^-10
    (1.0, [2.0 ** -11, 2.0 ** -24], 1.0 + 2 ** -10, 1.0),
])
def test_fp16_closed_form_rounding(c, prods, rne, rz):
    # products p = p * 1.0 exactly in FP16
    a = _f16(prods); b = _f16([1.0] * len(prods))
    cb = int(_f16([c])[0])
    for mode, want in ((False, rne), (True, rz)):
        got, _ = O.dot_fp(O.F16, a, b, cb, c_fmt=O.F16, out_fmt=O.F16, rz=mode)
        assert float(np.array([got], np.uint16).view(np.float16)[0]) == want, (c, prods, mode, hex(got))


def test_paper_zero_error_cells_fp16_cd():
    """Table FP16-FP16-numeric-profiling, CPU_FP32cvtFP16 / init_FP16 column = 0.00."""
    rng = np.random.default_rng(0)
    n = 4000
    a = rng.standard_normal((n, 2)).astype(np.float16)
    b = rng.standard_normal((n, 2)).astype(np.float16)
    c = rng.standard_normal(n).astype(np.float16)
    checked = 0
    for i in range(n):
        # multiplication: d0 = a0 * b0 (product exact in FP32) -> FP32 then FP16 on the CPU
        cpu = np.float16(np.float32(a[i, 0]) * np.float32(b[i, 0]))
        got, _ = O.dot_fp(O.F16, a[i, :1].view(np.uint16), b[i, :1].view(np.uint16), 0, O.F16, O.F16)
        assert got == int(np.array([cpu]).view(np.uint16)[0])
        # inner product and accumulation: equal to CPU FP32->FP16 whenever the FP32 sum is exact
        for K, cc in ((2, np.float16(0)), (1, c[i])):
            s32 = np.float32(np.float32(a[i, 0]) * np.float32(b[i, 0]) + (np.float32(a[i, 1]) * np.float32(b[i, 1]) if K == 2 else np.float32(cc)))
            exact = Fraction(float(a[i, 0])) * Fraction(float(b[i, 0])) + (
                Fraction(float(a[i, 1])) * Fraction(float(b[i, 1])) if K == 2 else Fraction(float(cc)))
            if Fraction(float(s32)) != exact:
                continue
            got, _ = O.dot_fp(O.F16, a[i, :K].view(np.uint16), b[i, :K].view(np.uint16),
                              int(np.array([cc]).view(np.uint16)[0]), O.F16, O.F16)
            assert got == int(np.array([np.float16(s32)]).view(np.uint16)[0])
            checked += 1
    assert checked > n          # most FP32 sums of two FP16 products are exact


def test_tiles_fp16_cd_matches_dot():
    rng = np.random.default_rng(5)
    count = 16
    A = rng.standard_normal((count, 16, 16)).astype(np.float16).view(np.uint16)
    B = rng.standard_normal((count, 8, 16)).astype(np.float16).view(np.uint16)
    C = rng.standard_normal((count, 16, 8)).astype(np.float16).view(np.uint16)
    D, absv = O.tiles(O.F16, 16, 8, 16, A, B, C, cd=O.F16)
    for t in range(count):
        for i in range(16):
            for j in range(8):
                want, _ = O.dot_fp(O.F16, A[t, i], B[t, j], int(C[t, i, j]), O.F16, O.F16)
                assert D[t, i, j] == want


@pytest.mark.parametrize("p", [-1, 3])
def test_model_fp16_acc_reduces_to_exact_and_rz(p):
    """M(g = Ki, p = inf, RNE) with an FP16 accumulator IS the FP16 oracle (SURVEY §8(c) special
    case); with RZ it is the exact sum rounded toward zero.  p = 3 is checked against the
    Fraction truncation model on the same inputs."""
    rng = np.random.default_rng(9)
    n = 2000
    a = rng.standard_normal((n, 16)).astype(np.float16).view(np.uint16)
    b = rng.standard_normal((n, 16)).astype(np.float16).view(np.uint16)
    c = rng.standard_normal(n).astype(np.float16).view(np.uint16).astype(np.uint32)
    for rz in (False, True):
        out = O.model_batch(O.F16, a, b, c, 16, 16, p, rz, emode=0, acc_fmt=O.F16)
        for i in range(0, n, 7):
            terms = [_fr(c[i])] + [_fr(x) * _fr(y) for x, y in zip(a[i], b[i])]
            if p >= 0:
                # exact leading-bit exponent of the largest addend
                big = max(map(abs, terms))
                e = 0
                while Fraction(2) ** e > big:
                    e -= 1
                while Fraction(2) ** (e + 1) <= big:
                    e += 1
                q = Fraction(2) ** (e - 10 - p)
                trunc = []
                for t in terms:
                    k = abs(t) / q
                    k = k.numerator // k.denominator
                    trunc.append((1 if t >= 0 else -1) * k * q)
                terms = trunc
            exact = sum(terms)
            want = 0 if exact == 0 else rne_f16_bits(exact, rz=rz)
            if exact == 0:
                assert out[i] & 0x7FFF == 0
            else:
                assert out[i] == want, (i, rz, hex(out[i]), hex(want))


def test_gemm_samples_fp16_cd_integer_exact():
    """integer-valued FP16 GEMM with |sums| < 2048: the FP16 result is exact, so it must equal
    numpy's exact float64 matmul cast to float16 (independent of the oracle's rounding code)."""
    rng = np.random.default_rng(21)
    M, N, K = 24, 20, 64
    A = rng.integers(-3, 4, (M, K)).astype(np.float16)
    B = rng.integers(-3, 4, (N, K)).astype(np.float16)
    C = rng.integers(-500, 500, (M, N)).astype(np.float16)
    ii, jj = np.meshgrid(np.arange(M), np.arange(N), indexing="ij")
    out, _ = O.gemm_samples(O.F16, A.view(np.uint16), B.view(np.uint16), C.view(np.uint16), ii.ravel(), jj.ravel(),
                            cd=O.F16)
    ref = (A.astype(np.float64) @ B.astype(np.float64).T + C.astype(np.float64)).astype(np.float16)
    assert np.array_equal(out.astype(np.uint16).reshape(M, N), ref.view(np.uint16))


def _model16(a_vals, b_vals, c, p, rz, win):
    a = _f16(a_vals)[None, :]
    b = _f16(b_vals)[None, :]
    cb = np.array([int(_f16([c])[0])], np.uint32)
    out = O.model_batch(O.F16, a, b, cb, Ki=len(a_vals), g=len(a_vals), p=p, rz=rz, emode=2, acc_fmt=O.F16,
                        win_fmt=win)
    return float(np.array([out[0]], np.uint16).view(np.float16)[0])


def test_fp32_window_single_rounding_closed_form():
    """M16 with the FP32 truncation window (win_fmt = FP32): c = 1, products 2^-11 and 2^-25.
    Exact sum 1 + 2^-11 + 2^-25 lies above FP16's tie at 1 + 2^-11 -> RNE up to 1 + 2^-10.
      * window p = 3 (bits down to 2^(1-23-3) = 2^-25, c's esum2 frame is 2^1) keeps 2^-25 -> one
        RNE into FP16 rounds up (the single-rounding model);
      * p = 2 drops 2^-25 -> an exact tie -> even -> 1.0;
      * the two-stage reading (FP32 RZ first) would land on the tie as well: 1.0 — which is what
        separates the two readings."""
    a, b = [2.0 ** -5, 2.0 ** -12], [2.0 ** -6, 2.0 ** -13]      # products 2^-11, 2^-25 exact in FP16 inputs
    assert _model16(a, b, 1.0, p=3, rz=False, win=O.F32) == 1.0 + 2 ** -10
    assert _model16(a, b, 1.0, p=2, rz=False, win=O.F32) == 1.0
    assert _model16(a, b, 1.0, p=3, rz=True, win=O.F32) == 1.0
    # the FP16-window family at p = 3 truncates at 2^(1-10-3) = 2^-12: both small products' bits
    # below it vanish (2^-11 survives) -> tie -> 1.0
    assert _model16(a, b, 1.0, p=3, rz=False, win=O.F16) == 1.0


def test_fp32_window_wide_p_is_exact_rne16():
    """with a window wider than any product/c spread (p = 60) nothing is truncated: the model is one
    RNE of the exact sum into FP16 — the pinned exact oracle (dot_fp)."""
    rng = np.random.default_rng(5)
    n, K = 400, 16
    A = np.stack([_rand_f16(rng, K, -8, 4) for _ in range(n)])
    B = np.stack([_rand_f16(rng, K, -8, 4) for _ in range(n)])
    C = np.array([_rand_f16(rng, 1, -6, 6)[0] for _ in range(n)], np.uint32)
    got = O.model_batch(O.F16, A, B, C, Ki=16, g=16, p=60, rz=False, emode=2, acc_fmt=O.F16, win_fmt=O.F32)
    for i in range(n):
        want, _ = O.dot_fp(O.F16, A[i], B[i], int(C[i]), c_fmt=O.F16, out_fmt=O.F16)
        assert got[i] == want, i
