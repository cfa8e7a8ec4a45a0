"""Pins for every branch of the C2 model family M(g, p, R, t, o, e) in oracle/models.c (-m "not gpu").

SURVEY.md §8(c) "Model family for the C2 classifier" defines the family; the classifier of
tests/test_gpu_numeric_probe.py searches all of it, so every branch must be pinned, not only the
ones the observed model uses (floor truncation, g < Ki, c_after with finite p
and emode 1 had no closed-form pin).

Two independent pins:
  1. closed forms derived by hand (tests/golden/model_branch_cases.txt, one row per branch, each
     chosen so the branch changes the result);
  2. a brute-force exact-rational re-statement of the family written from SURVEY §8(c) (and the
     emode definitions), evaluated with fractions.Fraction on random tiny tiles across the whole
     parameter space and compared bit for bit with the C oracle."""
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
from fp_ref import f32_bits_of, f32_from_bits, rne_f32_bits

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rows(name):
    with open(os.path.join(GOLD, name)) as f:
        for ln in f:
            ln = ln.strip()
            if ln and not ln.startswith("#"):
                yield ln.split()


def _f16(x):
    return O.quantize(float(x), O.F16)


def _pair(pr):
    """'a*b' -> (a, b); the factors may contain '**'"""
    a, b = pr.replace("**", "^").split("*")
    return eval(a.replace("^", "**")), eval(b.replace("^", "**"))


def _products(spec):
    """'16*[-0.5*0.5]' (sixteen copies) or '1*1;2**-12*2**-11' -> list of (a, b) exact values"""
    if spec.startswith("16*["):
        return [_pair(spec[4:-1])] * 16
    return [_pair(pr) for pr in spec.split(";")]


def test_model_branch_closed_forms():
    n = 0
    for name, Ki, g, p, R, t, o, em, c, prods, exp in _rows("model_branch_cases.txt"):
        Ki, g, p, em = int(Ki), int(g), int(p), int(em)
        pl = _products(prods)
        K = max(Ki, len(pl))
        a = np.array([_f16(x) for x, _ in pl] + [0] * (K - len(pl)), np.uint16)[None, :]
        b = np.array([_f16(y) for _, y in pl] + [0] * (K - len(pl)), np.uint16)[None, :]
        for (x, y), ab_, bb_ in zip(pl, a[0], b[0]):          # the factors are exact in FP16
            assert O.decode(O.F16, int(ab_)) == x and O.decode(O.F16, int(bb_)) == y, name
        cb = np.array([f32_bits_of(float(eval(c)))], np.uint32)
        assert float(f32_from_bits(int(cb[0]))) == float(Fraction(eval(c))), name
        out = O.model_batch(O.F16, a, b, cb, Ki=Ki, g=g, p=p, rz=(R == "RZ"), floor_mode=(t == "floor"),
                            c_after=(o == "c_after"), emode=em)
        assert float(f32_from_bits(int(out[0]))) == float(eval(exp)), (name, float(f32_from_bits(int(out[0]))))
        n += 1
    assert n == 15


# --------------------------------------------------------------------- brute-force re-statement
def _decode(fmt, bits):
    """(value, unbiased field exponent with subnormals at emin) of an input element"""
    if fmt == O.F16:
        e, f, fb, bias, sign = (bits >> 10) & 0x1F, bits & 0x3FF, 10, 15, bits >> 15
    else:                                                          # BF16
        e, f, fb, bias, sign = (bits >> 7) & 0xFF, bits & 0x7F, 7, 127, bits >> 15
    eu = (1 - bias) if e == 0 else e - bias
    mant = f if e == 0 else f | (1 << fb)
    v = Fraction(mant) * Fraction(2) ** (eu - fb)
    return (-v if sign else v), eu


def _f32_val(bits):
    return Fraction(float(f32_from_bits(bits)))


def _lead(x):
    ax = abs(x)
    e = ax.numerator.bit_length() - ax.denominator.bit_length()
    if Fraction(2) ** e > ax:
        e -= 1
    if Fraction(2) ** (e + 1) <= ax:
        e += 1
    return e


def _trunc(x, L, floor_mode):
    q = x / Fraction(2) ** L
    if floor_mode:
        k = q.numerator // q.denominator                           # floor
    else:
        k = abs(q).numerator // abs(q).denominator * (1 if q >= 0 else -1)
    return Fraction(k) * Fraction(2) ** L


def _rz_f32_bits(x):
    if x == 0:
        return 0
    sign = 1 if x < 0 else 0
    ax = abs(x)
    E = _lead(ax)
    q = max(E - 23, -149)
    k = (ax / Fraction(2) ** q)
    k = k.numerator // k.denominator
    v = Fraction(k) * Fraction(2) ** q
    if v >= Fraction(2) ** 128:
        v = Fraction((2 ** 24 - 1) * 2 ** 104)
    return f32_bits_of(float(v)) | (sign << 31)


def model_ref(fmt, a_bits, b_bits, c_bits, Ki, g, p, rz, floor_mode, c_after, emode):
    """blocks of g products within each Ki-instruction; addends {acc, products}
    (c_in) aligned to the largest leading exponent e_max, truncated to multiples of
    2^(e_max - 23 - p) (p = -1: none), summed exactly, rounded to FP32 (RNE / RZ).  c_after:
    products aligned among themselves, then R(acc + S).  emode 0: e_max from actual leading bits;
    >= 1: a product's nominal exponent is eu_a + eu_b + 1, the accumulator's its leading bit (1),
    that + 1 (2), or max(leading bit, field exponent) + 1 (3: a subnormal FP32 acc counts as -126)."""
    acc = int(c_bits)
    K = len(a_bits)
    for k0 in range(0, K, Ki):
        for kk in range(0, Ki, g):
            idx = [k0 + kk + j for j in range(g) if kk + j < Ki and k0 + kk + j < K]
            prods = []
            for i in idx:
                va, ea = _decode(fmt, int(a_bits[i]))
                vb, eb = _decode(fmt, int(b_bits[i]))
                prods.append((va * vb, ea + eb + 1))
            av = _f32_val(acc)
            terms = [(v, (_lead(v) if emode == 0 else nom)) for v, nom in prods if v != 0]
            if av != 0:
                le = _lead(av)
                if emode == 3:
                    fe = ((acc >> 23) & 0xFF) - 127 if (acc >> 23) & 0xFF else -126
                    le = max(le, fe)
                if emode >= 2:
                    le += 1
                acc_term = (av, le)
            else:
                acc_term = None
            group = terms + ([acc_term] if (acc_term and not c_after) else [])
            vals = [v for v, _ in group]
            if p >= 0 and group:
                L = max(le for _, le in group) - 23 - p
                vals = [_trunc(v, L, floor_mode) for v in vals]
            s = sum(vals, Fraction(0))
            if c_after:
                s += av
            elif acc_term is None:
                s += 0
            acc = _rz_f32_bits(s) if rz else rne_f32_bits(s)
    return acc


def _rand_bits(rng, fmt, n, lo, hi, p_zero=0.1, p_sub=0.05):
    out = []
    for _ in range(n):
        u = rng.random()
        if u < p_zero:
            out.append(0 if rng.random() < 0.5 else 0x8000)
            continue
        if u < p_zero + p_sub:
            m = int(rng.integers(1, 1 << (10 if fmt == O.F16 else 7)))
            out.append(m | (0x8000 if rng.random() < 0.5 else 0))
            continue
        x = float(rng.choice([-1, 1]) * (1 + rng.random()) * 2.0 ** int(rng.integers(lo, hi)))
        out.append(O.quantize(x, fmt))
    return np.array(out, np.uint16)


@pytest.mark.parametrize("fmt", [O.F16, O.BF16])
def test_model_family_equals_bruteforce(fmt):
    """the C model family == the Fraction re-statement on random tiles, every parameter branch"""
    rng = np.random.default_rng(77 + fmt)
    lo, hi = (-12, 8) if fmt == O.F16 else (-30, 20)
    n = 0
    for case in range(900):
        Ki = int(rng.choice([16, 8]))
        K = int(rng.choice([Ki, 2 * Ki]))
        g = int(rng.choice([x for x in (1, 2, 4, 8, 16) if x <= Ki]))
        p = int(rng.choice([-1, 0, 1, 3, 8]))
        rz, fl, ca = bool(rng.integers(2)), bool(rng.integers(2)), bool(rng.integers(2))
        em = int(rng.integers(4))
        a = _rand_bits(rng, fmt, K, lo, hi)
        b = _rand_bits(rng, fmt, K, lo, hi)
        r = rng.random()
        if r < 0.15:
            c = 0
        elif r < 0.3:                                             # FP32-subnormal accumulator
            c = int(rng.integers(1, 1 << 23)) | (int(rng.integers(2)) << 31)
        else:
            c = f32_bits_of(float(rng.choice([-1, 1]) * (1 + rng.random()) * 2.0 ** int(rng.integers(-20, 26))))
        if fmt == O.BF16 and r < 0.3 and case % 2:                  # push BF16 products into the subnormal range
            a = np.array([O.quantize(float(rng.choice([-1, 1]) * (1 + rng.random()) * 2.0 ** -70), fmt)
                          for _ in range(K)], np.uint16)
            b = np.array([O.quantize(float(rng.choice([-1, 1]) * (1 + rng.random()) * 2.0 ** -72), fmt)
                          for _ in range(K)], np.uint16)
        got = O.model_batch(fmt, a[None, :], b[None, :], np.array([c], np.uint32), Ki=Ki, g=g, p=p, rz=rz,
                            floor_mode=fl, c_after=ca, emode=em)[0]
        ref = model_ref(fmt, a, b, c, Ki, g, p, rz, fl, ca, em)
        assert int(got) == int(ref), dict(case=case, Ki=Ki, K=K, g=g, p=p, rz=rz, floor=fl, c_after=ca, emode=em,
                                          got=hex(int(got)), ref=hex(int(ref)))
        n += 1
    assert n == 900
