"""Pins for the oracle's 2:4 sparse helpers and the probe-model family (-m "not gpu").

Sparse: SPEC.md worked examples (tests/golden/sp24_pins.txt), decompress(compress(A)) = A
(SPEC.md:232,253), sparse oracle == dense oracle on expand(A) bitwise.
Models: the truncation discriminator table (tests/golden/truncation_cases.txt),
the special case "exact oracle = M(Ki, inf, RNE, c-in-block)", and seq32 == numpy binary32.
"""
import os

import numpy as np
import pytest
import torch

import oracle as O
import tcxgen
from fp_ref import f32_from_bits

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rows(name):
    with open(os.path.join(GOLD, name)) as f:
        for ln in f:
            ln = ln.strip()
            if ln and not ln.startswith("#"):
                yield ln.split()


def test_sp24_golden():
    n = 0
    for row in _rows("sp24_pins.txt"):
        if row[0] == "pair":
            i0, i1 = map(int, row[1].split(","))
            dense = np.zeros((1, 32), np.float16)
            dense[0, i0] = 1.0
            dense[0, i1] = 2.0
            vals, meta, bad = O.sp24_compress(dense.view(np.uint16))
            assert bad == -1
            assert meta[0, 0] & 0xF == int(row[2], 16)
            # the generator's packer agrees with the oracle's compress (shared definition)
            pi = tcxgen.PAIRS.index((i0, i1))
            m = tcxgen.sp24_canonical_meta(torch.full((1, 8), pi, dtype=torch.uint8))
            assert int(m[0, 0]) & 0xF == int(row[2], 16)
        elif row[0] == "group":
            g = [float(v) for v in row[1].split(",")]
            dense = np.zeros((1, 32), np.float16)
            dense[0, :4] = g
            vals, meta, bad = O.sp24_compress(dense.view(np.uint16))
            assert bad == -1
            assert [float(v) for v in vals.view(np.float16)[0, :2]] == [float(v) for v in row[3].split(",")]
            nib = int(meta[0, 0]) & 0xF
            assert (nib & 3, nib >> 2) == tuple(map(int, row[5].split(",")))
        elif row[0] in ("sp12", "sp12bad"):
            g = np.array([float(v) for v in row[1].split(",")], np.float32)
            dense = np.zeros((1, 32), np.float32)
            dense[0, :4] = g
            vals, meta, bad = O.sp12_compress(dense.view(np.uint32))
            if row[0] == "sp12bad":
                assert bad == 0
                n += 1
                continue
            assert bad == -1
            nib = int(meta[0, 0]) & 0xF
            i0, i1 = map(int, row[3].split(","))
            assert (nib & 3, nib >> 2) == (i0, i1)
            assert list(vals.view(np.float32)[0, :2]) == [g[i0], g[i1]]
        elif row[0] == "word":
            g = [float(v) for v in row[1].split(",")]
            dense = np.zeros((1, 32), np.float16)
            dense[0, :8] = g
            vals, meta, bad = O.sp24_compress(dense.view(np.uint16))
            assert bad == -1
            # groups 2..7 are all-zero -> padded (0,1) = 0x4 each
            assert int(meta[0, 0]) & 0xFF == int(row[2], 16)
        n += 1
    assert n == 15


def test_sp24_reject_and_roundtrip():
    rng = np.random.default_rng(11)
    M, K = 12, 64
    pairs = rng.integers(0, 6, (M, K // 4))
    dense = np.zeros((M, K), np.float16)
    for i in range(M):
        for g in range(K // 4):
            i0, i1 = tcxgen.PAIRS[pairs[i, g]]
            dense[i, 4 * g + i0] = rng.standard_normal() + 3
            dense[i, 4 * g + i1] = rng.standard_normal() - 3
    vals, meta, bad = O.sp24_compress(dense.view(np.uint16))
    assert bad == -1
    back = O.sp24_expand(vals, meta, K)
    assert np.array_equal(back, dense.view(np.uint16))
    # a 3-nonzero group is rejected, first violation in row-major order
    d2 = dense.copy()
    d2[5, 4 * 3: 4 * 3 + 4] = [1, 1, 1, 0]
    d2[7, 0:4] = [1, 1, 1, 1]
    _, _, bad = O.sp24_compress(d2.view(np.uint16))
    assert bad == 5 * (K // 4) + 3
    # -0 counts as zero, NaN as nonzero
    d3 = np.zeros((1, 32), np.float16)
    d3[0, :4] = [-0.0, np.nan, 1.0, -0.0]
    _, meta3, bad = O.sp24_compress(d3.view(np.uint16))
    assert bad == -1 and int(meta3[0, 0]) & 0xF == (1 | (2 << 2))


def test_sp12_roundtrip_and_first_violation():
    """TF32 1:2: expand(compress(A)) == A for one-nonzero-per-pair matrices (SPEC.md:232 analogue);
    the first pair with two nonzeros is reported in row-major order."""
    rng = np.random.default_rng(12)
    M, K = 9, 64
    dense = np.zeros((M, K), np.float32)
    pick = rng.integers(0, 2, (M, K // 2))
    keep = rng.random((M, K // 2)) < 0.9
    for i in range(M):
        for q in range(K // 2):
            if keep[i, q]:
                dense[i, 2 * q + pick[i, q]] = rng.standard_normal() + 5
    vals, meta, bad = O.sp12_compress(dense.view(np.uint32))
    assert bad == -1
    assert np.array_equal(O.sp24_expand(vals, meta, K), dense.view(np.uint32))
    nib = np.array([[(meta[i, g // 8] >> (4 * (g % 8))) & 0xF for g in range(K // 4)] for i in range(M)])
    assert np.all((nib & 3) <= 1) and np.all((nib >> 2) >= 2)
    d2 = dense.copy()
    d2[4, 10:12] = 1.0
    d2[6, 0:2] = 1.0
    _, _, bad = O.sp12_compress(d2.view(np.uint32))
    assert bad == 4 * (K // 4) + 10 // 4


def test_sparse_equals_dense_of_expanded():
    M, N, K = 16, 24, 128
    vals, meta = tcxgen.sp24_problem(M, K, seed=3)
    B = tcxgen.normal_matrix((N, K), "f16", 3, tcxgen.STREAM_B)
    v = vals.view(torch.int16).numpy().view(np.uint16)
    m = meta.numpy().view(np.uint32)
    dense = O.sp24_expand(v, m, K)
    # exactly 2 nonzeros per group, never +-0 among kept values
    nz = (dense.reshape(M, K // 4, 4) & 0x7FFF) != 0
    assert np.all(nz.sum(axis=2) == 2)
    # re-compress gives back the same canonical encoding
    v2, m2, bad = O.sp24_compress(dense)
    assert bad == -1 and np.array_equal(v2, v) and np.array_equal(m2, m)
    Bn = B.view(torch.int16).numpy().view(np.uint16)
    out_d, _ = O.gemm_full(O.F16, dense, Bn, None)
    # sparse oracle: only kept products (explicit 2:4 selection, exact zero skips)
    for i in range(M):
        for j in range(N):
            sel_a, sel_b = [], []
            for g in range(K // 4):
                nib = (m[i, g // 8] >> (4 * (g % 8))) & 0xF
                for s, idx in enumerate((nib & 3, nib >> 2)):
                    sel_a.append(v[i, 2 * g + s])
                    sel_b.append(Bn[j, 4 * g + idx])
            got, _ = O.dot_fp(O.F16, np.array(sel_a, np.uint16), np.array(sel_b, np.uint16), 0)
            assert got == out_d[i, j]


def _fp16_pair(p):
    from test_oracle_dot import _fp16_factor
    a, b = _fp16_factor(p)
    return O.quantize(a, O.F16), O.quantize(b, O.F16)


def test_truncation_discriminator_table():
    cols = [2, 3, 8, 11]
    for name, c, prods, *exp in _rows("truncation_cases.txt"):
        if prods.startswith("16*["):
            plist = [eval(prods[4:-1])] * 16
        else:
            plist = [eval(p) for p in prods.split(",")]
        ab = [_fp16_pair(p) for p in plist]
        a = np.array([x for x, _ in ab] + [0] * (16 - len(ab)), np.uint16)
        b = np.array([y for _, y in ab] + [0] * (16 - len(ab)), np.uint16)
        cb = int(np.array([float(eval(c))], np.float32).view(np.uint32)[0])
        for p, e in zip(cols, exp):
            got = O.model_dot(O.F16, a, b, cb, Ki=16, g=16, p=p, rz=True)
            assert float(f32_from_bits(got)) == float(eval(e)), (name, p)


@pytest.mark.parametrize("fmt,Ki", [(O.F16, 16), (O.BF16, 16), (O.TF32, 8)])
def test_exact_model_equals_oracle(fmt, Ki):
    rng = np.random.default_rng(12 + fmt)
    NPd = np.uint32 if fmt == O.TF32 else np.uint16
    for _ in range(2000):
        x = rng.standard_normal(2 * Ki) * 2.0 ** rng.integers(-8, 8, 2 * Ki)
        bits = np.array([O.quantize(v, fmt) for v in x], NPd)
        c = np.float32(rng.standard_normal() * 2.0 ** rng.integers(-5, 25))
        cb = int(np.array([c], np.float32).view(np.uint32)[0])
        a, b = bits[:Ki], bits[Ki:]
        ex, _ = O.dot_fp(fmt, a, b, cb)
        assert O.model_dot(fmt, a, b, cb, Ki=Ki, g=Ki, p=-1, rz=False) == ex
        # c-after with one block and infinite precision is the same single rounding
        assert O.model_dot(fmt, a, b, cb, Ki=Ki, g=Ki, p=-1, rz=False, c_after=True) == ex


def test_seq32_matches_numpy_binary32():
    rng = np.random.default_rng(13)
    for _ in range(200):
        a = rng.standard_normal(16).astype(np.float32)
        b = rng.standard_normal(16).astype(np.float32)
        c = np.float32(rng.standard_normal())
        acc = c
        for x, y in zip(a, b):
            acc = np.float32(acc + np.float32(x * y))
        assert O.seq32(a, b, float(c)) == float(acc)
        acc = np.float32(0)
        for x, y in zip(a, b):
            acc = np.float32(acc + np.float32(x * y))
        assert O.seq32(a, b, float(c), c_last=True) == float(np.float32(acc + c))


def _bf16_bits(x):
    return O.quantize(float(x), O.BF16)


def _emode_out(emode, a_vals, b_vals, c_val, p=3, Ki=16):
    a = np.array([_bf16_bits(x) for x in a_vals] + [0] * (Ki - len(a_vals)), np.uint16)[None, :]
    b = np.array([_bf16_bits(x) for x in b_vals] + [0] * (Ki - len(b_vals)), np.uint16)[None, :]
    cb = np.array([np.array([c_val], np.float32).view(np.uint32)[0]], np.uint32)
    out = O.model_batch(O.BF16, a, b, cb, Ki=Ki, g=Ki, p=p, rz=True, emode=emode)
    return float(f32_from_bits(out[0]))


def test_field_exponent_accumulator_closed_form():
    """emode 3 (the accumulator's exponent read from its exponent field): c = 2^-140 is an FP32
    subnormal, so its field exponent is emin = -126 (frame -125) while its leading bit is -140
    (frame -139).  Products: 2^-131 (a = 2^-65, b = 2^-66; nominal -130) and eight of 2^-152
    (2^-76 x 2^-76; nominal -151), whose sum 2^-149 is one FP32 subnormal ulp.
      * emode 2: e_max = -130 -> window 2^(-130-26) = 2^-156 keeps the 2^-152 products:
        2^-131 + 2^-140 + 2^-149 (RZ is exact on the 2^-149 grid);
      * emode 3: e_max = -125 (c) -> window 2^-151 truncates each 2^-152 product to 0:
        2^-131 + 2^-140."""
    a = [2.0 ** -65] + [2.0 ** -76] * 8
    b = [2.0 ** -66] + [2.0 ** -76] * 8
    c = 2.0 ** -140
    assert _emode_out(2, a, b, c) == 2.0 ** -131 + 2.0 ** -140 + 2.0 ** -149
    assert _emode_out(3, a, b, c) == 2.0 ** -131 + 2.0 ** -140
    # with a normal c the two readings coincide (field exponent == leading bit)
    assert _emode_out(3, a, b, 2.0 ** -120) == _emode_out(2, a, b, 2.0 ** -120)


@pytest.mark.parametrize("fmt,Ki", [(O.F16, 16), (O.BF16, 16), (O.TF32, 8)])
def test_field_exponent_equals_esum2_for_normal_c(fmt, Ki):
    """emode 3 differs from the pinned emode 2 only through a subnormal accumulator: identical on
    random tiles whose c (and every intermediate accumulator) is normal or zero."""
    rng = np.random.default_rng(31 + fmt)
    NPd = np.uint32 if fmt == O.TF32 else np.uint16
    n, K = 500, 2 * Ki
    A = np.array([[O.quantize(v, fmt) for v in rng.standard_normal(K) * 2.0 ** rng.integers(-6, 6, K)]
                  for _ in range(n)], NPd)
    B = np.array([[O.quantize(v, fmt) for v in rng.standard_normal(K) * 2.0 ** rng.integers(-6, 6, K)]
                  for _ in range(n)], NPd)
    C = (rng.standard_normal(n) * 2.0 ** rng.integers(-10, 10, n)).astype(np.float32).view(np.uint32)
    C[::7] = 0
    for p in (2, 3, 5):
        m2 = O.model_batch(fmt, A, B, C, Ki=Ki, g=Ki, p=p, rz=True, emode=2)
        m3 = O.model_batch(fmt, A, B, C, Ki=Ki, g=Ki, p=p, rz=True, emode=3)
        assert np.array_equal(m2, m3), p
