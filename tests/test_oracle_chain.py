"""Pins for the chain-matmul oracle functions — -m "not gpu".

  * chain_fp32 (the paper's CPU FP32 baseline) vs a plain Python loop of numpy float32 scalar
    operations (IEEE binary32, one rounding per * and +, ascending k, A_{i+1} = D_i);
  * quantize_f32_bits (the D -> A conversion) vs numpy's float32 -> float16 cast (RNE, overflow to
    inf) and vs the scalar quantize pinned in test_oracle_formats.py.
"""
import numpy as np

import oracle as O


def test_chain_fp32_vs_python_float32_loop():
    rng = np.random.default_rng(3)
    count, n_steps = 3, 4
    A0 = rng.standard_normal((count, 16, 8)).astype(np.float32)
    Bs = rng.standard_normal((count, n_steps, 8, 8)).astype(np.float32)
    Ds = O.chain_fp32(A0, Bs)
    for c in range(count):
        a = A0[c].copy()
        for s in range(n_steps):
            d = np.zeros((16, 8), np.float32)
            for i in range(16):
                for j in range(8):
                    acc = np.float32(0)
                    for k in range(8):
                        acc = np.float32(acc + np.float32(a[i, k] * Bs[c, s, j, k]))
                    d[i, j] = acc
            assert np.array_equal(d.view(np.uint32), Ds[c, s].view(np.uint32))
            a = d


def test_quantize_f32_bits_vs_numpy_f16_and_scalar():
    rng = np.random.default_rng(4)
    x = np.concatenate([rng.standard_normal(20000) * 2.0 ** rng.integers(-30, 20, 20000),
                        [65504.0, 65519.99, 65520.0, 1e6, -1e6, 2.0 ** -25, 0.0, -0.0, np.inf, -np.inf]]).astype(np.float32)
    bits = x.view(np.uint32)
    f16 = O.quantize_f32_bits(bits, O.F16)
    assert np.array_equal(f16, x.astype(np.float16).view(np.uint16))
    for fmt in (O.BF16, O.TF32):
        q = O.quantize_f32_bits(bits[:3000], fmt)
        assert all(int(q[i]) == O.quantize(float(x[i]), fmt) for i in range(3000))

