"""tcx_round_tf32 (include/tcx.h; DESIGN.md R-C1) on the GPU against the oracle's TF32 quantizer.

FP32 -> TF32 round-to-nearest-even: the oracle rounds the exact FP32 value to a
10-bit fraction (oracle.quantize_f32_bits, pinned in tests/test_oracle_formats.py against Fraction
brute force).  Crafted cases: exact ties with even and odd kept LSB, just above / below a tie,
carry out of the fraction into the exponent, max-finite -> +-inf, subnormals (ties among them
too), signed zeros, then NaN / inf pass-through (bit-identical, the header's definition) and the
in-place form.  Bit-exact."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2206_02874_b200 as tcx

pytestmark = pytest.mark.gpu


def _crafted():
    v = []
    for e in (0x3F8, 0x010, 0x7F0, 0x7F7, 0x001, 0x080):           # exponent-field bytes << 3: various binades
        base = e << 20
        for frac in (0x0000, 0x1000, 0x3000, 0x1001, 0x0FFF, 0x2FFF, 0x3001, 0x7FFFFF, 0x7FF000, 0x7FEFFF,
                     0x7FF001, 0x5000, 0x4FFF, 0x6000, 0x1FFF):
            v.append((base & 0x7F800000) | (frac & 0x7FFFFF))
    v += [0x7F7FFFFF, 0x7F7FF000, 0x7F7FEFFF, 0x7F7FF001,            # max finite -> inf, just below
          0x00000001, 0x00001000, 0x00003000, 0x00001001, 0x00002FFF, 0x007FFFFF, 0x007FF000,   # subnormals
          0x00000000]
    v += [x | 0x80000000 for x in v]                                 # negatives (-0 included)
    return np.array(v, np.uint32)


def _specials():
    return np.array([0x7F800000, 0xFF800000, 0x7FC00000, 0xFFC00000, 0x7F800001, 0x7FBFFFFF, 0x7FFFFFFF,
                     0xFF800FFF], np.uint32)


def test_round_tf32_matches_oracle():
    rng = np.random.default_rng(5)
    rand = rng.integers(0, 2 ** 32, 200_000, dtype=np.uint64).astype(np.uint32)
    rand = rand[(rand & 0x7F800000) != 0x7F800000]                    # finite random bit patterns
    x = np.concatenate([_crafted(), rand])
    xt = torch.from_numpy(x.view(np.int32)).cuda().view(torch.float32)
    out = tcx.round_tf32(xt)
    torch.cuda.synchronize()
    got = out.cpu().view(torch.int32).numpy().view(np.uint32)
    ref = O.quantize_f32_bits(x, O.TF32).astype(np.uint32)
    bad = np.nonzero(got != ref)[0]
    assert bad.size == 0, [(hex(x[i]), hex(got[i]), hex(ref[i])) for i in bad[:8]]
    # the defining property, restated on the crafted set: low 13 bits clear
    assert np.all(got & 0x1FFF == 0)
    # max finite rounds up to inf; the largest value that rounds down stays finite
    i = int(np.nonzero(x == 0x7F7FFFFF)[0][0])
    assert got[i] == 0x7F800000
    i = int(np.nonzero(x == 0x7F7FEFFF)[0][0])
    assert got[i] == 0x7F7FE000


def test_round_tf32_specials_and_in_place():
    s = _specials()
    t = torch.from_numpy(s.view(np.int32)).cuda().view(torch.float32)
    out = tcx.round_tf32(t)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().view(torch.int32).numpy().view(np.uint32), s)     # NaN / inf unchanged
    x = _crafted()
    t = torch.from_numpy(x.view(np.int32).copy()).cuda().view(torch.float32)
    r = tcx.round_tf32(t, out=t)                                                      # in = out
    torch.cuda.synchronize()
    assert r.data_ptr() == t.data_ptr()
    assert np.array_equal(t.cpu().view(torch.int32).numpy().view(np.uint32),
                          O.quantize_f32_bits(x, O.TF32).astype(np.uint32))


@pytest.mark.parametrize("n", [1, 255, 257, 148 * 32 * 256 + 3])
def test_round_tf32_sizes(n):
    """ragged sizes and more elements than the grid-stride launch covers in one pass"""
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n).astype(np.float32)
    t = torch.from_numpy(x).cuda()
    out = tcx.round_tf32(t)
    torch.cuda.synchronize()
    ref = O.quantize_f32_bits(x.view(np.uint32), O.TF32).astype(np.uint32)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), ref)
