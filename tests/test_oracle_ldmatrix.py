"""Pins for oracle.ldmatrix — -m "not gpu".

  * special case = the mma operand layout ("the data layout eventually fetched to the
    Register File matches arrangement of the inputs to the Tensor Cores mma"): ldmatrix.x4 of a
    16 x 16 A tile with lane l addressing row l % 16, column block 8 (l // 16) yields exactly the
    m16n8k16 A fragments a0..a3 (rows g / g+8, k pairs 2t / 2t+8; g = l/4, t = l%4), written here
    from the mma fragment definition, not from the oracle's ldmatrix code;
  * .trans of an 8 x 8 matrix = the non-trans load of its transpose;
  * Table ldmatrix-ld.shared: N x 128 bytes per warp, N x 4 bytes per thread,
    every element of the N matrices delivered exactly once;
  * lanes >= 8N do not matter (Fig. func_ldmatrix caption).
"""
import numpy as np
import pytest

import oracle as O


def test_x4_is_the_mma_a_fragment():
    rng = np.random.default_rng(1)
    A = rng.integers(0, 1 << 16, (16, 16), dtype=np.uint32).astype(np.uint16)
    smem = np.zeros(512, np.uint16)
    smem[:256] = A.ravel()
    row_elem = np.array([16 * (l % 16) + 8 * (l // 16) for l in range(32)])
    got = O.ldmatrix(4, False, smem, row_elem)
    for l in range(32):
        g, t = l // 4, l % 4
        want = [(g, 2 * t), (g + 8, 2 * t), (g, 2 * t + 8), (g + 8, 2 * t + 8)]      # a0, a1, a2, a3
        for j, (r, c) in enumerate(want):
            assert got[l, j] == int(A[r, c]) | (int(A[r, c + 1]) << 16)


@pytest.mark.parametrize("num", [1, 2, 4])
def test_trans_is_load_of_transpose_and_every_element_once(num):
    rng = np.random.default_rng(num)
    mats = rng.integers(0, 1 << 16, (num, 8, 8), dtype=np.uint32).astype(np.uint16)
    smem = np.zeros(512, np.uint16)
    smemT = np.zeros(512, np.uint16)
    for j in range(num):
        smem[64 * j: 64 * j + 64] = mats[j].ravel()
        smemT[64 * j: 64 * j + 64] = mats[j].T.ravel()
    row_elem = np.array([64 * (l // 8) + 8 * (l % 8) if l < 8 * num else 0 for l in range(32)])
    a = O.ldmatrix(num, True, smem, row_elem)
    b = O.ldmatrix(num, False, smemT, row_elem)
    assert np.array_equal(a, b)
    assert a.shape == (32, num) and a.nbytes == 128 * num                      # 128 N bytes per warp
    halves = np.concatenate([(a & 0xFFFF).ravel(), (a >> 16).ravel()]).astype(np.uint16)
    assert sorted(halves.tolist()) == sorted(mats.ravel().tolist())            # each element once
    # lanes >= 8N are ignored
    row2 = row_elem.copy()
    row2[8 * num:] = 448
    assert np.array_equal(O.ldmatrix(num, False, smemT, row2), b)
