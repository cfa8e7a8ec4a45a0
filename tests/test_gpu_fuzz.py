"""Seeded random-configuration fuzz of the GEMM front end and kernels: random shapes (ragged, tiny,
multi-tile), kinds and kernel options (CTA mode, wide tiles, multicast groups, raster, persistent-grid
caps, in-place D).  Every sampled output must equal the observed instruction model bit for bit
(FP) or the exact wrapped integer (INT8) — the strongest check there is, applied to
configurations nobody hand-picked."""
import numpy as np
import pytest
import torch

import oracle as O
import tcxgen
import paper_2206_02874_b200 as tcx
from parity import host_bits, model_predict, sp24_kept

pytestmark = pytest.mark.gpu
DEV = "cuda"
KI = {"bf16": 16, "f16": 16, "tf32": 8}
AB = {"bf16": O.BF16, "f16": O.F16, "tf32": O.TF32}


def _dense_case(rng, i):
    fmt = ["bf16", "f16", "tf32", "s8"][i % 4]
    kalign = {"bf16": 8, "f16": 8, "tf32": 4, "s8": 16}[fmt]
    M = int(rng.integers(1, 1100))
    N = int(rng.integers(1, 280)) * 4
    K = int(rng.integers(1, 80)) * kalign
    opts = {}
    r = rng.random()
    if r < 0.15:
        opts["cta_group"] = 1
    elif r < 0.3:
        opts["tile_n"] = 512
    elif r < 0.5:
        opts["pairs"] = [(1, 2), (2, 1), (2, 2)][int(rng.integers(3))]
    if rng.random() < 0.3:
        opts["group_m"] = int(rng.choice([-8, -2, 1, 3, 16]))
    if rng.random() < 0.3:
        opts["max_ctas"] = int(rng.choice([2, 8, 16]))
    return fmt, M, N, K, opts, rng.random() < 0.2


@pytest.mark.parametrize("i", range(32))
def test_dense_fuzz(i):
    rng = np.random.default_rng(1000 + i)
    fmt, M, N, K, opts, in_place = _dense_case(rng, i)
    seed = 77 + i
    if fmt == "s8":
        A = tcxgen.int8_matrix((M, K), seed, tcxgen.STREAM_A, DEV)
        B = tcxgen.int8_matrix((N, K), seed, tcxgen.STREAM_B, DEV)
        C = tcxgen.int32_matrix((M, N), seed, tcxgen.STREAM_C, device=DEV)
    else:
        A = tcxgen.normal_matrix((M, K), fmt, seed, tcxgen.STREAM_A, DEV)
        B = tcxgen.normal_matrix((N, K), fmt, seed, tcxgen.STREAM_B, DEV)
        C = tcxgen.normal_matrix((M, N), "f32", seed, tcxgen.STREAM_C, DEV)
    Cin = C.clone()
    D = tcx.gemm(A, B, C, C if in_place else None, tf32=(fmt == "tf32"), **opts)
    torch.cuda.synchronize()
    n = min(2048, M * N)
    rows, cols = rng.integers(0, M, n), rng.integers(0, N, n)
    Ah, Bh, Ch, Dh = host_bits(A), host_bits(B), host_bits(Cin), host_bits(D)
    if fmt == "s8":
        ref = (Ah[rows].astype(np.int64) * Bh[cols].astype(np.int64)).sum(1) + Ch[rows, cols].view(np.int32)
        want = (ref & 0xFFFFFFFF).astype(np.uint32)
    else:
        want = model_predict(AB[fmt], Ah[rows], Bh[cols], Ch[rows, cols].view(np.float32), KI[fmt])
    got = Dh[rows, cols]
    assert np.array_equal(want, got), (fmt, M, N, K, opts, in_place, int((want != got).sum()))


@pytest.mark.parametrize("i", range(12))
def test_sparse_fuzz(i):
    rng = np.random.default_rng(2000 + i)
    M = int(rng.integers(1, 6)) * 256
    N = int(rng.integers(1, 70)) * 16
    K = int(rng.integers(1, 6)) * 128
    opts = {}
    r = rng.random()
    if r < 0.25 and M % 512 == 0:
        opts["tile_m"] = 512
    elif r < 0.5:
        opts["pairs"] = [(1, 2), (2, 1), (2, 2)][int(rng.integers(3))]
    if rng.random() < 0.3:
        opts["max_ctas"] = int(rng.choice([2, 8]))
    if rng.random() < 0.3:
        opts["group_m"] = int(rng.choice([-4, 2, 16]))
    vals, meta = tcxgen.sp24_problem(M, K, 300 + i, "f16", DEV)
    B = tcxgen.normal_matrix((N, K), "f16", 300 + i, tcxgen.STREAM_B, DEV)
    C = tcxgen.normal_matrix((M, N), "f32", 300 + i, tcxgen.STREAM_C, DEV)
    hw = tcx.sp24_pack_meta(meta, M, K)
    D = tcx.gemm_sp24(vals, hw, B, C, **opts)
    torch.cuda.synchronize()
    n = 1024
    rows, cols = rng.integers(0, M, n), rng.integers(0, N, n)
    ka, kb = sp24_kept(host_bits(vals), host_bits(meta), host_bits(B), rows, cols, K)
    want = model_predict(O.F16, ka, kb, host_bits(C)[rows, cols].view(np.float32), 16)
    got = host_bits(D)[rows, cols]
    assert np.array_equal(want, got), (M, N, K, opts, int((want != got).sum()))


@pytest.mark.parametrize("i", range(12))
def test_tiles_fuzz(i):
    """tcx_mma_tiles over random formats / k / counts, C present or not, FP32 or FP16 C/D: every
    output of every tile equals the instruction model (C as the MMA's C operand) bit for bit."""
    rng = np.random.default_rng(3000 + i)
    fmt, k, cd16 = [("f16", 16, False), ("bf16", 16, False), ("f16", 8, False), ("bf16", 8, False),
                    ("tf32", 8, False), ("tf32", 16, False), ("f16", 16, True), ("f16", 8, True)][i % 8]
    count = int(rng.integers(1, 3000))
    A = tcxgen.uniform_matrix((count, 16, k), fmt, 40 + i, tcxgen.STREAM_A, device=DEV)
    B = tcxgen.uniform_matrix((count, 8, k), fmt, 40 + i, tcxgen.STREAM_B, device=DEV)
    with_c = rng.random() < 0.7
    C = tcxgen.uniform_matrix((count, 16, 8), "f16" if cd16 else "f32", 40 + i, tcxgen.STREAM_C, device=DEV) if with_c else None
    D = tcx.mma_tiles(A, B, C, tf32=(fmt == "tf32"), f16_acc=cd16)
    torch.cuda.synchronize()
    ii, jj = np.meshgrid(np.arange(16), np.arange(8), indexing="ij")
    Ah, Bh = host_bits(A), host_bits(B)
    a_rows = Ah[:, ii.ravel(), :].reshape(-1, k)
    b_rows = Bh[:, jj.ravel(), :].reshape(-1, k)
    if cd16:
        c = host_bits(C).reshape(-1).astype(np.uint32) if with_c else np.zeros(count * 128, np.uint32)
        want = O.model_batch(O.F16, a_rows, b_rows, c, Ki=k, g=k, p=3, rz=False, emode=2, acc_fmt=O.F16, win_fmt=O.F32)
        got = host_bits(D).reshape(-1).astype(np.uint32)
    else:
        c = host_bits(C).reshape(-1) if with_c else np.zeros(count * 128, np.uint32)
        ki = 8 if fmt == "tf32" else k
        want = O.model_batch(AB[fmt], a_rows, b_rows, c, Ki=ki, g=ki, p=3, rz=True, emode=3)
        got = host_bits(D).reshape(-1)
    assert np.array_equal(want, got), (fmt, k, cd16, count, with_c, int((want != got).sum()))
