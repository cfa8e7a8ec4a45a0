"""Seeded random-configuration fuzz of the GEMM front end and kernels: random shapes (ragged, tiny,
multi-tile), kinds and kernel options (CTA mode, wide and narrow tiles, multicast groups, raster,
persistent-grid caps, in-place D).  Two checks per sampled output:
  * PARITY against the exact oracle (oracle.gemm_samples): INT8 bit-exact (wrapped), FP within the
    north_star bound (K+2) 2^-23 (sum|ab| + |c|);
  * CROSS-VALIDATION against the instruction model DESIGN.md §7 observed on B200 (fitted to the
    numeric probe, so not parity): FP bit for bit."""
import numpy as np
import pytest
import torch

import oracle as O
import tcxgen
import paper_2206_02874_b200 as tcx
from parity import fp16_bound_check, fp_bound_check, host_bits, model_predict, sp24_kept

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
    elif r < 0.65:
        opts["tile_n"] = int(rng.choice([224, 192, 160, 128]))      # narrow (wave-aware) pair tiles
    if rng.random() < 0.3:
        opts["group_m"] = int(rng.choice([-8, -2, 1, 3, 16]))
    if rng.random() < 0.3:
        opts["max_ctas"] = int(rng.choice([2, 8, 16]))
    return fmt, M, N, K, opts, rng.random() < 0.2


@pytest.mark.parametrize("i", range(96))
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
    got = Dh[rows, cols]
    if fmt == "s8":
        ref, _ = O.gemm_samples(O.S8, Ah, Bh, Ch, rows, cols)                   # parity: bit-exact, wrapped
        assert np.array_equal(ref, got), (fmt, M, N, K, opts, in_place, int((ref != got).sum()))
        return
    ref, absv = O.gemm_samples(AB[fmt], Ah, Bh, Ch, rows, cols)                # parity: the FP bound
    fp_bound_check(got, ref, absv, K, f"dense fuzz {fmt} {M}x{N}x{K} {opts}")
    want = model_predict(AB[fmt], Ah[rows], Bh[cols], Ch[rows, cols].view(np.float32), KI[fmt])
    assert np.array_equal(want, got), (fmt, M, N, K, opts, in_place, int((want != got).sum()))


@pytest.mark.parametrize("i", range(32))
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
    got = host_bits(D)[rows, cols]
    dense = O.sp24_expand(host_bits(vals), host_bits(meta).view(np.uint32), K)
    ref, absv = O.gemm_samples(O.F16, dense, host_bits(B), host_bits(C), rows, cols)   # parity: the FP bound
    fp_bound_check(got, ref, absv, K, f"sparse fuzz {M}x{N}x{K} {opts}")
    ka, kb = sp24_kept(host_bits(vals), host_bits(meta), host_bits(B), rows, cols, K)
    want = model_predict(O.F16, ka, kb, host_bits(C)[rows, cols].view(np.float32), 16)
    assert np.array_equal(want, got), (M, N, K, opts, int((want != got).sum()))


@pytest.mark.parametrize("i", range(24))
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
    # parity: every output vs the exact oracle (FP32 bound, or the FP16-output bound R-F16)
    ref, absv = O.tiles(AB[fmt], 16, 8, k, Ah, Bh, host_bits(C) if with_c else None, cd=O.F16 if cd16 else O.F32)
    if cd16:
        fp16_bound_check(host_bits(D).reshape(ref.shape).astype(np.uint32), ref, absv, k, f"tiles fuzz f16acc k{k}")
    else:
        fp_bound_check(host_bits(D).reshape(ref.shape), ref, absv, k, f"tiles fuzz {fmt} k{k}")
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
