"""FP16-accumulate dense GEMM ("FP16-accumulate (C/D FP16) dense path in tiles
and GEMM (idesc D format F16)"): tcgen05.mma kind::f16 with an FP16 tensor-memory accumulator, C
preloaded into the accumulator (the MMA's own C operand), FP16 D through a TMA store.

Gate: the R-F16G bar of tests/parity.py against the exact oracle rounded once to FP16; integer-valued
inputs whose every partial is an exact FP16 value are bit-exact."""
import numpy as np
import pytest
import torch

import oracle as O
import tcxgen
import paper_2206_02874_b200 as tcx
from parity import host_bits, fp16acc_gemm_bound_check, gemm_sample_coords

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _problem(M, N, K, seed, with_c=True):
    A = tcxgen.normal_matrix((M, K), "f16", seed, tcxgen.STREAM_A, DEV)
    B = tcxgen.normal_matrix((N, K), "f16", seed, tcxgen.STREAM_B, DEV)
    C = tcxgen.normal_matrix((M, N), "f16", seed, tcxgen.STREAM_C, DEV) if with_c else None
    return A, B, C


def _check(A, B, C, D, rows=None, cols=None):
    M, K = A.shape
    N = B.shape[0]
    if rows is None:
        ii, jj = np.meshgrid(np.arange(M), np.arange(N), indexing="ij")
        rows, cols = ii.ravel(), jj.ravel()
    ref, absv = O.gemm_samples(O.F16, host_bits(A), host_bits(B), host_bits(C) if C is not None else None,
                               rows, cols, cd=O.F16)
    return fp16acc_gemm_bound_check(host_bits(D)[rows, cols], ref, absv, K, f"f16acc gemm {M}x{N}x{K}")


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("shape", [(256, 256, 64), (128, 256, 16), (512, 512, 512), (200, 136, 72), (264, 520, 40),
                                   (384, 64, 1024)])
def test_f16acc_gemm_small(shape, cg):
    M, N, K = shape
    A, B, C = _problem(M, N, K, M + N + K)
    D = tcx.gemm(A, B, C, f16_acc=True, cta_group=cg)
    torch.cuda.synchronize()
    assert D.dtype == torch.float16
    _check(A, B, C, D)


@pytest.mark.parametrize("cg", [1, 2])
def test_f16acc_gemm_integer_bit_exact(cg):
    """|a|, |b| <= 2, K = 128, |c| < 512: every partial sum is an integer below 2048, exact in FP16."""
    M, N, K = 512, 768, 128
    A = tcxgen.int32_matrix((M, K), 2, 1, -2, 2, DEV).to(torch.float16)
    B = tcxgen.int32_matrix((N, K), 2, 2, -2, 2, DEV).to(torch.float16)
    C = tcxgen.int32_matrix((M, N), 2, 3, -500, 500, DEV).to(torch.float16)
    for Cx in (C, None):
        D = tcx.gemm(A, B, Cx, f16_acc=True, cta_group=cg)
        ref = A.double() @ B.double().T + (Cx.double() if Cx is not None else 0)
        torch.cuda.synchronize()
        assert torch.equal(D.double(), ref)


def test_f16acc_gemm_persistent_determinism_and_k0():
    M, N, K = 1024, 1280, 512
    A, B, C = _problem(M, N, K, 9)
    D1 = tcx.gemm(A, B, C, f16_acc=True, max_ctas=2)
    D2 = tcx.gemm(A, B, C, f16_acc=True)
    torch.cuda.synchronize()
    assert torch.equal(D1.view(torch.int16), D2.view(torch.int16))
    rows, cols = gemm_sample_coords(M, N, 256, 256, nsamp=8192)
    _check(A, B, C, D1, rows, cols)
    D0 = tcx.gemm(A[:, :0], B[:, :0], C, f16_acc=True)       # K == 0: D = C
    torch.cuda.synchronize()
    assert torch.equal(D0, C)


def test_f16acc_gemm_c3_shape_sampled():
    """configs[2]'s shape (8192^3) with FP16 inputs and an FP16 accumulator (C = FP16 zeros)."""
    M = N = K = 8192
    A = tcxgen.normal_matrix((M, K), "f16", 0, tcxgen.STREAM_A, DEV)
    B = tcxgen.normal_matrix((N, K), "f16", 0, tcxgen.STREAM_B, DEV)
    C = torch.zeros(M, N, dtype=torch.float16, device=DEV)
    D = tcx.gemm(A, B, C, f16_acc=True)
    torch.cuda.synchronize()
    rows, cols = gemm_sample_coords(M, N, 256, 256, nsamp=16384, seed=3)
    worst = _check(A, B, C, D, rows, cols)
    assert worst > 0            # FP16 accumulation is inexact at this K (reported, within the bar)


def test_f16acc_gemm_in_place():
    M, N, K = 512, 512, 256
    A, B, C = _problem(M, N, K, 41)
    D = tcx.gemm(A, B, C, f16_acc=True)
    C2 = C.clone()
    tcx.gemm(A, B, C2, C2, f16_acc=True)
    torch.cuda.synchronize()
    assert torch.equal(D.view(torch.int16), C2.view(torch.int16))
