"""tcx_mma_tiles (mma.sync) vs the oracle — config 1 (BASELINE.json configs[0]) and variants."""
import numpy as np
import pytest
import torch

import oracle as O
import tcxgen
import paper_2206_02874_b200 as tcx
from parity import host_bits, fp_bound_check, fp16_bound_check

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _tiles_problem(count, fmt, seed=0, k=16, integer=False):
    if fmt == "s8":
        A = tcxgen.int8_matrix((count, 16, 32), seed, tcxgen.STREAM_A, DEV)
        B = tcxgen.int8_matrix((count, 8, 32), seed, tcxgen.STREAM_B, DEV)
        C = tcxgen.int32_matrix((count, 16, 8), seed, tcxgen.STREAM_C, device=DEV)
        return A, B, C
    if integer:   # integer-valued inputs, |a|,|b| <= 8: exact sums, so the GPU must be bit-exact
        A = (tcxgen.int32_matrix((count, 16, k), seed, 1, -8, 8, DEV)).to(torch.float32)
        B = (tcxgen.int32_matrix((count, 8, k), seed, 2, -8, 8, DEV)).to(torch.float32)
        C = (tcxgen.int32_matrix((count, 16, 8), seed, 3, -1000, 1000, DEV)).to(torch.float32)
        dt = {"f16": torch.float16, "bf16": torch.bfloat16, "tf32": torch.float32}[fmt]
        return A.to(dt), B.to(dt), C
    A = tcxgen.uniform_matrix((count, 16, k), fmt, seed, tcxgen.STREAM_A, device=DEV)
    B = tcxgen.uniform_matrix((count, 8, k), fmt, seed, tcxgen.STREAM_B, device=DEV)
    C = tcxgen.uniform_matrix((count, 16, 8), "f32", seed, tcxgen.STREAM_C, device=DEV)
    return A, B, C


OF = {"f16": O.F16, "bf16": O.BF16, "tf32": O.TF32, "s8": O.S8}


def _check(fmt, A, B, C, D, k):
    count = A.shape[0]
    ref, absv = O.tiles(OF[fmt], 16, 8, k, host_bits(A), host_bits(B), host_bits(C) if C is not None else None)
    got = host_bits(D)
    if fmt == "s8":
        assert np.array_equal(got.reshape(ref.shape), ref)
        return 0.0
    return fp_bound_check(got.reshape(ref.shape), ref, absv, k, f"tiles {fmt}")


def test_config1_whole_batch():
    """BASELINE configs[0]: 4096 m16n8k16 FP16 tiles, U[-1,1], C FP32 U[-1,1], seed 0."""
    A, B, C = _tiles_problem(4096, "f16", seed=0)
    D = tcx.mma_tiles(A, B, C)
    torch.cuda.synchronize()
    norm = _check("f16", A, B, C, D, 16)
    assert norm <= 18
    # bit for bit: all 524,288 outputs equal the observed instruction model with C as the MMA's C
    # operand (one m16n8k16: 16 products + c, window 3 bits below FP32's, RZ; DESIGN.md §7 finding 2)
    Ah, Bh, Ch = host_bits(A), host_bits(B), host_bits(C)
    ii, jj = np.meshgrid(np.arange(16), np.arange(8), indexing="ij")
    a_rows = Ah[:, ii.ravel(), :].reshape(-1, 16)
    b_rows = Bh[:, jj.ravel(), :].reshape(-1, 16)
    pred = O.model_batch(O.F16, a_rows, b_rows, Ch.reshape(-1), Ki=16, g=16, p=3, rz=True, emode=3)
    assert np.array_equal(pred, host_bits(D).reshape(-1))


@pytest.mark.parametrize("fmt,k", [("f16", 16), ("bf16", 16), ("tf32", 8), ("tf32", 16), ("s8", 32)])
@pytest.mark.parametrize("count", [1, 7, 1000, 4097])
def test_tiles_formats_and_ragged_counts(fmt, k, count):
    A, B, C = _tiles_problem(count, fmt, seed=count, k=k)
    D = tcx.mma_tiles(A, B, C, tf32=(fmt == "tf32"))
    torch.cuda.synchronize()
    _check(fmt, A, B, C, D, k)


@pytest.mark.parametrize("fmt,k", [("f16", 16), ("bf16", 16), ("tf32", 16)])
def test_tiles_integer_valued_bit_exact(fmt, k):
    A, B, C = _tiles_problem(2048, fmt, seed=5, k=k, integer=True)
    D = tcx.mma_tiles(A, B, C, tf32=(fmt == "tf32"))
    torch.cuda.synchronize()
    ref, _ = O.tiles(OF[fmt], 16, 8, k, host_bits(A), host_bits(B), host_bits(C))
    assert np.array_equal(host_bits(D).reshape(ref.shape), ref)


def test_tiles_no_c_and_empty_and_determinism():
    A, B, _ = _tiles_problem(333, "f16", seed=9)
    D1 = tcx.mma_tiles(A, B, None)
    D2 = tcx.mma_tiles(A, B, None)
    torch.cuda.synchronize()
    assert torch.equal(D1.view(torch.int32), D2.view(torch.int32))
    _check("f16", A, B, None, D1, 16)
    E = tcx.mma_tiles(A[:0], B[:0], None)
    assert E.shape[0] == 0


def test_tiles_unsupported_shape_raises():
    A = torch.zeros((4, 16, 4), dtype=torch.float16, device=DEV)
    B = torch.zeros((4, 8, 4), dtype=torch.float16, device=DEV)
    with pytest.raises(tcx.TcxError):
        tcx.mma_tiles(A, B, None)
    A = torch.zeros((4, 16, 16), dtype=torch.bfloat16, device=DEV)
    B = torch.zeros((4, 8, 16), dtype=torch.bfloat16, device=DEV)
    with pytest.raises(tcx.TcxError):               # FP16 accumulate exists for FP16 inputs only
        tcx.mma_tiles(A, B, None, f16_acc=True)


@pytest.mark.parametrize("fmt", ["f16", "bf16"])
@pytest.mark.parametrize("count", [1, 9, 3000])
def test_tiles_m16n8k8_f32(fmt, count):
    """m16n8k8 (the chain-matmul shape) with FP32 C/D."""
    A, B, C = _tiles_problem(count, fmt, seed=40 + count, k=8)
    D = tcx.mma_tiles(A, B, C)
    torch.cuda.synchronize()
    _check(fmt, A, B, C, D, 8)


def _f16acc_problem(count, k, seed, scale=1.0):
    A = tcxgen.normal_matrix((count, 16, k), "f16", seed, tcxgen.STREAM_A, DEV)
    B = tcxgen.normal_matrix((count, 8, k), "f16", seed, tcxgen.STREAM_B, DEV)
    C = (tcxgen.normal_matrix((count, 16, 8), "f32", seed, tcxgen.STREAM_C, DEV) * scale).to(torch.float16)
    return A, B, C


@pytest.mark.parametrize("k", [16, 8])
@pytest.mark.parametrize("count", [1, 7, 4097])
def test_tiles_fp16_accumulate_vs_oracle(k, count):
    """(F16, F16) tiles: D = A B + C with FP16 C/D vs RNE_fp16(exact)."""
    A, B, C = _f16acc_problem(count, k, seed=count + k)
    D = tcx.mma_tiles(A, B, C, f16_acc=True)
    torch.cuda.synchronize()
    assert D.dtype == torch.float16
    ref, absv = O.tiles(O.F16, 16, 8, k, host_bits(A), host_bits(B), host_bits(C), cd=O.F16)
    fp16_bound_check(host_bits(D).reshape(ref.shape), ref, absv, k, f"f16acc k{k}")


def test_tiles_fp16_accumulate_integer_bit_exact_and_no_c():
    """integer-valued FP16 inputs with |sum| < 2048: every partial and the result are exact FP16
    values, so D must equal the oracle bit for bit; C = NULL means zeros."""
    count = 2048
    A = tcxgen.int32_matrix((count, 16, 16), 3, 1, -4, 4, DEV).to(torch.float16)
    B = tcxgen.int32_matrix((count, 8, 16), 3, 2, -4, 4, DEV).to(torch.float16)
    C = tcxgen.int32_matrix((count, 16, 8), 3, 3, -1000, 1000, DEV).to(torch.float16)
    for Cx in (C, None):
        D = tcx.mma_tiles(A, B, Cx, f16_acc=True)
        torch.cuda.synchronize()
        ref, _ = O.tiles(O.F16, 16, 8, 16, host_bits(A), host_bits(B), host_bits(Cx) if Cx is not None else None,
                         cd=O.F16)
        assert np.array_equal(host_bits(D).reshape(ref.shape).astype(np.uint32), ref)


def test_tiles_fp16_accumulate_overflow_is_inf():
    """FP16 range: 8 products of 128*128 = 2^17 > 65504 must give +inf (the chain-matmul
    overflow the paper reports for FP16), as the oracle does."""
    A = torch.full((4, 16, 8), 128.0, dtype=torch.float16, device=DEV)
    B = torch.full((4, 8, 8), 128.0, dtype=torch.float16, device=DEV)
    D = tcx.mma_tiles(A, B, None, f16_acc=True)
    torch.cuda.synchronize()
    assert torch.isinf(D).all() and (D > 0).all()
