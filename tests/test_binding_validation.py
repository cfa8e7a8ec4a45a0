"""The Python binding's argument checks (-m "not gpu").

The C ABI takes plain pointers and row strides, so a tensor of the wrong dtype or shape would make
the TMA engine read or write past its allocation.  The binding therefore checks dtype, shape, inner
stride and device of every tensor before any pointer reaches the library; the checks run on CPU
tensors (a well-formed CPU call then fails on the device check: there is no CPU fallback)."""
import pytest
import torch

import paper_2206_02874_b200 as tcx


def _z(*shape, dtype=torch.float32):
    return torch.zeros(*shape, dtype=dtype)


def _raises(fn, match):
    with pytest.raises(ValueError, match=match):
        fn()


def test_gemm_checks():
    A, B = _z(256, 64, dtype=torch.bfloat16), _z(128, 64, dtype=torch.bfloat16)
    _raises(lambda: tcx.gemm(A, B, None, _z(256, 128, dtype=torch.bfloat16)), "D: expected dtype")     # 2-byte D
    _raises(lambda: tcx.gemm(A, B, _z(256, 128, dtype=torch.float16)), "C: expected dtype")
    _raises(lambda: tcx.gemm(A, B, _z(256, 127)), "C: expected shape")
    _raises(lambda: tcx.gemm(A, B, None, _z(255, 128)), "D: expected shape")
    _raises(lambda: tcx.gemm(A, _z(128, 64, dtype=torch.float16)), "B: expected dtype")               # bf16 vs f16
    _raises(lambda: tcx.gemm(A, _z(128, 32, dtype=torch.bfloat16)), "B: expected shape")
    _raises(lambda: tcx.gemm(A, B, _z(128, 256).t()), "C: expected shape|innermost")
    _raises(lambda: tcx.gemm(A, B, _z(256, 256)[:, ::2]), "innermost")
    _raises(lambda: tcx.gemm(A[:, ::2], B[:, ::2]), "innermost")
    s8 = _z(256, 64, dtype=torch.int8)
    _raises(lambda: tcx.gemm(s8, _z(128, 64, dtype=torch.int8), _z(256, 128)), "C: expected dtype")   # S32 C
    _raises(lambda: tcx.gemm(_z(256, 64, dtype=torch.float16), _z(128, 64, dtype=torch.float16), None,
                             _z(256, 128), f16_acc=True), "D: expected dtype")
    with pytest.raises(TypeError):
        tcx.gemm(_z(256, 64), _z(128, 64))                       # float32 without tf32=True
    # well-formed: reaches the device check
    _raises(lambda: tcx.gemm(A, B, _z(256, 128), _z(256, 128)), "CUDA tensors only")
    _raises(lambda: tcx.gemm(A, B, _z(512, 128)[:256], None), "CUDA tensors only")        # padded rows are fine


def test_sparse_checks():
    M, N, K = 256, 240, 256
    vals, B = _z(M, K // 2, dtype=torch.float16), _z(N, K, dtype=torch.float16)
    nbytes = M * K // 8                                         # the documented size (tcx.h), host-side
    hw = torch.zeros(nbytes, dtype=torch.uint8)
    _raises(lambda: tcx.gemm_sp24(vals, hw[:-16], B), "meta_hw has")
    _raises(lambda: tcx.gemm_sp24(vals, hw.view(torch.int32), B), "uint8")
    _raises(lambda: tcx.gemm_sp24(_z(M, K // 4, dtype=torch.float16), hw, B), "vals: expected shape|kept columns")
    _raises(lambda: tcx.gemm_sp24(vals, hw, _z(N, K, dtype=torch.bfloat16)), "B: expected dtype")
    _raises(lambda: tcx.gemm_sp24(vals, hw, B, _z(M, N, dtype=torch.float16)), "C: expected dtype")
    _raises(lambda: tcx.gemm_sp24(vals, hw, B, None, _z(M, N - 16)), "D: expected shape")
    _raises(lambda: tcx.gemm_sp24(vals.to(torch.int8), hw, B.to(torch.int8), _z(M, N)), "C: expected dtype")
    _raises(lambda: tcx.gemm_sp24(vals, hw, B, _z(M, N), _z(M, N)), "CUDA tensors only")


def test_tiles_pack_round_checks():
    A, B = _z(10, 16, 16, dtype=torch.float16), _z(10, 8, 16, dtype=torch.float16)
    _raises(lambda: tcx.mma_tiles(A, _z(10, 8, 8, dtype=torch.float16)), "B: expected shape")
    _raises(lambda: tcx.mma_tiles(A, B, _z(10, 16, 8, dtype=torch.float16)), "C: expected dtype")
    _raises(lambda: tcx.mma_tiles(A, B, None, _z(9, 16, 8)), "D: expected shape")
    _raises(lambda: tcx.mma_tiles(A, B, _z(10, 16, 8)), "CUDA tensors only")
    _raises(lambda: tcx.sp24_pack_meta(_z(256, 4, dtype=torch.int32), 256, 256), "meta_canon: expected shape")
    _raises(lambda: tcx.sp24_pack_meta(_z(256, 8, dtype=torch.int64), 256, 256), "meta_canon: expected dtype")
    _raises(lambda: tcx.round_tf32(_z(8, dtype=torch.float16)), "float32")
    _raises(lambda: tcx.round_tf32(_z(8), out=_z(7)), "out must")
    _raises(lambda: tcx.round_tf32(_z(8)), "CUDA tensors only")
