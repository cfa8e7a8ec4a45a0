"""C-ABI argument validation without a GPU (-m "not gpu"): every documented error of include/tcx.h is
detected before any device query or launch, so these calls return the stated status on a CPU-only
host.  Pointers are fake (aligned or not) device addresses — never dereferenced by host code.  The
one call with valid arguments reaches the device query and must report TCX_ERR_NO_DEVICE here."""
import ctypes

import pytest
import torch

import paper_2206_02874_b200 as tcx

OK, INVALID, UNSUPPORTED, MISALIGNED, NO_DEVICE = 0, 1, 2, 3, 5
P = 0x7F0000000000            # a 16-byte-aligned fake device address
F16, BF16, TF32, S8, F32, S32 = tcx.F16, tcx.BF16, tcx.TF32, tcx.S8, tcx.F32, tcx.S32


def _gemm(ab=BF16, cd=F32, M=256, N=256, K=64, A=P, lda=None, B=P, ldb=None, C=None, ldc=None, D=P, ldd=None,
          opts=None):
    L = tcx.lib()
    o = ctypes.byref(opts) if opts is not None else None
    return L.tcx_gemm_ex(ab, cd, M, N, K, A, lda if lda is not None else K, B, ldb if ldb is not None else K,
                         C, ldc if ldc is not None else N, D, ldd if ldd is not None else N, o, None)


def _opts(**kw):
    o = tcx.GemmOpts()
    for k, v in kw.items():
        setattr(o, k, v)
    return o


@pytest.mark.parametrize("kw,want", [
    (dict(ab=S8, cd=F32), UNSUPPORTED),              # INT8 needs S32 accumulate
    (dict(ab=BF16, cd=F16), UNSUPPORTED),            # FP16 accumulate is F16 inputs only
    (dict(M=-1), INVALID),
    (dict(M=0), OK),                                 # no-op
    (dict(N=0), OK),
    (dict(D=None), INVALID),
    (dict(A=None), INVALID),
    (dict(lda=32), INVALID),                         # lda < K
    (dict(ldd=128), INVALID),                        # ldd < N
    (dict(A=P + 8), MISALIGNED),
    (dict(K=60), MISALIGNED),                        # K * 2 bytes not a multiple of 16
    (dict(lda=68), MISALIGNED),
    (dict(M=1 << 31), UNSUPPORTED),
    (dict(opts=_opts(cta_group=3)), INVALID),
    (dict(opts=_opts(tile_n=384)), INVALID),
    (dict(opts=_opts(pairs_m=3)), INVALID),
    (dict(opts=_opts(pairs_m=2, cta_group=1)), INVALID),
    (dict(opts=_opts(pairs_n=2, tile_n=512)), INVALID),
    (dict(opts=_opts(tile_n=512, cta_group=1)), UNSUPPORTED),   # the wide tile needs the CTA pair
    (dict(ab=F16, cd=F16, opts=_opts(tile_n=512)), UNSUPPORTED),   # ... and a 32-bit accumulator
    (dict(opts=_opts(tile_n=224, cta_group=1)), UNSUPPORTED),   # the narrow tiles need the CTA pair
    (dict(opts=_opts(tile_n=192, pairs_n=2)), INVALID),         # multicast groups: 256-wide tiles only
    (dict(opts=_opts(tile_n=200)), INVALID),
])
def test_gemm_argument_errors(kw, want):
    assert _gemm(**kw) == want, tcx.lib().tcx_last_error()


def test_valid_gemm_reaches_the_device_query():
    if torch.cuda.is_available():
        pytest.skip("fake pointers must not reach a real launch")
    assert _gemm() == NO_DEVICE
    assert _gemm(opts=_opts(pairs_m=2, pairs_n=2, group_m=-4)) == NO_DEVICE
    assert b"device" in tcx.lib().tcx_last_error().lower() or b"cuda" in tcx.lib().tcx_last_error().lower()


def _sp(ab=F16, cd=F32, M=256, N=240, K=256, meta=P, opts=None):
    L = tcx.lib()
    o = ctypes.byref(opts) if opts is not None else None
    return L.tcx_gemm_sp24_ex(ab, cd, M, N, K, P, K // 2, meta, P, K, None, N, P, N, o, None)


@pytest.mark.parametrize("kw,want", [
    (dict(K=192), UNSUPPORTED),                      # K % 128 (f16)
    (dict(ab=S8, cd=S32, K=128), UNSUPPORTED),       # K % 256 (int8)
    (dict(N=250), UNSUPPORTED),                      # N % 16
    (dict(M=200), UNSUPPORTED),                      # M % 128
    (dict(meta=None), MISALIGNED),
    (dict(meta=P + 4), MISALIGNED),
    (dict(M=128), UNSUPPORTED),                      # the CTA pair needs M % 256
    (dict(ab=S8, cd=F32, K=256), UNSUPPORTED),
    (dict(opts=_opts(pairs_m=2, cta_group=1)), INVALID),       # multicast groups need the CTA pair
    (dict(M=256, opts=_opts(pairs_m=2, tile_n=512)), UNSUPPORTED),   # M-wide needs M % 512
    (dict(opts=_opts(tile_n=384)), INVALID),
    (dict(opts=_opts(cta_group=3)), INVALID),        # as tcx_gemm_ex
    (dict(opts=_opts(cta_group=-1)), INVALID),
    (dict(opts=_opts(tile_n=512, cta_group=1)), UNSUPPORTED),   # the M-wide tile needs the CTA pair,
    (dict(ab=S8, cd=S32, opts=_opts(tile_n=512)), UNSUPPORTED),  # a 16/32-bit kind
    (dict(M=768, opts=_opts(tile_n=512)), UNSUPPORTED),          # and M % 512 == 0
    (dict(M=0), OK),
])
def test_sparse_argument_errors(kw, want):
    assert _sp(**kw) == want, tcx.lib().tcx_last_error()


def test_tiles_and_chain_argument_errors():
    L = tcx.lib()
    assert L.tcx_mma_tiles(F16, F32, 16, 8, 16, -1, P, P, None, P, None) == INVALID
    assert L.tcx_mma_tiles(F16, F32, 16, 8, 16, 0, P, P, None, P, None) == OK
    assert L.tcx_mma_tiles(F16, F32, 16, 8, 4, 4, P, P, None, P, None) == UNSUPPORTED     # k = 4
    assert L.tcx_mma_tiles(S8, F32, 16, 8, 32, 4, P, P, None, P, None) == UNSUPPORTED     # S8 -> F32
    assert L.tcx_mma_chain(F16, -1, 4, P, P, P, None) == INVALID
    assert L.tcx_mma_chain(F16, 0, 4, P, P, P, None) == OK
    assert L.tcx_round_tf32(None, None, -1, None) == INVALID
    assert L.tcx_round_tf32(None, None, 0, None) == OK
    assert L.tcx_sm_clock_stamp(None, 4, None) == INVALID
    assert L.tcx_sm_clock_stamp(P, 0, None) == INVALID
    assert L.tcx_sm_clock_stamp(P + 4, 4, None) == MISALIGNED
