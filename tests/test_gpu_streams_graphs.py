"""The C ABI's stream contract (include/tcx.h: every call asynchronous on the caller's stream, no
allocation, programmatic dependent launch preserving stream order): GEMMs, sparse GEMMs and tile
batches on side streams and captured into one CUDA graph give the eager results bit for bit, and a
chain of dependent calls (each consuming the previous output) stays ordered."""
import numpy as np
import pytest
import torch

import tcxgen
import paper_2206_02874_b200 as tcx

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _inputs():
    A = tcxgen.normal_matrix((512, 256), "bf16", 5, tcxgen.STREAM_A, DEV)
    B = tcxgen.normal_matrix((768, 256), "bf16", 5, tcxgen.STREAM_B, DEV)
    C = tcxgen.normal_matrix((512, 768), "f32", 5, tcxgen.STREAM_C, DEV)
    vals, meta = tcxgen.sp24_problem(512, 256, 6, "f16", DEV)
    Bs = tcxgen.normal_matrix((480, 256), "f16", 6, tcxgen.STREAM_B, DEV)
    hw = tcx.sp24_pack_meta(meta, 512, 256)
    At = tcxgen.uniform_matrix((300, 16, 16), "f16", 0, 1, device=DEV)
    Bt = tcxgen.uniform_matrix((300, 8, 16), "f16", 0, 2, device=DEV)
    return A, B, C, vals, hw, Bs, At, Bt


def test_side_stream_and_graph_replay_match_eager():
    A, B, C, vals, hw, Bs, At, Bt = _inputs()
    ref = (tcx.gemm(A, B, C), tcx.gemm_sp24(vals, hw, Bs, None), tcx.mma_tiles(At, Bt, None))
    torch.cuda.synchronize()
    D1 = torch.empty_like(ref[0]); D2 = torch.empty_like(ref[1]); D3 = torch.empty_like(ref[2])
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        tcx.gemm(A, B, C, D1)
        tcx.gemm_sp24(vals, hw, Bs, None, D2)
        tcx.mma_tiles(At, Bt, None, D3)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    for r, d in zip(ref, (D1, D2, D3)):
        assert torch.equal(r.view(torch.int32), d.view(torch.int32))
    # one CUDA graph holding all three, replayed twice
    G1 = torch.zeros_like(D1); G2 = torch.zeros_like(D2); G3 = torch.zeros_like(D3)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        tcx.gemm(A, B, C, G1)
        tcx.gemm_sp24(vals, hw, Bs, None, G2)
        tcx.mma_tiles(At, Bt, None, G3)
    for _ in range(2):
        G1.zero_(); G2.zero_(); G3.zero_()
        g.replay()
        torch.cuda.synchronize()
        for r, d in zip(ref, (G1, G2, G3)):
            assert torch.equal(r.view(torch.int32), d.view(torch.int32))


def test_dependent_calls_stay_ordered():
    """D_{i+1} = A x B + D_i, 8 times in a row on one stream (each launch reads what the previous one
    wrote, with PDL overlapping their prologues): equals the same chain with a sync between calls."""
    A = tcxgen.int32_matrix((512, 256), 9, 1, -4, 4, DEV).to(torch.bfloat16)
    B = tcxgen.int32_matrix((512, 256), 9, 2, -4, 4, DEV).to(torch.bfloat16)
    D = torch.zeros(512, 512, dtype=torch.float32, device=DEV)
    for _ in range(8):
        tcx.gemm(A, B, D, D)                     # in place: D <- A B^T + D
    Dsync = torch.zeros_like(D)
    for _ in range(8):
        tcx.gemm(A, B, Dsync, Dsync)
        torch.cuda.synchronize()
    ref = 8 * (A.double() @ B.double().T)
    torch.cuda.synchronize()
    assert torch.equal(D, Dsync)
    assert torch.equal(D.double(), ref)         # integer-valued: exact
    # the tile batch: each call's C is the previous call's D
    At = tcxgen.int32_matrix((600, 16, 16), 3, 1, -3, 3, DEV).to(torch.float16)
    Bt = tcxgen.int32_matrix((600, 8, 16), 3, 2, -3, 3, DEV).to(torch.float16)
    Dt = torch.zeros(600, 16, 8, dtype=torch.float32, device=DEV)
    for _ in range(6):
        tcx.mma_tiles(At, Bt, Dt, Dt)
    ref_t = 6 * torch.einsum("tik,tjk->tij", At.double(), Bt.double())
    torch.cuda.synchronize()
    assert torch.equal(Dt.double(), ref_t)


def test_sm_clock_stamp_measures_the_sm_clock():
    """tcx_sm_clock_stamp (the bench's in-run clock): two stamps around a busy GEMM give every SM's
    average clock; it must be a sane B200 SM clock and agree with the probe's clock64/globaltimer
    ratio to within a generous margin (power management moves the clock between runs)."""
    import paper_2206_02874_b200 as tcx
    s0 = torch.zeros(2 * 256, dtype=torch.int64, device="cuda")
    s1 = torch.zeros_like(s0)
    A = torch.randn(4096, 4096, device="cuda").to(torch.bfloat16)
    tcx.sm_clock_stamp(s0)
    for _ in range(10):
        tcx.gemm(A, A)
    tcx.sm_clock_stamp(s1)
    torch.cuda.synchronize()
    mhz = tcx.sm_mhz_between(s0, s1)
    assert mhz is not None and 300 < mhz < 2200, mhz
    stamped = int(((s0.view(-1, 2)[:, 1] > 0) & (s1.view(-1, 2)[:, 1] > 0)).sum())
    assert stamped >= 140, stamped                     # (nearly) every SM ran a stamp CTA
