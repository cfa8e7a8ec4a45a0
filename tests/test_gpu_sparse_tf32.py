"""TF32 sparse GEMM (the paper's sparse TF32 mma.sp shapes, Table A100-mmasp
PAPER.md:619-620): tcgen05.mma.sp.kind::tf32 with the hardware's 1:2 rule (one element kept per
aligned pair, DESIGN.md R-C12), D = expand(sA, e) x B + C, FP32 accumulate.

Checks: 1:2 compress bit-exact vs the oracle (incl. the first-violation report); the packer's
kind::tf32 image (the kind::f16 layout over 2K, each kept TF32 element = two 16-bit halves) via
one-hot layout probes and integer-valued bit-exact GEMMs; FP results within the north_star bound
(K = logical K) of the exact oracle; sparse == dense TF32 GEMM of the expanded matrix."""
import numpy as np
import pytest
import torch

import oracle as O
import tcxgen
import paper_2206_02874_b200 as tcx
from parity import host_bits, fp_bound_check

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _sparse12(M, K, seed, integer=False):
    """1:2 TF32 matrix (every aligned pair keeps exactly one nonzero, position uniform)."""
    g = tcxgen
    pick = (g.uniform01(seed, g.STREAM_POS, 0, M * K // 2, DEV) < 0.5).view(M, K // 2)
    if integer:
        v = g.int32_matrix((M, K // 2), seed, g.STREAM_SPVAL, -8, 7, DEV)
        v = torch.where(v >= 0, v + 1, v).to(torch.float32)
    else:
        v = g.normal_matrix((M, K // 2), "tf32", seed, g.STREAM_SPVAL, DEV, redraw_zero=True)
    dense = torch.zeros(M, K // 2, 2, dtype=torch.float32, device=DEV)
    dense.scatter_(2, pick.long().unsqueeze(2), v.unsqueeze(2))
    return dense.view(M, K)


def test_tf32_compress_matches_oracle_and_reports_violation():
    M, K = 200, 256
    d = _sparse12(M, K, 3)
    d[::9, ::7] = 0                                     # some all-zero pairs: keep the lower element
    vals, meta = tcx.sp24_compress(d, tf32=True)
    rv, rm, bad = O.sp12_compress(host_bits(d))
    assert bad == -1
    assert np.array_equal(host_bits(vals), rv) and np.array_equal(host_bits(meta), rm)
    d[17, 40:42] = 1.0                                   # two nonzeros in one pair
    with pytest.raises(ValueError, match="row 17, group 10"):
        tcx.sp24_compress(d, tf32=True)


def test_tf32_pack_rejects_2of4_nibble():
    meta = torch.full((128, 4), 0x99999999 - 2 ** 32, dtype=torch.int32, device=DEV)   # nibble 0x9 = (1, 2): legal 1:2
    tcx.sp24_pack_meta(meta, 128, 128, ab=tcx.TF32)
    meta[5, 1] = 0x99999994 - 2 ** 32                   # nibble 0 of word 1 = 0x4 = (0, 1): both in pair 0
    with pytest.raises(ValueError, match="row 5, group 8"):
        tcx.sp24_pack_meta(meta, 128, 128, ab=tcx.TF32)


@pytest.mark.parametrize("cg", [1, 2])
def test_tf32_one_hot_layout_probe(cg):
    M, N, K = 256, 16, 512
    ks = (torch.arange(M, device=DEV) * 37 + 11) % K
    dense = torch.zeros(M, K, dtype=torch.float32, device=DEV)
    dense[torch.arange(M, device=DEV), ks] = 1.0
    vals, meta = tcx.sp24_compress(dense, tf32=True)
    hw = tcx.sp24_pack_meta(meta, M, K, ab=tcx.TF32)
    B = (torch.arange(K, device=DEV, dtype=torch.float32) + 1).expand(N, K).contiguous()
    D = tcx.gemm_sp24(vals, hw, B, None, cta_group=cg, tf32=True)
    torch.cuda.synchronize()
    got = D[:, 0].round().long() - 1
    wrong = (got != ks).nonzero().flatten().tolist()
    report = [(i, int(ks[i]), int(got[i])) for i in wrong[:24]]
    assert not wrong, f"{len(wrong)} rows pick the wrong k (row, expected k, got k): {report}"


@pytest.mark.parametrize("cg", [1, 2])
def test_tf32_sparse_integer_valued_bit_exact(cg):
    M, N, K = 512, 480, 1024
    dense = _sparse12(M, K, 5, integer=True)
    vals, meta = tcx.sp24_compress(dense, tf32=True)
    B = tcxgen.int32_matrix((N, K), 5, 2, -8, 8, DEV).to(torch.float32)
    C = tcxgen.int32_matrix((M, N), 5, 3, -1000, 1000, DEV).to(torch.float32)
    hw = tcx.sp24_pack_meta(meta, M, K, ab=tcx.TF32)
    D = tcx.gemm_sp24(vals, hw, B, C, cta_group=cg, tf32=True)
    ref = dense.double() @ B.double().T + C.double()
    torch.cuda.synchronize()
    assert torch.equal(D.double(), ref)


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("shape", [(256, 240, 64), (512, 496, 320), (768, 1024, 1024)])
def test_tf32_sparse_vs_oracle(shape, cg):
    M, N, K = shape
    dense = _sparse12(M, K, M + N + K)
    vals, meta = tcx.sp24_compress(dense, tf32=True)
    B = tcxgen.normal_matrix((N, K), "tf32", M + N, tcxgen.STREAM_B, DEV)
    C = tcxgen.normal_matrix((M, N), "f32", M + N, tcxgen.STREAM_C, DEV)
    hw = tcx.sp24_pack_meta(meta, M, K, ab=tcx.TF32)
    D = tcx.gemm_sp24(vals, hw, B, C, cta_group=cg, tf32=True)
    torch.cuda.synchronize()
    ii, jj = np.meshgrid(np.arange(M), np.arange(N), indexing="ij")
    ref, absv = O.gemm_samples(O.TF32, O.sp24_expand(host_bits(vals), host_bits(meta), K), host_bits(B),
                               host_bits(C), ii.ravel(), jj.ravel())
    fp_bound_check(host_bits(D).ravel(), ref, absv, K, f"sp tf32 {shape} cg{cg}")


def test_tf32_sparse_equals_dense_of_expanded():
    """integer-valued, so both are exact: sparse == dense tcx_gemm(tf32) on the expanded A."""
    M, N, K = 1024, 960, 2048
    dense = _sparse12(M, K, 7, integer=True)
    vals, meta = tcx.sp24_compress(dense, tf32=True)
    B = tcxgen.int32_matrix((N, K), 7, 2, -8, 8, DEV).to(torch.float32)
    hw = tcx.sp24_pack_meta(meta, M, K, ab=tcx.TF32)
    Ds = tcx.gemm_sp24(vals, hw, B, None, tf32=True)
    Dd = tcx.gemm(dense, B, None, tf32=True)
    torch.cuda.synchronize()
    assert torch.equal(Ds, Dd)


def test_tf32_sparse_m_wide_bit_exact():
    M, N, K = 1024, 480, 512
    dense = _sparse12(M, K, 9, integer=True)
    vals, meta = tcx.sp24_compress(dense, tf32=True)
    B = tcxgen.int32_matrix((N, K), 9, 2, -8, 8, DEV).to(torch.float32)
    hw = tcx.sp24_pack_meta(meta, M, K, ab=tcx.TF32)
    D = tcx.gemm_sp24(vals, hw, B, None, tf32=True, tile_m=512)
    ref = dense.double() @ B.double().T
    torch.cuda.synchronize()
    assert torch.equal(D.double(), ref)


@pytest.mark.parametrize("pairs", [(2, 1), (2, 2)])
def test_tf32_sparse_multicast_bit_exact(pairs):
    M, N, K = 768, 720, 512
    dense = _sparse12(M, K, 13, integer=True)
    vals, meta = tcx.sp24_compress(dense, tf32=True)
    B = tcxgen.int32_matrix((N, K), 13, 2, -8, 8, DEV).to(torch.float32)
    hw = tcx.sp24_pack_meta(meta, M, K, ab=tcx.TF32)
    D = tcx.gemm_sp24(vals, hw, B, None, tf32=True, pairs=pairs)
    ref = dense.double() @ B.double().T
    torch.cuda.synchronize()
    assert torch.equal(D.double(), ref)


def test_tf32_1to2_c3_shape_full_size_default_tile():
    """TF32 1:2 at C3's shape (8192^3, the bench's c3sptf32 operand): the library's default (the
    512 x 240 M-wide tile since K_eff = 16384) bit-identical to the 256-row tile over the whole D, and
    >= 65,536 sampled outputs (every 256-row tile's corner rows among them) within the bound of the
    exact oracle."""
    M = N = K = 8192
    vals, meta = tcxgen.sp12_problem_tf32(M, K, 0, DEV)
    B = tcxgen.normal_matrix((N, K), "tf32", 0, tcxgen.STREAM_B, DEV)
    hw = tcx.sp24_pack_meta(meta, M, K, ab=tcx.TF32)
    Dd = tcx.gemm_sp24(vals, hw, B, None, tf32=True)
    Dn = tcx.gemm_sp24(vals, hw, B, None, tf32=True, tile_m=256)
    torch.cuda.synchronize()
    assert torch.equal(Dd.view(torch.int32), Dn.view(torch.int32))
    del Dn
    rng = np.random.default_rng(1)
    corner = sorted({r for m0 in range(0, M, 256) for r in (m0, m0 + 255)})
    rows = np.array(sorted(set(corner) | set(rng.integers(0, M, 2048 - len(corner)).tolist())))
    idx = torch.from_numpy(rows).to(DEV)
    dense_rows = O.sp24_expand(host_bits(vals[idx]), host_bits(meta[idx]), K)
    ri = np.repeat(np.arange(len(rows)), -(-65536 // len(rows)))
    ci = rng.integers(0, N, ri.size)
    ref, absv = O.gemm_samples(O.TF32, dense_rows, host_bits(B), None, ri, ci)
    got = host_bits(Dd[idx])[ri, ci]
    assert ri.size >= 65536
    fp_bound_check(got, ref, absv, K, "TF32 1:2 8192^3")
