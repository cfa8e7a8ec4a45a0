"""INT8 2:4 sparse GEMM (the paper's sparse INT8 mma.sp shapes, Table
A100-mmasp PAPER.md:608-624, at GEMM scale): tcgen05.mma.sp.kind::i8, D = expand(sA, e) x B + C
with INT32 accumulation and two's-complement wraparound.  Integer work: bit-exact against the
oracle (expand then exact int64 dot, wrap).  The metadata image (sp24.cu, kind::i8: lane = row,
one canonical word per TMEM column) is verified by one-hot layout probes first."""
import numpy as np
import pytest
import torch

import oracle as O
import tcxgen
import paper_2206_02874_b200 as tcx
from parity import host_bits, gemm_sample_coords

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _sparse_i8(M, K, seed, lo=-128, hi=127):
    """exactly 2 nonzeros per aligned group of 4 along K (pairs uniform over the 6), values
    uniform in [lo, hi] \\ {0}; returns (vals (M, K/2) int8, canonical meta, dense)."""
    pairs = tcxgen.sp24_pairs(M, K, seed, device=DEV)
    meta = tcxgen.sp24_canonical_meta(pairs)
    v = tcxgen.int32_matrix((M, K // 2), seed, tcxgen.STREAM_SPVAL, lo, hi - 1, DEV)
    v = torch.where(v >= 0, v + 1, v)                          # [lo, hi] without 0
    vals = v.to(torch.int8)
    dense = torch.from_numpy(O.sp24_expand(host_bits(vals), host_bits(meta), K)).to(DEV)
    return vals, meta, dense


@pytest.mark.parametrize("cg", [1, 2])
def test_i8_one_hot_layout_probe(cg):
    """one kept 1 per row at logical column k_i, B[n][k] = k % 127 + 1: D[i][n] names the k the
    hardware paired with A's value, for every (row, group, position) class of the image."""
    M, N, K = 256, 16, 1024
    ks = (torch.arange(M, device=DEV) * 37 + 11) % K
    dense = torch.zeros(M, K, dtype=torch.int8, device=DEV)
    dense[torch.arange(M, device=DEV), ks] = 1
    vals, meta = tcx.sp24_compress(dense)
    hw = tcx.sp24_pack_meta(meta, M, K, ab=tcx.S8)
    B = (torch.arange(K, device=DEV) % 127 + 1).to(torch.int8).expand(N, K).contiguous()
    D = tcx.gemm_sp24(vals, hw, B, None, cta_group=cg)
    torch.cuda.synchronize()
    want = (ks % 127 + 1).to(torch.int32)
    wrong = (D[:, 0] != want).nonzero().flatten().tolist()
    report = [(i, int(ks[i]), int(D[i, 0])) for i in wrong[:24]]
    assert not wrong, f"{len(wrong)} rows pick the wrong k (row, k, got B value): {report}"
    assert torch.equal(D, D[:, :1].expand(M, N))


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("shape", [(256, 240, 256), (512, 496, 768), (768, 1024, 1024)])
def test_i8_sparse_bit_exact_small(shape, cg):
    M, N, K = shape
    vals, meta, dense = _sparse_i8(M, K, M + N + K)
    B = tcxgen.int8_matrix((N, K), M + N, tcxgen.STREAM_B, DEV)
    C = tcxgen.int32_matrix((M, N), M + N, tcxgen.STREAM_C, device=DEV)
    hw = tcx.sp24_pack_meta(meta, M, K, ab=tcx.S8)
    D = tcx.gemm_sp24(vals, hw, B, C, cta_group=cg)
    torch.cuda.synchronize()
    ii, jj = np.meshgrid(np.arange(M), np.arange(N), indexing="ij")
    ref, _ = O.gemm_samples(O.S8, host_bits(dense), host_bits(B), host_bits(C), ii.ravel(), jj.ravel())
    assert np.array_equal(host_bits(D).ravel(), ref)


def test_i8_sparse_wraparound():
    """INT32 two's-complement wrap (north_star; DESIGN.md R-C10): c = 2^31 - 1 plus positive products
    wraps negative; a saturating accumulator would stay at 2^31 - 1."""
    M, N, K = 256, 16, 256
    vals, meta, dense = _sparse_i8(M, K, 3, lo=1, hi=127)
    vals = vals.abs()
    dense = dense.abs()
    B = torch.full((N, K), 127, dtype=torch.int8, device=DEV)
    C = torch.full((M, N), 2 ** 31 - 1, dtype=torch.int32, device=DEV)
    hw = tcx.sp24_pack_meta(meta, M, K, ab=tcx.S8)
    D = tcx.gemm_sp24(vals, hw, B, C)
    torch.cuda.synchronize()
    ii, jj = np.meshgrid(np.arange(M), np.arange(N), indexing="ij")
    ref, _ = O.gemm_samples(O.S8, host_bits(dense), host_bits(B), host_bits(C), ii.ravel(), jj.ravel())
    assert np.array_equal(host_bits(D).ravel(), ref)
    assert (D < 0).all()


def test_i8_sparse_vs_dense_of_expanded_and_determinism():
    """sparse output == the dense INT8 GEMM (tcx_gemm) on expand(sA, e), bit for bit."""
    M, N, K = 1024, 960, 2048
    vals, meta, dense = _sparse_i8(M, K, 11)
    B = tcxgen.int8_matrix((N, K), 11, tcxgen.STREAM_B, DEV)
    C = tcxgen.int32_matrix((M, N), 11, tcxgen.STREAM_C, device=DEV)
    hw = tcx.sp24_pack_meta(meta, M, K, ab=tcx.S8)
    Ds = tcx.gemm_sp24(vals, hw, B, C)
    Ds2 = tcx.gemm_sp24(vals, hw, B, C, max_ctas=4)
    Dd = tcx.gemm(dense, B, C)
    torch.cuda.synchronize()
    assert torch.equal(Ds, Dd) and torch.equal(Ds, Ds2)


def test_i8_sparse_c4_shape_sampled():
    """the C4 shape (M=N=K=16384) with 2:4 A: >= 65,536 oracle samples incl. every CTA-tile corner."""
    M = N = K = 16384
    vals, meta, _ = _sparse_i8_nodense(M, K, 0)
    B = tcxgen.int8_matrix((N, K), 0, tcxgen.STREAM_B, DEV)
    C = tcxgen.int32_matrix((M, N), 0, tcxgen.STREAM_C, device=DEV)
    hw = tcx.sp24_pack_meta(meta, M, K, ab=tcx.S8)
    D = tcx.gemm_sp24(vals, hw, B, C)
    torch.cuda.synchronize()
    rows, cols = gemm_sample_coords(M, N, 256, 240, nsamp=65536, seed=1)
    ur = np.unique(rows)
    dense_rows = O.sp24_expand(host_bits(vals[torch.from_numpy(ur).to(DEV)]), host_bits(meta[torch.from_numpy(ur).to(DEV)]), K)
    pos = np.searchsorted(ur, rows)
    ref, _ = O.gemm_samples(O.S8, dense_rows, host_bits(B), host_bits(C[torch.from_numpy(ur).to(DEV)]), pos, cols)
    got = host_bits(D)[rows, cols]
    assert np.array_equal(got, ref)


def _sparse_i8_nodense(M, K, seed):
    pairs = tcxgen.sp24_pairs(M, K, seed, device=DEV)
    meta = tcxgen.sp24_canonical_meta(pairs)
    v = tcxgen.int32_matrix((M, K // 2), seed, tcxgen.STREAM_SPVAL, -128, 126, DEV)
    v = torch.where(v >= 0, v + 1, v)
    return v.to(torch.int8), meta, None


@pytest.mark.parametrize("pairs", [(2, 1), (1, 2), (2, 2)])
def test_i8_sparse_multicast_groups_bit_exact(pairs):
    M, N, K = 768, 1008, 768
    vals, meta, dense = _sparse_i8(M, K, 41)
    B = tcxgen.int8_matrix((N, K), 41, tcxgen.STREAM_B, DEV)
    C = tcxgen.int32_matrix((M, N), 41, tcxgen.STREAM_C, device=DEV)
    hw = tcx.sp24_pack_meta(meta, M, K, ab=tcx.S8)
    D = tcx.gemm_sp24(vals, hw, B, C, pairs=pairs)
    torch.cuda.synchronize()
    ii, jj = np.meshgrid(np.arange(M), np.arange(N), indexing="ij")
    ref, _ = O.gemm_samples(O.S8, host_bits(dense), host_bits(B), host_bits(C), ii.ravel(), jj.ravel())
    assert np.array_equal(host_bits(D).ravel(), ref)
