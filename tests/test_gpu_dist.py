"""Row sharding on the GPU: the shards computed separately are bit-identical to the 1-GPU D
(row sharding changes no per-element arithmetic).  One GPU emulates P ranks by
running each rank's slice through the same kernel (no inter-rank waiting is involved)."""
import pytest
import torch

import tcxgen
import paper_2206_02874_b200 as tcx
from paper_2206_02874_b200 import dist as tdist

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.mark.parametrize("P", [2, 4, 8])
def test_int8_row_shards_bit_identical(P):
    M, N, K = 4096, 2048, 1024
    A = tcxgen.int8_matrix((M, K), 1, 1, DEV)
    B = tcxgen.int8_matrix((N, K), 1, 2, DEV)
    C = tcxgen.int32_matrix((M, N), 1, 3, device=DEV)
    full = tcx.gemm(A, B, C)
    parts = []
    for r in range(P):
        m0, m1 = tdist.row_shard(M, P, r)
        parts.append(tdist.sharded_gemm(A[m0:m1], B, C[m0:m1]))
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(parts), full)


@pytest.mark.parametrize("P", [2, 8])
def test_bf16_and_sparse_row_shards_bit_identical(P):
    M, N, K = 4096, 1024, 2048
    A = tcxgen.normal_matrix((M, K), "bf16", 2, 1, DEV)
    B = tcxgen.normal_matrix((N, K), "bf16", 2, 2, DEV)
    full = tcx.gemm(A, B)
    parts = [tdist.sharded_gemm(A[m0:m1], B) for m0, m1 in (tdist.row_shard(M, P, r) for r in range(P))]
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(parts).view(torch.int32), full.view(torch.int32))
    vals, meta = tcxgen.sp24_problem(M, K, 3, "f16", DEV)
    Bs = tcxgen.normal_matrix((N, K), "f16", 3, 2, DEV)
    hw = tcx.sp24_pack_meta(meta, M, K)
    fulls = tcx.gemm_sp24(vals, hw, Bs)
    parts = []
    for r in range(P):
        m0, m1 = tdist.row_shard(M, P, r)
        parts.append(tdist.sharded_gemm_sp24(vals[m0:m1], tcx.sp24_pack_meta(meta[m0:m1].contiguous(), m1 - m0, K), Bs))
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(parts).view(torch.int32), fulls.view(torch.int32))
