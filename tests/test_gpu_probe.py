"""tcx_probe (clock-counter latency/throughput) and the tcgen05 numeric-probe
tile path (tcx_mma_tiles_tc05) on B200."""
import numpy as np
import pytest
import torch

import oracle as O
import tcxgen
import paper_2206_02874_b200 as tcx
from parity import host_bits, fp_bound_check

pytestmark = pytest.mark.gpu
DEV = "cuda"


def test_completion_latency_and_identity():
    r = tcx.probe("mma_sync", tcx.F16, tcx.F32, 16, 8, 16, warps=1, ilp=1, iters=2048, repeats=3)
    lat = r["latency_cycles"]
    assert 5 < lat < 200, r
    # the paper's throughput identity: warps * ILP * m*n*k / latency
    assert abs(r["fma_per_clk_per_sm"] - 16 * 8 * 16 / lat) < 1e-6 * r["fma_per_clk_per_sm"]
    assert 300 < r["sm_mhz"] < 2200


def test_throughput_grows_with_warps_and_ilp():
    lo = tcx.probe("mma_sync", tcx.BF16, tcx.F32, 16, 8, 16, warps=1, ilp=1, iters=1024)["fma_per_clk_per_sm"]
    hi = tcx.probe("mma_sync", tcx.BF16, tcx.F32, 16, 8, 16, warps=8, ilp=4, iters=1024)["fma_per_clk_per_sm"]
    assert hi > 2 * lo


@pytest.mark.parametrize("ab,m,n,k", [(tcx.F16, 16, 8, 8), (tcx.TF32, 16, 8, 8), (tcx.TF32, 16, 8, 4),
                                      (tcx.S8, 8, 8, 16), (tcx.S8, 16, 8, 32), (tcx.S8, 16, 8, 16)])
def test_every_dense_shape_runs(ab, m, n, k):
    cd = tcx.S32 if ab == tcx.S8 else tcx.F32
    r = tcx.probe("mma_sync", ab, cd, m, n, k, warps=4, ilp=2, iters=256, repeats=2)
    assert r["latency_cycles"] > 0


@pytest.mark.parametrize("ab,k", [(tcx.F16, 32), (tcx.F16, 16), (tcx.BF16, 32), (tcx.TF32, 16), (tcx.TF32, 8),
                                  (tcx.S8, 64), (tcx.S8, 32)])
def test_every_sparse_shape_runs(ab, k):
    cd = tcx.S32 if ab == tcx.S8 else tcx.F32
    r = tcx.probe("mma_sp_sync", ab, cd, 16, 8, k, warps=4, ilp=2, iters=256, repeats=2)
    assert r["latency_cycles"] > 0


@pytest.mark.parametrize("ab,k,cg,m", [(tcx.BF16, 16, 1, 128), (tcx.BF16, 16, 2, 256), (tcx.TF32, 8, 1, 128),
                                       (tcx.S8, 32, 1, 128), (tcx.S8, 32, 2, 256)])
def test_tc05_rate(ab, k, cg, m):
    """tcgen05 per-SM rate at depth: dense f16/bf16 ~4096, tf32 ~2048, i8 ~8192 FMA/clk/SM"""
    cd = tcx.S32 if ab == tcx.S8 else tcx.F32
    r = tcx.probe("tc05", ab, cd, m, 256, k, cta_group=cg, ilp=16, iters=200, repeats=3)
    expect = {tcx.BF16: 4096, tcx.TF32: 2048, tcx.S8: 8192}[ab]
    assert 0.5 * expect < r["fma_per_clk_per_sm"] < 1.2 * expect, r


def test_tc05_sparse_rate():
    r = tcx.probe("tc05_sp", tcx.F16, tcx.F32, 128, 256, 32, cta_group=1, ilp=16, iters=200, repeats=3)
    assert r["fma_per_clk_per_sm"] > 4096, r     # logical (dense-equivalent) FMAs exceed the dense rate


def _tiles(count, fmt, seed, k=16):
    A = tcxgen.uniform_matrix((count, 16, k), fmt, seed, tcxgen.STREAM_A, device=DEV)
    B = tcxgen.uniform_matrix((count, 8, k), fmt, seed, tcxgen.STREAM_B, device=DEV)
    C = tcxgen.uniform_matrix((count, 16, 8), "f32", seed, tcxgen.STREAM_C, device=DEV)
    return A, B, C


@pytest.mark.parametrize("fmt,k", [("f16", 16), ("bf16", 16), ("tf32", 8), ("tf32", 16)])
@pytest.mark.parametrize("count", [1, 9, 1000])
def test_tiles_tc05_vs_oracle(fmt, k, count):
    A, B, C = _tiles(count, fmt, count + k, k)
    D = tcx.mma_tiles_tc05(A, B, C, tf32=(fmt == "tf32"))
    torch.cuda.synchronize()
    of = {"f16": O.F16, "bf16": O.BF16, "tf32": O.TF32}[fmt]
    ref, absv = O.tiles(of, 16, 8, k, host_bits(A), host_bits(B), host_bits(C))
    fp_bound_check(host_bits(D).reshape(ref.shape), ref, absv, k, f"tc05 tiles {fmt}")


def test_tiles_tc05_integer_bit_exact():
    count = 512
    A = tcxgen.int32_matrix((count, 16, 16), 2, 1, -8, 8, DEV).to(torch.float16)
    B = tcxgen.int32_matrix((count, 8, 16), 2, 2, -8, 8, DEV).to(torch.float16)
    C = tcxgen.int32_matrix((count, 16, 8), 2, 3, -999, 999, DEV).to(torch.float32)
    D = tcx.mma_tiles_tc05(A, B, C)
    torch.cuda.synchronize()
    ref, _ = O.tiles(O.F16, 16, 8, 16, host_bits(A), host_bits(B), host_bits(C))
    assert np.array_equal(host_bits(D).reshape(ref.shape), ref)
