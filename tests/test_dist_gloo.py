"""The N>1 row-sharding path with world_size 2 over gloo on CPU: partition math, the one-time
broadcast of the replicated B, the verification all-gather, and max-over-ranks timing.  The
local GEMM is injected (a float64 CPU matmul) because the CPU has no tensor cores; the GPU side of
the same path is tests/test_gpu_dist.py."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2206_02874_b200 import dist as tdist


def test_row_shard_partition():
    for M in (1, 255, 256, 257, 8192, 16384, 65536, 1000):
        for world in (1, 2, 3, 4, 8):
            spans = [tdist.row_shard(M, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == M
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0
            for m0, m1 in spans:
                assert m0 % 256 == 0 and (m1 % 256 == 0 or m1 == M) and m0 <= m1
    # the configs of BASELINE.json shard evenly at 2/4/8
    for M in (16384, 65536, 8192):
        for world in (2, 4, 8):
            assert len({m1 - m0 for m0, m1 in (tdist.row_shard(M, world, r) for r in range(world))}) == 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        M, N, K = 1000, 48, 64
        g = torch.Generator().manual_seed(7)
        A = torch.randn(M, K, generator=g, dtype=torch.float64)
        Bfull = torch.randn(N, K, generator=g, dtype=torch.float64)
        C = torch.randn(M, N, generator=g, dtype=torch.float64)
        B = Bfull.clone() if rank == 0 else torch.zeros(N, K, dtype=torch.float64)
        tdist.broadcast_replicated(B, src=0)
        assert torch.equal(B, Bfull)
        m0, m1 = tdist.row_shard(M, world, rank)
        local = lambda a, b, c, d, **kw: a @ b.T + c                       # injected stand-in
        Dl = tdist.sharded_gemm(A[m0:m1], B, C[m0:m1], local_fn=local)
        D = tdist.gather_rows(Dl, M)
        ok = torch.equal(D, A @ Bfull.T + C)
        t = tdist.max_over_ranks(float(rank + 1))
        q.put((rank, ok, t))
    finally:
        dist.destroy_process_group()


def _strong_worker(rank, world, port, q):
    """bench.py's default multi-GPU mode (strong scaling): the config's rows split by shard_plan,
    uneven when the 256-row blocks do not divide evenly; whole-job work = SUM over ranks of each
    rank's own FLOPs (not world x this rank's), time = MAX over ranks; weak shards gather too."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        M, N, K = 1280, 32, 48                     # 5 blocks of 256 rows over 2 ranks: 512 + 768
        g = torch.Generator().manual_seed(11)
        A = torch.randn(M, K, generator=g, dtype=torch.float64)
        B = torch.randn(N, K, generator=g, dtype=torch.float64) if rank == 0 else torch.zeros(N, K, dtype=torch.float64)
        tdist.broadcast_replicated(B, src=0)
        m0, m1, seed, total = tdist.shard_plan(M, world, rank, "strong")
        local = lambda a, b, c, d, **kw: a @ b.T
        Dl = tdist.sharded_gemm(A[m0:m1], B, local_fn=local)
        flops = torch.tensor([2.0 * (m1 - m0) * N * K], dtype=torch.float64)
        dist.all_reduce(flops, op=dist.ReduceOp.SUM)
        D = tdist.gather_rows(Dl, M)
        ok = torch.equal(D, A @ B.T) and float(flops.item()) == 2.0 * M * N * K and total == M
        # weak plan: each rank a full M-row block of its own; gather_rows stacks them in rank order
        w0, w1, wseed, wtotal = tdist.shard_plan(M, world, rank, "weak")
        Aw = torch.randn(M, K, generator=torch.Generator().manual_seed(wseed), dtype=torch.float64)
        Dw = tdist.gather_rows(Aw @ B.T, wtotal)
        ref = torch.cat([torch.randn(M, K, generator=torch.Generator().manual_seed(tdist.shard_plan(M, world, r, "weak")[2]),
                                     dtype=torch.float64) for r in range(world)]) @ B.T
        ok = ok and torch.equal(Dw, ref) and (w0, w1) == (0, M)
        q.put((rank, ok, m1 - m0))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_gloo_world2_strong_plan_uneven_shards():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_strong_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=90) for _ in range(world))
    for p in ps:
        p.join(timeout=30)
    assert all(ok for _, ok, _ in res), res
    assert [rows for _, _, rows in res] == [512, 768]


@pytest.mark.timeout(120)
def test_gloo_world2_broadcast_shard_gather():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=90) for _ in range(world)]
    for p in ps:
        p.join(timeout=30)
    assert all(ok for _, ok, _ in res)
    assert all(t == 2.0 for _, _, t in res)       # max over ranks


def test_shard_plan_weak_and_strong():
    """bench.py's two multi-GPU modes: strong splits the config's rows (row_shard, one seed); weak
    gives every rank a full config-sized block of a world-times taller problem with its own row seed,
    so per-GPU work is fixed and no two ranks hold the same rows."""
    for M in (8192, 16384, 65536):
        for world in (1, 2, 4, 8):
            strong = [tdist.shard_plan(M, world, r, "strong") for r in range(world)]
            assert sum(m1 - m0 for m0, m1, _, _ in strong) == M
            assert all(seed == 0 and total == M for _, _, seed, total in strong)
            weak = [tdist.shard_plan(M, world, r, "weak") for r in range(world)]
            assert all((m0, m1) == (0, M) for m0, m1, _, _ in weak)
            assert all(total == M * world for *_, total in weak)
            seeds = [seed for _, _, seed, _ in weak]
            assert len(set(seeds)) == world and (world > 1 or seeds == [0])
    with pytest.raises(ValueError):
        tdist.shard_plan(256, 2, 0, "diagonal")
