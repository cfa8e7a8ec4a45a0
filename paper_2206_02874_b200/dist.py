"""Row-sharded GEMM across GPUs (north_star: "Large GEMMs are partitioned across the
8xB200 box by sharding rows of A (and C/D). B is replicated with one NCCL broadcast over NVLink,
and an NCCL all-gather of D runs only for verification").

Rank r owns rows [m0_r, m1_r) of A, C and D (and of sA + metadata for 2:4).  Row sharding changes no
per-element arithmetic, so the sharded D is bit-identical to the 1-GPU D for the same kernel
configuration (tests/test_gpu_dist.py checks it on one GPU; tests/test_dist_gloo.py checks the
plumbing with world_size 2 on CPU).  The only data-path collective is the one-time broadcast of
the replicated operand B; timing is reduced with MAX over ranks.  torch.distributed (NCCL on the
box, gloo in CPU tests) is the plumbing; every GEMM runs in libtcx.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

ROW_ALIGN = 256   # one CTA-pair output tile: no tile straddles two ranks


def row_shard(M: int, world: int, rank: int, align: int = ROW_ALIGN):
    """[m0, m1) of rank `rank`: contiguous, disjoint, covering [0, M); every boundary is a
    multiple of `align` except the final M (the last non-empty rank takes the ragged tail)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    blocks = (M + align - 1) // align
    b0 = blocks * rank // world
    b1 = blocks * (rank + 1) // world
    return min(M, b0 * align), min(M, b1 * align)


def shard_plan(M: int, world: int, rank: int, scaling: str = "strong", seed: int = 0):
    """(m0, m1, row_seed, M_total) for this rank.  strong: the M-row problem split by rows
    (row_shard), rows drawn from the one seeded matrix; weak: every rank owns a full M-row block of a
    world*M-row problem, its rows drawn with seed + 1000*rank (bench.py's default at N > 1)."""
    if scaling not in ("strong", "weak"):
        raise ValueError("scaling must be 'strong' or 'weak'")
    if scaling == "weak" and world > 1:
        if not 0 <= rank < world:
            raise ValueError("bad world/rank")
        return 0, M, seed + 1000 * rank, M * world
    m0, m1 = row_shard(M, world, rank)
    return m0, m1, seed, M


def broadcast_replicated(t: torch.Tensor, src: int = 0, group=None) -> torch.Tensor:
    """the one data-path collective: replicate B from `src` to every rank (NCCL over NVLink)."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(t, src=src, group=group)
    return t


def gather_rows(local: torch.Tensor, M: int | None = None, group=None) -> torch.Tensor:
    """verification only: all-gather every rank's row block of D, in rank order, into one matrix.
    The block sizes are exchanged first, so any shard plan works (strong: the M x N matrix; weak:
    the world x M-row problem); M, if given, is checked against the gathered row count."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return local
    rank = dist.get_rank(group)
    N = local.shape[1]
    mine = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
    all_sizes = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(all_sizes, mine, group=group)
    sizes = [int(t.item()) for t in all_sizes]
    if M is not None and sum(sizes) != M:
        raise ValueError(f"gather_rows: shards hold {sum(sizes)} rows, expected {M}")
    maxr = max(sizes)
    pad = torch.zeros(maxr, N, dtype=local.dtype, device=local.device)
    pad[: sizes[rank]] = local
    out = torch.empty(world * maxr, N, dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    return torch.cat([out[r * maxr: r * maxr + sizes[r]] for r in range(world)], dim=0)


def max_over_ranks(x: float, device=None, group=None) -> float:
    """device-timed numbers are reported as the max over ranks (bench contract)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sharded_gemm(A_local, B, C_local=None, D_local=None, local_fn=None, **kw):
    """D_local = A_local x B + C_local on this rank (B already replicated).
    local_fn defaults to the libtcx GEMM (paper_2206_02874_b200.gemm); tests may inject another."""
    if local_fn is None:
        from . import gemm as local_fn
    return local_fn(A_local, B, C_local, D_local, **kw)


def sharded_gemm_sp24(vals_local, meta_hw_local, B, C_local=None, D_local=None, local_fn=None, **kw):
    if local_fn is None:
        from . import gemm_sp24 as local_fn
    return local_fn(vals_local, meta_hw_local, B, C_local, D_local, **kw)
