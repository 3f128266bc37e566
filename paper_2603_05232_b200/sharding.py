"""Output-feature (N) sharding of the sparse linear across GPUs.

Rank r owns weight rows [lo, hi) of every layer (multiples of `align` so each
shard is whole 128-row metadata blocks); activations are replicated and lifted
locally, so the GEMM itself needs no collective. `gather_rows` /
`gather_cols` are the optional NCCL all-gathers for a consumer that needs the
full output row (one process per GPU, torch.distributed, backend nccl; the
same code runs on gloo for the CPU tests).
"""
from __future__ import annotations

import torch


def shard_rows(n: int, world: int, rank: int, align: int = 128) -> tuple[int, int]:
    """[lo, hi) of the rows owned by `rank`; equal `align`-multiple shards, the
    last one possibly shorter or empty."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    per = -(-n // world)
    per = -(-per // align) * align
    lo = min(n, rank * per)
    return lo, min(n, lo + per)


def shard_size(n: int, world: int, align: int = 128) -> int:
    per = -(-n // world)
    return -(-per // align) * align


def gather_rows(y_shard: torch.Tensor, n_total: int, world: int, group=None) -> torch.Tensor:
    """All-gather N x M (reference-orientation) shards into the full n_total x M."""
    import torch.distributed as dist

    per = shard_size(n_total, world)
    m = y_shard.shape[1]
    buf = torch.zeros((per, m), dtype=y_shard.dtype, device=y_shard.device)
    buf[: y_shard.shape[0]] = y_shard
    out = torch.empty((per * world, m), dtype=y_shard.dtype, device=y_shard.device)
    dist.all_gather_into_tensor(out, buf, group=group)
    return out[:n_total]


def gather_cols(y_shard: torch.Tensor, n_total: int, world: int, group=None) -> torch.Tensor:
    """All-gather M x N (token-major) shards into the full M x n_total."""
    import torch.distributed as dist

    per = shard_size(n_total, world)
    m = y_shard.shape[0]
    buf = torch.zeros((per, m), dtype=y_shard.dtype, device=y_shard.device)
    buf[: y_shard.shape[1]] = y_shard.t()
    out = torch.empty((per * world, m), dtype=y_shard.dtype, device=y_shard.device)
    dist.all_gather_into_tensor(out, buf, group=group)
    return out[:n_total].t().contiguous()
