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


# ---- K-sharded lift (the layer's input arrives feature-sharded) ------------------------
def shard_cols(k: int, world: int, rank: int, l: int = 8) -> tuple[int, int]:
    """[k0, k1) of the input columns rank `rank` holds and lifts: equal slices
    of whole quads (4 blocks of l, so every window and every 16-byte lifted
    vector belongs to one rank), the last one possibly shorter or empty."""
    return shard_rows(k, world, rank, align=4 * l)


def lifted_col(k0: int, z: int, l: int) -> int:
    """Byte column of source column k0 (a block boundary) in the INT8/FP8 payload row."""
    wc = (l - 4) // 2 + 1
    return k0 // l * wc * 4


class ShardedLift:
    """fused_quant_slide of an X whose columns are spread over the ranks,
    assembled in every rank's full payload without an all-gather.

    Rank r holds X[:, k0:k1] (shard_cols). Per call: its per-row |x|max
    (row_absmax, or the tok_amax its own sparse_gemm folded when it produced
    the slice) -> all_reduce(MAX) over the group (M floats; exact) ->
    fused_quant_slide_multi writes the slice's lifted bytes into every rank's
    payload (its own + the peers', mapped once through CUDA IPC), then a
    stream-ordered barrier (a 1-element all_reduce) before the GEMM reads the
    payload. Result on every rank: exactly fused_quant_slide(X) (the
    quantization of each element depends only on its row's global |x|max,
    quantize.hpp:151-163, and every window lies inside one quad). NVLink
    traffic: each rank sends its 1.5-byte lifted slice to world-1 peers
    (1.5 B/elem, vs 2 B/elem for an all-gather of BF16 X followed by a
    replicated lift).
    """

    def __init__(self, m: int, k: int, z: int, l: int, kp: int, world: int, rank: int, device,
                 group=None, kind: int | None = None):
        import torch.distributed as dist

        from . import _native as nat

        self.m, self.k, self.z, self.l, self.kp = m, k, z, l, kp
        self.world, self.rank, self.group = world, rank, group
        self.kind = nat.QUANT_INT8 if kind is None else kind
        self.k0, self.k1 = shard_cols(k, world, rank, l)
        self.col = lifted_col(self.k0, z, l)
        self.payload = torch.zeros((m, kp // 4), dtype=torch.int32, device=device)  # padding stays zero
        self.payload.slsp_kind = self.kind
        self.payload.slsp_pattern = (z, l)
        self.scales = torch.empty(m, dtype=torch.float32, device=device)
        self.amax = torch.empty(m, dtype=torch.float32, device=device)
        self.flag = torch.zeros(1, dtype=torch.float32, device=device)
        self.peers: list[int] = []
        self.mapped: list[tuple[int, int]] = []
        if world > 1:
            handles = [None] * world
            dist.all_gather_object(handles, nat.ipc_handle(self.payload), group=group)
            self.mapped = [nat.ipc_open(handles[r]) for r in range(world) if r != rank]
            self.peers = [ptr for _, ptr in self.mapped]
        self.dsts = [self.payload] + self.peers

    def __call__(self, x_slice: torch.Tensor, absmax: torch.Tensor | None = None, check: bool = False):
        import torch.distributed as dist

        from . import _native as nat

        if x_slice.shape != (self.m, self.k1 - self.k0):
            raise ValueError(f"rank {self.rank} expects its slice of {self.m} x {self.k1 - self.k0}")
        a = self.amax
        if absmax is not None:
            a.copy_(absmax)
        else:
            nat.row_absmax(x_slice, out=a)
        if self.world > 1:
            dist.all_reduce(a, op=dist.ReduceOp.MAX, group=self.group)
        if self.k1 > self.k0:
            nat.fused_quant_slide_multi(x_slice, self.z, self.l, a, self.dsts, self.kp, self.col, kind=self.kind,
                                        scales=self.scales, check=check)
        if self.world > 1:  # every slice has landed in every payload before any GEMM reads one
            dist.all_reduce(self.flag, group=self.group)
        return self.payload, self.scales

    def close(self) -> None:
        from . import _native as nat

        for base, _ in self.mapped:
            nat.ipc_close(base)
        self.peers, self.mapped = [], []
