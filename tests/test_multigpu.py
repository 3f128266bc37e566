"""Multi-rank logic of the N-sharded path on CPU (gloo, world_size 2).

The GEMM is stood in for by an exact int64 matmul (the sharding, not the
kernel, is under test here); the kernel's per-shard parity is covered by the
GPU tests, which call the same C ABI on row slices."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_05232_b200.sharding import gather_cols, gather_rows, shard_rows, shard_size


@pytest.mark.parametrize("n", [4608, 3584, 37888, 7168, 27648, 5120, 300, 1])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_shards_partition_rows(n, world):
    covered = []
    for r in range(world):
        lo, hi = shard_rows(n, world, r)
        assert hi == lo or lo % 128 == 0  # non-empty shards start on a 128-row block
        covered.extend(range(lo, hi))
    assert covered == list(range(n))
    assert shard_size(n, world) % 128 == 0


def test_qwen14b_shards_are_128_multiples():
    """every Qwen2.5-14B shard at 1/2/4/8 GPUs is whole."""
    for n in (7168, 5120, 27648, 13824):
        for world in (1, 2, 4, 8):
            sizes = {shard_rows(n, world, r)[1] - shard_rows(n, world, r)[0] for r in range(world)}
            assert all(s % 128 == 0 for s in sizes)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, k, m, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = torch.Generator().manual_seed(0)
    w = torch.randint(-127, 128, (n, k), generator=g, dtype=torch.int64)  # replicated seed
    x = torch.randint(-127, 128, (m, k), generator=g, dtype=torch.int64)
    lo, hi = shard_rows(n, world, rank)
    y_nm = w[lo:hi] @ x.t()                 # this rank's N x M shard
    full_nm = gather_rows(y_nm, n, world)
    full_mn = gather_cols(y_nm.t().contiguous(), n, world)
    ref = w @ x.t()
    q.put((rank, bool(torch.equal(full_nm, ref)), bool(torch.equal(full_mn, ref.t()))))
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [512, 300])
def test_gloo_world2_shard_and_gather(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, 64, 33, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    assert sorted(r for r, _, _ in results) == [0, 1]
    assert all(a and b for _, a, b in results)
