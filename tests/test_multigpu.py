"""Multi-rank logic of the N-sharded path on CPU (gloo, world_size 2).

The GEMM is stood in for by an exact int64 matmul (the sharding, not the
kernel, is under test here); the kernel's per-shard parity is covered by the
GPU tests, which call the same C ABI on row slices."""
import os

import numpy as np
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


# ---- K-sharded lift: the decomposition, checked on CPU ------------------------
def _lift_slice_np(bits: np.ndarray, amax: np.ndarray, l: int = 8) -> np.ndarray:
    """quantize.hpp:151-166 for a column slice of whole blocks, given each row's
    GLOBAL |x|max: r = 127/absmax and codes = nearbyint(x*r) in double, windows
    w = 0..wc-1 of every block at byte offset 2w. (Restatement for the
    multi-rank test; the GPU kernel's parity is test_gpu_sharded_lift.py.)"""
    x = (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    a = amax.astype(np.float64)
    r = np.where(a == 0, 0.0, 127.0 / np.where(a == 0, 1.0, a))
    codes = np.rint(x * r[:, None]).astype(np.int64).astype(np.int8).view(np.uint8)
    wc = (l - 4) // 2 + 1
    idx = np.array([2 * w + d for w in range(wc) for d in range(4)])
    m, kr = codes.shape
    return codes.reshape(m, kr // l, l)[..., idx].reshape(m, kr // l * wc * 4)


def _sharded_lift_worker(rank, world, port, m, k, q):
    import numpy as np

    from oracle_lib import DT_BF16, KIND_INT8, orc
    from paper_2603_05232_b200.sharding import shard_cols

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)  # same X on every rank; each keeps only its slice
    x = rng.standard_normal((m, k)).astype(np.float32) * 3
    bits = (x.view(np.uint32) >> 16).astype(np.uint16)  # truncation: any bf16 pattern will do
    k0, k1 = shard_cols(k, world, rank)
    mine = bits[:, k0:k1]
    xf = (mine.astype(np.uint32) << 16).view(np.float32)
    amax = torch.from_numpy(np.abs(xf).max(axis=1) if k1 > k0 else np.zeros(m, np.float32))
    dist.all_reduce(amax, op=dist.ReduceOp.MAX)  # M floats, exact
    part = torch.from_numpy(_lift_slice_np(mine, amax.numpy()))
    parts = [None] * world
    dist.all_gather_object(parts, part)  # stands in for the peer writes (same bytes, same columns)
    full = torch.cat(parts, dim=1).numpy()
    want, scales = orc().fused_quant_slide(bits, 6, 8, KIND_INT8, DT_BF16)
    sc = np.where(amax.numpy() == 0, 1.0, amax.numpy().astype(np.float64) / 127.0).astype(np.float32)
    q.put((rank, bool(np.array_equal(full, want.view(np.uint8))), bool(np.array_equal(sc, scales))))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,k", [(2, 3584), (2, 4096 + 32)])
def test_gloo_sharded_lift_matches_oracle(world, k):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_lift_worker, args=(r, world, port, 37, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    assert sorted(r for r, _, _ in results) == list(range(world))
    assert all(a and b for _, a, b in results)
