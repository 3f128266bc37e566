"""End-to-end ShardedLift with two real processes (gloo for the host
collectives) sharing cuda:0: the payload buffers are exchanged as CUDA IPC
handles and each rank's lift kernel writes its K-slice into both ranks'
payloads through the mapped peer pointer — the NVLink path of DESIGN §7,
here with the peer on the same device. Both payloads must equal
fused_quant_slide on the full X (quantize.hpp:122-174)."""
import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, m, k, q):
    import torch.distributed as dist

    import paper_2603_05232_b200 as slsp
    from paper_2603_05232_b200.sharding import ShardedLift

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    g = torch.Generator(device="cuda").manual_seed(1)
    x = (torch.randn(m, k, device="cuda", generator=g) * 2).to(torch.bfloat16)
    kp = slsp.round_up(slsp.lifted_width(k, 6, 8), 256)
    sl = ShardedLift(m, k, 6, 8, kp, world, rank, torch.device("cuda", 0))
    payload, scales = sl(x[:, sl.k0:sl.k1].contiguous(), check=True)
    torch.cuda.synchronize()
    dist.barrier()
    want_p, want_s = slsp.fused_quant_slide(x, 6, 8, kp=kp)
    ok = bool(torch.equal(payload, want_p)) and bool(torch.equal(scales, want_s))
    dist.barrier()
    sl.close()
    q.put((rank, ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,k", [(2, 3584), (3, 5120)])
def test_sharded_lift_ipc_two_processes(slsp, world, k):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 1000, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    assert sorted(r for r, _ in res) == list(range(world))
    assert all(ok for _, ok in res)
