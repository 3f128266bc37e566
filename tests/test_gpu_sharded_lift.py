"""The K-sharded lift on one GPU, world emulated.

Each emulated rank lifts its column slice (shard_cols) with the all-reduced
(here: elementwise max over the ranks' row_absmax) |x|max into EVERY rank's
payload buffer — the same multi-destination kernel the NVLink path runs with
peer pointers, here with all destinations on cuda:0. Every assembled payload
and every rank's scales must equal fused_quant_slide on the full X
(quantize.hpp:122-174), byte for byte.
"""
import pytest
import torch

from paper_2603_05232_b200.sharding import lifted_col, shard_cols

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,k,m", [(2, 3584, 300), (4, 3584, 8192), (8, 18944, 512), (8, 5120, 64),
                                       (3, 4096, 100), (8, 256, 16)])
def test_emulated_sharded_lift_equals_full(slsp, world, k, m):
    g = torch.Generator(device="cuda").manual_seed(world * 7 + k)
    x = (torch.randn(m, k, device="cuda", generator=g) * 3).to(torch.bfloat16)
    x[m // 2, k - 1] = 40.0  # a row max that lives in the last slice only
    kp = slsp.round_up(slsp.lifted_width(k, 6, 8), 256)
    want_p, want_s = slsp.fused_quant_slide(x, 6, 8, kp=kp)
    slices = [shard_cols(k, world, r) for r in range(world)]
    parts = [x[:, k0:k1].contiguous() for k0, k1 in slices]
    amax = torch.stack([slsp.row_absmax(p) if p.shape[1] else torch.zeros(m, device="cuda") for p in parts]).amax(0)
    assert torch.equal(amax, x.float().abs().amax(1))
    bufs = [torch.zeros((m, kp // 4), dtype=torch.int32, device="cuda") for _ in range(world)]
    for r, ((k0, k1), xr) in enumerate(zip(slices, parts)):
        if k1 == k0:
            continue
        dsts = [bufs[r]] + [bufs[j] for j in range(world) if j != r]
        s = slsp.fused_quant_slide_multi(xr, 6, 8, amax, dsts, kp, lifted_col(k0, 6, 8))
        assert torch.equal(s, want_s)
    for b in bufs:
        assert torch.equal(b, want_p)


def test_row_absmax_nan_and_unaligned(slsp):
    x = torch.rand(40, 100, device="cuda").to(torch.bfloat16)
    x[3, 7] = float("nan")
    a = slsp.row_absmax(x[:, 1:].contiguous())
    assert torch.isnan(a[3])
    keep = torch.arange(40, device="cuda") != 3
    assert torch.equal(a[keep], x[:, 1:].float().abs().amax(1)[keep])


def test_multi_rejects_misaligned_slices(slsp):
    x = torch.rand(8, 48, device="cuda").to(torch.bfloat16)  # 48 = 1.5 quads: not whole quads
    buf = torch.zeros((8, 256 // 4), dtype=torch.int32, device="cuda")
    with pytest.raises(slsp.DimensionMismatchError):
        slsp.fused_quant_slide_multi(x, 6, 8, slsp.row_absmax(x), [buf], 256, 0)
