"""GPU parity: Activation Lifting Ψ (fused_quant_slide, quantize_rows,
lift_rows) through the C ABI vs the CPU oracle — bit-exact codes and scales."""
import numpy as np
import pytest
import torch

from helpers import bf16_bits, lifted_width, pad_cols, round_up
from oracle_lib import DT_BF16, DT_F32, KIND_FP8, KIND_INT8

pytestmark = pytest.mark.gpu

PATTERNS = [(4, 6), (6, 8), (8, 10), (14, 16)]


def rows_f32(rng, rows, cols, scale=5.0):
    x = rng.uniform(-scale, scale, size=(rows, cols)).astype(np.float32)
    x[3 % rows] = 0.0  # an all-zero row -> scale 1 (quantize.hpp:151-153)
    return x


@pytest.mark.parametrize("z,l", PATTERNS)
@pytest.mark.parametrize("kind", [KIND_INT8, KIND_FP8])
def test_fused_quant_slide_f32(slsp, orc, z, l, kind):
    rng = np.random.default_rng(10 * l + kind)
    for cols in (l, 3 * l, 2 * l + 3, 517):  # last two need padding (quantize.hpp:130,162)
        x = rows_f32(rng, 19, cols)
        want_p, want_s = orc.fused_quant_slide(x, z, l, kind, DT_F32)
        kprime = want_p.shape[1] * 4
        kp = round_up(kprime, 16)
        p, s = slsp.fused_quant_slide(torch.from_numpy(x).cuda(), z, l, kind, kp=kp)
        got_p = p.cpu().numpy().view(np.uint32)
        assert np.array_equal(got_p[:, : want_p.shape[1]], want_p), (cols,)
        assert not got_p[:, want_p.shape[1]:].any()
        assert np.array_equal(s.cpu().numpy().view(np.uint32), want_s.view(np.uint32))


@pytest.mark.parametrize("kind", [KIND_INT8, KIND_FP8])
def test_fused_quant_slide_bf16_heavy_tails(slsp, orc, kind):
    """bf16 inputs with 1/7 of rows scaled x30 (SURVEY.md App. A parity probe)."""
    rng = np.random.default_rng(1234 + kind)
    x = rng.standard_normal((700, 4096)).astype(np.float32)
    x[::7] *= 30.0
    bits = bf16_bits(x)
    want_p, want_s = orc.fused_quant_slide(bits, 6, 8, kind, DT_BF16)
    t = torch.from_numpy(bits.view(np.int16)).cuda().view(torch.bfloat16)
    p, s = slsp.fused_quant_slide(t, 6, 8, kind)
    assert np.array_equal(p.cpu().numpy().view(np.uint32)[:, : want_p.shape[1]], want_p)
    assert np.array_equal(s.cpu().numpy().view(np.uint32), want_s.view(np.uint32))


def test_fused_quant_slide_known_answer(slsp):
    """test_quantize.cpp:265-276: 1..8 -> 3 words; unpack == lift(quantize(x))."""
    x = torch.arange(1, 9, dtype=torch.float32, device="cuda").view(1, 8)
    p, s = slsp.fused_quant_slide(x, 6, 8, slsp.QUANT_INT8, kp=16)
    q = [round(v * 127 / 8) for v in range(1, 9)]
    lifted = q[0:4] + q[2:6] + q[4:8]
    got = p.cpu().numpy().view(np.uint32)[0]
    for j in range(3):
        assert [(int(got[j]) >> (8 * d)) & 0xFF for d in range(4)] == lifted[4 * j: 4 * j + 4]
    assert got[3] == 0
    assert s.item() == np.float32(8.0 / 127.0)


def test_fused_quant_slide_rejects_non_finite(slsp):
    x = torch.zeros(4, 16, device="cuda")
    x[2, 5] = float("inf")
    x[3, 0] = float("nan")
    with pytest.raises(slsp.NonFiniteInputError, match="row 2"):
        slsp.fused_quant_slide(x, 6, 8)


@pytest.mark.parametrize("kind", [KIND_INT8, KIND_FP8])
def test_quantize_rows_matches_oracle(slsp, orc, kind):
    rng = np.random.default_rng(55 + kind)
    x = rows_f32(rng, 33, 300)
    want_q, want_s = orc.quantize_rows(x, kind, DT_F32)
    q, s = slsp.quantize_rows(torch.from_numpy(x).cuda(), kind, kpad=304)
    assert np.array_equal(q.cpu().numpy(), pad_cols(want_q, 304))
    assert np.array_equal(s.cpu().numpy().view(np.uint32), want_s.view(np.uint32))


def test_quantize_ties_to_even_and_never_minus_128(slsp):
    """test_quantize.cpp:62-82."""
    x = torch.tensor([[0.5, 1.5, 2.5, -0.5, -1.5, 127.0, -127.0, 0.0]], device="cuda")
    q, s = slsp.quantize_rows(x, slsp.QUANT_INT8, kpad=16)
    assert q.cpu().numpy().view(np.int8)[0, :8].tolist() == [0, 2, 2, 0, -2, 127, -127, 0]
    assert s.item() == 1.0


@pytest.mark.parametrize("z,l", PATTERNS)
def test_lift_rows_bf16_passthrough(slsp, orc, z, l):
    rng = np.random.default_rng(77 + l)
    x = rng.uniform(-1, 1, size=(21, 12 * l)).astype(np.float32)
    bits = bf16_bits(x)
    want = orc.lift_rows(bits, z, l, DT_BF16)
    got = slsp.lift_rows(torch.from_numpy(bits.view(np.int16)).cuda().view(torch.bfloat16), z, l)
    assert np.array_equal(got.view(torch.int16).cpu().numpy().view(np.uint16), want)
    want32 = orc.lift_rows(x, z, l, DT_F32)
    got32 = slsp.lift_rows(torch.from_numpy(x).cuda(), z, l)
    assert np.array_equal(got32.cpu().numpy(), want32)


def test_lift_six_eight_known_answer(slsp):
    """test_quantize.cpp:140-145."""
    x = torch.arange(10, 18, dtype=torch.float32, device="cuda").view(1, 8)
    got = slsp.lift_rows(x, 6, 8).cpu().numpy()[0].tolist()
    assert got == [10, 11, 12, 13, 12, 13, 14, 15, 14, 15, 16, 17]


def test_fused_full_shape_properties(slsp):
    """Full Qwen2.5-7B down_proj activations (M=8192, K=18944): size-independent
    properties — |code| <= 127, scale = absmax/127, and the lifted words equal a
    torch gather of quantize_rows' codes (two independent kernels)."""
    g = torch.Generator(device="cuda").manual_seed(3)
    x = (torch.rand(8192, 18944, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    p, s = slsp.fused_quant_slide(x, 6, 8)
    q, s2 = slsp.quantize_rows(x, slsp.QUANT_INT8)
    assert torch.equal(s, s2)
    amax = x.float().abs().amax(dim=1)
    assert torch.equal(s, (amax.double() / 127.0).float())
    k = 18944
    wins = k // 8 * 3
    j = torch.arange(wins, device="cuda")
    src = ((j // 3) * 8 + 2 * (j % 3))[:, None] + torch.arange(4, device="cuda")[None, :]
    lifted = q[:, :k][:, src.reshape(-1)]
    pb = p.view(torch.uint8)[:, : wins * 4]
    assert torch.equal(pb, lifted)
    assert int(q.view(torch.int8).min()) >= -127
