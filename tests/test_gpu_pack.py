"""GPU parity: weight transform Φ (pack_matrix, compress, fused pack_compress,
magnitude_prune) through the C ABI vs the CPU oracle — bit-exact."""
import numpy as np
import pytest
import torch

from helpers import compliant_matrix, lifted_width, mma_format, random_pruned_int8, round_up
from oracle_lib import DT_BF16, DT_E4M3, DT_F32, DT_I8

pytestmark = pytest.mark.gpu

PATTERNS = [(4, 6), (6, 8), (8, 10), (14, 16)]


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("z,l", PATTERNS)
def test_pack_matrix_matches_oracle(slsp, orc, z, l):
    rng = np.random.default_rng(100 + l)
    w = compliant_matrix(rng, 96, 40, z, l)
    got = slsp.pack_matrix(dev(w), z, l).cpu().numpy()
    want = orc.pack_matrix(w, z, l, DT_I8)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("z,l", PATTERNS)
def test_compress_matches_oracle(slsp, orc, z, l):
    rng = np.random.default_rng(200 + l)
    w = compliant_matrix(rng, 64, 24, z, l)
    slided = orc.pack_matrix(w, z, l, DT_I8)
    v, c = slsp.compress(dev(slided))
    wv, wc = orc.compress(slided, DT_I8)
    assert np.array_equal(v.cpu().numpy(), wv)
    assert np.array_equal(c.cpu().numpy(), wc)


@pytest.mark.parametrize("z,l", PATTERNS)
@pytest.mark.parametrize("exact", [False, True])
def test_pack_compress_int8_mma_format(slsp, orc, z, l, exact):
    rng = np.random.default_rng(300 + l + 7 * exact)
    w = compliant_matrix(rng, 130, 64, z, l, exact_z=exact)
    kp = round_up(lifted_width(w.shape[1], z, l), 256)
    pw = slsp.pack_compress(dev(w), z, l, kp=kp)
    vals, codes = orc.compress(orc.pack_matrix(w, z, l, DT_I8), DT_I8)
    want_v, want_m = mma_format(vals, codes, kp)
    assert np.array_equal(pw.values.cpu().numpy(), want_v)
    assert np.array_equal(pw.meta.cpu().numpy(), want_m)


def test_pack_compress_exact_kprime_layout(slsp, orc):
    """kp == K' reproduces compress() + pack_codes row by row (no padding)."""
    z, l = 6, 8
    rng = np.random.default_rng(7)
    w = compliant_matrix(rng, 50, 32, z, l)  # K' = 384, kp % 8 == 0
    kp = lifted_width(w.shape[1], z, l)
    pw = slsp.pack_compress(dev(w), z, l, kp=kp)
    vals, codes = orc.compress(orc.pack_matrix(w, z, l, DT_I8), DT_I8)
    assert np.array_equal(pw.values.cpu().numpy(), vals)
    packed = np.stack([orc.pack_codes(codes[r]) for r in range(codes.shape[0])])
    assert np.array_equal(pw.meta.cpu().numpy(), packed)


def test_pack_compress_pads_ragged_k(slsp, orc):
    """cols not a multiple of l: the tail block is zero-padded (4:6 on K=3584-like shapes)."""
    z, l = 4, 6
    rng = np.random.default_rng(8)
    w = compliant_matrix(rng, 40, 20, z, l)[:, :116]  # 116 = 19*6 + 2
    padded = np.zeros((40, 120), np.int8)
    padded[:, :116] = w
    kp = round_up(lifted_width(116, z, l), 256)
    pw = slsp.pack_compress(dev(w), z, l, kp=kp)
    vals, codes = orc.compress(orc.pack_matrix(padded, z, l, DT_I8), DT_I8)
    want_v, want_m = mma_format(vals, codes, kp)
    assert np.array_equal(pw.values.cpu().numpy(), want_v)
    assert np.array_equal(pw.meta.cpu().numpy(), want_m)


def test_pack_bf16_and_negative_zero(slsp, orc):
    z, l = 6, 8
    rng = np.random.default_rng(9)
    mask = compliant_matrix(rng, 64, 32, z, l) != 0
    vals = rng.uniform(-2, 2, size=mask.shape).astype(np.float32)
    w = np.where(mask, vals, 0).astype(np.float32)
    bits = (w.view(np.uint32) >> 16).astype(np.uint16)
    bits[~mask & (rng.random(mask.shape) < 0.3)] = 0x8000  # -0.0 counts as zero (matrix.hpp:63-67)
    t = torch.from_numpy(bits.view(np.int16)).cuda().view(torch.bfloat16)
    kp = round_up(lifted_width(w.shape[1], z, l), 256)
    pw = slsp.pack_compress(t, z, l, kp=kp)
    ov, oc = orc.compress(orc.pack_matrix(bits, z, l, DT_BF16), DT_BF16)
    want_v, want_m = mma_format(ov, oc, kp)
    assert np.array_equal(pw.values.view(torch.int16).cpu().numpy().view(np.uint16), want_v)
    assert np.array_equal(pw.meta.cpu().numpy(), want_m)
    sl = slsp.pack_matrix(t, z, l).view(torch.int16).cpu().numpy().view(np.uint16)
    assert np.array_equal(sl, orc.pack_matrix(bits, z, l, DT_BF16))


def test_pack_e4m3_codes(slsp, orc):
    z, l = 6, 8
    rng = np.random.default_rng(10)
    mask = compliant_matrix(rng, 64, 32, z, l) != 0
    codes = rng.integers(1, 0x7F, size=mask.shape).astype(np.uint8) | (rng.integers(0, 2, size=mask.shape) << 7).astype(np.uint8)
    w = np.where(mask, codes, np.where(rng.random(mask.shape) < 0.5, 0x80, 0)).astype(np.uint8)
    kp = round_up(lifted_width(w.shape[1], z, l), 256)
    pw = slsp.pack_compress(dev(w).view(torch.float8_e4m3fn), z, l, kp=kp)
    ov, oc = orc.compress(orc.pack_matrix(w, z, l, DT_E4M3), DT_E4M3)
    want_v, want_m = mma_format(ov, oc, kp)
    assert np.array_equal(pw.values.view(torch.uint8).cpu().numpy(), want_v)
    assert np.array_equal(pw.meta.cpu().numpy(), want_m)


def test_pack_reports_lowest_row_and_block(slsp):
    """pack.hpp:196-202 / test_pack.cpp:225-237: 'row 1, block 1' for a 7-nonzero block."""
    w = np.zeros((4, 32), np.int8)
    w[1, 8:15] = 1
    w[3, 0:8] = 1
    with pytest.raises(slsp.NotCompliantError, match=r"row 1, block 1"):
        slsp.pack_matrix(dev(w), 6, 8)
    with pytest.raises(slsp.NotCompliantError, match=r"row 1, block 1"):
        slsp.pack_compress(dev(w), 6, 8)


def test_pack_matrix_rejects_bad_length(slsp):
    with pytest.raises(slsp.DimensionMismatchError):
        slsp.pack_matrix(dev(np.zeros((2, 9), np.int8)), 6, 8)


def test_compress_rejects_overfull_window(slsp):
    s = np.zeros((3, 8), np.int8)
    s[2, 4:7] = 1
    with pytest.raises(slsp.NotCompliantError, match=r"window \(2, 1\)"):
        slsp.compress(dev(s))


@pytest.mark.parametrize("dt", ["i8", "f32"])
def test_magnitude_prune_matches_oracle(slsp, orc, dt):
    rng = np.random.default_rng(11)
    if dt == "i8":
        w = rng.integers(-127, 128, size=(64, 240)).astype(np.int8)
        w[:, ::7] = w[:, 1::7][:, : w[:, ::7].shape[1]]  # magnitude ties
        code = DT_I8
    else:
        w = rng.uniform(-1, 1, size=(64, 240)).astype(np.float32)
        code = DT_F32
    for z, l in PATTERNS[:3]:
        got = slsp.magnitude_prune(dev(w), z, l).cpu().numpy()
        assert np.array_equal(got, orc.magnitude_prune(w, z, l, code))


def test_prune_then_pack_full_shape_roundtrip(slsp):
    """Full Qwen2.5-7B o_proj shape: prune -> pack -> every window <= 2 nnz and
    the unpacked values reproduce W exactly (size-independent property)."""
    z, l = 6, 8
    g = torch.Generator(device="cuda").manual_seed(0)
    w = torch.randint(-127, 128, (3584, 3584), dtype=torch.int8, device="cuda", generator=g)
    w = slsp.magnitude_prune(w, z, l)
    pw = slsp.pack_compress(w, z, l)
    slided = slsp.pack_matrix(w, z, l)
    v, c = slsp.compress(slided)
    kprime = slided.shape[1]
    assert torch.equal(pw.values[:, : kprime // 2], v)
    # unslide on the GPU with torch: scatter values back to their source positions
    n = w.shape[0]
    wins = kprime // 4
    codes = c.view(n, wins, 2).long()
    win = torch.arange(wins, device="cuda")
    src_col = (win // 3) * 8 + 2 * (win % 3)
    rec = torch.zeros(w.shape, dtype=torch.int32, device="cuda")
    vals = v.view(n, wins, 2).to(torch.int32)
    for k in range(2):
        rec.scatter_add_(1, (src_col[None, :] + codes[:, :, k]).expand(n, wins), vals[:, :, k].contiguous())
    assert torch.equal(rec, w.to(torch.int32))
    # every 4-window of the packed format holds <= 2 nonzeros by construction;
    # check the metadata decodes to strictly increasing position pairs
    meta = pw.meta[:, : kprime // 8].to(torch.int32)
    nib = torch.stack([(meta >> (4 * i)) & 0xF for i in range(2)], dim=-1).reshape(n, -1)
    assert bool(((nib & 3) < (nib >> 2)).all())


def test_tile_meta_layout(slsp):
    """slsp_tile_meta: 4 KB blocks per (128-row block, 256-wide k-stage), two
    128x16B atoms each; padding rows canonical 0x44 (include/slsp_b200.h)."""
    rng = np.random.default_rng(12)
    rows, kp = 300, 768
    meta = rng.integers(0, 256, size=(rows, kp // 8)).astype(np.uint8)
    got = slsp.tile_meta(dev(meta), rows, kp).cpu().numpy()
    nb = -(-rows // 128)
    padded = np.full((nb * 128, kp // 8), 0x44, np.uint8)
    padded[:rows] = meta
    want = padded.reshape(nb, 128, kp // 256, 2, 16).transpose(0, 2, 3, 1, 4).reshape(-1)
    assert np.array_equal(got, want)
