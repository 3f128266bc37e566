"""GPU parity of exactly what bench.py times, against the CPU oracle.

bench.py's step (BASELINE.json configs[1]) runs, per Qwen2.5-7B linear layer
at M = 8192: slsp_fused_quant_slide on bf16 X, then slsp_sparse_gemm with the
BF16 [N][M] dequant epilogue — at M = 8192 the two-subtile (512 weight rows x
224 tokens, register-staged epilogue, TMA-box stores) configuration with a
128-token tail tile. These tests run that exact call on full-size inputs and
compare sampled blocks bit for bit with the oracle, rebuilt from scratch on
the CPU from the same W and X:

  vals, codes = compress(pack_matrix(W[rows]))           pack.hpp:171-204, gemm.hpp:70-110
  payload, s  = fused_quant_slide(X[tokens])             quantize.hpp:122-174
  acc         = sparse_gemm(vals, codes, payload)         gemm.hpp:199-233 (int32)
  y           = bf16((acc * s_ch[n]) * s_tok[t])          a18 epilogue, oracle/slsp_oracle.c

Rows are independent (gemm.hpp:215) and so are tokens, so sampled blocks pin
the whole output: the row blocks cover both CTAs of a pair and both M-subtiles
of a 512-row tile (first, a middle and the last 512-row block); the token
blocks cover the first two 224-token tiles, two tiles in the middle and the
last full tile plus the 128-token tail tile.
"""
import numpy as np
import pytest
import torch

from oracle_lib import DT_BF16, DT_I8, KIND_INT8

pytestmark = pytest.mark.gpu

QWEN7B = [("qkv", 4608, 3584), ("o", 3584, 3584), ("gate_up", 37888, 3584), ("down", 3584, 18944)]
M = 8192


def sample_rows(n):
    mid = (n // 2) // 512 * 512
    return np.unique(np.concatenate([np.arange(0, 512), np.arange(mid, mid + 512), np.arange(n - 512, n)]))


def sample_tokens(m):
    mid = (m // 2) // 224 * 224
    return np.unique(np.concatenate([np.arange(0, 448), np.arange(mid, mid + 448), np.arange(m - 352, m)]))


def ix(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(a).cuda()


def bf16_bits(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def layer_inputs(slsp, n, k, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    w = slsp.magnitude_prune(torch.randint(-127, 128, (n, k), dtype=torch.int8, device="cuda", generator=g), 6, 8)
    x = (torch.rand(M, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    s_ch = (torch.rand(n, device="cuda", generator=g) * 0.01 + 0.001).float()
    return w, x, s_ch


def oracle_block(orc, w, x, rows, toks):
    vals, codes = orc.compress(orc.pack_matrix(w[ix(rows)].cpu().numpy(), 6, 8, DT_I8), DT_I8)
    payload, scales = orc.fused_quant_slide(bf16_bits(x[ix(toks)]), 6, 8, KIND_INT8, DT_BF16)
    return vals, codes, payload, scales


@pytest.mark.parametrize("name,n,k", QWEN7B, ids=[q[0] for q in QWEN7B])
def test_benched_step_bf16_nm_vs_oracle(slsp, orc, name, n, k):
    """The bench's exact call sequence and configuration, full size, sampled
    blocks bit-exact vs the oracle: packed weights, payload words, scale bits
    and the BF16 outputs of the two-subtile register-staged epilogue."""
    w, x, s_ch = layer_inputs(slsp, n, k, seed=n + k)
    pw = slsp.pack_compress(w, 6, 8)
    cfg = slsp.sparse_gemm_config(pw, M, slsp.OUT_BF16_NM)
    assert (cfg["subtiles"], cfg["tokens_per_tile"], cfg["epilogue"], cfg["ksplit"]) == (2, 224, 1, 1), cfg
    payload, s_tok = slsp.fused_quant_slide(x, 6, 8, kp=pw.kp, check=False)
    y = slsp.sparse_gemm(pw, payload, s_ch=s_ch, s_tok=s_tok, out_mode=slsp.OUT_BF16_NM)
    torch.cuda.synchronize()

    rows, toks = sample_rows(n), sample_tokens(M)
    vals, codes, pay_o, sc_o = oracle_block(orc, w, x, rows, toks)
    kprime = vals.shape[1] * 2
    # the offline packer Φ and the lift, on the sampled rows / tokens
    assert np.array_equal(pw.values[ix(rows)].cpu().numpy()[:, : kprime // 2], vals)
    assert np.array_equal(payload[ix(toks)].cpu().numpy().view(np.uint32)[:, : kprime // 4], pay_o)
    assert np.array_equal(s_tok[ix(toks)].cpu().numpy().view(np.uint32), sc_o.view(np.uint32))
    # the GEMM + a18 epilogue
    acc = orc.sparse_gemm_words(vals, codes, pay_o)
    want = orc.dequant_bf16(acc, s_ch[ix(rows)].cpu().numpy(), sc_o)
    got = bf16_bits(y[ix(rows)][:, ix(toks)])
    bad = np.argwhere(got != want)
    assert bad.size == 0, f"{len(bad)} mismatches, first at (row {rows[bad[0][0]]}, token {toks[bad[0][1]]})"


@pytest.mark.parametrize("name,n,k", [QWEN7B[1], QWEN7B[2]], ids=["o", "gate_up"])
def test_full_shape_raw_int32_vs_oracle(slsp, orc, name, n, k):
    """RAW int32 [N][M] at M = 8192 (two-subtile tiles, chunked TMEM drain,
    TMA-box int32 stores): sampled blocks equal the oracle's accumulators."""
    w, x, _ = layer_inputs(slsp, n, k, seed=7 + n)
    pw = slsp.pack_compress(w, 6, 8)
    cfg = slsp.sparse_gemm_config(pw, M, slsp.OUT_RAW_NM)
    assert cfg["subtiles"] == 2 and cfg["epilogue"] == 0, cfg
    payload, _ = slsp.fused_quant_slide(x, 6, 8, kp=pw.kp, check=False)
    y = slsp.sparse_gemm(pw, payload)
    rows, toks = sample_rows(n), sample_tokens(M)
    vals, codes, pay_o, _ = oracle_block(orc, w, x, rows, toks)
    want = orc.sparse_gemm_words(vals, codes, pay_o)
    assert np.array_equal(y[ix(rows)][:, ix(toks)].cpu().numpy(), want)


def test_benched_step_bf16_mn_vs_oracle(slsp, orc):
    """Token-major BF16 output ([M][N], what a next layer consumes) at full
    size: o_proj, sampled blocks bit-exact."""
    n, k = 3584, 3584
    w, x, s_ch = layer_inputs(slsp, n, k, seed=5)
    pw = slsp.pack_compress(w, 6, 8)
    payload, s_tok = slsp.fused_quant_slide(x, 6, 8, kp=pw.kp, check=False)
    y = slsp.sparse_gemm(pw, payload, s_ch=s_ch, s_tok=s_tok, out_mode=slsp.OUT_BF16_MN)
    rows, toks = sample_rows(n), sample_tokens(M)
    vals, codes, pay_o, sc_o = oracle_block(orc, w, x, rows, toks)
    want = orc.dequant_bf16(orc.sparse_gemm_words(vals, codes, pay_o), s_ch[ix(rows)].cpu().numpy(), sc_o)
    assert np.array_equal(bf16_bits(y[ix(toks)][:, ix(rows)]).T, want)


def test_config1_full_vs_oracle(slsp, orc):
    """BASELINE.json configs[0]: 6:8 INT8, K = N = 4096, M = 128 —
    decompose + lift + sparse GEMM on the GPU vs the CPU oracle, every output
    (int32 accumulators and the BF16 epilogue)."""
    n = k = 4096
    m = 128
    g = torch.Generator(device="cuda").manual_seed(0)
    w = slsp.magnitude_prune(torch.randint(-127, 128, (n, k), dtype=torch.int8, device="cuda", generator=g), 6, 8)
    x = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    s_ch = (torch.rand(n, device="cuda", generator=g) * 0.01 + 0.001).float()
    pw = slsp.pack_compress(w, 6, 8)
    payload, s_tok = slsp.fused_quant_slide(x, 6, 8, kp=pw.kp)
    y_raw = slsp.sparse_gemm(pw, payload)
    y_bf = slsp.sparse_gemm(pw, payload, s_ch=s_ch, s_tok=s_tok, out_mode=slsp.OUT_BF16_NM)
    vals, codes = orc.compress(orc.pack_matrix(w.cpu().numpy(), 6, 8, DT_I8), DT_I8)
    pay_o, sc_o = orc.fused_quant_slide(bf16_bits(x), 6, 8, KIND_INT8, DT_BF16)
    kprime = vals.shape[1] * 2
    assert np.array_equal(pw.values.cpu().numpy()[:, : kprime // 2], vals)
    assert np.array_equal(payload.cpu().numpy().view(np.uint32)[:, : kprime // 4], pay_o)
    acc = orc.sparse_gemm_words(vals, codes, pay_o)
    assert np.array_equal(y_raw.cpu().numpy(), acc)
    assert np.array_equal(bf16_bits(y_bf), orc.dequant_bf16(acc, s_ch.cpu().numpy(), sc_o))


@pytest.mark.parametrize("m", [300, 8192])
def test_lift_long_rows_vs_oracle(slsp, orc, m):
    """fused_quant_slide at K = 18944 (down_proj; the QPT=2 row-resident
    kernel) vs the oracle: payload words and scale bits, including rows with
    heavy tails (one element x1000) that push codes onto the exact-fallback
    path."""
    k = 18944
    g = torch.Generator(device="cuda").manual_seed(m)
    x = torch.rand(m, k, device="cuda", generator=g) * 2 - 1
    x[::7, 5] *= 1000.0
    x = x.to(torch.bfloat16)
    payload, s_tok = slsp.fused_quant_slide(x, 6, 8)
    rows = np.arange(m) if m <= 512 else sample_tokens(m)
    pay_o, sc_o = orc.fused_quant_slide(bf16_bits(x[ix(rows)]), 6, 8, KIND_INT8, DT_BF16)
    words = pay_o.shape[1]
    assert np.array_equal(payload[ix(rows)].cpu().numpy().view(np.uint32)[:, :words], pay_o)
    assert np.array_equal(s_tok[ix(rows)].cpu().numpy().view(np.uint32), sc_o.view(np.uint32))


@pytest.mark.parametrize("n,k,m", [(512, 1024, 448), (300, 2048, 64), (256, 3584, 1000)])
def test_dense_fp8_within_tolerance(slsp, orc, n, k, m):
    """dense_gemm<e4m3> (gemm.hpp:142-162; config 3's speedup denominator) vs a
    float64 oracle on the decoded codes. Stated tolerance: |err| <= 2^-12 *
    sum|w*x| per output — e4m3 products are exact in fp32, and K fp32
    additions (K <= 4096 here) err by at most K * 2^-24 * sum|w*x|. Covers
    256-token and 64-token tile configs."""
    rng = np.random.default_rng(n + k + m)
    lut = np.array([orc.fp8_decode(c) for c in range(256)], dtype=np.float64)
    lut[np.isnan(lut)] = 0.0
    wc = rng.integers(0, 256, size=(n, k), dtype=np.uint8)
    xc = rng.integers(0, 256, size=(m, k), dtype=np.uint8)
    wc[(wc & 0x7F) == 0x7F] = 0  # no NaN codes
    xc[(xc & 0x7F) == 0x7F] = 0
    w = torch.from_numpy(wc).cuda().view(torch.float8_e4m3fn)
    x = torch.from_numpy(xc).cuda().view(torch.float8_e4m3fn)
    got = slsp.dense_gemm(w, x).double().cpu().numpy()
    wd, xd = lut[wc], lut[xc]
    want = wd @ xd.T
    absum = np.abs(wd) @ np.abs(xd).T
    print(f"fp8 dense max |err|/sum|w*x| = {(np.abs(got - want) / np.maximum(absum, 1e-30)).max():.3e}")
    assert np.all(np.abs(got - want) <= 2.0 ** -12 * absum + 1e-30)


def test_dense_int8_full_shape_vs_oracle(slsp, orc):
    """The bench's dense denominator (quantize_rows + dense_gemm, BF16 [N][M])
    at o_proj M = 8192, sampled blocks bit-exact vs the oracle's dense_gemm
    (gemm.hpp:142-162) on its own quantize_row codes (quantize.hpp:52-68)."""
    n = k = 3584
    w, x, s_ch = layer_inputs(slsp, n, k, seed=3)
    q, q_s = slsp.quantize_rows(x, check=False)
    y = slsp.dense_gemm(w, q.view(torch.int8), s_ch=s_ch, s_tok=q_s, out_mode=slsp.OUT_BF16_NM)
    rows, toks = sample_rows(n), sample_tokens(M)
    qo, so = orc.quantize_rows(bf16_bits(x[ix(toks)]), KIND_INT8, DT_BF16)
    assert np.array_equal(q[ix(toks)].cpu().numpy()[:, :k], qo)
    acc = orc.dense_gemm_i8(w[ix(rows)].cpu().numpy(), qo.view(np.int8).T.copy())
    assert np.array_equal(bf16_bits(y[ix(rows)][:, ix(toks)]), orc.dequant_bf16(acc, s_ch[ix(rows)].cpu().numpy(), so))


def test_payload_pairing_checked(slsp):
    """gemm.hpp:203-208: a payload lifted for another pattern or quantised to
    another kind is rejected, not multiplied."""
    g = torch.Generator(device="cuda").manual_seed(2)
    w = slsp.magnitude_prune(torch.randint(-127, 128, (256, 768), dtype=torch.int8, device="cuda", generator=g), 6, 8)
    pw = slsp.pack_compress(w, 6, 8)
    x = (torch.rand(64, 768, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    p8, _ = slsp.fused_quant_slide(x, 6, 8, kind=slsp.QUANT_FP8E4M3, kp=pw.kp)
    with pytest.raises(slsp.DimensionMismatchError):
        slsp.sparse_gemm(pw, p8)
    ok, _ = slsp.fused_quant_slide(x, 6, 8, kp=pw.kp)
    slsp.sparse_gemm(pw, ok)


def test_out_buffer_validated(slsp):
    """A caller-provided output of the wrong shape/dtype is rejected before the
    kernel could write past it."""
    g = torch.Generator(device="cuda").manual_seed(4)
    w = slsp.magnitude_prune(torch.randint(-127, 128, (512, 512), dtype=torch.int8, device="cuda", generator=g), 6, 8)
    pw = slsp.pack_compress(w, 6, 8)
    x = (torch.rand(256, 512, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    payload, s_tok = slsp.fused_quant_slide(x, 6, 8, kp=pw.kp)
    s_ch = torch.ones(512, device="cuda")
    with pytest.raises(ValueError):
        slsp.sparse_gemm(pw, payload, s_ch=s_ch, s_tok=s_tok, out_mode=slsp.OUT_BF16_NM,
                         out=torch.empty((256, 512), dtype=torch.bfloat16, device="cuda"))
    with pytest.raises(TypeError):
        slsp.sparse_gemm(pw, payload, out=torch.empty((512, 256), dtype=torch.float32, device="cuda"))
    with pytest.raises(ValueError):
        slsp.sparse_gemm(pw, payload, s_ch=s_ch[:100], s_tok=s_tok, out_mode=slsp.OUT_BF16_NM)
