"""the next layer's lift fused upstream.

Layer i's sparse GEMM (BF16 epilogue) also writes each token's max |y| over
its output features (sparse_gemm(..., tok_amax=a)); layer i+1's
fused_quant_slide(y, absmax=a) then quantizes + lifts without an |x|max pass
of its own. The reference computes the same thing in one call per layer
(quantize.hpp:122-174 on the previous output), so the chained result must be
bit-identical to the unfused chain, and the final int32 result must match
the CPU oracle (pack -> compress -> fused_quant_slide(y) -> sparse_gemm).
"""
import numpy as np
import pytest
import torch

from oracle_lib import DT_BF16, DT_I8, KIND_INT8

pytestmark = pytest.mark.gpu


def bf16_bits(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def layer(slsp, n, k, g):
    w = slsp.magnitude_prune(torch.randint(-127, 128, (n, k), dtype=torch.int8, device="cuda", generator=g), 6, 8)
    s_ch = (torch.rand(n, device="cuda", generator=g) * 0.01 + 0.001).float()
    return w, slsp.pack_compress(w, 6, 8), s_ch


@pytest.mark.parametrize("m,mode", [(8192, "mn"), (300, "mn"), (8192, "nm"), (1000, "nm")])
def test_gemm_token_amax_is_exact(slsp, m, mode):
    """tok_amax == max_n |y[t][n]| of the BF16 outputs, and y is unchanged by the fold."""
    g = torch.Generator(device="cuda").manual_seed(11)
    n, k = 3584, 3584
    _, pw, s_ch = layer(slsp, n, k, g)
    x = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    pay, s_tok = slsp.fused_quant_slide(x, 6, 8)
    om = slsp.OUT_BF16_MN if mode == "mn" else slsp.OUT_BF16_NM
    y_ref = slsp.sparse_gemm(pw, pay, s_ch=s_ch, s_tok=s_tok, out_mode=om)
    amax = torch.full((m,), 123.0, device="cuda")  # stale contents are reset by the call
    y = slsp.sparse_gemm(pw, pay, s_ch=s_ch, s_tok=s_tok, out_mode=om, tok_amax=amax)
    assert torch.equal(y, y_ref)
    yt = y if mode == "mn" else y.t()
    want = yt.float().abs().amax(dim=1)
    assert torch.equal(amax, want)


@pytest.mark.parametrize("m", [8192, 448])
def test_two_layer_chain_matches_unfused_and_oracle(slsp, orc, m):
    """Layer 1 (o-shaped) -> fused lift of its output -> layer 2 (gate-shaped, rows sampled)."""
    g = torch.Generator(device="cuda").manual_seed(5)
    n1, k1, n2 = 3584, 3584, 2048
    _, pw1, s1 = layer(slsp, n1, k1, g)
    w2, pw2, s2 = layer(slsp, n2, n1, g)
    x = (torch.rand(m, k1, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    pay1, t1 = slsp.fused_quant_slide(x, 6, 8)
    amax = torch.empty(m, device="cuda")
    y1 = slsp.sparse_gemm(pw1, pay1, s_ch=s1, s_tok=t1, out_mode=slsp.OUT_BF16_MN, tok_amax=amax)
    # fused: the lift takes the upstream |x|max
    pay2, t2 = slsp.fused_quant_slide(y1, 6, 8, kp=pw2.kp, absmax=amax)
    # unfused: the plain lift of the same y1
    pay2_ref, t2_ref = slsp.fused_quant_slide(y1, 6, 8, kp=pw2.kp)
    assert torch.equal(pay2, pay2_ref)
    assert torch.equal(t2, t2_ref)
    acc = slsp.sparse_gemm(pw2, pay2)
    # CPU oracle on sampled tokens and rows of layer 2, from y1's BF16 bits
    toks = np.unique(np.concatenate([np.arange(0, 64), np.arange(m - 64, m)]))
    rows = np.concatenate([np.arange(0, 128), np.arange(n2 - 128, n2)])
    vals, codes = orc.compress(orc.pack_matrix(w2[torch.from_numpy(rows).cuda()].cpu().numpy(), 6, 8, DT_I8), DT_I8)
    payload, scales = orc.fused_quant_slide(bf16_bits(y1[torch.from_numpy(toks).cuda()]), 6, 8, KIND_INT8, DT_BF16)
    want = orc.sparse_gemm_words(vals, codes, payload)
    got = acc.cpu().numpy()[np.ix_(rows, toks)]
    assert np.array_equal(got, want)
    assert np.array_equal(t2.cpu().numpy()[toks].view(np.uint32), scales.view(np.uint32))


def test_scaled_lift_reports_nonfinite_row(slsp):
    x = (torch.rand(64, 1024, device="cuda") * 2 - 1).to(torch.bfloat16)
    a = x.float().abs().amax(dim=1)
    a[17] = float("inf")
    with pytest.raises(slsp.NonFiniteInputError, match="row 17"):
        slsp.fused_quant_slide(x, 6, 8, absmax=a)


@pytest.mark.parametrize("z,l", [(4, 6), (8, 10)])
def test_scaled_lift_other_patterns(slsp, z, l):
    """The warp-path kernels (patterns other than 6:8) take the upstream |x|max too."""
    g = torch.Generator(device="cuda").manual_seed(3)
    k = 30 * l * 4
    x = (torch.rand(200, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    a = x.float().abs().amax(dim=1)
    p0, s0 = slsp.fused_quant_slide(x, z, l)
    p1, s1 = slsp.fused_quant_slide(x, z, l, absmax=a)
    assert torch.equal(p0, p1) and torch.equal(s0, s1)


@pytest.mark.parametrize("n,m", [(1000, 500), (1536, 8192 - 97), (256, 224 * 3 + 5)])
def test_token_major_epilogue_ragged(slsp, n, m):
    """Two-subtile tiles with token-major output (the register epilogue's
    in-smem transpose) at ragged shapes: identical to the [N][M] output
    transposed, and the |y|max fold exact."""
    g = torch.Generator(device="cuda").manual_seed(n + m)
    k = 1024
    _, pw, s_ch = layer(slsp, n, k, g)
    x = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    pay, s_tok = slsp.fused_quant_slide(x, 6, 8)
    with slsp.knobs(SLSP_GEMM_MSUB="2", SLSP_GEMM_BN256_MAXM="0"):
        assert slsp.sparse_gemm_config(pw, m, slsp.OUT_BF16_MN)["subtiles"] == 2
        y_nm = slsp.sparse_gemm(pw, pay, s_ch=s_ch, s_tok=s_tok, out_mode=slsp.OUT_BF16_NM)
        y_mn = slsp.sparse_gemm(pw, pay, s_ch=s_ch, s_tok=s_tok, out_mode=slsp.OUT_BF16_MN)
        amax = torch.empty(m, device="cuda")
        y_mn2 = slsp.sparse_gemm(pw, pay, s_ch=s_ch, s_tok=s_tok, out_mode=slsp.OUT_BF16_MN, tok_amax=amax)
    assert torch.equal(y_mn, y_nm.t().contiguous())
    assert torch.equal(y_mn2, y_mn)
    assert torch.equal(amax, y_mn.float().abs().amax(dim=1))
