"""the BF16 lift inside the GEMM (decode-shaped M).

sparse_gemm_lift(w, x) takes the UNLIFTED BF16 activations; the kernel's lift
warps read each window's four source elements (quantize.hpp:72-89 lift_row)
from x and write them straight into the shared-memory B stage. It must equal
sparse_gemm(w, lift_rows(x, z, l, kp)) on the same tile configuration bit for
bit (same MMAs on the same operands in the same order), including split-K and
every output mode, and W @ X^T within the BF16 GEMM's stated tolerance.
"""
import pytest
import torch

pytestmark = pytest.mark.gpu


def case(slsp, n, k, m, z, l, seed, x_ld=None):
    g = torch.Generator(device="cuda").manual_seed(seed)
    w = slsp.magnitude_prune((torch.rand(n, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16), z, l)
    pw = slsp.pack_compress(w, z, l)
    big = (torch.rand(m, x_ld or k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    x = big[:, :k]
    s_ch = (torch.rand(n, device="cuda", generator=g) + 0.5).float()
    s_tok = (torch.rand(m, device="cuda", generator=g) + 0.5).float()
    return w, pw, x, s_ch, s_tok


def reference(slsp, pw, x, s_ch, s_tok, out_mode):
    """The unfused pair on the same (64-token, one-subtile) tiles."""
    lifted = slsp.lift_rows(x.contiguous(), pw.z, pw.l, kp=pw.kp)
    with slsp.knobs(SLSP_GEMM_DECODE_M="1000000"):
        return slsp.sparse_gemm(pw, lifted, s_ch=s_ch, s_tok=s_tok, out_mode=out_mode)


@pytest.mark.parametrize("n,k,m", [(3584, 3584, 1), (3584, 3584, 16), (4608, 3584, 64), (1000, 1024, 7),
                                   (512, 2048, 33), (3584, 18944, 16), (768, 4096, 200)])
@pytest.mark.parametrize("out_mode", ["raw", "nm", "mn"])
def test_glift_equals_lift_then_gemm(slsp, n, k, m, out_mode):
    om = {"raw": slsp.OUT_RAW_NM, "nm": slsp.OUT_BF16_NM, "mn": slsp.OUT_BF16_MN}[out_mode]
    w, pw, x, s_ch, s_tok = case(slsp, n, k, m, 6, 8, n + k + m)
    kw = {} if om == slsp.OUT_RAW_NM else {"s_ch": s_ch, "s_tok": s_tok}
    got = slsp.sparse_gemm_lift(pw, x, out_mode=om, **kw)
    want = reference(slsp, pw, x, kw.get("s_ch"), kw.get("s_tok"), om)
    assert torch.equal(got, want)


@pytest.mark.parametrize("z,l", [(4, 6), (8, 10), (2, 4), (4, 8)])
def test_glift_other_patterns(slsp, z, l):
    k = 60 * l * 4
    w, pw, x, _, _ = case(slsp, 640, k, 24, z, l, z * 100 + l)
    got = slsp.sparse_gemm_lift(pw, x)
    assert torch.equal(got, reference(slsp, pw, x, None, None, slsp.OUT_RAW_NM))


@pytest.mark.parametrize("pad,off", [(96, 0), (2, 0), (8, 2), (0, 2)])
def test_glift_strided_rows_and_tolerance(slsp, pad, off):
    """x as a column slice of a wider buffer (row stride k + pad, first column
    off: the 16-byte-aligned 6:8 path and the 4-byte window path); the result
    equals the contiguous call and a float64 W @ X^T within the BF16 GEMM's
    bound (|err| <= 2^-14 sum|w x|)."""
    n, k, m = 768, 2048, 40
    w, pw, xb, _, _ = case(slsp, n, k, m, 6, 8, 9 + pad + off, x_ld=k + pad + off)
    x = xb if off == 0 else torch.as_strided(xb, (m, k), (k + pad + off, 1), off)
    got = slsp.sparse_gemm_lift(pw, x)
    assert torch.equal(got, slsp.sparse_gemm_lift(pw, x.contiguous()))
    got = got.double().cpu()
    wd, xd = w.double().cpu(), x.double().cpu()
    want = wd @ xd.T
    assert torch.all((got - want).abs() <= 2.0 ** -14 * (wd.abs() @ xd.abs().T) + 1e-30)


def test_glift_rejects_bad_inputs(slsp):
    _, pw, x, _, _ = case(slsp, 256, 1024, 8, 6, 8, 1)
    with pytest.raises(slsp.DimensionMismatchError):
        slsp.sparse_gemm_lift(pw, x[:, :1016])
    with pytest.raises(slsp.UnsupportedError):
        slsp.sparse_gemm_lift(pw, x.float())
    odd = torch.zeros(8, 1025, dtype=torch.bfloat16, device="cuda")[:, :1024]  # odd row stride
    with pytest.raises(ValueError):
        slsp.sparse_gemm_lift(pw, odd)
    empty = slsp.sparse_gemm_lift(pw, x[:0])
    assert empty.shape == (256, 0)
