"""GPU parity of the in-SM-lifting sparse GEMM (slsp_sparse_gemm_x, 6:8).

The activation operand is the UNLIFTED quantize_rows output; the window-
duplicating rearrangement of fused_quant_slide (quantize.hpp:122-174) happens
in shared memory and the weights are in slsp_gemm_order's window order. The
contract: int32 accumulators bit-exact vs the oracle's packed-word
sparse_gemm (gemm.hpp:199-233) on fused_quant_slide's payload, and the BF16
dequant epilogue bit-identical to slsp_sparse_gemm's."""

import numpy as np
import pytest
import torch

from helpers import compliant_matrix, round_up
from oracle_lib import DT_F32, DT_I8, KIND_INT8

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.fixture(params=["1", "2"], ids=["msub1", "msub2"])
def msub(request, slsp):
    with slsp.knobs(SLSP_GEMM_MSUB=request.param):
        yield request.param


@pytest.mark.parametrize("n,k,m", [(256, 512, 224), (512, 1024, 448), (300, 1000, 250), (1024, 3584, 700),
                                   (640, 1536, 1)])
def test_gemm_x_int8_bit_exact(slsp, orc, msub, n, k, m):
    rng = np.random.default_rng(n * 7 + k + m)
    w = compliant_matrix(rng, n, k // 8, 6, 8)
    x = rng.uniform(-1, 1, size=(m, k)).astype(np.float32)
    vals, codes = orc.compress(orc.pack_matrix(w, 6, 8, DT_I8), DT_I8)
    payload, _ = orc.fused_quant_slide(x, 6, 8, KIND_INT8, DT_F32)
    want = orc.sparse_gemm_words(vals, codes, payload)

    pw = slsp.pack_compress(dev(w), 6, 8)
    xq, s_tok = slsp.quantize_rows(dev(x), kpad=round_up(k, 512))
    got = slsp.sparse_gemm_x(pw, xq).cpu().numpy()
    assert np.array_equal(got, want)


@pytest.mark.parametrize("n,k,m", [(512, 3584, 448), (768, 2048, 300)])
def test_gemm_x_bf16_matches_lifted_path(slsp, msub, n, k, m):
    """Same accumulators, same fp32 epilogue: BF16 outputs identical to the
    HBM-lifted path, both output layouts."""
    g = torch.Generator(device="cuda").manual_seed(n + k + m)
    w = slsp.magnitude_prune(torch.randint(-127, 128, (n, k), dtype=torch.int8, device="cuda", generator=g), 6, 8)
    x = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    s_ch = torch.rand(n, device="cuda", generator=g) * 0.01 + 0.001
    pw = slsp.pack_compress(w, 6, 8)
    payload, s_tok = slsp.fused_quant_slide(x, 6, 8)
    xq, s_tok2 = slsp.quantize_rows(x, kpad=round_up(k, 512))
    assert torch.equal(s_tok, s_tok2)
    for mode in (slsp.OUT_BF16_NM, slsp.OUT_BF16_MN):
        want = slsp.sparse_gemm(pw, payload, s_ch=s_ch, s_tok=s_tok, out_mode=mode)
        got = slsp.sparse_gemm_x(pw, xq, s_ch=s_ch, s_tok=s_tok2, out_mode=mode)
        torch.cuda.synchronize()
        assert torch.equal(got.view(torch.int16), want.view(torch.int16))


def test_gemm_x_fp8_matches_lifted_path(slsp, msub):
    n, k, m = 512, 2048, 448
    g = torch.Generator(device="cuda").manual_seed(3)
    wf = (torch.rand(n, k, device="cuda", generator=g) * 2 - 1)
    w8 = slsp.magnitude_prune(wf.to(torch.float8_e4m3fn), 6, 8)
    x = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    pw = slsp.pack_compress(w8, 6, 8)
    payload, s_tok = slsp.fused_quant_slide(x, 6, 8, kind=slsp.QUANT_FP8E4M3)
    xq, _ = slsp.quantize_rows(x, kind=slsp.QUANT_FP8E4M3, kpad=round_up(k, 512))
    want = slsp.sparse_gemm(pw, payload)
    got = slsp.sparse_gemm_x(pw, xq)
    # fp32 accumulation in a different k order: equal up to fp32 reassociation
    # (|err| <= 2^-14 * sum |w*x| is the FP8 tolerance of test_gpu_gemm.py)
    assert torch.allclose(got, want, rtol=0, atol=float(want.abs().max()) * 2 ** -14 + 1e-3)


def test_gemm_x_rejects_bad_width(slsp):
    g = torch.Generator(device="cuda").manual_seed(0)
    w = slsp.magnitude_prune(torch.randint(-127, 128, (256, 512), dtype=torch.int8, device="cuda", generator=g), 6, 8)
    pw = slsp.pack_compress(w, 6, 8)
    xq = torch.zeros((128, 640), dtype=torch.uint8, device="cuda")
    with pytest.raises(slsp.DimensionMismatchError):
        slsp.sparse_gemm_x(pw, xq)
