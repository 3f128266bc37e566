"""Cluster split-K for the decode tiles (Params::ksc).

ksc CTA pairs of one cluster take consecutive k-ranges of the same tile; the
partial accumulators meet in distributed shared memory and every CTA sums its
row share in slice order. The k-ranges and the summation order are those of
a ksc-way workspace split (splitk_finish_kernel), so:
  * INT8: the int32 sums equal the CPU oracle's (gemm.hpp:199-233) exactly;
  * BF16 / FP8 (fp32 accumulators): the outputs equal the workspace split's
    with the same slice count bit for bit, in every output mode;
  * the in-GEMM lift (sparse_gemm_lift) equals lift_rows + sparse_gemm under
    the same split.
"""
import numpy as np
import pytest
import torch

from oracle_lib import DT_I8, orc

pytestmark = pytest.mark.gpu


def _int8_case(slsp, n, k, m, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    w = slsp.magnitude_prune(torch.randint(-127, 128, (n, k), dtype=torch.int8, device="cuda", generator=g), 6, 8)
    x = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    s_ch = torch.rand(n, device="cuda", generator=g) * 0.01 + 0.001
    return w, x, s_ch


@pytest.mark.parametrize("n,k,m", [(4096, 4096, 128), (2048, 4096, 64), (1000, 3584, 1), (768, 18944, 16)])
@pytest.mark.parametrize("ksc", [2, 3, 4])
def test_int8_cluster_split_equals_oracle(slsp, n, k, m, ksc):
    w, x, s_ch = _int8_case(slsp, n, k, m, n + m + ksc)
    pw = slsp.pack_compress(w, 6, 8)
    payload, s_tok = slsp.fused_quant_slide(x, 6, 8)
    with slsp.knobs(SLSP_GEMM_KSC=str(ksc)):
        cfg = slsp.sparse_gemm_config(pw, m, slsp.OUT_RAW_NM)
        assert cfg["cluster_ksplit"] == ksc and cfg["cluster_ctas"] == 2 * ksc and cfg["workspace_bytes"] == 0, cfg
        raw = slsp.sparse_gemm(pw, payload)
        nm = slsp.sparse_gemm(pw, payload, s_ch=s_ch, s_tok=s_tok, out_mode=slsp.OUT_BF16_NM)
        mn = slsp.sparse_gemm(pw, payload, s_ch=s_ch, s_tok=s_tok, out_mode=slsp.OUT_BF16_MN)
    with slsp.knobs(SLSP_GEMM_KSC="1", SLSP_GEMM_KSPLIT="1"):
        assert slsp.sparse_gemm_config(pw, m, slsp.OUT_BF16_NM)["ksplit"] == 1
        nm1 = slsp.sparse_gemm(pw, payload, s_ch=s_ch, s_tok=s_tok, out_mode=slsp.OUT_BF16_NM)
    torch.cuda.synchronize()
    O = orc()
    vals, codes = O.compress(O.pack_matrix(w.cpu().numpy(), 6, 8, DT_I8), DT_I8)
    kprime = vals.shape[1] * 2
    pay = np.ascontiguousarray(payload.cpu().numpy().view(np.uint32)[:, : kprime // 4])
    want = O.sparse_gemm_words(vals, codes, pay)
    assert np.array_equal(raw.cpu().numpy(), want)
    # same int32 sums -> the same fp32 epilogue, whatever the split
    assert torch.equal(nm.view(torch.int16), nm1.view(torch.int16))
    assert torch.equal(mn.t().contiguous().view(torch.int16), nm1.view(torch.int16))


@pytest.mark.parametrize("n,k,m", [(6144, 4096, 1), (4096, 4096, 16), (3000, 2048, 64), (4096, 14336, 5)])
@pytest.mark.parametrize("ksc", [2, 3, 4])
def test_bf16_cluster_split_equals_workspace_split(slsp, n, k, m, ksc):
    """fp32 accumulators: cluster split == workspace split of the same slice
    count, bit for bit (same k-ranges, same slice-order sum, same epilogue);
    sparse, in-GEMM lift and dense."""
    g = torch.Generator(device="cuda").manual_seed(n + k + m + ksc)
    w = slsp.magnitude_prune((torch.rand(n, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16), 6, 8)
    pw = slsp.pack_compress(w, 6, 8)
    x = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    s_ch = (torch.rand(n, device="cuda", generator=g) + 0.5).float()
    s_tok = (torch.rand(m, device="cuda", generator=g) + 0.5).float()
    lifted = slsp.lift_rows(x, 6, 8, kp=pw.kp)
    outs = {}
    for tag, kn in (("cl", {"SLSP_GEMM_KSC": str(ksc)}), ("ws", {"SLSP_GEMM_KSPLIT": str(ksc)})):
        with slsp.knobs(**kn):
            cfg = slsp.sparse_gemm_config(pw, m, slsp.OUT_BF16_NM)
            assert cfg["ksplit"] == ksc and cfg["cluster_ksplit"] == (ksc if tag == "cl" else 1), (tag, cfg)
            for mode in (slsp.OUT_RAW_NM, slsp.OUT_BF16_NM, slsp.OUT_BF16_MN):
                kw = {} if mode == slsp.OUT_RAW_NM else {"s_ch": s_ch, "s_tok": s_tok}
                outs[(tag, mode, "s")] = slsp.sparse_gemm(pw, lifted, out_mode=mode, **kw)
                outs[(tag, mode, "g")] = slsp.sparse_gemm_lift(pw, x, out_mode=mode, **kw)
                outs[(tag, mode, "d")] = slsp.dense_gemm(w, x, out_mode=mode, **kw)
    torch.cuda.synchronize()
    for mode in (slsp.OUT_RAW_NM, slsp.OUT_BF16_NM, slsp.OUT_BF16_MN):
        for kind in ("s", "g", "d"):
            a, b = outs[("cl", mode, kind)], outs[("ws", mode, kind)]
            assert torch.equal(a.view(torch.int16 if a.element_size() == 2 else torch.int32),
                               b.view(torch.int16 if b.element_size() == 2 else torch.int32)), (mode, kind)
        assert torch.equal(outs[("cl", mode, "s")], outs[("cl", mode, "g")])
    # and against W @ X^T in fp32 (the BF16 GEMM's stated tolerance, test_gpu_gemm)
    ref = (w.float() @ x.float().t())
    got = outs[("cl", slsp.OUT_RAW_NM, "s")]
    tol = 2.0 ** -14 * (w.float().abs() @ x.float().abs().t()) + 1e-6
    assert torch.all((got - ref).abs() <= tol)


def test_cluster_split_cost_model(slsp):
    """Default (cost model): decode shapes whose tiles leave clusters idle take
    the cluster split (no workspace), large M never does; SLSP_GEMM_KSC=1
    turns it off."""
    g = torch.Generator(device="cuda").manual_seed(7)
    w = slsp.magnitude_prune(torch.randint(-127, 128, (4096, 4096), dtype=torch.int8, device="cuda", generator=g), 6, 8)
    pw = slsp.pack_compress(w, 6, 8)
    c1 = slsp.sparse_gemm_config(pw, 128, slsp.OUT_BF16_NM)
    assert c1["cluster_ksplit"] > 1 and c1["workspace_bytes"] == 0, c1
    c2 = slsp.sparse_gemm_config(pw, 8192, slsp.OUT_BF16_NM)
    assert c2["cluster_ksplit"] == 1 and c2["ksplit"] == 1, c2
    with slsp.knobs(SLSP_GEMM_KSC="1"):
        assert slsp.sparse_gemm_config(pw, 128, slsp.OUT_BF16_NM)["cluster_ksplit"] == 1


@pytest.mark.parametrize("m", [1, 16, 64])
@pytest.mark.parametrize("ksc", [2, 4])
def test_fp8_cluster_split_equals_workspace_split(slsp, m, ksc):
    """FP8 (e4m3 weights and lifted activations, fp32 accumulators): cluster
    split == workspace split of the same slice count, bit for bit, in every
    output mode."""
    g = torch.Generator(device="cuda").manual_seed(100 + m + ksc)
    n, k = 2048, 4096
    w = slsp.magnitude_prune(((torch.rand(n, k, device="cuda", generator=g) * 2 - 1) * 200).to(torch.float8_e4m3fn),
                             6, 8)
    pw = slsp.pack_compress(w, 6, 8)
    x = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    payload, s_tok = slsp.fused_quant_slide(x, 6, 8, kind=slsp.QUANT_FP8E4M3)
    s_ch = torch.rand(n, device="cuda", generator=g) * 0.01 + 0.001
    outs = {}
    for tag, kn in (("cl", {"SLSP_GEMM_KSC": str(ksc)}), ("ws", {"SLSP_GEMM_KSPLIT": str(ksc)})):
        with slsp.knobs(**kn):
            cfg = slsp.sparse_gemm_config(pw, m, slsp.OUT_BF16_NM)
            assert cfg["ksplit"] == ksc and cfg["cluster_ksplit"] == (ksc if tag == "cl" else 1), (tag, cfg)
            for mode in (slsp.OUT_RAW_NM, slsp.OUT_BF16_NM, slsp.OUT_BF16_MN):
                kw = {} if mode == slsp.OUT_RAW_NM else {"s_ch": s_ch, "s_tok": s_tok}
                outs[(tag, mode)] = slsp.sparse_gemm(pw, payload, out_mode=mode, **kw)
    torch.cuda.synchronize()
    for mode in (slsp.OUT_RAW_NM, slsp.OUT_BF16_NM, slsp.OUT_BF16_MN):
        a, b = outs[("cl", mode)], outs[("ws", mode)]
        iv = torch.int16 if a.element_size() == 2 else torch.int32
        assert torch.equal(a.view(iv), b.view(iv)), mode
