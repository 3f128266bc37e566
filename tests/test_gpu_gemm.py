"""GPU parity: tcgen05 sparse / dense GEMMs through the C ABI.

INT8: bit-exact int32 accumulators vs the oracle's packed-word sparse_gemm
(gemm.hpp:199-233) and dense_gemm (gemm.hpp:142-162). BF16 dequant epilogue:
bit-exact vs the oracle's fp32 restatement (same operation order). FP8:
relative tolerance vs the double-precision oracle (stated per test)."""
import numpy as np
import pytest
import torch

from helpers import compliant_matrix, lifted_width, mma_format, pad_cols, random_pruned_int8, round_up
from oracle_lib import DT_E4M3, DT_F32, DT_I8, KIND_FP8, KIND_INT8

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def sparse_case(orc, rng, n, k, m, z=6, l=8, exact=False):
    w = compliant_matrix(rng, n, k // l, z, l, exact_z=exact)
    x = rng.uniform(-1, 1, size=(m, k)).astype(np.float32)
    vals, codes = orc.compress(orc.pack_matrix(w, z, l, DT_I8), DT_I8)
    payload, scales = orc.fused_quant_slide(x, z, l, KIND_INT8, DT_F32)
    kp = round_up(lifted_width(k, z, l), 256)
    return w, x, vals, codes, payload, scales, kp


def run_sparse_raw(slsp, vals, codes, payload, kp, n, z=6, l=8):
    v, meta = mma_format(vals, codes, kp)
    pw = slsp.PackedWeights(dev(v), dev(meta), n, 0, kp, z, l)
    act = dev(pad_cols(payload.view(np.uint8).reshape(payload.shape[0], -1), kp))
    return slsp.sparse_gemm(pw, act).cpu().numpy()


@pytest.mark.parametrize("n,k,m", [(256, 256, 224), (512, 1024, 448), (300, 400, 250), (1024, 2048, 700),
                                   (512, 1024, 512), (384, 4096, 256), (256, 2048, 1000), (256, 16384, 256),
                                   (384, 2048, 120)])
def test_sparse_int8_bit_exact(slsp, orc, n, k, m):
    """Token counts cover every tile shape: 224-token tiles (one or two weight
    subtiles), 256-token tiles (moderate M where they need fewer token tiles:
    250, 256, 512, 700, 1000), split-K on them (k = 16384, one tile) and
    64-token tiles at M = 120 (short K, few weight tiles)."""
    rng = np.random.default_rng(n + k + m)
    w, x, vals, codes, payload, scales, kp = sparse_case(orc, rng, n, k, m)
    got = run_sparse_raw(slsp, vals, codes, payload, kp, n)
    want = orc.sparse_gemm_words(vals, codes, payload)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("z,l", [(4, 6), (8, 10), (14, 16)])
def test_sparse_int8_other_patterns(slsp, orc, z, l):
    rng = np.random.default_rng(l)
    n, m = 256, 224
    k = l * 40
    w, x, vals, codes, payload, scales, kp = sparse_case(orc, rng, n, k, m, z, l)
    got = run_sparse_raw(slsp, vals, codes, payload, kp, n, z, l)
    assert np.array_equal(got, orc.sparse_gemm_words(vals, codes, payload))


def test_sparse_equals_dense_on_quantized(slsp, orc):
    """test_gemm.cpp:299-323: the packed-word sparse path equals dense_gemm on
    per-row-quantized X, exactly — here both sides on the GPU kernels."""
    rng = np.random.default_rng(5)
    n, k, m = 512, 1024, 448
    w = random_pruned_int8(rng, n, k, 6, 8)
    x = torch.from_numpy(rng.uniform(-2, 2, size=(m, k)).astype(np.float32)).cuda()
    pw = slsp.pack_compress(dev(w), 6, 8)
    payload, s_tok = slsp.fused_quant_slide(x, 6, 8)
    ys = slsp.sparse_gemm(pw, payload)
    q, s2 = slsp.quantize_rows(x)
    yd = slsp.dense_gemm(dev(w), q.view(torch.int8))
    assert torch.equal(s_tok, s2)
    assert torch.equal(ys, yd)
    want = orc.dense_gemm_i8(w, q.view(torch.int8).cpu().numpy().T.copy())
    assert np.array_equal(yd.cpu().numpy(), want)


@pytest.mark.parametrize("n,k,m", [(256, 128, 256), (512, 1024, 512), (300, 384, 260)])
def test_dense_int8_bit_exact(slsp, orc, n, k, m):
    rng = np.random.default_rng(n * 3 + k + m)
    w = rng.integers(-127, 128, size=(n, k)).astype(np.int8)
    x = rng.integers(-127, 128, size=(m, k)).astype(np.int8)
    got = slsp.dense_gemm(dev(w), dev(x)).cpu().numpy()
    assert np.array_equal(got, orc.dense_gemm_i8(w, x.T.copy()))


@pytest.mark.parametrize("mode", ["nm", "mn"])
def test_sparse_bf16_dequant_epilogue(slsp, orc, mode):
    rng = np.random.default_rng(17)
    n, k, m = 512, 1024, 300
    w, x, vals, codes, payload, scales, kp = sparse_case(orc, rng, n, k, m)
    s_ch = rng.uniform(0.001, 0.02, size=n).astype(np.float32)
    v, meta = mma_format(vals, codes, kp)
    pw = slsp.PackedWeights(dev(v), dev(meta), n, k, kp, 6, 8)
    act = dev(pad_cols(payload.view(np.uint8).reshape(m, -1), kp))
    out_mode = slsp.OUT_BF16_NM if mode == "nm" else slsp.OUT_BF16_MN
    y = slsp.sparse_gemm(pw, act, s_ch=dev(s_ch), s_tok=dev(scales), out_mode=out_mode)
    acc = orc.sparse_gemm_words(vals, codes, payload)
    want = orc.dequant_bf16(acc, s_ch, scales)
    got = y.view(torch.int16).cpu().numpy().view(np.uint16)
    if mode == "mn":
        got = got.T
    assert np.array_equal(got, want)


@pytest.mark.parametrize("m", [448, 250, 120])
def test_sparse_fp8_within_tolerance(slsp, orc, m):
    """FP8 e4m3 weights and activations, fp32 accumulation in TMEM vs the
    double oracle on decoded values. Stated tolerance: |err| <= 2^-14 * sum|w*x|
    per output (products of e4m3 values are exact in fp32; the bound covers the
    tensor core's fp32 accumulation order over K'/2 = 768 products). M covers
    the 224-token (two-subtile), 256-token and 64-token tile configs."""
    rng = np.random.default_rng(23)
    n, k = 512, 1024
    mask = compliant_matrix(rng, n, k // 8, 6, 8) != 0
    wf = np.where(mask, rng.uniform(-1, 1, size=mask.shape), 0.0)
    wcode = np.array([orc.fp8_encode(v) for v in (wf * 200).ravel()], np.uint8).reshape(n, k)
    wcode[wcode == 0x80] = 0
    x = rng.uniform(-1, 1, size=(m, k)).astype(np.float32)
    payload, scales = orc.fused_quant_slide(x, 6, 8, KIND_FP8, DT_F32)
    vals, codes = orc.compress(orc.pack_matrix(wcode, 6, 8, DT_E4M3), DT_E4M3)
    kp = round_up(lifted_width(k, 6, 8), 256)
    v, meta = mma_format(vals, codes, kp)
    pw = slsp.PackedWeights(dev(v).view(torch.float8_e4m3fn), dev(meta), n, k, kp, 6, 8)
    act = dev(pad_cols(payload.view(np.uint8).reshape(m, -1), kp))
    got = slsp.sparse_gemm(pw, act).cpu().numpy().astype(np.float64)
    dec = np.vectorize(orc.fp8_decode, otypes=[np.float64])
    vd = dec(vals)
    ad = dec(payload.view(np.uint8).reshape(m, -1))
    want = orc.sparse_gemm_f64(vd, codes, ad)
    absum = orc.sparse_gemm_f64(np.abs(vd), codes, np.abs(ad))
    rel = np.abs(got - want) / np.maximum(absum, 1e-30)
    print(f"fp8 max relative error {rel.max():.3e}")
    assert np.all(np.abs(got - want) <= 2.0 ** -14 * absum + 1e-30)


def test_gemm_rejects_bad_kp(slsp):
    pw = slsp.PackedWeights(torch.zeros(256, 100, dtype=torch.int8, device="cuda"),
                            torch.zeros(256, 25, dtype=torch.uint8, device="cuda"), 256, 0, 200, 6, 8)
    with pytest.raises(slsp.DimensionMismatchError):
        slsp.sparse_gemm(pw, torch.zeros(224, 200, dtype=torch.uint8, device="cuda"))


def test_full_shape_sparse_equals_dense(slsp):
    """Qwen2.5-7B o_proj at M=8192 (full size): sparse(lifted) == dense(quantized)
    elementwise, exactly (size-independent equivalence, gemm.hpp:258-286)."""
    g = torch.Generator(device="cuda").manual_seed(1)
    n = k = 3584
    m = 8192
    w = torch.randint(-127, 128, (n, k), dtype=torch.int8, device="cuda", generator=g)
    w = slsp.magnitude_prune(w, 6, 8)
    x = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    pw = slsp.pack_compress(w, 6, 8)
    payload, s_tok = slsp.fused_quant_slide(x, 6, 8)
    q, _ = slsp.quantize_rows(x)
    ys = slsp.sparse_gemm(pw, payload)
    yd = slsp.dense_gemm(w, q.view(torch.int8))
    assert torch.equal(ys, yd)


@pytest.mark.parametrize("n,k,m", [(512, 1024, 448), (300, 2048, 64), (768, 4096, 1), (512, 1024, 256),
                                   (256, 1024, 500), (256, 2048, 100)])
def test_sparse_bf16_within_tolerance(slsp, n, k, m):
    """BF16 6:8 weights (kind::f16 .sp, one metadata column per K=32 MMA) and
    lifted BF16 activations (lift_row, quantize.hpp:72-89) vs a float64
    reference of W @ X^T (sparse_gemm<T>, gemm.hpp:164-197, accumulates in
    double). Stated tolerance: |err| <= 2^-14 * sum|w*x| per output (bf16
    products are exact in fp32; the bound covers fp32 accumulation)."""
    g = torch.Generator(device="cuda").manual_seed(n + k + m)
    w = slsp.magnitude_prune((torch.rand(n, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16), 6, 8)
    x = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    pw = slsp.pack_compress(w, 6, 8)
    lifted = slsp.lift_rows(x, 6, 8, kp=pw.kp)
    got = slsp.sparse_gemm(pw, lifted).double().cpu()
    wd, xd = w.double().cpu(), x.double().cpu()
    want = wd @ xd.T
    absum = wd.abs() @ xd.abs().T
    assert torch.all((got - want).abs() <= 2.0 ** -14 * absum + 1e-30)
    # the same-precision dense kernel agrees to the same bound
    yd = slsp.dense_gemm(w, x).double().cpu()
    assert torch.all((yd - want).abs() <= 2.0 ** -14 * absum + 1e-30)


@pytest.mark.parametrize("m", [1, 16, 64, 600])
def test_decode_split_k_int8_bit_exact(slsp, orc, m):
    """Decode-shaped and moderate M: the tiles do not fill the GPU, so K is
    split across CTAs (long K: 96 k-blocks), slices store int32 partial sums
    and a finishing kernel adds them in order — exact, so the result is still
    bit-identical to the oracle (gemm.hpp:199-233)."""
    rng = np.random.default_rng(m)
    n, k = 1024, 16384
    w, x, vals, codes, payload, scales, kp = sparse_case(orc, rng, n, k, m)
    got = run_sparse_raw(slsp, vals, codes, payload, kp, n)
    assert np.array_equal(got, orc.sparse_gemm_words(vals, codes, payload))


@pytest.mark.parametrize("m", [1, 16, 64, 512])
def test_decode_split_k_bf16_epilogue_identical(slsp, m):
    """BF16 outputs of a split-K GEMM (workspace + finishing kernel) equal the
    unsplit GEMM's bit for bit (INT8: same int32 sums, same fp32 epilogue)."""
    g = torch.Generator(device="cuda").manual_seed(m)
    n, k = 2048, 4096
    w = slsp.magnitude_prune(torch.randint(-127, 128, (n, k), dtype=torch.int8, device="cuda", generator=g), 6, 8)
    x = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    s_ch = torch.rand(n, device="cuda", generator=g) * 0.01 + 0.001
    pw = slsp.pack_compress(w, 6, 8)
    payload, s_tok = slsp.fused_quant_slide(x, 6, 8)
    q, q_s = slsp.quantize_rows(x)
    outs = {}
    for ks in ("1", "4"):  # forced unsplit, then a 4-way split
        with slsp.knobs(SLSP_GEMM_KSPLIT=ks):
            for mode in (slsp.OUT_BF16_NM, slsp.OUT_BF16_MN):
                assert slsp.sparse_gemm_config(pw, m, mode)["ksplit"] == int(ks)
                outs[(ks, mode, "s")] = slsp.sparse_gemm(pw, payload, s_ch=s_ch, s_tok=s_tok, out_mode=mode)
                outs[(ks, mode, "d")] = slsp.dense_gemm(w, q.view(torch.int8), s_ch=s_ch, s_tok=q_s, out_mode=mode)
    torch.cuda.synchronize()
    for mode in (slsp.OUT_BF16_NM, slsp.OUT_BF16_MN):
        for kind in ("s", "d"):
            assert torch.equal(outs[("1", mode, kind)].view(torch.int16), outs[("4", mode, kind)].view(torch.int16))


@pytest.mark.parametrize("z,l,n,k,m", [(6, 8, 512, 1024, 300), (4, 6, 256, 600, 100), (6, 8, 3584, 3584, 8192)])
def test_gpu_check_equivalence(slsp, z, l, n, k, m):
    """gemm.hpp:258-286 on the GPU: dense vs the full sparse pipeline, exact
    (last case: Qwen2.5-7B o_proj at M=8192)."""
    g = torch.Generator(device="cuda").manual_seed(n + m)
    kk = -(-k // l) * l
    w = slsp.magnitude_prune(torch.randint(-127, 128, (n, kk), dtype=torch.int8, device="cuda", generator=g), z, l)
    w = w[:, :k].contiguous()
    x = torch.randint(-127, 128, (k, m), dtype=torch.int8, device="cuda", generator=g)
    rep = slsp.check_equivalence(w, x, z, l)
    assert rep.exact and rep.max_abs_diff == 0
    # op-count ratio = gamma * hw_m / hw_n on whole blocks (acceptance.cpp:335-357)
    if k % l == 0:
        wc = (l - 4) // 2 + 1
        assert rep.sparse_multiplies * l == rep.dense_multiplies * wc * 2


def test_gpu_check_equivalence_rejects_noncompliant(slsp):
    w = torch.ones((128, 64), dtype=torch.int8, device="cuda")
    x = torch.ones((64, 32), dtype=torch.int8, device="cuda")
    with pytest.raises(slsp.NotCompliantError, match="row 0, block 0"):
        slsp.check_equivalence(w, x, 6, 8)


@pytest.mark.parametrize("kind", ["int8", "fp8"])
def test_half_k_stage_config_identical(slsp, kind):
    """The half-k-stage two-subtile config (SLSP_GEMM_KHALF: 64-byte A rows,
    one metadata atom and two MMAs per stage and subtile) reproduces the
    default two-subtile config's BF16 output bit for bit (INT8: same exact
    sums; FP8: same MMA order). Both runs are forced onto two-subtile tiles
    (SLSP_GEMM_MSUB=2) and the test asserts that the two launches really are
    different configurations."""
    g = torch.Generator(device="cuda").manual_seed(11)
    n, k, m = 1536, 3584, 1000
    if kind == "int8":
        w = slsp.magnitude_prune(torch.randint(-127, 128, (n, k), dtype=torch.int8, device="cuda", generator=g), 6, 8)
        qk = slsp.QUANT_INT8
    else:
        w = slsp.magnitude_prune(((torch.rand(n, k, device="cuda", generator=g) * 2 - 1) * 200).to(torch.float8_e4m3fn),
                                 6, 8)
        qk = slsp.QUANT_FP8E4M3
    x = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    s_ch = torch.rand(n, device="cuda", generator=g) * 0.01 + 0.001
    pw = slsp.pack_compress(w, 6, 8)
    payload, s_tok = slsp.fused_quant_slide(x, 6, 8, kind=qk)
    outs, cfgs = [], []
    for kh in ("0", "1"):
        # M = 1000 would take 256-token one-subtile tiles: keep it on the two-subtile ones
        with slsp.knobs(SLSP_GEMM_BN256_MAXM=0, SLSP_GEMM_MSUB=2, SLSP_GEMM_KHALF=kh):
            cfgs.append(slsp.sparse_gemm_config(pw, m, slsp.OUT_BF16_NM))
            outs.append(slsp.sparse_gemm(pw, payload, s_ch=s_ch, s_tok=s_tok, out_mode=slsp.OUT_BF16_NM))
    torch.cuda.synchronize()
    assert cfgs[0]["subtiles"] == cfgs[1]["subtiles"] == 2
    assert (cfgs[0]["half_k_stages"], cfgs[1]["half_k_stages"]) == (0, 1)
    assert cfgs[0]["stages"] < cfgs[1]["stages"]
    if kind == "int8":
        assert torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16))
    else:  # fp32 accumulation: the per-MMA k order is the same, so equal in practice; allow 1 bf16 ulp
        diff = (outs[0].float() - outs[1].float()).abs()
        assert torch.all(diff <= outs[0].float().abs() * 2 ** -7 + 1e-6)


def test_empty_inputs(slsp):
    """Empty shapes behave like the reference's (empty results, no error):
    zero tokens, zero weight rows."""
    g = torch.Generator(device="cuda").manual_seed(3)
    w = slsp.magnitude_prune(torch.randint(-127, 128, (256, 512), dtype=torch.int8, device="cuda", generator=g), 6, 8)
    pw = slsp.pack_compress(w, 6, 8)
    x0 = torch.empty((0, 512), dtype=torch.bfloat16, device="cuda")
    payload, s_tok = slsp.fused_quant_slide(x0, 6, 8)
    assert payload.shape == (0, pw.kp // 4) and s_tok.numel() == 0
    y = slsp.sparse_gemm(pw, payload)
    assert y.shape == (256, 0)
    q, qs = slsp.quantize_rows(x0)
    assert slsp.dense_gemm(w, q.view(torch.int8)).shape == (256, 0)
    w0 = torch.empty((0, 512), dtype=torch.int8, device="cuda")
    pw0 = slsp.pack_compress(w0, 6, 8)
    x = (torch.rand(64, 512, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    payload, s_tok = slsp.fused_quant_slide(x, 6, 8)
    assert slsp.sparse_gemm(pw0, payload).shape == (0, 64)
