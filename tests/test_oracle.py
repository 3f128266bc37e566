"""Pins the CPU oracle (oracle/slsp_oracle.c) — runs on CPU, no GPU.

1. Known-answer vectors restated from the reference's own tests
   (proj/tests/test_pack.cpp, test_quantize.cpp, test_gemm.cpp).
2. Golden fixtures generated from the reference library itself
   (tests/golden/gen_golden.py over oracle/_ref/libslsp_ref.so).
3. Randomised bit-for-bit agreement with the reference compiled from
   /root/reference (skipped where that build is absent, e.g. the GPU box).
"""
from pathlib import Path

import numpy as np
import pytest

from oracle_lib import (DT_BF16, DT_E4M3, DT_F32, DT_I8, KIND_FP8, KIND_INT8, OracleError, compliant_matrix,
                        f32_to_bf16_bits)

GOLDEN = Path(__file__).resolve().parent / "golden"
PATTERNS = [(4, 6), (6, 8), (8, 10), (14, 16)]


# ---------------------------------------------------------------- 1. KATs --
def test_plan_geometry(orc):
    """test_pattern.cpp:24-30 and pattern.hpp:131-154."""
    assert orc.plan(6, 8) == (3, [0, 2, 4])
    assert orc.plan(4, 6) == (2, [0, 2])
    assert orc.plan(8, 10) == (4, [0, 2, 4, 6])
    assert orc.plan(14, 16)[0] == 7
    with pytest.raises(OracleError):
        orc.plan(1, 4)  # already 2:4 compliant
    with pytest.raises(OracleError):
        orc.plan(6, 7)  # non-integral window count


def test_pack_worked_example(orc):
    """test_pack.cpp:48-59, test_gemm.cpp:114-127."""
    w = np.array([[1, 2, 3, 0, 4, 5, 0, 6]], np.int8)
    s = orc.pack_matrix(w, 6, 8, DT_I8)
    assert s.tolist() == [[1, 2, 0, 0, 3, 0, 4, 0, 0, 5, 0, 6]]
    lifted = np.array([[1, 2, 3, 4, 3, 4, 5, 6, 5, 6, 7, 8]])
    assert int((s.astype(np.int64) * lifted).sum()) == 112


def test_pack_residual_forwarding_and_zero(orc):
    """test_pack.cpp:67-78."""
    w = np.array([[1, 1, 1, 1, 1, 1, 0, 0], [0] * 8], np.int8)
    s = orc.pack_matrix(w, 6, 8, DT_I8)
    assert s[0].tolist() == [1, 1, 0, 0, 1, 1, 0, 0, 1, 1, 0, 0]
    assert s[1].tolist() == [0] * 12


def test_pack_identity_pattern_rejected_and_overfull(orc):
    """test_pack.cpp:80-90 (overfull -> NotCompliant, bad length -> DimensionMismatch)."""
    with pytest.raises(OracleError) as e:
        orc.pack_matrix(np.array([[1, 1, 1, 1, 1, 1, 1, 0]], np.int8), 6, 8, DT_I8)
    assert e.value.status == 1
    with pytest.raises(OracleError) as e:
        orc.pack_matrix(np.zeros((1, 9), np.int8), 6, 8, DT_I8)
    assert e.value.status == 2


def test_pack_reports_row_and_block(orc):
    """test_pack.cpp:225-237."""
    w = np.zeros((2, 16), np.int8)
    w[1, 8:15] = 1
    with pytest.raises(OracleError) as e:
        orc.pack_matrix(w, 6, 8, DT_I8)
    assert e.value.where == (1, 1)


def test_pack_negative_zero_is_zero(orc):
    """test_pack.cpp:92-99 (double) and the same rule for f32/bf16."""
    w = np.array([[-0.0, -0.0, 1, 2, 3, 4, 5, 6]], np.float32)
    assert np.count_nonzero(orc.pack_matrix(w, 6, 8, DT_F32)) == 6
    wb = f32_to_bf16_bits(w)
    assert np.count_nonzero(orc.pack_matrix(wb, 6, 8, DT_BF16)) == 6


def test_pack_lossless_dot_property(orc):
    """test_pack.cpp:101-116 (window dot == dense dot), vectorised."""
    rng = np.random.default_rng(11)
    for z, l in PATTERNS:
        wc, starts = orc.plan(z, l)
        w = compliant_matrix(rng, 500, 3, z, l)
        x = rng.integers(-9, 10, size=w.shape).astype(np.int64)
        s = orc.pack_matrix(w, z, l, DT_I8).astype(np.int64)
        idx = np.array([g * l + st + d for g in range(3) for st in starts for d in range(4)])
        assert np.array_equal((s * x[:, idx]).sum(1), (w.astype(np.int64) * x).sum(1))


def test_compress_window_examples(orc):
    """test_gemm.cpp:44-61: canonical padding (smallest unused positions)."""
    s = np.array([[1, 2, 0, 0, 3, 0, 4, 0, 0, 0, 0, 0, 0, 0, 7, 0]], np.int8)
    v, c = orc.compress(s, DT_I8)
    assert v.tolist() == [[1, 2, 3, 4, 0, 0, 0, 7]]
    assert c.tolist() == [[0, 1, 0, 2, 0, 1, 0, 2]]
    with pytest.raises(OracleError):
        orc.compress(np.array([[1, 2, 3, 0]], np.int8), DT_I8)


def test_quantize_worked_example_and_ties(orc):
    """test_quantize.cpp:32-71."""
    q, s = orc.quantize_rows(np.array([[1.0, -2.0, 0.5, 4.0]]), KIND_INT8, 4)  # f64
    assert q.view(np.int8).tolist() == [[32, -64, 16, 127]]
    assert s[0] == np.float32(4.0 / 127.0)
    q, s = orc.quantize_rows(np.array([[0.5, 1.5, 2.5, -0.5, -1.5, 127.0]]), KIND_INT8, 4)
    assert q.view(np.int8).tolist()[0][:5] == [0, 2, 2, 0, -2]
    q, s = orc.quantize_rows(np.zeros((1, 16), np.float32), KIND_INT8, DT_F32)
    assert s[0] == 1.0 and not q.any()


def test_quantize_never_minus_128_and_non_finite(orc):
    """test_quantize.cpp:73-103."""
    rng = np.random.default_rng(5)
    q, _ = orc.quantize_rows(rng.uniform(-100, 100, size=(200, 64)), KIND_INT8, 4)
    assert q.view(np.int8).min() >= -127
    with pytest.raises(OracleError) as e:
        orc.quantize_rows(np.array([[1.0, np.inf]]), KIND_INT8, 4)
    assert e.value.status == 4


def test_fp8_known_values(orc):
    """test_quantize.cpp:105-124."""
    kv = {448.0: 0x7E, -448.0: 0xFE, 1.0: 0x38, 0.015625: 0x08, 0.001953125: 0x01, 1000.0: 0x7E, 432.0: 0x7E,
          0.0: 0x00}
    for x, c in kv.items():
        assert orc.fp8_encode(x) == c, x
    for c in range(256):
        if (c & 0x7F) == 0x7F:
            assert np.isnan(orc.fp8_decode(c))
        else:
            assert orc.fp8_encode(orc.fp8_decode(c)) == c
    assert orc.quantize_value(-1e-9, KIND_FP8) == 0x80  # tiny negative keeps its sign
    assert orc.quantize_value(-0.0, KIND_FP8) == 0x00


def test_lift_examples(orc):
    """test_quantize.cpp:140-163."""
    x = np.arange(10, 18, dtype=np.float32)[None]
    assert orc.lift_rows(x, 6, 8, DT_F32).tolist() == [[10, 11, 12, 13, 12, 13, 14, 15, 14, 15, 16, 17]]
    x = np.arange(6, dtype=np.float32)[None]
    assert orc.lift_rows(x, 4, 6, DT_F32).tolist() == [[0, 1, 2, 3, 2, 3, 4, 5]]


def test_fused_smallest_instance_and_pack_word(orc):
    """test_quantize.cpp:198-205, 265-276."""
    x = np.arange(1, 9, dtype=np.float32)[None]
    p, s = orc.fused_quant_slide(x, 6, 8, KIND_INT8, DT_F32)
    assert p.shape == (1, 3)
    q, _ = orc.quantize_rows(x, KIND_INT8, DT_F32)
    lifted = np.concatenate([q[0, 0:4], q[0, 2:6], q[0, 4:8]])
    assert p.view(np.uint8).tolist()[0] == lifted.tolist()
    assert orc.pack_codes(np.array([1, 2, 3, 0], np.uint8)).tolist() == [1 | 2 << 2 | 3 << 4]


def test_fused_equals_composition(orc):
    """test_quantize.cpp:241-263: fused == quantize -> lift -> pack, incl. padding."""
    rng = np.random.default_rng(9)
    for z, l in PATTERNS:
        for kind in (KIND_INT8, KIND_FP8):
            for cols in (l, 3 * l, 2 * l + 3):
                x = rng.uniform(-5, 5, size=(16, cols)).astype(np.float32)
                x[3] = 0
                p, s = orc.fused_quant_slide(x, z, l, kind, DT_F32)
                groups = -(-cols // l)
                padded = np.zeros((16, groups * l), np.float32)
                padded[:, :cols] = x
                q, qs = orc.quantize_rows(padded, kind, DT_F32)
                lifted = orc.lift_rows(q, z, l, DT_E4M3)
                assert np.array_equal(p.view(np.uint8).reshape(16, -1), lifted)
                assert np.array_equal(s.view(np.uint32), qs.view(np.uint32))


def test_sparse_equals_dense_quantized(orc):
    """test_gemm.cpp:299-323 (and acceptance.cpp:45-71 for several patterns)."""
    rng = np.random.default_rng(13)
    for z, l in PATTERNS:
        w = compliant_matrix(rng, 12, 3, z, l)
        x = rng.uniform(-2, 2, size=(5, w.shape[1])).astype(np.float32)
        v, c = orc.compress(orc.pack_matrix(w, z, l, DT_I8), DT_I8)
        p, _ = orc.fused_quant_slide(x, z, l, KIND_INT8, DT_F32)
        q, _ = orc.quantize_rows(x, KIND_INT8, DT_F32)
        assert np.array_equal(orc.sparse_gemm_words(v, c, p), orc.dense_gemm_i8(w, q.view(np.int8).T.copy()))


def test_op_count_ratio_matches_expansion(orc):
    """test_gemm.cpp:283-297: sparse/dense multiplies = gamma * hw_m/hw_n."""
    from fractions import Fraction

    for z, l in PATTERNS:
        wc, _ = orc.plan(z, l)
        gamma = Fraction(wc * 4, l)
        assert Fraction(wc * 2, l) == gamma * Fraction(2, 4)


def test_dequant_epilogue_restatement(orc):
    acc = np.array([[1000, -7, 0]], np.int32)
    y = orc.dequant_bf16(acc, np.array([0.5], np.float32), np.array([2.0, 1.0, 3.0], np.float32))
    assert y.tolist() == [[f32_to_bf16_bits(np.float32(1000.0))[()], f32_to_bf16_bits(np.float32(-3.5))[()], 0]]


# ------------------------------------------------------------- 2. goldens --
@pytest.mark.parametrize("z,l", PATTERNS)
def test_golden_pack(orc, z, l):
    g = np.load(GOLDEN / f"pack_{z}_{l}.npz")
    assert np.array_equal(orc.pack_matrix(g["w"], z, l, DT_I8), g["slided"])
    v, c = orc.compress(g["slided"], DT_I8)
    assert np.array_equal(v, g["values"]) and np.array_equal(c, g["codes"])
    assert np.array_equal(orc.pack_matrix(g["w_bf16"], z, l, DT_BF16), g["slided_bf16"])
    v, c = orc.compress(g["slided_bf16"], DT_BF16)
    assert np.array_equal(v, g["values_bf16"]) and np.array_equal(c, g["codes_bf16"])


@pytest.mark.parametrize("z,l", PATTERNS)
@pytest.mark.parametrize("tag,kind", [("int8", KIND_INT8), ("fp8", KIND_FP8)])
def test_golden_fused_quant_slide(orc, z, l, tag, kind):
    g = np.load(GOLDEN / f"fqs_{z}_{l}_{tag}.npz")
    p, s = orc.fused_quant_slide(g["x"], z, l, kind, DT_F32)
    assert np.array_equal(p, g["payload"])
    assert np.array_equal(s.view(np.uint32), g["scales"].view(np.uint32))


def test_golden_gemms(orc):
    g = np.load(GOLDEN / "gemm_6_8.npz")
    assert np.array_equal(orc.sparse_gemm_words(g["values"], g["codes"], g["payload"]), g["y_sparse"])
    q, qs = orc.quantize_rows(g["x"], KIND_INT8, DT_F32)
    assert np.array_equal(q, g["q"]) and np.array_equal(qs, g["q_scales"])
    assert np.array_equal(orc.dense_gemm_i8(g["w"], q.view(np.int8).T.copy()), g["y_dense"])
    assert np.array_equal(g["y_sparse"], g["y_dense"])


def test_golden_codec_and_prune(orc):
    g = np.load(GOLDEN / "codec_prune.npz")
    assert [orc.fp8_encode(v) for v in g["xs"]] == g["enc"].tolist()
    dec = np.array([orc.fp8_decode(c) for c in range(256)], np.float32)
    assert np.array_equal(dec.view(np.uint32), g["dec"].view(np.uint32))
    assert np.array_equal(orc.magnitude_prune(g["wp"], 6, 8, DT_I8), g["pruned"])


# -------------------------------------------- 3. vs the compiled reference --
def test_randomised_vs_reference(orc, ref):
    rng = np.random.default_rng(77)
    for z, l in PATTERNS:
        w = compliant_matrix(rng, 64, 16, z, l)
        so, sr = orc.pack_matrix(w, z, l, DT_I8), ref.pack_matrix(w, z, l, DT_I8)
        assert np.array_equal(so, sr)
        (vo, co), (vr, cr) = orc.compress(so, DT_I8), ref.compress(sr, DT_I8)
        assert np.array_equal(vo, vr) and np.array_equal(co, cr)
        codes = rng.integers(0, 256, size=w.shape).astype(np.uint8)
        e = np.where(w != 0, codes | 1, np.where(rng.random(w.shape) < 0.5, 0x80, 0)).astype(np.uint8)
        assert np.array_equal(orc.pack_matrix(e, z, l, DT_E4M3), ref.pack_matrix(e, z, l, DT_E4M3))
        for kind in (KIND_INT8, KIND_FP8):
            x = (rng.standard_normal((24, 16 * l + 5)) * np.where(rng.random((24, 1)) < 0.2, 30, 1)).astype(np.float32)
            po, sco = orc.fused_quant_slide(x, z, l, kind, DT_F32)
            pr, scr = ref.fused_quant_slide(x, z, l, kind, DT_F32)
            assert np.array_equal(po, pr) and np.array_equal(sco.view(np.uint32), scr.view(np.uint32))
            xb = f32_to_bf16_bits(x)
            po, _ = orc.fused_quant_slide(xb, z, l, kind, DT_BF16)
            pr, _ = ref.fused_quant_slide(xb, z, l, kind, DT_BF16)
            assert np.array_equal(po, pr)
        x = rng.uniform(-1, 1, size=(7, w.shape[1])).astype(np.float32)
        p, _ = orc.fused_quant_slide(x, z, l, KIND_INT8, DT_F32)
        assert np.array_equal(orc.sparse_gemm_words(vo, co, p), ref.sparse_gemm_words(vr, cr, p))
        wp = rng.integers(-127, 128, size=(16, 4 * l)).astype(np.int8)
        assert np.array_equal(orc.magnitude_prune(wp, z, l, DT_I8), ref.magnitude_prune(wp, z, l, DT_I8))
    xs = rng.uniform(-600, 600, 20000)
    assert all(orc.fp8_encode(v) == ref.fp8_encode(v) for v in xs)


def test_error_locations_vs_reference(orc, ref):
    w = np.zeros((5, 24), np.int8)
    w[2, 9:16] = 3
    w[4, 0:8] = 1
    for lib in (orc, ref):
        with pytest.raises(OracleError) as e:
            lib.pack_matrix(w, 6, 8, DT_I8)
        assert e.value.where == (2, 1)
    x = np.zeros((4, 8), np.float32)
    x[1, 2] = np.nan
    x[3, 0] = np.inf
    for lib in (orc, ref):
        with pytest.raises(OracleError) as e:
            lib.fused_quant_slide(x, 6, 8, KIND_INT8, DT_F32)
        assert e.value.where == 1
