"""Generates tests/golden/*.npz from the REFERENCE implementation.

Runs the reference headers compiled unmodified (oracle/_ref/libslsp_ref.so,
built by `make -C oracle ref` from /root/reference/proj/include) on seeded
inputs and stores inputs + outputs. These fixtures pin the plain-C oracle
(tests/test_oracle.py) on machines where /root/reference does not exist
(the GPU box). Re-run: `python tests/golden/gen_golden.py`.
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))

from oracle_lib import (DT_BF16, DT_E4M3, DT_F32, DT_I8, KIND_FP8, KIND_INT8,  # noqa: E402
                        compliant_matrix, f32_to_bf16_bits, ref)

PATTERNS = [(4, 6), (6, 8), (8, 10), (14, 16)]


def main():
    R = ref()
    if R is None:
        raise SystemExit("oracle/_ref/libslsp_ref.so missing: run `make -C oracle ref` where /root/reference exists")
    rng = np.random.default_rng(20261017)

    # --- packer / compress, all four patterns, int8 and bf16 ---------------
    for z, l in PATTERNS:
        w = compliant_matrix(rng, 48, 12, z, l)
        slided = R.pack_matrix(w, z, l, DT_I8)
        values, codes = R.compress(slided, DT_I8)
        wb = f32_to_bf16_bits(np.where(w != 0, rng.uniform(-3, 3, w.shape), 0).astype(np.float32))
        sb = R.pack_matrix(wb, z, l, DT_BF16)
        vb, cb = R.compress(sb, DT_BF16)
        np.savez_compressed(HERE / f"pack_{z}_{l}.npz", w=w, slided=slided, values=values, codes=codes,
                            w_bf16=wb, slided_bf16=sb, values_bf16=vb, codes_bf16=cb)

    # --- fused_quant_slide: int8 + fp8, padded widths, an all-zero row -------
    for z, l in PATTERNS:
        for kind, tag in ((KIND_INT8, "int8"), (KIND_FP8, "fp8")):
            x = rng.uniform(-5, 5, size=(12, 2 * l + 3)).astype(np.float32)
            x[3] = 0
            payload, scales = R.fused_quant_slide(x, z, l, kind, DT_F32)
            np.savez_compressed(HERE / f"fqs_{z}_{l}_{tag}.npz", x=x, payload=payload, scales=scales)

    # --- sparse_gemm (packed words) and dense_gemm: int32 exact --------------
    z, l = 6, 8
    w = compliant_matrix(rng, 24, 16, z, l)
    x = rng.uniform(-1, 1, size=(9, w.shape[1])).astype(np.float32)
    values, codes = R.compress(R.pack_matrix(w, z, l, DT_I8), DT_I8)
    payload, scales = R.fused_quant_slide(x, z, l, KIND_INT8, DT_F32)
    y = R.sparse_gemm_words(values, codes, payload, threads=1)
    q, qs = R.quantize_rows(x, KIND_INT8, DT_F32)
    yd = R.dense_gemm_i8(w, q.view(np.int8).T.copy(), threads=1)
    np.savez_compressed(HERE / "gemm_6_8.npz", w=w, x=x, values=values, codes=codes, payload=payload,
                        scales=scales, y_sparse=y, q=q, q_scales=qs, y_dense=yd)

    # --- fp8 codec and magnitude_prune ----------------------------------------
    xs = np.concatenate([rng.uniform(-500, 500, 2000), rng.uniform(-0.01, 0.01, 2000),
                         np.array([448.0, -448.0, 1.0, 2.0 ** -6, 2.0 ** -9, 1000.0, 432.0, 0.0, -0.0, -1e-9])])
    enc = np.array([R.fp8_encode(v) for v in xs], np.uint8)
    dec = np.array([R.fp8_decode(c) for c in range(256)], np.float32)
    wp = rng.integers(-127, 128, size=(16, 48)).astype(np.int8)
    pruned = R.magnitude_prune(wp, 6, 8, DT_I8)
    np.savez_compressed(HERE / "codec_prune.npz", xs=xs, enc=enc, dec=dec, wp=wp, pruned=pruned)
    # --- SLSP containers (container.hpp) written by the reference: kind 2 ----
    # (compressed weights, even and odd windows per row) and kind 3 (lifted
    # activations); pin the loader of SURVEY.md §8f #1
    for tag, rows, groups in (("even", 40, 64), ("odd", 7, 5)):
        w = compliant_matrix(rng, rows, groups, 6, 8)
        values, codes = R.compress(R.pack_matrix(w, 6, 8, DT_I8), DT_I8)
        (HERE / f"container_6_8_{tag}.slsp").write_bytes(R.serialize_compressed_i8(values, codes, 6, 8))
        np.savez_compressed(HERE / f"container_6_8_{tag}.npz", w=w, values=values, codes=codes)
    x = rng.uniform(-2, 2, size=(9, 96)).astype(np.float32)
    payload, scales = R.fused_quant_slide(x, 6, 8, KIND_INT8, DT_F32)
    (HERE / "container_fqs_6_8.slsp").write_bytes(R.serialize_quantized(payload, scales, 6, 8, KIND_INT8))
    np.savez_compressed(HERE / "container_fqs_6_8.npz", x=x, payload=payload, scales=scales)
    print("wrote", sorted(p.name for p in HERE.glob("*.npz")))


if __name__ == "__main__":
    main()
