"""Diagnostic driver for the tcgen05 GEMMs (run on a B200 under `timeout`).

Prints, per configuration, whether the int32 result matches the CPU oracle and
a small mismatch summary. Test infrastructure only (uses the oracle)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))

import paper_2603_05232_b200 as slsp  # noqa: E402
from helpers import compliant_matrix, lifted_width, mma_format, pad_cols, round_up  # noqa: E402
from oracle_lib import DT_F32, DT_I8, KIND_INT8, orc  # noqa: E402

O = orc()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def summary(name, got, want):
    eq = got == want
    print(f"[{name}] match={eq.all()} frac_equal={eq.mean():.4f} shape={got.shape}", flush=True)
    if not eq.all():
        idx = np.argwhere(~eq)[:6]
        for i in idx:
            print("   at", tuple(i), "got", got[tuple(i)], "want", want[tuple(i)])
        rows_bad = (~eq).any(axis=1)
        cols_bad = (~eq).any(axis=0)
        print("   bad rows:", np.flatnonzero(rows_bad)[:20], "count", rows_bad.sum())
        print("   bad cols:", np.flatnonzero(cols_bad)[:20], "count", cols_bad.sum())


def dense(n, k, m, seed=0):
    rng = np.random.default_rng(seed)
    w = rng.integers(-127, 128, size=(n, k)).astype(np.int8)
    x = rng.integers(-127, 128, size=(m, k)).astype(np.int8)
    t = time.time()
    got = slsp.dense_gemm(dev(w), dev(x)).cpu().numpy()
    print(f"dense {n}x{k}x{m} ran in {time.time() - t:.3f}s", flush=True)
    summary(f"dense {n},{k},{m}", got, O.dense_gemm_i8(w, x.T.copy()))


def sparse(n, k, m, seed=0):
    rng = np.random.default_rng(seed)
    w = compliant_matrix(rng, n, k // 8, 6, 8)
    x = rng.uniform(-1, 1, size=(m, k)).astype(np.float32)
    vals, codes = O.compress(O.pack_matrix(w, 6, 8, DT_I8), DT_I8)
    payload, _ = O.fused_quant_slide(x, 6, 8, KIND_INT8, DT_F32)
    kp = round_up(lifted_width(k, 6, 8), 256)
    v, meta = mma_format(vals, codes, kp)
    pw = slsp.PackedWeights(dev(v), dev(meta), n, k, kp, 6, 8)
    act = dev(pad_cols(payload.view(np.uint8).reshape(m, -1), kp))
    t = time.time()
    got = slsp.sparse_gemm(pw, act).cpu().numpy()
    print(f"sparse {n}x{k}x{m} (kp={kp}) ran in {time.time() - t:.3f}s", flush=True)
    want = O.sparse_gemm_words(vals, codes, payload)
    summary(f"sparse {n},{k},{m}", got, want)
    if not (got == want).all():
        # Hypothesis checks on the metadata semantics: every window taking
        # positions (0,1) regardless of codes, or codes read per 4-col offset.
        c01 = np.zeros_like(codes)
        c01[:, 1::2] = 1
        alt = O.sparse_gemm_words(vals, c01, payload)
        print("   == result if metadata ignored (codes (0,1)):", (got == alt).mean())


if __name__ == "__main__":
    print(torch.cuda.get_device_name(), flush=True)
    dense(256, 128, 256)
    dense(512, 1024, 512, 1)
    sparse(256, 168, 224)
    sparse(512, 1024, 448, 2)
    sparse(300, 400, 250, 3)
