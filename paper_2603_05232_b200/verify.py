"""GPU check_equivalence (gemm.hpp:258-286).

Runs the dense product and the full sparse pipeline (pack -> compress -> lift
-> sparse GEMM) on the same integer operands, all on the B200, and compares
elementwise on the device — the reference's dual-path oracle at full model
shapes, without the CPU oracle's minutes per layer.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _native as N


@dataclass
class EquivalenceReport:
    """gemm.hpp EquivalenceReport: integer inputs must agree exactly."""
    exact: bool
    max_abs_diff: float
    sparse_multiplies: int  # OpCounts of the two paths (gemm.hpp:51-53)
    dense_multiplies: int


def check_equivalence(w: torch.Tensor, x: torch.Tensor, z: int, l: int) -> EquivalenceReport:
    """w: int8 N x K (device), x: int8 K x M (the reference's orientation, columns
    are tokens). Raises NotCompliantError for weights that violate z:l
    (gemm.hpp:265-270, the packer reports the first (row, block))."""
    if w.dtype != torch.int8 or x.dtype != torch.int8:
        raise TypeError("check_equivalence: int8 operands (the exact-arithmetic case)")
    n, k = w.shape
    if x.shape[0] != k:
        raise N.DimensionMismatchError("W.cols must equal X.rows")
    m = x.shape[1]
    xt = x.t().contiguous()  # token rows
    pw = N.pack_compress(w, z, l)  # raises NotCompliantError("row R, block B violates pattern z:l")
    # lift_activations on int8: the gather through our lift kernel on the exact
    # bf16 image of the codes (|v| <= 127 is exact in bf16), cast back
    lifted = N.lift_rows(xt.to(torch.bfloat16), z, l, kp=pw.kp).to(torch.int8)
    ys = N.sparse_gemm(pw, lifted)
    kpad = N.round_up(k, 128)
    xd = torch.zeros((m, kpad), dtype=torch.int8, device=x.device)
    xd[:, :k] = xt
    wd = w if kpad == k else torch.nn.functional.pad(w, (0, kpad - k))
    yd = N.dense_gemm(wd.contiguous(), xd)
    diff = (ys.to(torch.int64) - yd.to(torch.int64)).abs()
    wc = (l - 4) // 2 + 1
    windows = -(-k // l) * wc
    return EquivalenceReport(bool(torch.equal(ys, yd)), float(diff.max().item()) if diff.numel() else 0.0,
                             n * windows * 2 * m, n * k * m)
