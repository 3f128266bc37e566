"""Shared test utilities: input synthesis and reference-format <-> MMA-format maps."""
from __future__ import annotations

import numpy as np

from oracle_lib import compliant_matrix  # noqa: F401  (re-export)


def round_up(x: int, a: int) -> int:
    return -(-x // a) * a


def lifted_width(cols: int, z: int, l: int) -> int:
    wc = (l - 4) // 2 + 1
    return -(-cols // l) * wc * 4


def mma_format(values: np.ndarray, codes: np.ndarray, kp: int) -> tuple[np.ndarray, np.ndarray]:
    """Reference compress() output (values, one code per byte) -> the packed
    sparse-MMA format: values n x kp/2, meta n x kp/8 with 2-bit codes LSB
    first (container.hpp:330-336), padding windows = zero values, codes (0,1)."""
    n, half = values.shape
    v = np.zeros((n, kp // 2), dtype=values.dtype)
    v[:, :half] = values
    c = np.zeros((n, kp // 2), dtype=np.uint8)
    c[:, 0::2] = 0
    c[:, 1::2] = 1
    c[:, :half] = codes
    c4 = c.reshape(n, kp // 8, 4).astype(np.uint8)
    meta = (c4[..., 0] | (c4[..., 1] << 2) | (c4[..., 2] << 4) | (c4[..., 3] << 6)).astype(np.uint8)
    return v, meta


def pad_cols(a: np.ndarray, width: int) -> np.ndarray:
    out = np.zeros((a.shape[0], width), dtype=a.dtype)
    out[:, : a.shape[1]] = a
    return out


def bf16_round(x: np.ndarray) -> np.ndarray:
    """float32 -> nearest bf16 value, returned as float32 (RNE)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return (u.astype(np.uint32) << 16).view(np.float32)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(bf16_round(x)).view(np.uint32) >> 16).astype(np.uint16)


def random_pruned_int8(rng: np.random.Generator, rows: int, cols: int, z: int, l: int) -> np.ndarray:
    """magnitude_prune(U[-127,127], z:l) restated in numpy (pack.hpp:238-261):
    zero the l-z smallest |v| per block, ties prune the lower index first."""
    w = rng.integers(-127, 128, size=(rows, cols)).astype(np.int8)
    blocks = w.reshape(rows, cols // l, l)
    mag = np.abs(blocks.astype(np.int16))
    order = np.argsort(mag, axis=-1, kind="stable")
    prune = order[..., : l - z]
    np.put_along_axis(blocks, prune, 0, axis=-1)
    return blocks.reshape(rows, cols)
