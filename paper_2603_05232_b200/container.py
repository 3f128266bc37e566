"""SLSP tensor containers (container.hpp) -> device operands.

The paper's offline -> load flow: weights are packed once and stored as a
kind-2 ("compressed") container; at load time they become the sparse GEMM's
operands. Host side (this module): the file format of container.hpp:1-19 —
header, u64-length sections, CRC-32 tail — with the reference's validation and
ContainerError messages (deserialize :205-247, validate_payload :168-203).
Device side: `slsp_load_compressed` re-lays the values and the packed 2-bit code
stream into the MMA layout (the codes already are the 2:4 hardware nibbles, so
loading is a retile, not a re-encode), then `slsp_tile_meta_ex`.
"""
from __future__ import annotations

import ctypes as C
import os
import struct
import zlib
from dataclasses import dataclass, field
from pathlib import Path

import torch

from . import _native as N

MAGIC = b"SLSP"
VERSION = 1
KIND_DENSE, KIND_SLIDED, KIND_COMPRESSED, KIND_QUANTIZED = 0, 1, 2, 3
DT_INT8, DT_INT32, DT_FP32, DT_FP64, DT_FP8 = 0, 1, 2, 3, 4
_DT_SIZE = {DT_INT8: 1, DT_INT32: 4, DT_FP32: 4, DT_FP64: 8, DT_FP8: 1}
_TORCH = {DT_INT8: torch.int8, DT_INT32: torch.int32, DT_FP32: torch.float32, DT_FP64: torch.float64,
          DT_FP8: torch.float8_e4m3fn}


class ContainerError(N.SlspError):
    """container.hpp ContainerError (pattern.hpp error hierarchy)."""


@dataclass
class Container:
    """container.hpp:61-77 Container: raw sections, no interpretation."""
    kind: int = KIND_DENSE
    dtype: int = DT_INT8
    z: int = 0
    l: int = 0
    hw_m: int = 0
    hw_n: int = 0
    rows: int = 0
    cols: int = 0
    values: bytes = b""
    metadata: bytes = b""
    scales: list = field(default_factory=list)


def _validate(c: Container) -> None:
    """container.hpp:168-203 validate_payload."""
    elem = _DT_SIZE[c.dtype]
    if c.kind in (KIND_DENSE, KIND_SLIDED):
        if len(c.values) != c.rows * c.cols * elem:
            raise ContainerError("values payload does not match shape")
    elif c.kind == KIND_COMPRESSED:
        if c.hw_m == 0 or c.hw_n == 0:
            raise ContainerError("compressed container needs a pattern")
        codes = c.rows * c.cols * c.hw_m
        if len(c.values) != codes * elem:
            raise ContainerError("values payload does not match shape")
        if len(c.metadata) != (codes + 3) // 4:
            raise ContainerError("metadata payload does not match shape")
    else:
        if len(c.values) != c.rows * c.cols * 4:
            raise ContainerError("word payload does not match shape")
        if len(c.scales) != c.rows:
            raise ContainerError("scale count does not match rows")
        if c.dtype not in (DT_INT8, DT_FP8):
            raise ContainerError("quantized container must be int8 or fp8e4m3")
    if c.kind == KIND_DENSE:
        if c.z or c.l or c.hw_m or c.hw_n:
            raise ContainerError("dense container must zero pattern")
    elif c.z == 0 or c.l == 0 or c.hw_m == 0 or c.hw_n == 0:
        raise ContainerError("transformed container needs a pattern")


def deserialize(data: bytes) -> Container:
    """container.hpp:205-247 deserialize (same checks, same order, same messages)."""
    if len(data) < 36:
        raise ContainerError("container truncated")
    if data[:4] != MAGIC:
        raise ContainerError("bad magic; not a tensor container")
    body, tail = data[:-4], data[-4:]
    if zlib.crc32(body) & 0xFFFFFFFF != struct.unpack("<I", tail)[0]:
        raise ContainerError("checksum mismatch")
    pos = 4

    def take(n):
        nonlocal pos
        if pos + n > len(body):
            raise ContainerError("container truncated")
        out = body[pos:pos + n]
        pos += n
        return out

    (version,) = struct.unpack("<H", take(2))
    if version != VERSION:
        raise ContainerError(f"unsupported container version {version}")
    c = Container()
    c.kind = take(1)[0]
    if c.kind > 3:
        raise ContainerError("unknown kind")
    c.dtype = take(1)[0]
    if c.dtype > 4:
        raise ContainerError("unknown dtype")
    c.z, c.l, c.hw_m, c.hw_n = struct.unpack("<4H", take(8))
    c.rows, c.cols = struct.unpack("<2Q", take(16))

    def block():
        (n,) = struct.unpack("<Q", take(8))
        return take(n)

    c.values = block()
    if c.kind == KIND_COMPRESSED:
        c.metadata = block()
    if c.kind == KIND_QUANTIZED:
        raw = block()
        if len(raw) % 4 != 0:
            raise ContainerError("scale payload not a multiple of 4 bytes")
        c.scales = list(struct.unpack(f"<{len(raw) // 4}f", raw))
    if pos != len(body):
        raise ContainerError("trailing bytes after payload")
    _validate(c)
    return c


def serialize(c: Container) -> bytes:
    """container.hpp:141-166 serialize."""
    _validate(c)
    out = bytearray(MAGIC)
    out += struct.pack("<HBB4H2Q", VERSION, c.kind, c.dtype, c.z, c.l, c.hw_m, c.hw_n, c.rows, c.cols)
    out += struct.pack("<Q", len(c.values)) + c.values
    if c.kind == KIND_COMPRESSED:
        out += struct.pack("<Q", len(c.metadata)) + c.metadata
    if c.kind == KIND_QUANTIZED:
        out += struct.pack("<Q", 4 * len(c.scales)) + struct.pack(f"<{len(c.scales)}f", *c.scales)
    out += struct.pack("<I", zlib.crc32(bytes(out)) & 0xFFFFFFFF)
    return bytes(out)


def load_container(path) -> Container:
    """container.hpp:264-275 load_container."""
    try:
        data = Path(path).read_bytes()
    except OSError as e:
        raise ContainerError(f"cannot read {path}: {e}") from e
    return deserialize(data)


def save_container(path, c: Container) -> None:
    """container.hpp:249-262 save_container: written to a temporary file in the
    destination directory, flushed, then renamed over the destination, so a
    failed write never leaves a truncated container or destroys the old one."""
    path = Path(path)
    data = serialize(c)
    tmp = path.with_name(f"{path.name}.tmp{os.getpid()}")
    try:
        with open(tmp, "wb") as f:
            f.write(data)
            f.flush()
            os.fsync(f.fileno())
        os.replace(tmp, path)
    except OSError as e:
        tmp.unlink(missing_ok=True)
        raise ContainerError(f"cannot write {path}: {e}") from e


# ---- device side ---------------------------------------------------------------------
def compressed_to_device(c: Container, device=None, kp: int | None = None) -> N.PackedWeights:
    """A kind-2 container -> GEMM-ready PackedWeights (values + tiled metadata),
    the device counterpart of container.hpp:424-435 compressed_from."""
    if c.kind != KIND_COMPRESSED:
        raise ContainerError("expected a compressed container")
    if c.hw_m != 2 or c.hw_n != 4:
        raise N.UnsupportedError("the sparse tensor core path is 2:4")
    if c.dtype not in (DT_INT8, DT_FP8):
        raise N.UnsupportedError("device load: int8 / fp8e4m3 weights (the GEMM operand types)")
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    rows, windows = c.rows, c.cols
    kp = N.round_up(4 * windows, 256) if kp is None else kp
    tdt = _TORCH[c.dtype]
    vals_in = torch.frombuffer(bytearray(c.values), dtype=torch.uint8).to(device)
    stream_in = torch.frombuffer(bytearray(c.metadata), dtype=torch.uint8).to(device)
    values = torch.empty((rows, kp // 2), dtype=tdt, device=device)
    meta = torch.empty((rows, kp // 8), dtype=torch.uint8, device=device)
    N._check(N.lib().slsp_load_compressed(N.DT_I8 if c.dtype == DT_INT8 else N.DT_E4M3, N._ptr(vals_in),
                                          N._ptr(stream_in), rows, windows, kp, N._ptr(N._raw(values)),
                                          N._ptr(meta), N._stream(device)), "load_compressed")
    # K of the source matrix: windows per row = ceil(K/l) * wc; the lifted width is 4*windows
    wc = (c.l - 4) // 2 + 1
    k = windows // wc * c.l
    pw = N.PackedWeights(values, meta, rows, k, kp, c.z, c.l)
    pw.tiled()
    return pw


def quantized_to_device(c: Container, device=None, kp: int | None = None):
    """A kind-3 container -> (payload rows x kp/4 words, scales): the GEMM's
    lifted-activation operand (container.hpp:437-449 quantized_from)."""
    if c.kind != KIND_QUANTIZED:
        raise ContainerError("expected a quantized container")
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    words = c.cols
    kp = N.round_up(4 * words, 256) if kp is None else kp
    host = torch.zeros((c.rows, kp // 4), dtype=torch.int32)
    if words:
        host[:, :words] = torch.frombuffer(bytearray(c.values), dtype=torch.int32).view(c.rows, words)
    scales = torch.tensor(c.scales, dtype=torch.float32)
    return host.to(device), scales.to(device)


def compressed_from_device(pw: N.PackedWeights, windows: int | None = None) -> Container:
    """PackedWeights -> a kind-2 container (container.hpp:379-390 to_container),
    for the round trip: the real windows of each row, codes re-packed as one
    contiguous stream."""
    wc = (pw.l - 4) // 2 + 1
    windows = -(-pw.k // pw.l) * wc if windows is None else windows
    vals = pw.values.view(torch.uint8).reshape(pw.n, -1)[:, : 2 * windows * pw.values.element_size()].cpu()
    meta = pw.meta.cpu()
    # row-major nibbles -> one stream of rows*windows nibbles
    lo, hi = meta & 0xF, meta >> 4
    nib = torch.stack([lo, hi], dim=-1).reshape(pw.n, -1)[:, :windows].reshape(-1)
    if nib.numel() % 2:
        nib = torch.cat([nib, torch.zeros(1, dtype=nib.dtype)])
    stream = (nib[0::2] | (nib[1::2] << 4)).to(torch.uint8)
    dt = DT_INT8 if pw.values.dtype == torch.int8 else DT_FP8
    return Container(KIND_COMPRESSED, dt, pw.z, pw.l, 2, 4, pw.n, windows, bytes(vals.contiguous().numpy()),
                     bytes(stream.numpy()))


def load_compressed(path, device=None, kp: int | None = None) -> N.PackedWeights:
    """File -> GEMM-ready weights in one call."""
    return compressed_to_device(load_container(path), device, kp)
