"""ctypes binding of the C ABI (include/slsp_b200.h) over torch device tensors.

This is the Python host side of the drop-in boundary. Every function takes
and returns CUDA tensors and calls exactly one ``slsp_*`` C entry point; the
library is ``paper_2603_05232_b200/libslsp_b200.so`` (built in-tree by
``paper_2603_05232_b200/build.py``). There is no CPU fallback: if the library
or a B200 is missing, calls raise.
"""
from __future__ import annotations

import contextlib
import ctypes as C
import os
import threading
from dataclasses import dataclass
from pathlib import Path

import torch

LIB_PATH = Path(os.environ.get("SLSP_LIB") or Path(__file__).resolve().parent / "libslsp_b200.so")

# ---- constants mirrored from include/slsp_b200.h -----------------------------
DT_I8, DT_BF16, DT_E4M3, DT_F32, DT_F64 = 0, 1, 2, 3, 4
QUANT_INT8, QUANT_FP8E4M3 = 0, 1
OUT_RAW_NM, OUT_BF16_NM, OUT_BF16_MN = 0, 1, 2
OK, ERR_NOT_COMPLIANT, ERR_DIMENSION, ERR_PLAN, ERR_NON_FINITE, ERR_INVALID, ERR_MALFORMED, \
    ERR_UNSUPPORTED, ERR_CUDA = range(9)
STATUS_WS_BYTES = 64


# ---- error hierarchy (pattern.hpp:24-57) -------------------------------------
class SlspError(RuntimeError):
    """slsp::Error"""


class NotCompliantError(SlspError):
    pass


class DimensionMismatchError(SlspError):
    pass


class PlanError(SlspError):
    """AlreadyCompliantError / NonIntegralWindowCountError / InsufficientCapacityError."""


class NonFiniteInputError(SlspError):
    pass


class MalformedMetadataError(SlspError):
    pass


class UnsupportedError(SlspError):
    pass


class CudaError(SlspError):
    pass


_ERRORS = {
    ERR_NOT_COMPLIANT: NotCompliantError,
    ERR_DIMENSION: DimensionMismatchError,
    ERR_PLAN: PlanError,
    ERR_NON_FINITE: NonFiniteInputError,
    ERR_INVALID: ValueError,
    ERR_MALFORMED: MalformedMetadataError,
    ERR_UNSUPPORTED: UnsupportedError,
    ERR_CUDA: CudaError,
}


class GemmConfig(C.Structure):
    """slsp_gemm_config (include/slsp_b200.h): the tile configuration a GEMM call launches."""
    _fields_ = [("tokens_per_tile", C.c_int), ("weight_rows_per_tile", C.c_int), ("subtiles", C.c_int),
                ("half_k_stages", C.c_int), ("stages", C.c_int), ("cluster_ctas", C.c_int), ("ksplit", C.c_int),
                ("epilogue", C.c_int), ("clusters", C.c_int), ("cluster_ksplit", C.c_int),
                ("workspace_bytes", C.c_int64)]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


_lib = None
_lock = threading.Lock()


def lib() -> C.CDLL:
    """Loads the native library (fails loudly; there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2603_05232_b200.build` "
                                  "(the B200 path has no CPU fallback)")
            L = C.CDLL(str(LIB_PATH))
            i64, vp, i32 = C.c_int64, C.c_void_p, C.c_int
            sigs = {
                "slsp_version": (i32, []),
                "slsp_status_string": (C.c_char_p, [i32]),
                "slsp_last_cuda_error": (C.c_char_p, []),
                "slsp_device_supported": (i32, [i32]),
                "slsp_plan_decomposition": (i32, [i32, i32, i32, i32, vp, vp, i32]),
                "slsp_pack_matrix": (i32, [i32, vp, i64, i64, i32, i32, vp, vp, vp, vp, vp]),
                "slsp_compress": (i32, [i32, vp, i64, i64, vp, vp, vp, vp, vp, vp]),
                "slsp_pack_compress": (i32, [i32, vp, i64, i64, i32, i32, i64, vp, vp, vp, vp, vp, vp]),
                "slsp_magnitude_prune": (i32, [i32, vp, i64, i64, i32, i32, vp, vp]),
                "slsp_fused_quant_slide": (i32, [i32, vp, i64, i64, i32, i32, i32, i64, vp, vp, vp, vp, vp]),
                "slsp_quantize_rows": (i32, [i32, vp, i64, i64, i32, i64, vp, vp, vp, vp, vp]),
                "slsp_lift_rows": (i32, [i32, vp, i64, i64, i32, i32, i64, vp, vp]),
                "slsp_sparse_gemm": (i32, [i32, vp, vp, i64, i64, vp, i64, vp, vp, i32, vp, i64, vp]),
                "slsp_dense_gemm": (i32, [i32, vp, i64, i64, vp, i64, vp, vp, i32, vp, i64, vp]),
                "slsp_sparse_gemm_ws": (i32, [i32, vp, vp, i64, i64, vp, i64, vp, vp, i32, vp, i64, vp, i64, vp]),
                "slsp_dense_gemm_ws": (i32, [i32, vp, i64, i64, vp, i64, vp, vp, i32, vp, i64, vp, i64, vp]),
                "slsp_gemm_workspace_bytes": (i64, [i64, i64]),
                "slsp_tile_meta": (i32, [vp, i64, i64, vp, vp]),
                "slsp_tile_meta_ex": (i32, [vp, i64, i64, i32, vp, vp]),
                "slsp_load_compressed": (i32, [i32, vp, vp, i64, i64, i64, vp, vp, vp]),
                "slsp_gemm_order": (i32, [i32, vp, vp, i64, i64, i64, vp, vp, i64, vp]),
                "slsp_sparse_gemm_x": (i32, [i32, vp, vp, i64, i64, vp, i64, vp, vp, i32, vp, i64, vp]),
                "slsp_sparse_gemm_amax": (i32, [i32, vp, vp, i64, i64, vp, i64, vp, vp, i32, vp, i64, vp, vp]),
                "slsp_fused_quant_slide_scaled": (i32, [i32, vp, i64, i64, i32, i32, i32, i64, vp, vp, vp, vp, vp,
                                                        vp]),
                "slsp_fused_quant_slide_scaled_multi": (i32, [i32, vp, i64, i64, i32, i32, i32, vp, vp, i32, i64,
                                                              i64, vp, vp, vp, vp]),
                "slsp_row_absmax": (i32, [i32, vp, i64, i64, vp, vp]),
                "slsp_ipc_get_handle": (i32, [vp, vp, vp]),
                "slsp_ipc_open_handle": (i32, [vp, vp]),
                "slsp_ipc_close": (i32, [vp]),
                "slsp_tiled_meta_bytes": (i64, [i64, i64]),
                "slsp_reload_knobs": (None, []),
                "slsp_sparse_gemm_config": (i32, [i32, i64, i64, i64, i32, i64, C.POINTER(GemmConfig)]),
                "slsp_sparse_gemm_lift": (i32, [i32, vp, vp, i64, i64, vp, i64, i64, i64, i32, i32, vp, vp, i32, vp,
                                                i64, vp, i64, vp]),
                "slsp_sparse_gemm_lift_config": (i32, [i32, i64, i64, i64, i64, i32, i32, i32, i64,
                                                       C.POINTER(GemmConfig)]),
                "slsp_dense_gemm_config": (i32, [i32, i64, i64, i64, i32, i64, C.POINTER(GemmConfig)]),
            }
            for name, (res, args) in sigs.items():
                if os.environ.get("SLSP_LIB") and not hasattr(L, name):
                    continue  # an older library build under test (perf probing): only what it exports
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def _check(status: int, what: str, msg: str | None = None) -> None:
    if status == OK:
        return
    cls = _ERRORS.get(status, SlspError)
    text = msg or f"{what}: {lib().slsp_status_string(status).decode()}"
    if status == ERR_CUDA:
        text += f" ({lib().slsp_last_cuda_error().decode()})"
    raise cls(text)


def _ptr(t: torch.Tensor | None):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(device: torch.device | None = None):
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _status_ws(device) -> torch.Tensor:
    return torch.empty(STATUS_WS_BYTES, dtype=torch.uint8, device=device)


_DT_OF = {torch.int8: DT_I8, torch.bfloat16: DT_BF16, torch.uint8: DT_E4M3, torch.float32: DT_F32,
          torch.float64: DT_F64, torch.float8_e4m3fn: DT_E4M3}


def dtype_code(t: torch.Tensor) -> int:
    try:
        return _DT_OF[t.dtype]
    except KeyError:
        raise TypeError(f"unsupported element type {t.dtype}") from None


def _raw(t: torch.Tensor) -> torch.Tensor:
    """fp8 tensors travel as their uint8 codes."""
    return t.view(torch.uint8) if t.dtype == torch.float8_e4m3fn else t


def _require_cuda(*ts: torch.Tensor) -> None:
    for t in ts:
        if t is not None and (not t.is_cuda or not t.is_contiguous()):
            raise ValueError("slsp_b200 operates on contiguous CUDA tensors")


def _require_buffer(t: torch.Tensor, name: str, dtypes, shape: tuple, device) -> None:
    """A caller-provided output buffer: CUDA, contiguous, on `device`, of one of
    `dtypes` and exactly `shape` — the kernels write shape-derived extents, so
    a smaller buffer would be overrun (the reference allocates its own results)."""
    if not t.is_cuda or not t.is_contiguous() or t.device != device:
        raise ValueError(f"{name} must be a contiguous CUDA tensor on {device}")
    if t.dtype not in dtypes:
        raise TypeError(f"{name} must have dtype {' or '.join(str(d) for d in dtypes)}, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")


def _require_scales(t: torch.Tensor | None, name: str, count: int, device) -> None:
    if t is None:
        return
    if not t.is_cuda or not t.is_contiguous() or t.device != device or t.dtype != torch.float32:
        raise ValueError(f"{name} must be a contiguous float32 CUDA tensor on {device}")
    if t.numel() < count:
        raise ValueError(f"{name} holds {t.numel()} scales, needs >= {count}")


def reload_knobs() -> None:
    """Re-read the SLSP_* tuning/probing environment variables (snapshotted by
    the library once per process otherwise)."""
    lib().slsp_reload_knobs()


@contextlib.contextmanager
def knobs(**kv):
    """Temporarily set SLSP_* knobs, e.g. ``with knobs(SLSP_GEMM_MSUB=2): ...``."""
    old = {k: os.environ.get(k) for k in kv}
    try:
        for k, v in kv.items():
            os.environ[k] = str(v)
        reload_knobs()
        yield
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        reload_knobs()


# ---- a1: geometry --------------------------------------------------------------
def plan_decomposition(z: int, l: int, hw_m: int = 2, hw_n: int = 4) -> tuple[int, list[int]]:
    """pattern.hpp:131-154 -> (window_count, window_starts)."""
    wc = C.c_int(0)
    starts = (C.c_int * 64)()
    _check(lib().slsp_plan_decomposition(z, l, hw_m, hw_n, C.byref(wc), starts, 64), "plan_decomposition")
    return wc.value, list(starts[: wc.value])


def lifted_width(cols: int, z: int, l: int) -> int:
    """K' = ceil(cols/l) * wc * 4 (quantize.hpp:130-133)."""
    wc, _ = plan_decomposition(z, l)
    return -(-cols // l) * wc * 4


def round_up(x: int, a: int) -> int:
    return -(-x // a) * a


# ---- a3-a5: packer -----------------------------------------------------------
def pack_matrix(w: torch.Tensor, z: int, l: int) -> torch.Tensor:
    """pack.hpp:171-204 pack_matrix -> slided rows x K' (same dtype)."""
    _require_cuda(w)
    rows, cols = w.shape
    wc, _ = plan_decomposition(z, l)
    if cols % l:
        raise DimensionMismatchError(f"matrix cols {cols} not divisible by block length {l}")
    out = torch.empty((rows, cols // l * wc * 4), dtype=w.dtype, device=w.device)
    er, eb = C.c_int64(-1), C.c_int64(-1)
    st = lib().slsp_pack_matrix(dtype_code(w), _ptr(_raw(w)), rows, cols, z, l, _ptr(_raw(out)),
                                _ptr(_status_ws(w.device)), C.byref(er), C.byref(eb), _stream(w.device))
    _check(st, "pack_matrix", f"row {er.value}, block {eb.value} violates pattern {z}:{l}"
           if st == ERR_NOT_COMPLIANT else None)
    return out


def compress(slided: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """gemm.hpp:70-110 compress -> (values rows x K'/2, codes rows x K'/2 bytes)."""
    _require_cuda(slided)
    rows, cexp = slided.shape
    values = torch.empty((rows, cexp // 2), dtype=slided.dtype, device=slided.device)
    codes = torch.empty((rows, cexp // 2), dtype=torch.uint8, device=slided.device)
    er, ew = C.c_int64(-1), C.c_int64(-1)
    st = lib().slsp_compress(dtype_code(slided), _ptr(_raw(slided)), rows, cexp, _ptr(_raw(values)), _ptr(codes),
                             _ptr(_status_ws(slided.device)), C.byref(er), C.byref(ew), _stream(slided.device))
    _check(st, "compress", f"window ({er.value}, {ew.value}) holds more than 2 nonzeros"
           if st == ERR_NOT_COMPLIANT else None)
    return values, codes


@dataclass
class PackedWeights:
    """MMA-ready compressed weights: values n x kp/2, meta n x kp/8 (row-major
    2-bit codes, the interchange format) and meta_tiled (slsp_tile_meta, the
    GEMM operand; built on first use if absent)."""
    values: torch.Tensor
    meta: torch.Tensor
    n: int
    k: int
    kp: int
    z: int
    l: int
    meta_tiled: torch.Tensor | None = None

    @property
    def dtype(self) -> int:
        return dtype_code(self.values)

    def tiled(self) -> torch.Tensor:
        if self.meta_tiled is None:
            self.meta_tiled = tile_meta(self.meta, self.n, self.kp, self.dtype)
        return self.meta_tiled

    def gemm_order(self) -> "GemmOrderWeights":
        """The in-SM-lifting operand (slsp_gemm_order + slsp_tile_meta), built once."""
        if getattr(self, "_gemm_order", None) is None:
            self._gemm_order = gemm_order(self)
        return self._gemm_order


@dataclass
class GemmOrderWeights:
    """Weights in the window order of slsp_sparse_gemm_x (6:8): values n x kp/2,
    tiled metadata; kx = round_up(k, 512) activation bytes per token, kp = 3kx/2."""
    values: torch.Tensor
    meta_tiled: torch.Tensor
    n: int
    k: int
    kx: int
    kp: int

    @property
    def dtype(self) -> int:
        return dtype_code(self.values)


def gemm_order(w: PackedWeights) -> GemmOrderWeights:
    """slsp_gemm_order: reference window order -> the in-SM-lifting GEMM order (6:8 only)."""
    if (w.z, w.l) != (6, 8):
        raise UnsupportedError("in-SM lifting is implemented for the 6:8 pattern")
    kx = round_up(w.k, 512)
    kp = kx * 3 // 2
    values = torch.empty((w.n, kp // 2), dtype=w.values.dtype, device=w.values.device)
    codes = torch.empty((w.n, kp // 8), dtype=torch.uint8, device=w.values.device)
    _check(lib().slsp_gemm_order(w.dtype, _ptr(_raw(w.values)), _ptr(w.meta), w.n, w.k, w.kp, _ptr(_raw(values)),
                                 _ptr(codes), kp, _stream(values.device)), "gemm_order")
    return GemmOrderWeights(values, tile_meta(codes, w.n, kp), w.n, w.k, kx, kp)


def tile_meta(meta: torch.Tensor, rows: int, kp: int, dtype: int = DT_I8) -> torch.Tensor:
    """Row-major codes -> the MMA-tiled metadata layout of operand type `dtype` (slsp_tile_meta_ex)."""
    _require_cuda(meta)
    out = torch.empty(int(lib().slsp_tiled_meta_bytes(rows, kp)), dtype=torch.uint8, device=meta.device)
    _check(lib().slsp_tile_meta_ex(_ptr(meta), rows, kp, dtype, _ptr(out), _stream(meta.device)), "tile_meta")
    return out


def pack_compress(w: torch.Tensor, z: int, l: int, kp: int | None = None, check: bool = True) -> PackedWeights:
    """Fused Φ: pack_matrix + compress + pack_codes straight into the sparse-MMA format."""
    _require_cuda(w)
    rows, cols = w.shape
    kprime = lifted_width(cols, z, l)
    kp = round_up(kprime, 256) if kp is None else kp
    values = torch.empty((rows, kp // 2), dtype=w.dtype, device=w.device)
    meta = torch.empty((rows, kp // 8), dtype=torch.uint8, device=w.device)
    er, eb = C.c_int64(-1), C.c_int64(-1)
    ws = _status_ws(w.device) if check else None
    st = lib().slsp_pack_compress(dtype_code(w), _ptr(_raw(w)), rows, cols, z, l, kp, _ptr(_raw(values)),
                                  _ptr(meta), _ptr(ws), C.byref(er), C.byref(eb), _stream(w.device))
    _check(st, "pack_compress", f"row {er.value}, block {eb.value} violates pattern {z}:{l}"
           if st == ERR_NOT_COMPLIANT else None)
    pw = PackedWeights(values, meta, rows, cols, kp, z, l)
    if kp % 256 == 0:  # GEMM-ready: tile the metadata once, offline
        pw.tiled()
    return pw


def magnitude_prune(w: torch.Tensor, z: int, l: int) -> torch.Tensor:
    """pack.hpp:238-261 magnitude_prune."""
    _require_cuda(w)
    out = torch.empty_like(w)
    _check(lib().slsp_magnitude_prune(dtype_code(w), _ptr(_raw(w)), w.shape[0], w.shape[1], z, l, _ptr(_raw(out)),
                                      _stream(w.device)), "magnitude_prune")
    return out


# ---- a6-a12: activations -----------------------------------------------------------
def _in_dtype(x: torch.Tensor) -> int:
    if x.dtype == torch.float32:
        return DT_F32
    if x.dtype == torch.bfloat16:
        return DT_BF16
    raise TypeError(f"activations must be float32 or bfloat16, got {x.dtype}")


def fused_quant_slide(x: torch.Tensor, z: int, l: int, kind: int = QUANT_INT8, kp: int | None = None,
                      check: bool = True, payload: torch.Tensor | None = None,
                      scales: torch.Tensor | None = None,
                      absmax: torch.Tensor | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    """quantize.hpp:122-174 -> (payload rows x kp/4 uint32 words as int32 storage, scales fp32).

    absmax (fp32, one per row): each row's |x|max computed upstream — the
    tok_amax of sparse_gemm(..., tok_amax=...) on the layer that produced x
    (SURVEY §8f #3); the kernel then skips its own |x|max pass. The result is
    identical to the call without it."""
    _require_cuda(x, absmax)
    rows, cols = x.shape
    kprime = lifted_width(cols, z, l)
    kp = round_up(kprime, 256) if kp is None else kp
    if kp < kprime or kp % 4:
        raise DimensionMismatchError(f"payload width kp={kp} must be >= K'={kprime} and a multiple of 4")
    if payload is None:
        payload = torch.empty((rows, kp // 4), dtype=torch.int32, device=x.device)
    else:
        _require_buffer(payload, "payload", (torch.int32, torch.uint32), (rows, kp // 4), x.device)
    if scales is None:
        scales = torch.empty(rows, dtype=torch.float32, device=x.device)
    else:
        _require_buffer(scales, "scales", (torch.float32,), (rows,), x.device)
    bad = C.c_int64(-1)
    ws = _status_ws(x.device) if check else None
    if absmax is not None:
        _require_scales(absmax, "absmax", rows, x.device)
        st = lib().slsp_fused_quant_slide_scaled(_in_dtype(x), _ptr(x), rows, cols, z, l, kind, kp, _ptr(absmax),
                                                 _ptr(payload), _ptr(scales), _ptr(ws), C.byref(bad),
                                                 _stream(x.device))
    else:
        st = lib().slsp_fused_quant_slide(_in_dtype(x), _ptr(x), rows, cols, z, l, kind, kp, _ptr(payload),
                                          _ptr(scales), _ptr(ws), C.byref(bad), _stream(x.device))
    _check(st, "fused_quant_slide", f"non-finite activation value in row {bad.value}"
           if st == ERR_NON_FINITE else None)
    # QuantizedLiftedActivation's kind and pattern (quantize.hpp:101-116) travel
    # with the payload so sparse_gemm can reject a mismatched pairing
    # (gemm.hpp:203-208) instead of computing garbage
    payload.slsp_kind = kind
    payload.slsp_pattern = (z, l)
    return payload, scales


def row_absmax(x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Per-row max |x| (fp32; NaN propagates): a rank's partial |x|max in the sharded lift."""
    _require_cuda(x)
    rows, cols = x.shape
    if out is None:
        out = torch.empty(rows, dtype=torch.float32, device=x.device)
    else:
        _require_buffer(out, "out", (torch.float32,), (rows,), x.device)
    _check(lib().slsp_row_absmax(_in_dtype(x), _ptr(x), rows, cols, _ptr(out), _stream(x.device)), "row_absmax")
    return out


def fused_quant_slide_multi(x: torch.Tensor, z: int, l: int, absmax: torch.Tensor, dsts: list, dst_ld: int,
                            dst_col: int, kind: int = QUANT_INT8, scales: torch.Tensor | None = None,
                            check: bool = True) -> torch.Tensor:
    """Lift a K-slice of X (rows x cols) with the global per-row |x|max into the
    byte column dst_col (row stride dst_ld bytes) of every payload in `dsts`
    (device pointers or tensors; the first is this device's, the rest may be
    peer mappings from ipc_open). Returns the scales (identical on every rank)."""
    _require_cuda(x, absmax)
    rows, cols = x.shape
    _require_scales(absmax, "absmax", rows, x.device)
    if scales is None:
        scales = torch.empty(rows, dtype=torch.float32, device=x.device)
    ptrs = (C.c_void_p * len(dsts))(*[d.data_ptr() if isinstance(d, torch.Tensor) else int(d) for d in dsts])
    bad = C.c_int64(-1)
    ws = _status_ws(x.device) if check else None
    st = lib().slsp_fused_quant_slide_scaled_multi(_in_dtype(x), _ptr(x), rows, cols, z, l, kind, _ptr(absmax), ptrs,
                                                   len(dsts), dst_ld, dst_col, _ptr(scales), _ptr(ws), C.byref(bad),
                                                   _stream(x.device))
    _check(st, "fused_quant_slide_multi", f"non-finite activation value in row {bad.value}"
           if st == ERR_NON_FINITE else None)
    return scales


def ipc_handle(t: torch.Tensor) -> tuple[bytes, int]:
    """(CUDA IPC handle of the allocation holding t, byte offset of t in it)."""
    buf = C.create_string_buffer(64)
    off = C.c_int64(0)
    _check(lib().slsp_ipc_get_handle(C.c_void_p(t.data_ptr()), buf, C.byref(off)), "ipc_handle")
    return buf.raw, int(off.value)


def ipc_open(handle: tuple[bytes, int]) -> tuple[int, int]:
    """Maps a peer's (handle, offset) into this process -> (base, tensor pointer)."""
    raw, off = handle
    ptr = C.c_void_p()
    _check(lib().slsp_ipc_open_handle(C.create_string_buffer(raw, 64), C.byref(ptr)), "ipc_open")
    return int(ptr.value), int(ptr.value) + off


def ipc_close(base: int) -> None:
    _check(lib().slsp_ipc_close(C.c_void_p(base)), "ipc_close")


def quantize_rows(x: torch.Tensor, kind: int = QUANT_INT8, kpad: int | None = None,
                  check: bool = True, out: torch.Tensor | None = None,
                  scales: torch.Tensor | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    """quantize.hpp:52-68 quantize_row for every token row -> (bytes rows x kpad, scales)."""
    _require_cuda(x)
    rows, cols = x.shape
    kpad = round_up(cols, 128) if kpad is None else kpad
    if kpad < cols:
        raise DimensionMismatchError(f"kpad={kpad} must be >= cols={cols}")
    if out is None:
        out = torch.empty((rows, kpad), dtype=torch.uint8, device=x.device)
    else:
        _require_buffer(out, "out", (torch.uint8, torch.int8, torch.float8_e4m3fn), (rows, kpad), x.device)
    if scales is None:
        scales = torch.empty(rows, dtype=torch.float32, device=x.device)
    else:
        _require_buffer(scales, "scales", (torch.float32,), (rows,), x.device)
    bad = C.c_int64(-1)
    ws = _status_ws(x.device) if check else None
    st = lib().slsp_quantize_rows(_in_dtype(x), _ptr(x), rows, cols, kind, kpad, _ptr(_raw(out)), _ptr(scales),
                                  _ptr(ws), C.byref(bad), _stream(x.device))
    _check(st, "quantize_rows", f"non-finite activation value in row {bad.value}"
           if st == ERR_NON_FINITE else None)
    return out, scales


def lift_rows(x: torch.Tensor, z: int, l: int, kp: int | None = None) -> torch.Tensor:
    """quantize.hpp:72-89 lift_row per token row (bf16/fp32 passthrough)."""
    _require_cuda(x)
    rows, cols = x.shape
    kprime = lifted_width(cols, z, l)
    kp = kprime if kp is None else kp
    out = torch.empty((rows, kp), dtype=x.dtype, device=x.device)
    _check(lib().slsp_lift_rows(dtype_code(x), _ptr(x), rows, cols, z, l, kp, _ptr(out), _stream(x.device)),
           "lift_rows")
    return out


# ---- a13-a15: GEMMs ------------------------------------------------------------------
def _gemm_out(out_mode: int, n: int, m: int, acc_int: bool, device, out: torch.Tensor | None):
    """The GEMM's result buffer: allocated, or the caller's checked against the
    exact extents the kernel writes (n x m / m x n, dtype of the mode)."""
    if out_mode == OUT_RAW_NM:
        dt, shape = (torch.int32 if acc_int else torch.float32), (n, m)
    elif out_mode == OUT_BF16_NM:
        dt, shape = torch.bfloat16, (n, m)
    elif out_mode == OUT_BF16_MN:
        dt, shape = torch.bfloat16, (m, n)
    else:
        raise ValueError(f"unknown out_mode {out_mode}")
    if out is None:
        return torch.empty(shape, dtype=dt, device=device)
    _require_buffer(out, "out", (dt,), shape, device)
    return out


def sparse_gemm_config(w: "PackedWeights", m: int, out_mode: int = OUT_RAW_NM) -> dict:
    """The tile configuration sparse_gemm(w, act[m], out_mode=...) launches."""
    cfg = GemmConfig()
    _check(lib().slsp_sparse_gemm_config(w.dtype, w.n, w.kp, m, out_mode, int(lib().slsp_gemm_workspace_bytes(w.n, m)),
                                         C.byref(cfg)), "sparse_gemm_config")
    return cfg.as_dict()


def dense_gemm_config(dtype: int, n: int, k: int, m: int, out_mode: int = OUT_RAW_NM) -> dict:
    cfg = GemmConfig()
    _check(lib().slsp_dense_gemm_config(dtype, n, k, m, out_mode, int(lib().slsp_gemm_workspace_bytes(n, m)),
                                        C.byref(cfg)), "dense_gemm_config")
    return cfg.as_dict()


_WS: dict = {}
_WS_MAX = 64 << 20  # the split-K slice cap (slsp_gemm_workspace_bytes bound)


def _workspace(query, device):
    """Split-K workspace for a call that splits (None when it does not): one
    buffer per device, allocated once at the library's upper bound and kept
    for the process lifetime (no per-call allocation, and CUDA graphs that
    captured it stay valid). Calls on one stream are ordered; concurrent
    streams must not split at the same time."""
    cfg = GemmConfig()
    _check(query(C.byref(cfg)), "gemm_config")
    nb = int(cfg.workspace_bytes)
    if nb == 0:
        return None, 0
    key = device.index if device.index is not None else torch.cuda.current_device()
    buf = _WS.get(key)
    if buf is None:
        buf = _WS[key] = torch.zeros(max(nb, _WS_MAX), dtype=torch.uint8, device=device)
    if buf.numel() < nb:
        raise UnsupportedError(f"split-K workspace of {nb} bytes exceeds the {buf.numel()}-byte bound")
    return buf, nb


def _check_pairing(w: "PackedWeights", act: torch.Tensor) -> None:
    """gemm.hpp:203-208: the payload's quant kind and pattern must match the weights."""
    kind = getattr(act, "slsp_kind", None)
    pattern = getattr(act, "slsp_pattern", None)
    if pattern is not None and tuple(pattern) != (w.z, w.l):
        raise DimensionMismatchError(f"activation lifted for pattern {pattern[0]}:{pattern[1]}, "
                                     f"weights packed for {w.z}:{w.l}")
    if kind is not None:
        want = QUANT_INT8 if w.values.dtype == torch.int8 else QUANT_FP8E4M3 if w.dtype == DT_E4M3 else None
        if want is None or kind != want:
            raise DimensionMismatchError(f"activation quant kind {kind} does not match {w.values.dtype} weights")


def sparse_gemm(w: PackedWeights, act: torch.Tensor, s_ch: torch.Tensor | None = None,
                s_tok: torch.Tensor | None = None, out_mode: int = OUT_RAW_NM,
                out: torch.Tensor | None = None, tok_amax: torch.Tensor | None = None) -> torch.Tensor:
    """gemm.hpp:199-233 on tcgen05.mma.sp. act: m x kp bytes (or the uint32 payload).

    tok_amax (fp32, m; BF16 outputs only): also written with each token's
    max |y| over the n outputs, the |x|max the next layer's
    fused_quant_slide(y, ..., absmax=tok_amax) needs."""
    _require_cuda(act, s_ch, s_tok, tok_amax)
    m = act.shape[0]
    if act.shape[1] * act.element_size() != w.kp * w.values.element_size():
        raise DimensionMismatchError("lifted activation width does not match compressed weights")
    _check_pairing(w, act)
    _require_scales(s_ch, "s_ch", w.n, act.device)
    _require_scales(s_tok, "s_tok", m, act.device)
    o = _gemm_out(out_mode, w.n, m, w.values.dtype == torch.int8, act.device, out)
    ldo = o.shape[1]
    if tok_amax is not None:
        if out_mode == OUT_RAW_NM:
            raise ValueError("tok_amax needs a BF16 output mode")
        _require_scales(tok_amax, "tok_amax", m, act.device)
        _check(lib().slsp_sparse_gemm_amax(w.dtype, _ptr(_raw(w.values)), _ptr(w.tiled()), w.n, w.kp, _ptr(act), m,
                                           _ptr(s_ch), _ptr(s_tok), out_mode, _ptr(o), ldo, _ptr(tok_amax),
                                           _stream(act.device)), "sparse_gemm")
        return o
    wsb0 = int(lib().slsp_gemm_workspace_bytes(w.n, m))
    ws, wsb = _workspace(lambda q: lib().slsp_sparse_gemm_config(w.dtype, w.n, w.kp, m, out_mode, wsb0, q),
                         act.device)
    _check(lib().slsp_sparse_gemm_ws(w.dtype, _ptr(_raw(w.values)), _ptr(w.tiled()), w.n, w.kp, _ptr(act), m,
                                     _ptr(s_ch), _ptr(s_tok), out_mode, _ptr(o), ldo, _ptr(ws), wsb,
                                     _stream(act.device)), "sparse_gemm")
    return o


def sparse_gemm_lift(w: PackedWeights, x: torch.Tensor, s_ch: torch.Tensor | None = None,
                     s_tok: torch.Tensor | None = None, out_mode: int = OUT_RAW_NM,
                     out: torch.Tensor | None = None) -> torch.Tensor:
    """BF16 sparse GEMM on the UNLIFTED activations x (m x w.k BF16): the
    lift (quantize.hpp:72-89 lift_row) runs inside the GEMM's lift warps, so
    no lifted copy of x is written (decode-shaped M). Equals
    sparse_gemm(w, lift_rows(x, w.z, w.l, w.kp)) bit for bit."""
    _require_cuda(s_ch, s_tok)
    if not x.is_cuda:
        raise ValueError("slsp_b200 operates on CUDA tensors")
    if w.values.dtype != torch.bfloat16 or x.dtype != torch.bfloat16:
        raise UnsupportedError("sparse_gemm_lift: BF16 weights and activations")
    if x.dim() != 2 or x.shape[1] != w.k:
        raise DimensionMismatchError(f"activation rows must hold k = {w.k} BF16 values")
    if x.stride(1) != 1:
        x = x.contiguous()
    m = x.shape[0]
    _require_scales(s_ch, "s_ch", w.n, x.device)
    _require_scales(s_tok, "s_tok", m, x.device)
    o = _gemm_out(out_mode, w.n, m, False, x.device, out)
    ldo = o.shape[1]
    wsb0 = int(lib().slsp_gemm_workspace_bytes(w.n, m))
    ws, wsb = _workspace(lambda q: lib().slsp_sparse_gemm_lift_config(w.dtype, w.n, w.kp, m, w.k, w.z, w.l, out_mode,
                                                                      wsb0, q), x.device)
    _check(lib().slsp_sparse_gemm_lift(w.dtype, _ptr(w.values), _ptr(w.tiled()), w.n, w.kp, _ptr(x), x.stride(0), m,
                                       w.k, w.z, w.l, _ptr(s_ch), _ptr(s_tok), out_mode, _ptr(o), ldo, _ptr(ws), wsb,
                                       _stream(x.device)), "sparse_gemm_lift")
    return o


def sparse_gemm_x(w: "PackedWeights | GemmOrderWeights", act: torch.Tensor, s_ch: torch.Tensor | None = None,
                  s_tok: torch.Tensor | None = None, out_mode: int = OUT_RAW_NM,
                  out: torch.Tensor | None = None) -> torch.Tensor:
    """Sparse GEMM with in-SM lifting: act = quantize_rows(x, kpad=w.kx) (m x kx
    bytes, UNLIFTED); equals sparse_gemm(w, fused_quant_slide(x)) bit for bit."""
    g = w.gemm_order() if isinstance(w, PackedWeights) else w
    _require_cuda(act, s_ch, s_tok)
    m = act.shape[0]
    if act.shape[1] * act.element_size() != g.kx:
        raise DimensionMismatchError(f"activation rows must be kx = {g.kx} bytes (quantize_rows(x, kpad=kx))")
    _require_scales(s_ch, "s_ch", g.n, act.device)
    _require_scales(s_tok, "s_tok", m, act.device)
    o = _gemm_out(out_mode, g.n, m, g.values.dtype == torch.int8, act.device, out)
    ldo = o.shape[1]
    _check(lib().slsp_sparse_gemm_x(g.dtype, _ptr(_raw(g.values)), _ptr(g.meta_tiled), g.n, g.kx, _ptr(act), m,
                                    _ptr(s_ch), _ptr(s_tok), out_mode, _ptr(o), ldo, _stream(act.device)),
           "sparse_gemm_x")
    return o


def dense_gemm(w: torch.Tensor, act: torch.Tensor, s_ch: torch.Tensor | None = None,
               s_tok: torch.Tensor | None = None, out_mode: int = OUT_RAW_NM,
               out: torch.Tensor | None = None) -> torch.Tensor:
    """gemm.hpp:142-162 on tcgen05.mma. w: n x k, act: m x k (token rows)."""
    _require_cuda(w, act, s_ch, s_tok)
    n, k = w.shape
    m = act.shape[0]
    if act.shape[1] * act.element_size() != k * w.element_size():
        raise DimensionMismatchError("dense_gemm: W.cols must equal X.rows")
    _require_scales(s_ch, "s_ch", n, act.device)
    _require_scales(s_tok, "s_tok", m, act.device)
    o = _gemm_out(out_mode, n, m, w.dtype == torch.int8, act.device, out)
    ldo = o.shape[1]
    wsb0 = int(lib().slsp_gemm_workspace_bytes(n, m))
    ws, wsb = _workspace(lambda q: lib().slsp_dense_gemm_config(dtype_code(w), n, k, m, out_mode, wsb0, q),
                         act.device)
    _check(lib().slsp_dense_gemm_ws(dtype_code(w), _ptr(_raw(w)), n, k, _ptr(act), m, _ptr(s_ch), _ptr(s_tok),
                                    out_mode, _ptr(o), ldo, _ptr(ws), wsb, _stream(act.device)), "dense_gemm")
    return o


def device_supported(dev: int = 0) -> bool:
    return bool(lib().slsp_device_supported(dev))
