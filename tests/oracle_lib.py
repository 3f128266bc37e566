"""ctypes front-end to the CPU oracle libraries — TEST INFRASTRUCTURE ONLY.

Loads oracle/_build/libslsp_oracle.so (the plain-C restatement, prefix
``orc_``) and, when present, oracle/_ref/libslsp_ref.so (the reference headers
compiled unmodified, prefix ``ref_``). Both expose the interface declared in
oracle/slsp_oracle.h. Only tests/, ``__graft_entry__.smoke()`` and bench.py's
CPU-baseline legs import this module; the B200 product never does.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORC_PATH = ROOT / "oracle" / "_build" / "libslsp_oracle.so"
REF_PATH = ROOT / "oracle" / "_ref" / "libslsp_ref.so"

DT_I8, DT_BF16, DT_E4M3, DT_F32, DT_F64 = 0, 1, 2, 3, 4
KIND_INT8, KIND_FP8 = 0, 1
ST_OK, ST_NOT_COMPLIANT, ST_DIM, ST_PLAN, ST_NONFINITE, ST_INVALID, ST_MALFORMED = range(7)

_NP_OF = {DT_I8: np.int8, DT_BF16: np.uint16, DT_E4M3: np.uint8, DT_F32: np.float32, DT_F64: np.float64}


class OracleError(RuntimeError):
    def __init__(self, status: int, where=None):
        super().__init__(f"oracle status {status} at {where}")
        self.status = status
        self.where = where


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class Oracle:
    """One of the two CPU implementations of the path (``orc_`` or ``ref_``)."""

    def __init__(self, path: Path, prefix: str):
        self.lib = C.CDLL(str(path))
        self.prefix = prefix
        self.path = path
        i64, vp, i32 = C.c_int64, C.c_void_p, C.c_int
        sig = {
            "plan": (i32, [i32, i32, i32, i32, vp, vp, i32]),
            "pack_matrix": (i32, [i32, vp, i64, i64, i32, i32, vp, vp, vp, i32]),
            "compress": (i32, [i32, vp, i64, i64, vp, vp, vp, vp]),
            "fused_quant_slide": (i32, [i32, vp, i64, i64, i32, i32, i32, vp, vp, vp, i32]),
            "quantize_rows": (i32, [i32, vp, i64, i64, i32, vp, vp, vp]),
            "lift_rows": (i32, [i32, vp, i64, i64, i32, i32, vp]),
            "sparse_gemm_words": (i32, [vp, vp, i64, i64, vp, i64, vp, i32]),
            "sparse_gemm_f64": (i32, [vp, vp, i64, i64, vp, i64, vp, i32]),
            "dense_gemm_i8": (i32, [vp, i64, i64, vp, i64, vp, i32]),
            "magnitude_prune": (i32, [i32, vp, i64, i64, i32, i32, vp]),
            "fp8_encode": (C.c_uint8, [C.c_double]),
            "fp8_decode": (C.c_float, [C.c_uint8]),
            "quantize_value": (C.c_uint8, [C.c_double, i32]),
            "pack_codes": (None, [vp, i64, vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(self.lib, prefix + name)
            fn.restype = res
            fn.argtypes = args
            setattr(self, "_" + name, fn)
        if prefix == "ref_":  # container.hpp serialization (the reference only)
            self.lib.ref_serialize_compressed_i8.restype = i64
            self.lib.ref_serialize_compressed_i8.argtypes = [vp, vp, i64, i64, i32, i32, vp, i64]
            self.lib.ref_serialize_quantized.restype = i64
            self.lib.ref_serialize_quantized.argtypes = [vp, vp, i64, i64, i32, i32, i32, vp, i64]
        if prefix == "orc_":
            for name in ("orc_dequant_bf16", "orc_dequant_f32_bf16"):
                fn = getattr(self.lib, name)
                fn.restype = None
                fn.argtypes = [vp, i64, i64, vp, vp, vp]

    # ---- geometry -------------------------------------------------------
    def plan(self, z, l, hw_m=2, hw_n=4):
        wc = C.c_int(0)
        starts = (C.c_int * 64)()
        st = self._plan(z, l, hw_m, hw_n, C.byref(wc), starts, 64)
        if st:
            raise OracleError(st)
        return wc.value, list(starts[: wc.value])

    # ---- packer ---------------------------------------------------------
    def pack_matrix(self, w: np.ndarray, z: int, l: int, dtype: int, threads: int = 0):
        rows, cols = w.shape
        wc, _ = self.plan(z, l)
        out = np.zeros((rows, cols // l * wc * 4), dtype=w.dtype)
        er, eb = C.c_int64(-1), C.c_int64(-1)
        w = np.ascontiguousarray(w)
        st = self._pack_matrix(dtype, _p(w), rows, cols, z, l, _p(out), C.byref(er), C.byref(eb), threads)
        if st:
            raise OracleError(st, (er.value, eb.value))
        return out

    def compress(self, slided: np.ndarray, dtype: int):
        rows, cexp = slided.shape
        values = np.zeros((rows, cexp // 2), dtype=slided.dtype)
        codes = np.zeros((rows, cexp // 2), dtype=np.uint8)
        er, ew = C.c_int64(-1), C.c_int64(-1)
        slided = np.ascontiguousarray(slided)
        st = self._compress(dtype, _p(slided), rows, cexp, _p(values), _p(codes), C.byref(er), C.byref(ew))
        if st:
            raise OracleError(st, (er.value, ew.value))
        return values, codes

    def magnitude_prune(self, w: np.ndarray, z: int, l: int, dtype: int):
        out = np.empty_like(w)
        w = np.ascontiguousarray(w)
        st = self._magnitude_prune(dtype, _p(w), w.shape[0], w.shape[1], z, l, _p(out))
        if st:
            raise OracleError(st)
        return out

    # ---- activations ----------------------------------------------------
    def fused_quant_slide(self, x: np.ndarray, z: int, l: int, kind: int, in_dtype: int, threads: int = 0):
        rows, cols = x.shape
        wc, _ = self.plan(z, l)
        words = (cols + l - 1) // l * wc
        payload = np.zeros((rows, words), dtype=np.uint32)
        scales = np.ones(rows, dtype=np.float32)
        bad = C.c_int64(-1)
        x = np.ascontiguousarray(x)
        st = self._fused_quant_slide(in_dtype, _p(x), rows, cols, z, l, kind, _p(payload), _p(scales),
                                     C.byref(bad), threads)
        if st:
            raise OracleError(st, bad.value)
        return payload, scales

    def quantize_rows(self, x: np.ndarray, kind: int, in_dtype: int):
        rows, cols = x.shape
        out = np.zeros((rows, cols), dtype=np.uint8)
        scales = np.ones(rows, dtype=np.float32)
        bad = C.c_int64(-1)
        x = np.ascontiguousarray(x)
        st = self._quantize_rows(in_dtype, _p(x), rows, cols, kind, _p(out), _p(scales), C.byref(bad))
        if st:
            raise OracleError(st, bad.value)
        return out, scales

    def lift_rows(self, x: np.ndarray, z: int, l: int, dtype: int):
        rows, cols = x.shape
        wc, _ = self.plan(z, l)
        out = np.zeros((rows, cols // l * wc * 4), dtype=x.dtype)
        x = np.ascontiguousarray(x)
        st = self._lift_rows(dtype, _p(x), rows, cols, z, l, _p(out))
        if st:
            raise OracleError(st)
        return out

    # ---- GEMMs ------------------------------------------------------------
    def sparse_gemm_words(self, values, codes, payload, threads: int = 0):
        rows = values.shape[0]
        wpr = values.shape[1] // 2
        tokens = payload.shape[0]
        y = np.zeros((rows, tokens), dtype=np.int32)
        values, codes, payload = (np.ascontiguousarray(a) for a in (values, codes, payload))
        st = self._sparse_gemm_words(_p(values), _p(codes), rows, wpr, _p(payload), tokens, _p(y), threads)
        if st:
            raise OracleError(st)
        return y

    def sparse_gemm_f64(self, values, codes, lifted, threads: int = 0):
        rows = values.shape[0]
        wpr = values.shape[1] // 2
        tokens = lifted.shape[0]
        y = np.zeros((rows, tokens), dtype=np.float64)
        values = np.ascontiguousarray(values, dtype=np.float64)
        lifted = np.ascontiguousarray(lifted, dtype=np.float64)
        codes = np.ascontiguousarray(codes)
        st = self._sparse_gemm_f64(_p(values), _p(codes), rows, wpr, _p(lifted), tokens, _p(y), threads)
        if st:
            raise OracleError(st)
        return y

    def dense_gemm_i8(self, w: np.ndarray, x_km: np.ndarray, threads: int = 0):
        n, k = w.shape
        m = x_km.shape[1]
        y = np.zeros((n, m), dtype=np.int32)
        w, x_km = np.ascontiguousarray(w), np.ascontiguousarray(x_km)
        st = self._dense_gemm_i8(_p(w), n, k, _p(x_km), m, _p(y), threads)
        if st:
            raise OracleError(st)
        return y

    # ---- scalars / formats ------------------------------------------------
    def fp8_encode(self, x: float) -> int:
        return int(self._fp8_encode(float(x)))

    def fp8_decode(self, code: int) -> float:
        return float(self._fp8_decode(int(code)))

    def quantize_value(self, scaled: float, kind: int) -> int:
        return int(self._quantize_value(float(scaled), kind))

    def pack_codes(self, codes: np.ndarray) -> np.ndarray:
        codes = np.ascontiguousarray(codes.reshape(-1), dtype=np.uint8)
        out = np.zeros((codes.size + 3) // 4, dtype=np.uint8)
        self._pack_codes(_p(codes), codes.size, _p(out))
        return out

    # ---- reference-only: container.hpp serialize(to_container(...)) ---------
    def serialize_compressed_i8(self, values: np.ndarray, codes: np.ndarray, z: int, l: int) -> bytes:
        rows, wx2 = values.shape
        values = np.ascontiguousarray(values, dtype=np.int8)
        codes = np.ascontiguousarray(codes, dtype=np.uint8)
        out = np.zeros(64 + values.nbytes + codes.size, dtype=np.uint8)
        n = self.lib.ref_serialize_compressed_i8(_p(values), _p(codes), rows, wx2 // 2, z, l, _p(out), out.size)
        assert n > 0
        return out[:n].tobytes()

    def serialize_quantized(self, payload: np.ndarray, scales: np.ndarray, z: int, l: int, kind: int) -> bytes:
        rows, words = payload.shape
        payload = np.ascontiguousarray(payload, dtype=np.uint32)
        scales = np.ascontiguousarray(scales, dtype=np.float32)
        out = np.zeros(64 + payload.nbytes + scales.nbytes, dtype=np.uint8)
        n = self.lib.ref_serialize_quantized(_p(payload), _p(scales), rows, words, z, l, kind, _p(out), out.size)
        assert n > 0
        return out[:n].tobytes()

    # ---- restatement-only: a18 dequant epilogue -----------------------------
    def dequant_bf16(self, acc: np.ndarray, s_ch: np.ndarray, s_tok: np.ndarray) -> np.ndarray:
        n, m = acc.shape
        y = np.zeros((n, m), dtype=np.uint16)
        acc = np.ascontiguousarray(acc)
        s_ch = np.ascontiguousarray(s_ch, dtype=np.float32)
        s_tok = np.ascontiguousarray(s_tok, dtype=np.float32)
        fn = self.lib.orc_dequant_bf16 if acc.dtype == np.int32 else self.lib.orc_dequant_f32_bf16
        if acc.dtype not in (np.int32, np.float32):
            raise TypeError(acc.dtype)
        fn(_p(acc), n, m, _p(s_ch), _p(s_tok), _p(y))
        return y


def build_oracle() -> None:
    """Compiles the restatement (and the reference bridge when /root/reference exists)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle")], check=True)
    if Path(os.environ.get("SLSP_REF_INC", "/root/reference/proj/include")).is_dir():
        subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "ref"], check=True)


_cache: dict = {}


def orc() -> Oracle:
    if "orc" not in _cache:
        if not ORC_PATH.exists():
            build_oracle()
        _cache["orc"] = Oracle(ORC_PATH, "orc_")
    return _cache["orc"]


def ref() -> Oracle | None:
    """The reference compiled from its own headers, or None if not built here."""
    if "ref" not in _cache:
        _cache["ref"] = Oracle(REF_PATH, "ref_") if REF_PATH.exists() else None
    return _cache["ref"]


# ---- helpers shared by tests (numpy-side restatements of trivial maps) ------
def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16_bits(f: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bf16 bit pattern."""
    u = np.ascontiguousarray(f, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = u + 0x7FFF + ((u >> 16) & 1)
    return (u >> 16).astype(np.uint16)


def compliant_matrix(rng: np.random.Generator, rows: int, groups: int, z: int, l: int,
                     exact_z: bool = False) -> np.ndarray:
    """int8 rows with a random number (<= z) of nonzeros per block at random
    positions, values in [-127,127]\\{0} (proj/tests/test_util.hpp:14-60)."""
    nnz = np.full((rows, groups, 1), z) if exact_z else rng.integers(0, z + 1, size=(rows, groups, 1))
    rank = np.argsort(rng.random((rows, groups, l)), axis=-1).argsort(axis=-1)
    v = rng.integers(-127, 127, size=(rows, groups, l))
    v = np.where(v >= 0, v + 1, v)
    return np.where(rank < nnz, v, 0).astype(np.int8).reshape(rows, groups * l)
