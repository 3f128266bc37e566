"""C-ABI boundary checks that run without a GPU: the native library loads,
exports every symbol include/slsp_b200.h declares, host-only geometry matches
the reference plan, and argument validation rejects bad shapes before any
device work. No kernels are launched here."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "slsp_b200.h"


def declared_symbols():
    return re.findall(r"SLSP_API\s+[\w\s\*]+?\b(slsp_\w+)\s*\(", HEADER.read_text())


@pytest.fixture(scope="module")
def native():
    from paper_2603_05232_b200 import build as b

    b.build()
    from paper_2603_05232_b200 import _native

    return _native.lib()


def test_header_declares_the_path():
    syms = set(declared_symbols())
    for s in ("slsp_pack_matrix", "slsp_compress", "slsp_pack_compress", "slsp_fused_quant_slide",
              "slsp_quantize_rows", "slsp_lift_rows", "slsp_sparse_gemm", "slsp_dense_gemm",
              "slsp_plan_decomposition", "slsp_magnitude_prune"):
        assert s in syms


def test_library_exports_every_declared_symbol(native):
    from paper_2603_05232_b200._native import LIB_PATH

    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (slsp_\w+)", out))
    missing = set(declared_symbols()) - exported
    assert not missing, missing
    for s in declared_symbols():
        assert getattr(native, s) is not None


def test_library_is_sm100a_only(native):
    from paper_2603_05232_b200._native import LIB_PATH

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(LIB_PATH)], capture_output=True,
                         text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_plan_matches_reference_geometry(native, orc):
    from paper_2603_05232_b200 import plan_decomposition

    for z, l in [(4, 6), (6, 8), (8, 10), (14, 16)]:
        assert plan_decomposition(z, l) == orc.plan(z, l)
    assert native.slsp_plan_decomposition(1, 4, 2, 4, None, None, 0) == 3  # already compliant
    assert native.slsp_plan_decomposition(6, 7, 2, 4, None, None, 0) == 3  # non-integral
    assert native.slsp_plan_decomposition(0, 4, 2, 4, None, None, 0) == 5  # invalid pattern


def test_status_strings(native):
    assert native.slsp_status_string(0) == b"ok"
    assert native.slsp_status_string(1) == b"not compliant"
    assert native.slsp_version() >= 100


def test_host_side_validation_before_device(native):
    i64 = C.c_int64
    # pack_matrix: cols % l != 0 -> DIMENSION (pack.hpp:174-177), decided on the host
    assert native.slsp_pack_matrix(0, None, 4, 9, 6, 8, None, None, None, None, None) == 2
    # compress: width not a multiple of 4 -> DIMENSION (gemm.hpp:78-80)
    assert native.slsp_compress(0, None, 1, 6, None, None, C.c_void_p(1), None, None, None) == 2
    # sparse GEMM: kp not a multiple of the 256-wide k-block -> DIMENSION
    assert native.slsp_sparse_gemm(0, None, None, 256, 200, None, 224, None, None, 0, C.c_void_p(1), 224,
                                   None) == 2
    # dense GEMM: bad element type -> UNSUPPORTED
    assert native.slsp_dense_gemm(4, None, 256, 128, None, 256, None, None, 0, C.c_void_p(1), 256, None) == 7
    # fused_quant_slide: kp narrower than K' -> DIMENSION
    assert native.slsp_fused_quant_slide(3, None, 4, 16, 6, 8, 0, i64(16), None, None, None, None, None) == 2


def test_no_device_fails_loudly(native):
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    assert native.slsp_device_supported(0) == 0


def test_cpp_dropin_headers_compile():
    """include/slsp/*.hpp (the C++ drop-in) compile against the C ABI header."""
    import subprocess

    r = subprocess.run(["make", "-s", "-C", str(ROOT / "tests" / "cpp")], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
