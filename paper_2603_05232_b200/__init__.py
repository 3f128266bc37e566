"""B200-native SlideSparse hot path (pack -> lift -> 2:4-sparse GEMM on sm_100a).

The product is the native library ``libslsp_b200.so`` behind the C ABI in
``include/slsp_b200.h``; this package is its Python host binding (ctypes over
torch CUDA tensors) plus the build recipe. See DESIGN.md.
"""
from ._native import (  # noqa: F401
    DT_BF16, DT_E4M3, DT_F32, DT_F64, DT_I8, OUT_BF16_MN, OUT_BF16_NM, OUT_RAW_NM, QUANT_FP8E4M3, QUANT_INT8,
    CudaError, DimensionMismatchError, GemmOrderWeights, MalformedMetadataError, NonFiniteInputError, NotCompliantError,
    PackedWeights, PlanError, SlspError, UnsupportedError, compress, dense_gemm, dense_gemm_config, device_supported,
    fused_quant_slide, fused_quant_slide_multi, gemm_order, ipc_close, ipc_handle, ipc_open, knobs, lib, lift_rows,
    lifted_width, magnitude_prune, pack_compress, pack_matrix, plan_decomposition, quantize_rows, reload_knobs,
    round_up, row_absmax, sparse_gemm, sparse_gemm_config, sparse_gemm_lift, sparse_gemm_x, tile_meta,
)

from . import container  # noqa: F401,E402
from .verify import EquivalenceReport, check_equivalence  # noqa: F401,E402

__version__ = "0.2.0"
