/*
 * slsp_b200.h — C ABI of the B200-native SlideSparse hot path.
 *
 * This is the drop-in boundary: plain pointers, sizes and a
 * cudaStream_t, no C++ or torch types. Every entry point replaces one
 * function of the reference's header-only C++ library (namespace slsp in
 * /root/reference/proj/include/slsp/); the citation is given per function.
 * The C++ drop-in headers in include/slsp/ are implemented on top of this
 * ABI, and INTEGRATION.md shows the ctypes / C++ bindings.
 *
 * Conventions
 *  - All data pointers are DEVICE pointers on the current device, except
 *    where a parameter says "host". Buffers are caller-allocated; the library
 *    keeps no pointer past the call (reference value semantics).
 *  - Calls are stream-ordered on `stream`. Entry points that report data
 *    errors (non-compliant weights, non-finite activations) take a device
 *    scratch `status_ws` of SLSP_STATUS_WS_BYTES bytes; when it is non-NULL
 *    the call synchronises `stream` and returns the error with its location,
 *    mirroring the reference's exceptions. When NULL the check is skipped
 *    (the hot path) and the call is fully asynchronous.
 *  - Row-major everywhere. "Lifted width" kp is the padded width of the
 *    lifted/slided K dimension: kp >= K' = ceil(K/l)*(l-2)/2*4, kp % 8 == 0
 *    for the MMA-ready formats, kp % 256 == 0 for the GEMM entry points.
 *    Padding windows hold zero values and the canonical codes (0,1).
 *  - The library fails loudly: a missing device, wrong architecture or a
 *    CUDA error is returned as SLSP_ERR_CUDA; there is no CPU fallback.
 */
#ifndef SLSP_B200_H
#define SLSP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define SLSP_API __attribute__((visibility("default")))
#else
#define SLSP_API
#endif

typedef struct CUstream_st* slsp_stream_t; /* == cudaStream_t */

/* Element types (weights / activations). */
enum {
  SLSP_DT_I8 = 0,   /* int8 two's complement                          */
  SLSP_DT_BF16 = 1, /* bfloat16 bit patterns                          */
  SLSP_DT_E4M3 = 2, /* fp8 e4m3fn codes (fp8.hpp)                     */
  SLSP_DT_F32 = 3,
  SLSP_DT_F64 = 4,
  SLSP_DT_I32 = 5   /* int32 (the reference's generic Matrix<int>)        */
};

/* Activation quantization kinds (quantize.hpp:16 QuantKind). */
enum { SLSP_QUANT_INT8 = 0, SLSP_QUANT_FP8E4M3 = 1 };

/* GEMM output modes. */
enum {
  SLSP_OUT_RAW_NM = 0,   /* accumulators, N x M (int32 for I8, fp32 otherwise) — gemm.hpp:214 */
  SLSP_OUT_BF16_NM = 1,  /* bf16((acc*s_ch[n])*s_tok[t]), N x M                                */
  SLSP_OUT_BF16_MN = 2   /* same values, M x N (token-major, what the next layer consumes)     */
};

/* Status codes; the C++ shim maps each to the reference's exception type. */
enum {
  SLSP_OK = 0,
  SLSP_ERR_NOT_COMPLIANT = 1, /* slsp::NotCompliantError       (pattern.hpp:40) */
  SLSP_ERR_DIMENSION = 2,     /* slsp::DimensionMismatchError  (pattern.hpp:43) */
  SLSP_ERR_PLAN = 3,          /* AlreadyCompliant / NonIntegralWindowCount / InsufficientCapacity */
  SLSP_ERR_NON_FINITE = 4,    /* slsp::NonFiniteInputError     (pattern.hpp:49) */
  SLSP_ERR_INVALID = 5,       /* std::invalid_argument / std::overflow_error    */
  SLSP_ERR_MALFORMED = 6,     /* slsp::MalformedMetadataError  (pattern.hpp:46) */
  SLSP_ERR_UNSUPPORTED = 7,   /* shape/type outside what the sm_100a kernels handle */
  SLSP_ERR_CUDA = 8           /* CUDA runtime/driver failure, no device, wrong arch */
};

#define SLSP_STATUS_WS_BYTES 64

/* Version / diagnostics. */
SLSP_API int slsp_version(void);
SLSP_API const char* slsp_status_string(int status);
/* Last CUDA error text seen by this thread (for SLSP_ERR_CUDA). */
SLSP_API const char* slsp_last_cuda_error(void);
/* 1 if device `dev` is an sm_100 part the kernels run on, else 0. */
SLSP_API int slsp_device_supported(int dev);
/* Re-reads the SLSP_* tuning/probing environment variables (snapshotted once
 * per process otherwise; probes and tests that change them call this). */
SLSP_API void slsp_reload_knobs(void);

/* a1 — pattern.hpp:107-154 plan_status + plan_decomposition (host only).
 * Hardware window fixed at hw_m:hw_n. Fills window_count and up to `cap`
 * window starts. */
SLSP_API int slsp_plan_decomposition(int z, int l, int hw_m, int hw_n, int* window_count, int* window_starts,
                            int cap);

/* a3/a4 — pack.hpp:171-204 pack_matrix. W (rows x cols, dtype) -> slided
 * (rows x K', same dtype), K' = cols/l*wc*4. cols % l != 0 -> DIMENSION.
 * Errors: NOT_COMPLIANT with (*err_row, *err_block) of the lowest row. */
SLSP_API int slsp_pack_matrix(int dtype, const void* w, int64_t rows, int64_t cols, int z, int l, void* slided,
                     void* status_ws, int64_t* err_row, int64_t* err_block, slsp_stream_t stream);

/* a5 — gemm.hpp:70-110 compress. slided (rows x cols_exp) -> values
 * (rows x cols_exp/2, dtype) + codes (rows x cols_exp/2 bytes, one 2-bit
 * position per byte, the reference's in-memory format). */
SLSP_API int slsp_compress(int dtype, const void* slided, int64_t rows, int64_t cols_exp, void* values, uint8_t* codes,
                  void* status_ws, int64_t* err_row, int64_t* err_window, slsp_stream_t stream);

/* a3+a4+a5 fused, the offline packer Φ in MMA-ready form:
 *   values: rows x kp/2 (dtype), meta: rows x kp/8 bytes, four 2-bit codes per
 *   byte LSB-first (== container.hpp:330-336 pack_codes per row == the 2:4
 *   sparse-MMA metadata nibbles). cols need not be a multiple of l: the tail
 *   block is zero-padded like quantize.hpp:130,162 does for activations. */
SLSP_API int slsp_pack_compress(int dtype, const void* w, int64_t rows, int64_t cols, int z, int l, int64_t kp,
                       void* values, uint8_t* meta, void* status_ws, int64_t* err_row, int64_t* err_block,
                       slsp_stream_t stream);

/* MMA-tiled metadata (the operand format of slsp_sparse_gemm): re-tiles the
 * row-major codes (rows x kp/8 bytes, as written by slsp_pack_compress) into
 * contiguous 4 KB blocks, one per (128-row block b, 256-wide k-stage s):
 *   tiled[((b*(kp/256) + s)*2 + c)*2048 + r*16 + j] = meta[(b*128 + r)*(kp/8) + s*32 + c*16 + j]
 * i.e. two 128x16-byte tcgen05.cp atoms per stage. Rows past `rows` up to the
 * next multiple of 128 are filled with canonical codes (0,1) = 0x44. `tiled`
 * holds ceil(rows/128)*128 * kp/8 bytes. kp % 256 == 0. */
SLSP_API int slsp_tile_meta(const uint8_t* meta, int64_t rows, int64_t kp, uint8_t* tiled, slsp_stream_t stream);

/* slsp_tile_meta for the operand type `dtype` of the sparse GEMM: I8/E4M3
 * use the row-major atom above; BF16 (kind::f16) uses the 16-bit atom, the
 * same bytes with byte-offset bits 1 and 7 of each 2 KB atom exchanged. */
SLSP_API int slsp_tile_meta_ex(const uint8_t* meta, int64_t rows, int64_t kp, int dtype, uint8_t* tiled,
                      slsp_stream_t stream);

/* Bytes of the tiled metadata buffer for `rows` x `kp`. */
SLSP_API int64_t slsp_tiled_meta_bytes(int64_t rows, int64_t kp);

/* a8 — pack.hpp:238-261 magnitude_prune (synthesises compliant weights). */
SLSP_API int slsp_magnitude_prune(int dtype, const void* w, int64_t rows, int64_t cols, int z, int l, void* out,
                         slsp_stream_t stream);

/* a12 — quantize.hpp:122-174 fused_quant_slide. x (rows x cols, F32|BF16)
 * -> payload (rows x kp/4 uint32 words; word j = window j, byte d = position
 * d, pack_word :91-94) + scales (rows, fp32). kp >= K' and kp % 4 == 0;
 * kp == K' reproduces QuantizedLiftedActivation::payload exactly. */
SLSP_API int slsp_fused_quant_slide(int in_dtype, const void* x, int64_t rows, int64_t cols, int z, int l, int kind,
                           int64_t kp, uint32_t* payload, float* scales, void* status_ws, int64_t* bad_row,
                           slsp_stream_t stream);

/* a8 — quantize.hpp:52-68 quantize_row for every token row (the dense
 * GEMM's activations): out rows x kpad bytes (zero padded), scales fp32. */
SLSP_API int slsp_quantize_rows(int in_dtype, const void* x, int64_t rows, int64_t cols, int kind, int64_t kpad,
                       uint8_t* out, float* scales, void* status_ws, int64_t* bad_row, slsp_stream_t stream);

/* a9 — quantize.hpp:72-89 lift_row per token row (gemm.hpp:240-256
 * lift_activations with tokens as rows). Pure gather, any dtype; cols % l == 0;
 * out rows x kp (zero padded past K'). */
SLSP_API int slsp_lift_rows(int dtype, const void* x, int64_t rows, int64_t cols, int z, int l, int64_t kp, void* out,
                   slsp_stream_t stream);

/* a13/a14 — gemm.hpp:164-233 sparse_gemm on tcgen05.mma.sp (sm_100a).
 *   dtype I8  : values int8,  act = quantized payload bytes (int8), acc int32
 *   dtype E4M3: values e4m3,  act = e4m3 payload bytes,              acc fp32
 *   dtype BF16: values bf16,  act = lifted bf16,                     acc fp32
 * values: n x kp/2 (slsp_pack_compress), meta: the slsp_tile_meta layout
 * (slsp_tiled_meta_bytes(n, kp) bytes), act: m x kp.
 * kp % 256 == 0. s_ch (n) / s_tok (m) are required for the BF16 outputs.
 * out: SLSP_OUT_RAW_NM / BF16_NM -> n x m (row stride ldo elements);
 *      SLSP_OUT_BF16_MN -> m x n (row stride ldo). */
SLSP_API int slsp_sparse_gemm(int dtype, const void* values, const uint8_t* meta, int64_t n, int64_t kp, const void* act,
                     int64_t m, const float* s_ch, const float* s_tok, int out_mode, void* out, int64_t ldo,
                     slsp_stream_t stream);

/* §8f #3 — the next layer's lift fused upstream. slsp_sparse_gemm with BF16
 * outputs that also writes tok_amax[t] = max over this call's n output
 * features of |y[t][.]| (the BF16-rounded outputs; zeroed first, then
 * max-accumulated with atomics; NaN wins over Inf). Feeding y and tok_amax
 * to slsp_fused_quant_slide_scaled gives exactly slsp_fused_quant_slide(y)
 * (quantize.hpp:122-174) without its |x|max pass. No split-K. */
SLSP_API int slsp_sparse_gemm_amax(int dtype, const void* values, const uint8_t* meta, int64_t n, int64_t kp,
                                   const void* act, int64_t m, const float* s_ch, const float* s_tok, int out_mode,
                                   void* out, int64_t ldo, float* tok_amax, slsp_stream_t stream);

/* fused_quant_slide (quantize.hpp:122-174) given each row's |x|max
 * (tok_amax, e.g. from slsp_sparse_gemm_amax): r = qmax/absmax, scale =
 * float(absmax/qmax) in double exactly as the reference; a non-finite
 * tok_amax[row] reports SLSP_ERR_NON_FINITE for that row like the
 * unscaled entry. Same layouts and requirements as slsp_fused_quant_slide. */
SLSP_API int slsp_fused_quant_slide_scaled(int in_dtype, const void* x, int64_t rows, int64_t cols, int z, int l,
                                           int kind, int64_t kp, const float* tok_amax, uint32_t* payload,
                                           float* scales, void* status_ws, int64_t* bad_row, slsp_stream_t stream);

/* Sharded lift. The input X of an N-sharded layer
 * arrives K-sharded (rank r holds columns [k0, k0+cols) — the previous
 * layer's output features it computed). Each rank:
 *   slsp_row_absmax          its slice's per-row |x|max (or the tok_amax of
 *                            slsp_sparse_gemm_amax when it produced the slice),
 *   all-reduce(MAX) over ranks (M floats; exact),
 *   slsp_fused_quant_slide_scaled_multi
 *                            quantizes + lifts its slice with the global
 *                            |x|max and writes the lifted bytes — byte column
 *                            dst_col = k0*K'/K of the full payload row (row
 *                            stride dst_ld = kp) — into EVERY rank's payload
 *                            (dsts: this rank's buffer first, then the peers',
 *                            opened with slsp_ipc_open_handle), so no
 *                            all-gather follows; a stream-ordered barrier
 *                            before the GEMM reads the assembled payload.
 * The assembled payload and scales equal slsp_fused_quant_slide on the full
 * X byte for byte. cols % (4*l) == 0; padding past K' (kp > K') is the
 * caller's (zero it once). */
SLSP_API int slsp_row_absmax(int in_dtype, const void* x, int64_t rows, int64_t cols, float* amax,
                             slsp_stream_t stream);
SLSP_API int slsp_fused_quant_slide_scaled_multi(int in_dtype, const void* x, int64_t rows, int64_t cols, int z, int l,
                                                 int kind, const float* tok_amax, void* const* dsts, int ndst,
                                                 int64_t dst_ld, int64_t dst_col, float* scales, void* status_ws,
                                                 int64_t* bad_row, slsp_stream_t stream);
SLSP_API int slsp_ipc_get_handle(const void* ptr, void* handle_out, int64_t* offset_out);
SLSP_API int slsp_ipc_open_handle(const void* handle, void** ptr_out);
SLSP_API int slsp_ipc_close(void* ptr);

/* SLSP kind-2 container payload -> MMA-ready weights (
 * container.hpp:379-390 to_container / :424-435 compressed_from). values:
 * the container's values section on the device (rows x windows x 2 elements);
 * codes_stream: its metadata section (2-bit codes, four per byte LSB-first,
 * container.hpp:330-336, contiguous over the whole matrix). Writes values_out
 * (rows x kp/2) and meta_out (rows x kp/8, the slsp_pack_compress layout; tile
 * it with slsp_tile_meta_ex), padding windows = value 0 / codes (0,1).
 * kp >= 4*windows, kp % 8 == 0 (the GEMM needs kp % 256 == 0). The host side
 * (file I/O, header, CRC-32, the reference's ContainerError checks) is
 * paper_2603_05232_b200/container.py. */
SLSP_API int slsp_load_compressed(int dtype, const void* values, const uint8_t* codes_stream, int64_t rows,
                         int64_t windows, int64_t kp, void* values_out, uint8_t* meta_out, slsp_stream_t stream);

/* GEMM window order for in-SM lifting (6:8). Permutes the windows of
 * slsp_pack_compress output (values rows x kp_ref/2, row-major codes
 * rows x kp_ref/8; K' = 3*ceil(cols/8)*4 real lifted positions) into the
 * order slsp_sparse_gemm_x consumes: per period of 64 source blocks (512
 * source bytes), the 128 windows (block b: window 0, window 2) for b = 0..63,
 * then the 64 windows 1. Output width kp_out = 3/2 * round_up(cols, 512);
 * blocks past the real ones are padding windows (values 0, codes (0,1)).
 * values_out: rows x kp_out/2, codes_out: rows x kp_out/8 (row-major, to be
 * tiled with slsp_tile_meta(codes_out, rows, kp_out, ...)). The sum over the
 * lifted dimension is order-independent, so slsp_sparse_gemm_x reproduces
 * slsp_sparse_gemm (== gemm.hpp:199-233) bit for bit. */
SLSP_API int slsp_gemm_order(int dtype, const void* values, const uint8_t* codes, int64_t rows, int64_t cols, int64_t kp_ref,
                    void* values_out, uint8_t* codes_out, int64_t kp_out, slsp_stream_t stream);

/* Sparse GEMM with in-SM activation lifting (6:8). act is the UNLIFTED
 * quantized activation (slsp_quantize_rows output, m x kx bytes, kx =
 * round_up(cols, 512), zero padded); values/meta from slsp_gemm_order +
 * slsp_tile_meta with kp = 3*kx/2. The window-duplicating rearrangement of
 * fused_quant_slide (quantize.hpp:122-174) happens in shared memory inside
 * the GEMM. Results equal slsp_sparse_gemm on fused_quant_slide's payload
 * bit for bit (int32) / to the same fp32 epilogue (BF16). */
SLSP_API int slsp_sparse_gemm_x(int dtype, const void* values, const uint8_t* meta, int64_t n, int64_t kx, const void* act,
                       int64_t m, const float* s_ch, const float* s_tok, int out_mode, void* out, int64_t ldo,
                       slsp_stream_t stream);

/* Workspace budget of the *_ws GEMM variants for m <= 1024: 8 slices of
 * n*m*4 bytes, capped at 64 MiB (whole slices; 0 if that holds < 2 slices);
 * 0 for m > 1024. slsp_*_gemm_config reports what a call actually needs.
 * With it, GEMMs whose tiles do not fill the 148 SMs
 * split K across CTAs (up to ws_bytes / (n*m*4) slices, <= 16): each slice
 * stores its raw int32/fp32 partial sums, a finishing kernel sums the slices
 * in slice order (exact for INT8, so results stay bit-identical;
 * deterministic for FP8/BF16) and applies the same epilogue. Stream-ordered;
 * the workspace must not be shared by concurrent calls. */
SLSP_API int64_t slsp_gemm_workspace_bytes(int64_t n, int64_t m);
SLSP_API int slsp_sparse_gemm_ws(int dtype, const void* values, const uint8_t* meta, int64_t n, int64_t kp, const void* act,
                        int64_t m, const float* s_ch, const float* s_tok, int out_mode, void* out, int64_t ldo,
                        void* workspace, int64_t ws_bytes, slsp_stream_t stream);
SLSP_API int slsp_dense_gemm_ws(int dtype, const void* w, int64_t n, int64_t k, const void* act, int64_t m,
                       const float* s_ch, const float* s_tok, int out_mode, void* out, int64_t ldo, void* workspace,
                       int64_t ws_bytes, slsp_stream_t stream);

/* The tile configuration a GEMM call with these arguments launches (nothing
 * is launched; no device memory is touched). ws_bytes is the workspace the
 * caller would pass to the *_ws variant (0: none). workspace_bytes is what
 * the chosen split-K actually uses (0 when unsplit), so callers can size
 * the workspace exactly: query with slsp_gemm_workspace_bytes(n, m), then
 * allocate cfg.workspace_bytes. */
typedef struct slsp_gemm_config {
  int tokens_per_tile;      /* MMA N across the CTA pair (tokens of one tile) */
  int weight_rows_per_tile; /* 256 x subtiles */
  int subtiles;             /* M=256 UMMA subtiles per tile (1 or 2) */
  int half_k_stages;        /* 1: 128 lifted bytes per ring stage */
  int stages;               /* shared-memory ring depth */
  int cluster_ctas;         /* CTAs per cluster */
  int ksplit;               /* split-K slices (1: none) */
  int epilogue;             /* 0: chunked TMEM drain, 1: register-staged two-subtile drain */
  int clusters;             /* persistent clusters launched */
  int cluster_ksplit;       /* k-slices reduced inside a cluster through DSMEM (1: none); included in ksplit */
  int64_t workspace_bytes;  /* workspace the split needs (0 when ksplit == 1) */
} slsp_gemm_config;
SLSP_API int slsp_sparse_gemm_config(int dtype, int64_t n, int64_t kp, int64_t m, int out_mode, int64_t ws_bytes,
                                     slsp_gemm_config* cfg);
SLSP_API int slsp_dense_gemm_config(int dtype, int64_t n, int64_t k, int64_t m, int out_mode, int64_t ws_bytes,
                                    slsp_gemm_config* cfg);

/* BF16 sparse GEMM with the activation lift inside the kernel (decode-shaped
 * M). x is the UNLIFTED BF16 activation (m x cols, row
 * stride x_ld elements, even; x 4-byte aligned; cols % l == 0); values/meta
 * as for slsp_sparse_gemm (slsp_pack_compress + slsp_tile_meta, kp lifted
 * columns). Lift warps in the GEMM read each window's four source elements
 * (quantize.hpp:72-89 lift_row) from x and write them straight into the
 * shared-memory B stage, so no lifted copy of x is ever written. Equals
 * slsp_sparse_gemm(values, meta, slsp_lift_rows(x, z, l, kp)) bit for bit.
 * Replaces the lift_row + gemm.hpp:199-233 pair of the reference's BF16 path.
 * workspace: split-K slices as for slsp_sparse_gemm_ws (NULL: no split). */
SLSP_API int slsp_sparse_gemm_lift(int dtype, const void* values, const uint8_t* meta, int64_t n, int64_t kp,
                                   const void* x, int64_t x_ld, int64_t m, int64_t cols, int z, int l,
                                   const float* s_ch, const float* s_tok, int out_mode, void* out, int64_t ldo,
                                   void* workspace, int64_t ws_bytes, slsp_stream_t stream);
SLSP_API int slsp_sparse_gemm_lift_config(int dtype, int64_t n, int64_t kp, int64_t m, int64_t cols, int z, int l,
                                          int out_mode, int64_t ws_bytes, slsp_gemm_config* out);

/* gemm.hpp:142-197 generic instantiations (T = int32 -> int64 accumulators,
 * T = float -> double) on the CUDA cores, for the drop-in's Matrix<int> /
 * Matrix<float> calls: one thread per output element sums in the reference's
 * left-to-right order with exact products, so results are bit-identical to
 * the reference at any size. Not the hot path (that is tcgen05, above).
 *   dense : w n x k, x k x m (one token per column), y n x m (int64|double)
 *   sparse: values rows x windows x hw_m, codes same shape (one position
 *           code per byte, gemm.hpp:49-58), lifted m x windows*hw_n (one token
 *           per row), y rows x m; a code >= hw_n reports SLSP_ERR_MALFORMED. */
SLSP_API int slsp_generic_dense_gemm(int dtype, const void* w, int64_t n, int64_t k, const void* x, int64_t m, void* y,
                                     slsp_stream_t stream);
SLSP_API int slsp_generic_sparse_gemm(int dtype, const void* values, const uint8_t* codes, int64_t rows,
                                      int64_t windows, int hw_m, int hw_n, const void* lifted, int64_t m, void* y,
                                      void* status_ws, int64_t* bad_row, slsp_stream_t stream);

/* a15 — gemm.hpp:142-162 dense_gemm on tcgen05.mma (the speedup
 * denominator). w: n x k, act: m x k (token rows; the reference's X is k x m,
 * the C++ shim transposes), k % 128 == 0. Outputs as slsp_sparse_gemm. */
SLSP_API int slsp_dense_gemm(int dtype, const void* w, int64_t n, int64_t k, const void* act, int64_t m,
                    const float* s_ch, const float* s_tok, int out_mode, void* out, int64_t ldo,
                    slsp_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* SLSP_B200_H */
