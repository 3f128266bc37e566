/*
 * CPU oracle interface — TEST INFRASTRUCTURE ONLY.
 *
 * Two libraries implement this interface:
 *   oracle/_build/libslsp_oracle.so  prefix orc_  plain-C restatement of the
 *                                    reference algorithm (oracle/slsp_oracle.c)
 *   oracle/_ref/libslsp_ref.so       prefix ref_  the reference headers under
 *                                    /root/reference/proj/include compiled
 *                                    unmodified (oracle/ref_bridge.cpp)
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load either library. The product
 * (paper_2603_05232_b200/) never links or calls them.
 *
 * Conventions (match include/slsp_b200.h):
 *   dtype: 0 int8, 1 bf16 (raw bits), 2 e4m3 (raw codes), 3 fp32, 4 fp64
 *   kind : 0 int8, 1 fp8e4m3                       (quantize.hpp:16)
 *   status: 0 ok, 1 not compliant, 2 dimension mismatch, 3 plan error,
 *           4 non-finite input, 5 invalid argument, 6 malformed metadata,
 *           7 unsupported by this implementation
 */
#ifndef SLSP_ORACLE_H
#define SLSP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_DECLARE(P)                                                                          \
  int P##plan(int z, int l, int hw_m, int hw_n, int* window_count, int* starts, int cap);       \
  int P##pack_matrix(int dtype, const void* w, int64_t rows, int64_t cols, int z, int l,        \
                     void* slided, int64_t* err_row, int64_t* err_block, int threads);          \
  int P##compress(int dtype, const void* slided, int64_t rows, int64_t cols_exp, void* values,  \
                  uint8_t* codes, int64_t* err_row, int64_t* err_window);                       \
  int P##fused_quant_slide(int in_dtype, const void* x, int64_t rows, int64_t cols, int z,      \
                           int l, int kind, uint32_t* payload, float* scales,                   \
                           int64_t* bad_row, int threads);                                      \
  int P##quantize_rows(int in_dtype, const void* x, int64_t rows, int64_t cols, int kind,       \
                       uint8_t* bytes, float* scales, int64_t* bad_row);                        \
  int P##lift_rows(int dtype, const void* x, int64_t rows, int64_t cols, int z, int l,          \
                   void* out);                                                                  \
  int P##sparse_gemm_words(const int8_t* values, const uint8_t* codes, int64_t rows,            \
                           int64_t wpr, const uint32_t* payload, int64_t tokens, int32_t* y,    \
                           int threads);                                                        \
  int P##sparse_gemm_f64(const double* values, const uint8_t* codes, int64_t rows,              \
                         int64_t wpr, const double* lifted, int64_t tokens, double* y,          \
                         int threads);                                                          \
  int P##dense_gemm_i8(const int8_t* w, int64_t n, int64_t k, const int8_t* x, int64_t m,       \
                       int32_t* y, int threads);                                                \
  int P##magnitude_prune(int dtype, const void* w, int64_t rows, int64_t cols, int z, int l,    \
                         void* out);                                                            \
  uint8_t P##fp8_encode(double x);                                                              \
  float P##fp8_decode(uint8_t code);                                                            \
  uint8_t P##quantize_value(double scaled, int kind);                                           \
  void P##pack_codes(const uint8_t* codes, int64_t count, uint8_t* out);

ORC_DECLARE(orc_)
ORC_DECLARE(ref_)

/* Restatement-only helpers (no reference counterpart): the B200 additions. */
/* a18: per-token x per-channel dequant epilogue, y = bf16(((float)acc*s_ch[n])*s_tok[t]). */
void orc_dequant_bf16(const int32_t* acc, int64_t n, int64_t m, const float* s_ch,
                      const float* s_tok, uint16_t* y);
/* Same epilogue, fp32 accumulator input (FP8/BF16 kernels). */
void orc_dequant_f32_bf16(const float* acc, int64_t n, int64_t m, const float* s_ch,
                          const float* s_tok, uint16_t* y);

#ifdef __cplusplus
}
#endif
#endif
