/*
 * slsp CPU oracle: a plain-C restatement of the reference SlideSparse hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This file is the checker, never the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs load it. The B200 library in paper_2603_05232_b200/
 * does not link it and has no CPU fallback.
 *
 * Every function cites the reference file:line it restates (paths relative
 * to /root/reference/proj/include/slsp/). Parity of this restatement is
 * pinned two ways (tests/test_oracle.py):
 *   1. the known-answer vectors of the reference's own tests
 *      (proj/tests/test_pack.cpp, test_quantize.cpp, test_gemm.cpp);
 *   2. bit-for-bit agreement with the reference headers compiled unmodified
 *      into oracle/_ref/libslsp_ref.so (oracle/ref_bridge.cpp), and with the
 *      golden fixtures in tests/golden/ generated from that library.
 */
#include "slsp_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

enum { DT_I8 = 0, DT_BF16 = 1, DT_E4M3 = 2, DT_F32 = 3, DT_F64 = 4 };
enum { ST_OK = 0, ST_NOT_COMPLIANT = 1, ST_DIM = 2, ST_PLAN = 3, ST_NONFINITE = 4,
       ST_INVALID = 5, ST_MALFORMED = 6 };

static int elem_size(int dtype) {
  switch (dtype) {
    case DT_I8: case DT_E4M3: return 1;
    case DT_BF16: return 2;
    case DT_F32: return 4;
    case DT_F64: return 8;
    default: return 0;
  }
}

static float bf16_to_f32(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* fp8.hpp:15-23 fp8_e4m3_decode */
float orc_fp8_decode(uint8_t code) {
  const int neg = (code & 0x80) != 0;
  const int exp_field = (code >> 3) & 0xF;
  const int mant = code & 0x7;
  if (exp_field == 15 && mant == 7) return NAN;
  const double v = exp_field == 0 ? ldexp(mant / 8.0, -6) : ldexp(1.0 + mant / 8.0, exp_field - 7);
  return (float)(neg ? -v : v);
}

/* fp8.hpp:25-52 fp8_e4m3_encode: RNE via nearbyint in double, saturating at 448. */
uint8_t orc_fp8_encode(double x) {
  if (isnan(x)) return 0x7F;
  const uint8_t sign = signbit(x) ? 0x80 : 0x00;
  const double a = fabs(x);
  if (a == 0.0) return sign;
  if (a >= 448.0) return sign | 0x7E;
  int exp2 = 0;
  frexp(a, &exp2);
  int e = exp2 - 1;
  if (e < -6) {
    const double m = nearbyint(ldexp(a, 9));
    if (m >= 8.0) return sign | 0x08;
    return sign | (uint8_t)m;
  }
  double q = nearbyint(ldexp(a, 3 - e));
  if (q >= 16.0) {
    q = 8.0;
    ++e;
  }
  if (e > 8) return sign | 0x7E;
  const uint8_t exp_field = (uint8_t)(e + 7);
  const uint8_t mant = (uint8_t)q & 0x7;
  if (exp_field == 15 && mant == 7) return sign | 0x7E;
  return sign | (uint8_t)(exp_field << 3) | mant;
}

/* matrix.hpp:63-67 is_nonzero: v != T{} (so -0.0 is zero, NaN is nonzero).
 * e4m3 has no reference element type; its codes are judged by decoded value,
 * i.e. 0x00 and 0x80 are zero (SURVEY.md §8c "FP8 weights"). */
static int is_nonzero(int dtype, const void* base, int64_t idx) {
  switch (dtype) {
    case DT_I8: return ((const int8_t*)base)[idx] != 0;
    case DT_E4M3: return (((const uint8_t*)base)[idx] & 0x7F) != 0;
    case DT_BF16: return bf16_to_f32(((const uint16_t*)base)[idx]) != 0.0f;
    case DT_F32: return ((const float*)base)[idx] != 0.0f;
    case DT_F64: return ((const double*)base)[idx] != 0.0;
  }
  return 0;
}

static double as_double(int dtype, const void* base, int64_t idx) {
  switch (dtype) {
    case DT_I8: return (double)((const int8_t*)base)[idx];
    case DT_E4M3: return (double)orc_fp8_decode(((const uint8_t*)base)[idx]);
    case DT_BF16: return (double)bf16_to_f32(((const uint16_t*)base)[idx]);
    case DT_F32: return (double)((const float*)base)[idx];
    case DT_F64: return ((const double*)base)[idx];
  }
  return 0.0;
}

/* pattern.hpp:107-117 plan_status and pattern.hpp:131-154 plan_decomposition.
 * density() < hw_density() compares z/l < hw_m/hw_n exactly (cross-multiply). */
int orc_plan(int z, int l, int hw_m, int hw_n, int* window_count, int* starts, int cap) {
  if (z <= 0 || l <= 0 || z > l || hw_m <= 0 || hw_m >= hw_n) return ST_INVALID;
  if ((int64_t)z * hw_n < (int64_t)hw_m * l) return ST_PLAN; /* already_compliant */
  const int stride = hw_n - hw_m;
  if (l < hw_n || (l - hw_n) % stride != 0) return ST_PLAN; /* non_integral_window_count */
  const int wc = (l - hw_n) / stride + 1;
  if ((int64_t)wc * hw_m < z) return ST_PLAN; /* insufficient_capacity */
  if (wc > cap) return ST_INVALID;
  *window_count = wc;
  for (int j = 0; j < wc; ++j) starts[j] = j * stride;
  return ST_OK;
}

/* ---- parallel_rows (detail/parallel.hpp:18-34): static round-robin rows ---- */
typedef void (*row_fn)(void* ctx, int64_t row);
typedef struct { row_fn fn; void* ctx; int64_t n; int64_t w; int64_t workers; } row_job;

static void* row_worker(void* p) {
  row_job* j = (row_job*)p;
  for (int64_t i = j->w; i < j->n; i += j->workers) j->fn(j->ctx, i);
  return NULL;
}

static void parallel_rows(int64_t n, int threads, row_fn fn, void* ctx) {
  if (threads <= 0) {
    long hc = sysconf(_SC_NPROCESSORS_ONLN);
    threads = hc > 0 ? (int)hc : 1;
  }
  if (threads <= 1 || n <= 1) {
    for (int64_t i = 0; i < n; ++i) fn(ctx, i);
    return;
  }
  int64_t workers = threads < n ? threads : n;
  pthread_t* pool = (pthread_t*)malloc(sizeof(pthread_t) * workers);
  row_job* jobs = (row_job*)malloc(sizeof(row_job) * workers);
  for (int64_t w = 0; w < workers; ++w) {
    jobs[w] = (row_job){fn, ctx, n, w, workers};
    pthread_create(&pool[w], NULL, row_worker, &jobs[w]);
  }
  for (int64_t w = 0; w < workers; ++w) pthread_join(pool[w], NULL);
  free(pool);
  free(jobs);
}

/* ---- weight packer Φ ---- */
typedef struct {
  int dtype, esz, z, l, wc, starts[64];
  const uint8_t* w;
  uint8_t* out;
  int64_t cols, cols_exp;
  int64_t* row_err; /* per-row error block or -1 */
} pack_ctx;

/* pack.hpp:124-133 first_overfull_block, then pack.hpp:83-122 greedy_pack_row.
 * Walk (group g, window w, offset d); accept an unused nonzero while the
 * window holds fewer than hw_m(=2) values, writing it at slot g*wc*4+4w+d. */
static void pack_row_fn(void* vctx, int64_t r) {
  pack_ctx* c = (pack_ctx*)vctx;
  const int64_t groups = c->cols / c->l;
  const uint8_t* src = c->w + r * c->cols * c->esz;
  uint8_t* dst = c->out + r * c->cols_exp * c->esz;
  memset(dst, 0, (size_t)(c->cols_exp * c->esz));
  c->row_err[r] = -1;
  for (int64_t g = 0; g < groups; ++g) { /* first_overfull_block, pack.hpp:127-131 */
    int nnz = 0;
    for (int k = 0; k < c->l; ++k) nnz += is_nonzero(c->dtype, src, g * c->l + k);
    if (nnz > c->z) {
      c->row_err[r] = g;
      return;
    }
  }
  int64_t leftover = -1;
  char used[256];
  const int64_t out_group = (int64_t)c->wc * 4;
  for (int64_t g = 0; g < groups; ++g) {
    const int64_t base = g * c->l;
    memset(used, 0, (size_t)c->l);
    for (int w = 0; w < c->wc; ++w) {
      const int b = c->starts[w];
      int cnt = 0;
      for (int d = 0; d < 4; ++d) {
        const int k = b + d;
        if (!is_nonzero(c->dtype, src, base + k) || used[k]) continue;
        if (cnt < 2) {
          memcpy(dst + (g * out_group + w * 4 + d) * c->esz, src + (base + k) * c->esz,
                 (size_t)c->esz);
          used[k] = 1;
          ++cnt;
        }
      }
    }
    if (leftover < 0) { /* pack.hpp:112-119 */
      for (int k = 0; k < c->l; ++k) {
        if (is_nonzero(c->dtype, src, base + k) && !used[k]) {
          leftover = base + k;
          break;
        }
      }
    }
  }
  if (leftover >= 0) c->row_err[r] = leftover / c->l; /* pack.hpp:192-194 */
}

/* pack.hpp:171-204 pack_matrix; errors report the lowest offending row
 * (row_errors scanned in order, pack.hpp:196-202). Only hw 2:4 is supported
 * by the B200 path (the MMA window), so the oracle fixes hw_m=2, hw_n=4. */
int orc_pack_matrix(int dtype, const void* w, int64_t rows, int64_t cols, int z, int l,
                    void* slided, int64_t* err_row, int64_t* err_block, int threads) {
  pack_ctx c;
  c.dtype = dtype;
  c.esz = elem_size(dtype);
  if (!c.esz || l > 256) return ST_INVALID;
  int st = orc_plan(z, l, 2, 4, &c.wc, c.starts, 64);
  if (st) return st;
  if (cols % l != 0) return ST_DIM; /* pack.hpp:174-177 */
  c.z = z;
  c.l = l;
  c.w = (const uint8_t*)w;
  c.out = (uint8_t*)slided;
  c.cols = cols;
  c.cols_exp = cols / l * c.wc * 4;
  c.row_err = (int64_t*)malloc(sizeof(int64_t) * (size_t)(rows > 0 ? rows : 1));
  parallel_rows(rows, threads, pack_row_fn, &c);
  st = ST_OK;
  for (int64_t r = 0; r < rows; ++r) {
    if (c.row_err[r] >= 0) {
      if (err_row) *err_row = r;
      if (err_block) *err_block = c.row_err[r];
      st = ST_NOT_COMPLIANT;
      break;
    }
  }
  free(c.row_err);
  return st;
}

/* gemm.hpp:70-110 compress: per 4-window, nonzero positions padded with the
 * smallest unused positions (value T{}), sorted; values in position order and
 * one byte per 2-bit code. Single-threaded, like the reference. */
int orc_compress(int dtype, const void* slided, int64_t rows, int64_t cols_exp, void* values,
                 uint8_t* codes, int64_t* err_row, int64_t* err_window) {
  const int esz = elem_size(dtype);
  if (!esz) return ST_INVALID;
  if (cols_exp % 4 != 0) return ST_DIM;
  const int64_t wpr = cols_exp / 4;
  const uint8_t* s = (const uint8_t*)slided;
  uint8_t* v = (uint8_t*)values;
  int64_t o = 0;
  for (int64_t r = 0; r < rows; ++r) {
    for (int64_t w = 0; w < wpr; ++w) {
      const int64_t base = r * cols_exp + w * 4;
      int pos[4], np = 0;
      for (int d = 0; d < 4; ++d)
        if (is_nonzero(dtype, s, base + d)) pos[np++] = d;
      if (np > 2) {
        if (err_row) *err_row = r;
        if (err_window) *err_window = w;
        return ST_NOT_COMPLIANT;
      }
      for (int d = 0; np < 2; ++d) { /* gemm.hpp:99-101 */
        int found = 0;
        for (int i = 0; i < np; ++i) found |= pos[i] == d;
        if (!found) pos[np++] = d;
      }
      if (pos[0] > pos[1]) { /* sort, gemm.hpp:102 */
        int t = pos[0];
        pos[0] = pos[1];
        pos[1] = t;
      }
      for (int i = 0; i < 2; ++i) {
        memcpy(v + o * esz, s + (base + pos[i]) * esz, (size_t)esz);
        codes[o] = (uint8_t)pos[i];
        ++o;
      }
    }
  }
  return ST_OK;
}

/* container.hpp:330-336 pack_codes: four 2-bit codes per byte, LSB first. */
void orc_pack_codes(const uint8_t* codes, int64_t count, uint8_t* out) {
  memset(out, 0, (size_t)((count + 3) / 4));
  for (int64_t i = 0; i < count; ++i) out[i / 4] |= (uint8_t)((codes[i] & 0x3) << (2 * (i % 4)));
}

/* quantize.hpp:26-37 quant_max + quantize_value: int8 = clamp(rne(s), ±127),
 * never -128; fp8: exact 0 (incl. -0.0) -> 0x00, else encode(clamp(s, ±448)). */
static double quant_max(int kind) { return kind == 0 ? 127.0 : 448.0; }

uint8_t orc_quantize_value(double scaled, int kind) {
  if (kind == 0) {
    double q = nearbyint(scaled);
    if (q < -127.0) q = -127.0;
    if (q > 127.0) q = 127.0;
    return (uint8_t)(int8_t)q;
  }
  if (scaled == 0.0) return 0;
  if (scaled < -448.0) scaled = -448.0;
  if (scaled > 448.0) scaled = 448.0;
  return orc_fp8_encode(scaled);
}

typedef struct {
  int dtype, kind, l, wc, starts[64];
  const void* x;
  int64_t cols, words;
  uint32_t* payload;
  float* scales;
  char* bad;
} fqs_ctx;

/* quantize.hpp:122-174 fused_quant_slide, one token row: pass 1 absmax in
 * double with a non-finite flag (:142-150); r = qmax/absmax and
 * scale = float(absmax/qmax) (:151-153); pass 2 over output words
 * j -> (g = j/wc, w = j%wc), b = l*g + start[w], zero padding past cols. */
static void fqs_row_fn(void* vctx, int64_t i) {
  fqs_ctx* c = (fqs_ctx*)vctx;
  double absmax = 0.0;
  c->bad[i] = 0;
  for (int64_t k = 0; k < c->cols; ++k) {
    const double d = as_double(c->dtype, c->x, i * c->cols + k);
    if (!isfinite(d)) {
      c->bad[i] = 1;
      return;
    }
    if (fabs(d) > absmax) absmax = fabs(d);
  }
  const double qmax = quant_max(c->kind);
  const double r = absmax == 0.0 ? 0.0 : qmax / absmax;
  c->scales[i] = absmax == 0.0 ? 1.0f : (float)(absmax / qmax);
  uint32_t* words = c->payload + i * c->words;
  for (int64_t j = 0; j < c->words; ++j) {
    const int64_t g = j / c->wc;
    const int w = (int)(j % c->wc);
    const int64_t b = (int64_t)c->l * g + c->starts[w];
    uint32_t word = 0;
    for (int d = 0; d < 4; ++d) {
      const int64_t k = b + d;
      const double v = k < c->cols ? as_double(c->dtype, c->x, i * c->cols + k) : 0.0;
      word |= (uint32_t)orc_quantize_value(v * r, c->kind) << (8 * d); /* pack_word :91-94 */
    }
    words[j] = word;
  }
}

int orc_fused_quant_slide(int in_dtype, const void* x, int64_t rows, int64_t cols, int z, int l,
                          int kind, uint32_t* payload, float* scales, int64_t* bad_row,
                          int threads) {
  fqs_ctx c;
  if (in_dtype != DT_F32 && in_dtype != DT_F64 && in_dtype != DT_BF16) return ST_INVALID;
  if (kind != 0 && kind != 1) return ST_INVALID;
  int st = orc_plan(z, l, 2, 4, &c.wc, c.starts, 64);
  if (st) return st;
  c.dtype = in_dtype;
  c.kind = kind;
  c.l = l;
  c.x = x;
  c.cols = cols;
  c.words = (cols + l - 1) / l * c.wc; /* quantize.hpp:130-133 */
  c.payload = payload;
  c.scales = scales;
  c.bad = (char*)calloc((size_t)(rows > 0 ? rows : 1), 1);
  for (int64_t i = 0; i < rows; ++i) scales[i] = 1.0f;
  memset(payload, 0, (size_t)(rows * c.words * 4));
  parallel_rows(rows, threads, fqs_row_fn, &c);
  st = ST_OK;
  for (int64_t i = 0; i < rows; ++i) {
    if (c.bad[i]) { /* quantize.hpp:168-172: first bad row */
      if (bad_row) *bad_row = i;
      st = ST_NONFINITE;
      break;
    }
  }
  free(c.bad);
  return st;
}

/* quantize.hpp:52-68 quantize_row applied per token row (the dense side's
 * activations, tools/slsp.cpp:610-614). */
int orc_quantize_rows(int in_dtype, const void* x, int64_t rows, int64_t cols, int kind,
                      uint8_t* bytes, float* scales, int64_t* bad_row) {
  if (in_dtype != DT_F32 && in_dtype != DT_F64 && in_dtype != DT_BF16) return ST_INVALID;
  for (int64_t i = 0; i < rows; ++i) {
    double absmax = 0.0;
    for (int64_t k = 0; k < cols; ++k) {
      const double d = as_double(in_dtype, x, i * cols + k);
      if (!isfinite(d)) {
        if (bad_row) *bad_row = i;
        return ST_NONFINITE;
      }
      if (fabs(d) > absmax) absmax = fabs(d);
    }
    const double qmax = quant_max(kind);
    const double r = absmax == 0.0 ? 0.0 : qmax / absmax;
    scales[i] = absmax == 0.0 ? 1.0f : (float)(absmax / qmax);
    for (int64_t k = 0; k < cols; ++k)
      bytes[i * cols + k] = orc_quantize_value(as_double(in_dtype, x, i * cols + k) * r, kind);
  }
  return ST_OK;
}

/* quantize.hpp:72-89 lift_row per token row: window j of group g holds
 * x[l*g + stride*j .. +4). Pure index remapping, any element type. */
int orc_lift_rows(int dtype, const void* x, int64_t rows, int64_t cols, int z, int l, void* out) {
  int wc, starts[64];
  const int esz = elem_size(dtype);
  if (!esz) return ST_INVALID;
  int st = orc_plan(z, l, 2, 4, &wc, starts, 64);
  if (st) return st;
  if (cols % l != 0) return ST_DIM;
  const int64_t groups = cols / l;
  const int64_t ocols = groups * wc * 4;
  const uint8_t* s = (const uint8_t*)x;
  uint8_t* o = (uint8_t*)out;
  for (int64_t i = 0; i < rows; ++i) {
    int64_t p = 0;
    for (int64_t g = 0; g < groups; ++g)
      for (int j = 0; j < wc; ++j)
        for (int d = 0; d < 4; ++d, ++p)
          memcpy(o + (i * ocols + p) * esz, s + (i * cols + g * l + starts[j] + d) * esz,
                 (size_t)esz);
  }
  return ST_OK;
}

/* gemm.hpp:199-233 int8 packed-word sparse_gemm: Y[i][t] = sum_w sum_k
 * val[i][w][k] * int8(byte(payload[t][w], meta[i][w][k])), int32, N x M. */
typedef struct {
  const int8_t* values;
  const uint8_t* codes;
  const uint32_t* payload;
  int64_t wpr, tokens;
  int32_t* y;
} spw_ctx;

static void spw_row_fn(void* vctx, int64_t i) {
  spw_ctx* c = (spw_ctx*)vctx;
  const int8_t* vals = c->values + i * c->wpr * 2;
  const uint8_t* meta = c->codes + i * c->wpr * 2;
  for (int64_t t = 0; t < c->tokens; ++t) {
    const uint32_t* words = c->payload + t * c->wpr;
    int32_t acc = 0;
    for (int64_t w = 0; w < c->wpr; ++w) {
      const uint32_t word = words[w];
      for (int k = 0; k < 2; ++k) {
        const int8_t b = (int8_t)((word >> (8 * meta[w * 2 + k])) & 0xFFu);
        acc += (int32_t)vals[w * 2 + k] * (int32_t)b;
      }
    }
    c->y[i * c->tokens + t] = acc;
  }
}

int orc_sparse_gemm_words(const int8_t* values, const uint8_t* codes, int64_t rows, int64_t wpr,
                          const uint32_t* payload, int64_t tokens, int32_t* y, int threads) {
  spw_ctx c = {values, codes, payload, wpr, tokens, y};
  if (wpr * 4 > ((int64_t)1 << 23)) return ST_INVALID; /* gemm.hpp:56 overflow guard */
  parallel_rows(rows, threads, spw_row_fn, &c);
  return ST_OK;
}

/* gemm.hpp:164-197 generic sparse_gemm<T> restated on doubles (accum_type
 * float -> double, gemm.hpp:39-42): the FP8/BF16 tolerance oracle. */
typedef struct {
  const double* values;
  const uint8_t* codes;
  const double* lifted;
  int64_t wpr, tokens;
  double* y;
} spf_ctx;

static void spf_row_fn(void* vctx, int64_t i) {
  spf_ctx* c = (spf_ctx*)vctx;
  const double* vals = c->values + i * c->wpr * 2;
  const uint8_t* meta = c->codes + i * c->wpr * 2;
  for (int64_t t = 0; t < c->tokens; ++t) {
    const double* act = c->lifted + t * c->wpr * 4;
    double acc = 0.0;
    for (int64_t w = 0; w < c->wpr; ++w)
      for (int k = 0; k < 2; ++k) acc += vals[w * 2 + k] * act[w * 4 + meta[w * 2 + k]];
    c->y[i * c->tokens + t] = acc;
  }
}

int orc_sparse_gemm_f64(const double* values, const uint8_t* codes, int64_t rows, int64_t wpr,
                        const double* lifted, int64_t tokens, double* y, int threads) {
  spf_ctx c = {values, codes, lifted, wpr, tokens, y};
  parallel_rows(rows, threads, spf_row_fn, &c);
  return ST_OK;
}

/* gemm.hpp:142-162 dense_gemm: Y = W X with X holding one token per column
 * (K x M), fixed left-to-right k order, int8 -> int32. */
typedef struct {
  const int8_t* w;
  const int8_t* x;
  int64_t k, m;
  int32_t* y;
} dg_ctx;

static void dg_row_fn(void* vctx, int64_t i) {
  dg_ctx* c = (dg_ctx*)vctx;
  for (int64_t t = 0; t < c->m; ++t) {
    int32_t acc = 0;
    for (int64_t k = 0; k < c->k; ++k) acc += (int32_t)c->w[i * c->k + k] * (int32_t)c->x[k * c->m + t];
    c->y[i * c->m + t] = acc;
  }
}

int orc_dense_gemm_i8(const int8_t* w, int64_t n, int64_t k, const int8_t* x, int64_t m,
                      int32_t* y, int threads) {
  dg_ctx c = {w, x, k, m, y};
  if (k > ((int64_t)1 << 23)) return ST_INVALID; /* gemm.hpp:147-149 */
  parallel_rows(n, threads, dg_row_fn, &c);
  return ST_OK;
}

/* pack.hpp:238-261 magnitude_prune: zero the l-z smallest-|v| elements of
 * every block; ties prune the lower index first (stable sort by magnitude). */
int orc_magnitude_prune(int dtype, const void* w, int64_t rows, int64_t cols, int z, int l,
                        void* out) {
  const int esz = elem_size(dtype);
  if (!esz || l > 256 || z > l) return ST_INVALID;
  if (cols % l != 0) return ST_DIM;
  memcpy(out, w, (size_t)(rows * cols * esz));
  const int prune = l - z;
  uint8_t* o = (uint8_t*)out;
  int order[256];
  double mag[256];
  for (int64_t r = 0; r < rows; ++r) {
    for (int64_t g = 0; g * l < cols; ++g) {
      const int64_t base = r * cols + g * l;
      for (int k = 0; k < l; ++k) {
        order[k] = k;
        mag[k] = fabs(as_double(dtype, w, base + k));
      }
      for (int a = 1; a < l; ++a) { /* stable insertion sort by magnitude */
        const int key = order[a];
        int b = a - 1;
        while (b >= 0 && mag[order[b]] > mag[key]) {
          order[b + 1] = order[b];
          --b;
        }
        order[b + 1] = key;
      }
      for (int k = 0; k < prune; ++k) memset(o + (base + order[k]) * esz, 0, (size_t)esz);
    }
  }
  return ST_OK;
}

/* ---- B200 addition a18: dequant epilogue, restated with the
 * exact fp32 operation order the CUDA epilogue uses. ---- */
static uint16_t f32_to_bf16_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40);
  const uint32_t lsb = (u >> 16) & 1u;
  u += 0x7fffu + lsb;
  return (uint16_t)(u >> 16);
}

void orc_dequant_bf16(const int32_t* acc, int64_t n, int64_t m, const float* s_ch,
                      const float* s_tok, uint16_t* y) {
  for (int64_t i = 0; i < n; ++i)
    for (int64_t t = 0; t < m; ++t) {
      volatile float a = (float)acc[i * m + t];
      volatile float p = a * s_ch[i];
      volatile float q = p * s_tok[t];
      y[i * m + t] = f32_to_bf16_rne(q);
    }
}

void orc_dequant_f32_bf16(const float* acc, int64_t n, int64_t m, const float* s_ch,
                          const float* s_tok, uint16_t* y) {
  for (int64_t i = 0; i < n; ++i)
    for (int64_t t = 0; t < m; ++t) {
      volatile float p = acc[i * m + t] * s_ch[i];
      volatile float q = p * s_tok[t];
      y[i * m + t] = f32_to_bf16_rne(q);
    }
}
