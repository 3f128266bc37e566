// Activation Lifting Ψ on sm_100a: per-token absmax + quantization fused with
// the window-duplicating rearrangement K -> K'.
//
// One CTA per token row (grid-stride). Pass 1 streams the row into shared
// memory with 16-byte coalesced loads while reducing |x| (warp shuffles +
// one smem hop). Pass 2 quantizes every SOURCE element exactly once in
// double precision (the reference computes x*r in double, quantize.hpp:151,
// :163 — fp32 math would flip ~4e-4 of the codes). Pass 3
// emits the lifted words: word j = window j of group g = j/wc, source offset
// l*g + 2*(j%wc), written as 16-byte vector stores.
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace {

using namespace slsp_dev;

constexpr int kThreads = 256;

enum : int { IN_F32 = 0, IN_BF16 = 1 };
enum : int { K_INT8 = 0, K_FP8 = 1, K_NONE = 2 };

template <int IN>
SLSP_DEVINL float in_value(const uint8_t* s, int64_t k) {
  if constexpr (IN == IN_F32) return reinterpret_cast<const float*>(s)[k];
  return __uint_as_float(static_cast<uint32_t>(reinterpret_cast<const uint16_t*>(s)[k]) << 16);
}

struct ActArgs {
  const uint8_t* x;
  int64_t rows, cols;
  int l, wc, kind;
  int64_t in_cols_pad;  // ceil(cols/l)*l: zero-padded source width (quantize.hpp:130,162)
  int64_t words_real;   // lifted windows per row (LIFT) — unused otherwise
  int64_t out_bytes;    // bytes written per row (kp or kpad, times element size for K_NONE)
  uint8_t* out;
  float* scales;
  unsigned long long* status;
  // §8f #3: each row's |x|max computed upstream (slsp_sparse_gemm_amax);
  // when set, the kernels skip their own |x|max pass / block reduction
  const float* amax_in;
  // Row stride of the output(s) in bytes (== out_bytes except for the
  // K-sharded multi-destination lift, where a rank writes its column slice
  // of every rank's full payload: out and dst[0..ndst) all at the slice's
  // byte column, ld = the full payload row, SURVEY §8e / DESIGN §7)
  int64_t out_ld;
  int ndst;
  uint8_t* dst[7];
};

// 16-byte store of output vector `i` of row `row` to the output and every
// extra destination (peer payloads over NVLink in the sharded lift).
SLSP_DEVINL void store_out_vec(const ActArgs& a, int64_t row, int i, uint4 v) {
  reinterpret_cast<uint4*>(a.out + row * a.out_ld)[i] = v;
  for (int d = 0; d < a.ndst; ++d) reinterpret_cast<uint4*>(a.dst[d] + row * a.out_ld)[i] = v;
}

// Launch-path selection (env SLSP_LIFT_ROW, perf probing): 0 = warp path,
// else (default) the row-resident path where it applies. (Measured and
// dropped: persistent CTAs with a register double buffer, and a coalesced
// one-block-per-lane layout — both slower on the Qwen/Llama K values.)
int env_row_path() { return static_cast<int>(slsp_host::knob("SLSP_LIFT_ROW", 1)); }

template <int IN, int KIND, bool LIFT>
__global__ void __launch_bounds__(kThreads) act_kernel(ActArgs a) {
  constexpr int ESZ = IN == IN_F32 ? 4 : 2;
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ float s_red[kThreads / 32];
  __shared__ int s_bad[kThreads / 32];
  uint8_t* s_x = smem;                                       // raw source row, padded
  uint8_t* s_q = smem + ((a.in_cols_pad * ESZ + 15) & ~15);  // quantized codes (KIND != NONE)
  const int warp = threadIdx.x >> 5;

  for (int64_t row = blockIdx.x; row < a.rows; row += gridDim.x) {
    const uint8_t* src = a.x + row * a.cols * ESZ;
    // ---- pass 1: row -> smem, |x| max, finiteness ----
    float amax = 0.f;
    int bad = 0;
    const int64_t nbytes = a.cols * ESZ;
    const bool vec = ((reinterpret_cast<uintptr_t>(src) & 15u) == 0);
    int64_t done = 0;
    if (vec) {
      const int64_t nvec = nbytes >> 4;
      for (int64_t i = threadIdx.x; i < nvec; i += kThreads) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(src) + i);
        reinterpret_cast<uint4*>(s_x)[i] = v;
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if constexpr (IN == IN_F32) {
            const float f = __uint_as_float(w[j]);
            bad |= !isfinite(f);
            amax = fmaxf(amax, fabsf(f));
          } else {
            const float f0 = __uint_as_float(w[j] << 16), f1 = __uint_as_float(w[j] & 0xFFFF0000u);
            bad |= !isfinite(f0) | !isfinite(f1);
            amax = fmaxf(amax, fmaxf(fabsf(f0), fabsf(f1)));
          }
        }
      }
      done = nvec << 4;
    }
    for (int64_t b = done / ESZ + threadIdx.x; b < a.cols; b += kThreads) {
      const float f = in_value<IN>(src, b);
      if constexpr (IN == IN_F32) reinterpret_cast<float*>(s_x)[b] = f;
      else reinterpret_cast<uint16_t*>(s_x)[b] = reinterpret_cast<const uint16_t*>(src)[b];
      bad |= !isfinite(f);
      amax = fmaxf(amax, fabsf(f));
    }
    for (int64_t b = a.cols + threadIdx.x; b < a.in_cols_pad; b += kThreads) {  // zero pad
      if constexpr (IN == IN_F32) reinterpret_cast<float*>(s_x)[b] = 0.f;
      else reinterpret_cast<uint16_t*>(s_x)[b] = 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if ((threadIdx.x & 31) == 0) {
      s_red[warp] = amax;
      s_bad[warp] = bad;
    }
    __syncthreads();
    amax = 0.f;
    bad = 0;
#pragma unroll
    for (int i = 0; i < kThreads / 32; ++i) {
      amax = fmaxf(amax, s_red[i]);
      bad |= s_bad[i];
    }
    if (a.amax_in) {
      amax = a.amax_in[row];
      bad = !isfinite(amax);
    }
    if (bad && threadIdx.x == 0 && a.status) atomicMin(a.status, static_cast<unsigned long long>(row) << 32);

    if constexpr (KIND != K_NONE) {
      // quantize.hpp:151-153: r = qmax/absmax, scale = float(absmax/qmax), in double.
      const double qmax = KIND == K_INT8 ? 127.0 : 448.0;
      const double absmax = static_cast<double>(amax);
      const double r = absmax == 0.0 ? 0.0 : qmax / absmax;
      if (threadIdx.x == 0) a.scales[row] = absmax == 0.0 ? 1.0f : __double2float_rn(absmax / qmax);
      // ---- pass 2: quantize each source element once ----
      for (int64_t k = threadIdx.x; k < a.in_cols_pad; k += kThreads)
        s_q[k] = quantize_value(static_cast<double>(in_value<IN>(s_x, k)) * r, KIND);
    }
    __syncthreads();

    // ---- pass 3: emit the row, 16 bytes per thread per step ----
    uint8_t* dst = a.out + row * a.out_ld;
    const int64_t nchunks = a.out_bytes >> 4;
    for (int64_t c = threadIdx.x; c < nchunks; c += kThreads) {
      uint32_t o[4];
      if constexpr (KIND != K_NONE && LIFT) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t j = c * 4 + i;  // lifted word = window j
          uint32_t word = 0;
          if (j < a.words_real) {
            const int64_t g = j / a.wc;
            const int64_t b = g * a.l + 2 * (j - g * a.wc);
            const uint16_t lo = *reinterpret_cast<const uint16_t*>(s_q + b);
            const uint16_t hi = *reinterpret_cast<const uint16_t*>(s_q + b + 2);
            word = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
          }
          o[i] = word;
        }
      } else if constexpr (KIND != K_NONE) {  // quantize_rows: identity layout
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint32_t word = 0;
          for (int d = 0; d < 4; ++d) {
            const int64_t k = c * 16 + i * 4 + d;
            if (k < a.cols) word |= static_cast<uint32_t>(s_q[k]) << (8 * d);
          }
          o[i] = word;
        }
      } else {  // BF16/FP32 passthrough lift (lift_row, quantize.hpp:72-89)
        constexpr int PER = 16 / ESZ;  // elements per 16-byte chunk
        uint8_t* ob = reinterpret_cast<uint8_t*>(o);
#pragma unroll
        for (int e = 0; e < PER; ++e) {
          const int64_t p = c * PER + e;  // lifted element index
          const int64_t j = p >> 2;
          if (j < a.words_real) {
            const int64_t g = j / a.wc;
            const int64_t b = g * a.l + 2 * (j - g * a.wc) + (p & 3);
            if constexpr (ESZ == 2)
              reinterpret_cast<uint16_t*>(ob)[e] = reinterpret_cast<const uint16_t*>(s_x)[b];
            else
              reinterpret_cast<uint32_t*>(ob)[e] = reinterpret_cast<const uint32_t*>(s_x)[b];
          } else {
            if constexpr (ESZ == 2) reinterpret_cast<uint16_t*>(ob)[e] = 0;
            else reinterpret_cast<uint32_t*>(ob)[e] = 0;
          }
        }
      }
      reinterpret_cast<uint4*>(dst)[c] = make_uint4(o[0], o[1], o[2], o[3]);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Fast path: one WARP per token row, no shared memory. A lane owns "quads" of
// 4 consecutive source blocks (4*L elements, a whole number of 16-byte
// vectors for every (2N-2):2N pattern), so every lifted window of a quad is
// built from registers: window w of block g covers bytes [g*L + 2w, +4) of
// the quad's codes. Pass 1 streams the row for |x|max (vector loads, warp
// shuffle reduce); pass 2 re-reads it (L1/L2-resident), quantizes each source
// element once in double and emits the quad's lifted words as 16-byte stores.
// Requirements (host-checked): cols % (4*L) == 0, 16-byte aligned rows.
template <int IN, int KIND, int L>
struct WarpGeom {
  static constexpr int ESZ = IN == IN_F32 ? 4 : 2;
  static constexpr int WC = (L - 4) / 2 + 1;
  static constexpr int ELEMS = 4 * L;               // source elements per quad
  static constexpr int IN_VEC = ELEMS * ESZ / 16;   // 16-byte loads per quad
  static constexpr int OUT_ELEMS = 4 * WC * 4;      // lifted elements per quad
  static constexpr int OESZ = KIND == K_NONE ? ESZ : 1;
  static constexpr int OUT_VEC = OUT_ELEMS * OESZ / 16;
  static_assert(ELEMS * ESZ % 16 == 0 && OUT_ELEMS * OESZ % 16 == 0, "quad must be whole vectors");
};

template <int IN, int N>
SLSP_DEVINL float elem(const uint4 (&v)[N], int e) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(v);
  if constexpr (IN == IN_F32) return __uint_as_float(w[e]);
  return __uint_as_float(((w[e >> 1] >> (16 * (e & 1))) & 0xFFFFu) << 16);
}

// Exact f32 -> f64 widening on the integer pipes (the FP64 pipe is the
// lifting kernel's bottleneck). Zero/subnormal/non-finite inputs take the
// conversion instruction.
SLSP_DEVINL double widen_exact(float f) {
  const uint32_t u = __float_as_uint(f);
  const uint32_t e = (u >> 23) & 0xFFu;
  if (e == 0u || e == 0xFFu) return static_cast<double>(f);
  const uint32_t hi = (u & 0x80000000u) | ((e + 896u) << 20) | ((u >> 3) & 0xFFFFFu);
  return __hiloint2double(static_cast<int>(hi), static_cast<int>(u << 29));
}

// quantize.hpp:30-37 for one element. INT8: |x| <= absmax implies
// |x*r| <= fl(absmax*fl(127/absmax)) < 127.5, so the reference's clamp never
// binds and rint+convert is one cvt.rni (ties-to-even, like nearbyint).
template <int KIND>
SLSP_DEVINL uint32_t quant_code(float x, double r) {
  if constexpr (KIND == K_INT8) return static_cast<uint32_t>(__double2int_rn(widen_exact(x) * r)) & 0xFFu;
  return quantize_value(static_cast<double>(x) * r, KIND);
}

// INT8 fast path, exact: y = fl32(x * fl32(r)) differs from the reference's
// fl64(x * r) by < 1.6e-5 (|y| <= 127.0001, two fp32 roundings); rounding y
// with the 1.5*2^23 magic constant therefore gives rint(fl64(x*r)) unless y is
// within 3e-5 of a half-integer, in which case the FP64 path decides. The
// code byte is the low byte of the magic sum (0x4B400000 + q).
SLSP_DEVINL uint32_t quant_int8_fast(float x, float r32, double r) {
  const float y = __fmul_rn(x, r32);
  const float t = __fadd_rn(y, 12582912.0f);
  const float frac = __fsub_rn(y, __fsub_rn(t, 12582912.0f));
  if (fabsf(frac) >= 0.49997f) return quant_code<K_INT8>(x, r);
  return __float_as_uint(t) & 0xFFu;
}

__device__ __noinline__ uint32_t quant4_bf16_int8_slow(uint32_t wa, uint32_t wb, double r) {
  uint32_t c[4];
  c[0] = quant_code<K_INT8>(__uint_as_float(wa << 16), r);
  c[1] = quant_code<K_INT8>(__uint_as_float(wa & 0xFFFF0000u), r);
  c[2] = quant_code<K_INT8>(__uint_as_float(wb << 16), r);
  c[3] = quant_code<K_INT8>(__uint_as_float(wb & 0xFFFF0000u), r);
  return __byte_perm(__byte_perm(c[0], c[1], 0x0040), __byte_perm(c[2], c[3], 0x0040), 0x5410);
}

// quant_int8_fast for 4 BF16 elements (two bf16x2 words) with packed f32x2
// math: byte d of the result = code of element d. Any element within 3e-5 of
// a half-integer sends all four to the exact FP64 path (out of line: rare).
SLSP_DEVINL uint32_t quant4_bf16_int8(uint32_t wa, uint32_t wb, float r32, double r, bool exact_r = false) {
  const float2 M = make_float2(12582912.0f, 12582912.0f), R = make_float2(r32, r32);
  const float2 y0 = fmul2_rn(make_float2(__uint_as_float(wa << 16), __uint_as_float(wa & 0xFFFF0000u)), R);
  const float2 y1 = fmul2_rn(make_float2(__uint_as_float(wb << 16), __uint_as_float(wb & 0xFFFF0000u)), R);
  const float2 t0 = fadd2_rn(y0, M), t1 = fadd2_rn(y1, M);
  const float2 f0 = fsub2_rn(y0, fsub2_rn(t0, M)), f1 = fsub2_rn(y1, fsub2_rn(t1, M));
  const float m = fmaxf(fmaxf(fabsf(f0.x), fabsf(f0.y)), fmaxf(fabsf(f1.x), fabsf(f1.y)));
  if (!exact_r && m >= 0.49997f) return quant4_bf16_int8_slow(wa, wb, r);
  return __byte_perm(__byte_perm(__float_as_uint(t0.x), __float_as_uint(t0.y), 0x0040),
                     __byte_perm(__float_as_uint(t1.x), __float_as_uint(t1.y), 0x0040), 0x5410);
}

// One quad (4 source blocks) -> its lifted output words (quantize.hpp:130-166
// for the quad's groups): quantize every source element once, then window w
// of block g = bytes [g*L + 2w, +4) of the quad's codes.
template <int IN, int KIND, int L>
SLSP_DEVINL void emit_quad(const uint4 (&v)[WarpGeom<IN, KIND, L>::IN_VEC], float r32, double r, bool exact_r,
                           uint32_t (&o)[WarpGeom<IN, KIND, L>::OUT_VEC * 4]) {
  using G = WarpGeom<IN, KIND, L>;
      if constexpr (KIND != K_NONE) {
        uint32_t qw[G::ELEMS / 4 + 1];
        qw[G::ELEMS / 4] = 0;
#pragma unroll
        for (int i = 0; i < G::ELEMS / 4; ++i) {
          if constexpr (KIND == K_INT8 && IN == IN_BF16) {
            const uint32_t* iw = reinterpret_cast<const uint32_t*>(v);
            qw[i] = quant4_bf16_int8(iw[2 * i], iw[2 * i + 1], r32, r, exact_r);
          } else {
            uint32_t b[4];
#pragma unroll
            for (int d = 0; d < 4; ++d) {
              const float x = elem<IN>(v, 4 * i + d);
              if constexpr (KIND == K_INT8) b[d] = quant_int8_fast(x, r32, r);
              else b[d] = quant_code<KIND>(x, r);
            }
            // byte 0 of each b[d] -> byte d of the word
            qw[i] = __byte_perm(__byte_perm(b[0], b[1], 0x0040), __byte_perm(b[2], b[3], 0x0040), 0x5410);
          }
        }
#pragma unroll
        for (int g = 0; g < 4; ++g)
#pragma unroll
          for (int w = 0; w < G::WC; ++w) {
            const int b = g * L + 2 * w;  // even byte offset of the window in the quad
            o[g * G::WC + w] = (b & 3) ? __byte_perm(qw[b >> 2], qw[(b >> 2) + 1], 0x5432) : qw[b >> 2];
          }
      } else {  // passthrough lift of raw elements
        const uint32_t* iw = reinterpret_cast<const uint32_t*>(v);
#pragma unroll
        for (int g = 0; g < 4; ++g)
#pragma unroll
          for (int w = 0; w < G::WC; ++w) {
            const int b = g * L + 2 * w;  // element offset
            if constexpr (G::ESZ == 2) {
              o[(g * G::WC + w) * 2] = iw[b >> 1];
              o[(g * G::WC + w) * 2 + 1] = iw[(b >> 1) + 1];
            } else {
#pragma unroll
              for (int d = 0; d < 4; ++d) o[(g * G::WC + w) * 4 + d] = iw[b + d];
            }
          }
      }
}

template <int IN, int KIND, int L>
__global__ void __launch_bounds__(256) act_warp_kernel(ActArgs a) {
  using G = WarpGeom<IN, KIND, L>;
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int nquads = static_cast<int>(a.cols / G::ELEMS);
  const int out_vecs = static_cast<int>(a.out_bytes >> 4);
  for (int64_t row = warp0; row < a.rows; row += nwarps) {
    const uint4* src = reinterpret_cast<const uint4*>(a.x + row * a.cols * G::ESZ);
    double r = 0.0;
    float r32 = 0.f;
    bool exact_r = false;
    if constexpr (KIND != K_NONE) {
      float amax = 0.f;
      int bad = 0;
      if (a.amax_in) {
        amax = a.amax_in[row];
        bad = !isfinite(amax);
      } else if constexpr (IN == IN_BF16) {
        // packed bf16x2 |x| max; NaN propagates and Inf wins, so the row is
        // non-finite iff the final max is
        __nv_bfloat162 m2 = __float2bfloat162_rn(0.f);
#pragma unroll 2
        for (int q = lane; q < nquads; q += 32) {
          uint4 v[G::IN_VEC];
#pragma unroll
          for (int i = 0; i < G::IN_VEC; ++i) v[i] = __ldg(src + q * G::IN_VEC + i);
          const uint32_t* w = reinterpret_cast<const uint32_t*>(v);
#pragma unroll
          for (int e = 0; e < G::IN_VEC * 4; ++e)
            m2 = __hmax2_nan(m2, __habs2(*reinterpret_cast<const __nv_bfloat162*>(&w[e])));
        }
        amax = fmaxf(__low2float(m2), __high2float(m2));
        bad = !isfinite(__low2float(m2)) || !isfinite(__high2float(m2));
      } else {
#pragma unroll 2
        for (int q = lane; q < nquads; q += 32) {
          uint4 v[G::IN_VEC];
#pragma unroll
          for (int i = 0; i < G::IN_VEC; ++i) v[i] = __ldg(src + q * G::IN_VEC + i);
#pragma unroll
          for (int e = 0; e < G::ELEMS; ++e) {
            const float f = elem<IN>(v, e);
            bad |= !isfinite(f);
            amax = fmaxf(amax, fabsf(f));
          }
        }
      }
      if (!a.amax_in) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
          bad |= __shfl_xor_sync(0xffffffffu, bad, o);
        }
      }
      if (bad && lane == 0 && a.status) atomicMin(a.status, static_cast<unsigned long long>(row) << 32);
      // quantize.hpp:151-153, in double
      const double qmax = KIND == K_INT8 ? 127.0 : 448.0;
      const double absmax = static_cast<double>(amax);
      r = absmax == 0.0 ? 0.0 : qmax / absmax;
      r32 = __double2float_rn(r);
      // r exactly representable with <= 16 significant bits (e.g. absmax a power
      // of two): every bf16 x times r32 is exact in fp32, ties included
      exact_r = IN == IN_BF16 && KIND == K_INT8 && r32 != 0.f &&
                fmaf(r32, static_cast<float>(absmax), -127.0f) == 0.f && (__float_as_uint(r32) & 0xFFu) == 0u;
      if (lane == 0) a.scales[row] = absmax == 0.0 ? 1.0f : __double2float_rn(absmax / qmax);
    }
#pragma unroll 2
    for (int q = lane; q < nquads; q += 32) {
      uint4 v[G::IN_VEC];
#pragma unroll
      for (int i = 0; i < G::IN_VEC; ++i) v[i] = __ldg(src + q * G::IN_VEC + i);
      uint32_t o[G::OUT_VEC * 4];
      emit_quad<IN, KIND, L>(v, r32, r, exact_r, o);
#pragma unroll
      for (int i = 0; i < G::OUT_VEC; ++i)
        store_out_vec(a, row, q * G::OUT_VEC + i, make_uint4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]));
    }
    for (int i = nquads * G::OUT_VEC + lane; i < out_vecs; i += 32)
      store_out_vec(a, row, i, make_uint4(0, 0, 0, 0));  // kp padding
  }
}

// ---------------------------------------------------------------------------
// Row-resident path (the default where it applies): one CTA per token row,
// every thread loads its QPT quads (4L source elements each) into registers
// in one shot — the row is read from HBM exactly once and every load is in
// flight before the first use — then a block-wide |x|max (warp shuffles + one
// smem hop), then each quad is quantized from registers and its lifted
// windows stored as 16-byte vectors (48 B per quad for 6:8: a warp writes
// 1.5 KB contiguous). Requirements as the warp path, plus cols / 4L <= 1024*QPT.
template <int IN, int KIND, int L, int QPT>
SLSP_DEVINL void row_load(const ActArgs& a, int64_t row, int nquads, uint4 (&v)[QPT][WarpGeom<IN, KIND, L>::IN_VEC]) {
  using G = WarpGeom<IN, KIND, L>;
  const uint4* src = reinterpret_cast<const uint4*>(a.x + row * a.cols * G::ESZ);
#pragma unroll
  for (int j = 0; j < QPT; ++j) {
    const int q = threadIdx.x + j * blockDim.x;
#pragma unroll
    for (int i = 0; i < G::IN_VEC; ++i)
      v[j][i] = (row < a.rows && q < nquads) ? __ldg(src + q * G::IN_VEC + i) : make_uint4(0, 0, 0, 0);
  }
}

template <int IN, int KIND, int L, int QPT>
SLSP_DEVINL void row_emit(const ActArgs& a, int64_t row, int nquads, float* s_max,
                          const uint4 (&v)[QPT][WarpGeom<IN, KIND, L>::IN_VEC]) {
  using G = WarpGeom<IN, KIND, L>;
  const int tid = threadIdx.x;
  const int nthr = blockDim.x;
  double r = 0.0;
  float r32 = 0.f;
  bool exact_r = false;
  if constexpr (KIND != K_NONE) {
    float amax;
    if (a.amax_in) {
      // |x|max from upstream: no block reduction, every warp runs on
      amax = a.amax_in[row];
    } else {
    if constexpr (IN == IN_BF16) {
      // packed bf16x2 |x| max; NaN propagates and Inf wins, so the row is
      // non-finite iff the final max is (zero-filled tail slots are neutral)
      __nv_bfloat162 m2 = __float2bfloat162_rn(0.f);
#pragma unroll
      for (int j = 0; j < QPT; ++j) {
        const uint32_t* w = reinterpret_cast<const uint32_t*>(v[j]);
#pragma unroll
        for (int e = 0; e < G::IN_VEC * 4; ++e)
          m2 = __hmax2_nan(m2, __habs2(*reinterpret_cast<const __nv_bfloat162*>(&w[e])));
      }
      const float lo = __low2float(m2), hi = __high2float(m2);
      amax = (isnan(lo) || isnan(hi)) ? __int_as_float(0x7fc00000) : fmaxf(lo, hi);
    } else {
      amax = 0.f;
      bool bad = false;
#pragma unroll
      for (int j = 0; j < QPT; ++j)
#pragma unroll
        for (int e = 0; e < G::ELEMS; ++e) {
          const float f = elem<IN>(v[j], e);
          bad |= isnan(f);
          amax = fmaxf(amax, fabsf(f));
        }
      if (bad) amax = __int_as_float(0x7fc00000);
    }
    // block max with NaN propagation (fmaxf would drop NaN)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float t = __shfl_xor_sync(0xffffffffu, amax, o);
      amax = (isnan(t) || t > amax) ? t : amax;
    }
    if ((tid & 31) == 0) s_max[tid >> 5] = amax;
    __syncthreads();
    amax = s_max[0];
    for (int w = 1; w < (nthr >> 5); ++w) {
      const float t = s_max[w];
      amax = (isnan(t) || t > amax) ? t : amax;
    }
    __syncthreads();  // s_max is reused by the next row
    }
    if (!isfinite(amax) && tid == 0 && a.status) atomicMin(a.status, static_cast<unsigned long long>(row) << 32);
    // quantize.hpp:151-153, in double
    const double qmax = KIND == K_INT8 ? 127.0 : 448.0;
    const double absmax = static_cast<double>(amax);
    r = absmax == 0.0 ? 0.0 : qmax / absmax;
    r32 = __double2float_rn(r);
    // r exactly representable with <= 16 significant bits (e.g. absmax a power
    // of two): every bf16 x times r32 is exact in fp32, ties included
    exact_r = IN == IN_BF16 && KIND == K_INT8 && r32 != 0.f &&
              fmaf(r32, static_cast<float>(absmax), -127.0f) == 0.f && (__float_as_uint(r32) & 0xFFu) == 0u;
    if (tid == 0) a.scales[row] = absmax == 0.0 ? 1.0f : __double2float_rn(absmax / qmax);
  }
#pragma unroll
  for (int j = 0; j < QPT; ++j) {
    const int q = tid + j * nthr;
    if (q >= nquads) break;
    uint32_t o[G::OUT_VEC * 4];
    emit_quad<IN, KIND, L>(v[j], r32, r, exact_r, o);
#pragma unroll
    for (int i = 0; i < G::OUT_VEC; ++i)
      store_out_vec(a, row, q * G::OUT_VEC + i, make_uint4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]));
  }
  const int out_vecs = static_cast<int>(a.out_bytes >> 4);
  for (int i = nquads * G::OUT_VEC + tid; i < out_vecs; i += nthr)
    store_out_vec(a, row, i, make_uint4(0, 0, 0, 0));  // kp padding
}

// MAXT/MINB: launch bounds; the <=128-thread instantiation asks for 16
// resident CTAs (<= 32 registers) so more rows are in flight per SM.
template <int IN, int KIND, int L, int QPT, int MAXT = 1024, int MINB = 1>
__global__ void __launch_bounds__(MAXT, MINB) act_row1_kernel(ActArgs a) {  // one row per CTA, grid = rows
  using G = WarpGeom<IN, KIND, L>;
  __shared__ float s_max[32];
  const int nquads = static_cast<int>(a.cols / G::ELEMS);
  uint4 v[QPT][G::IN_VEC];
  pdl_wait();  // the activations may come from the previous kernel (PDL launch)
  pdl_trigger();
  row_load<IN, KIND, L, QPT>(a, blockIdx.x, nquads, v);
  row_emit<IN, KIND, L, QPT>(a, blockIdx.x, nquads, s_max, v);
}

template <int IN, int KIND, int L, int QPT>
int launch_row_q(ActArgs& a, int threads, cudaStream_t s) {
  if (a.rows >= (int64_t{1} << 31)) return SLSP_ERR_UNSUPPORTED;
  if (threads <= 128 && env_row_path() != 2)
    return slsp_host::launch_pdl(a.rows, act_row1_kernel<IN, KIND, L, QPT, 128, 16>, dim3(static_cast<unsigned>(a.rows)),
                                 dim3(threads), 0, s, a);
  return slsp_host::launch_pdl(a.rows, act_row1_kernel<IN, KIND, L, QPT>, dim3(static_cast<unsigned>(a.rows)), dim3(threads),
                               0, s, a);
}

// Row-resident launch when the row fits (<= 4 quads per thread, <= 1024
// threads); returns 0 when the caller should use the warp path.
template <int IN, int KIND, int L>
int launch_row(ActArgs& a, cudaStream_t s, int* st) {
  // BF16 input, 6:8 lift or quantize_rows (the hot path); the rest use the warp path
  if constexpr (IN != IN_BF16 || (L != 8 && L != 4)) return 0;
  using G = WarpGeom<IN, KIND, L>;
  const int64_t nquads = a.cols / G::ELEMS;
  // >= 64 input bytes per thread in flight (a quad is 4L elements), <= 1024 threads
  constexpr int QMIN = G::IN_VEC >= 4 ? 1 : 4 / G::IN_VEC;
  // (measured on the Qwen/Llama K values: 1 quad per thread up to 256 quads,
  // then 2 up to 1024, then 4)
  int qpt = nquads <= 256 ? 1 : nquads <= 1024 ? 2 : nquads <= 4096 ? 4 : 0;
  if (const int f = static_cast<int>(slsp_host::knob("SLSP_LIFT_QPT", 0))) {  // perf probing
    if ((f == 1 || f == 2 || f == 4) && qpt) qpt = f;
  }
  if (qpt && qpt < QMIN) qpt = QMIN;
  if (qpt && nquads > 1024 * qpt) qpt = 0;
  if (!qpt || nquads == 0) return 0;
  const int threads = static_cast<int>(((nquads + qpt - 1) / qpt + 31) / 32 * 32);
  *st = qpt == 1 ? launch_row_q<IN, KIND, L, 1>(a, threads, s)
        : qpt == 2 ? launch_row_q<IN, KIND, L, 2>(a, threads, s)
                   : launch_row_q<IN, KIND, L, 4>(a, threads, s);
  return 1;
}

template <int IN, int KIND, int L>
int launch_warp(ActArgs& a, cudaStream_t s) {
  static slsp_host::PerDevice<int> grid_caps;
  auto k = act_warp_kernel<IN, KIND, L>;
  int grid_cap = 0;
  int st = grid_caps.get(&grid_cap, [&](int& v) -> int {
    int per_sm = 0;
    SLSP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 256, 0));
    v = slsp_host::num_sms() * (per_sm > 0 ? per_sm : 1);
    return v > 0 ? SLSP_OK : SLSP_ERR_CUDA;
  });
  if (st) return st;
  const int64_t blocks = (a.rows + 7) / 8;
  k<<<static_cast<unsigned>(blocks < grid_cap ? blocks : grid_cap), 256, 0, s>>>(a);
  SLSP_LAUNCH_CHECK();
  return SLSP_OK;
}

// Returns 1 and launches when the warp fast path applies, 0 to fall back.
template <int IN, int KIND>
int try_warp_path(ActArgs& a, cudaStream_t s, int* st) {
  const int esz = IN == IN_F32 ? 4 : 2;
  const int oesz = KIND == K_NONE ? esz : 1;
  if (a.rows == 0) return 0;
  if ((reinterpret_cast<uintptr_t>(a.x) & 15u) || (reinterpret_cast<uintptr_t>(a.out) & 15u)) return 0;
  if (a.cols % (4 * a.l) != 0 || (a.cols * esz) % 16 != 0 || a.out_bytes % 16 != 0) return 0;
  if (a.words_real * 4 * oesz > a.out_bytes) return 0;
  const bool row = env_row_path() != 0;
  switch (a.l) {
    case 6: return (row && launch_row<IN, KIND, 6>(a, s, st)) || (*st = launch_warp<IN, KIND, 6>(a, s), 1);
    case 8: return (row && launch_row<IN, KIND, 8>(a, s, st)) || (*st = launch_warp<IN, KIND, 8>(a, s), 1);
    case 10: return (row && launch_row<IN, KIND, 10>(a, s, st)) || (*st = launch_warp<IN, KIND, 10>(a, s), 1);
    case 16: return (row && launch_row<IN, KIND, 16>(a, s, st)) || (*st = launch_warp<IN, KIND, 16>(a, s), 1);
    default: return 0;
  }
}

// quantize_rows on the warp path: the 2:4 "identity" geometry (L = 4, one
// window per block at offset 0) maps every source byte to itself.
template <int IN, int KIND>
int try_warp_identity(ActArgs& a, cudaStream_t s, int* st) {
  const int esz = IN == IN_F32 ? 4 : 2;
  if (a.rows == 0) return 0;
  if ((reinterpret_cast<uintptr_t>(a.x) & 15u) || (reinterpret_cast<uintptr_t>(a.out) & 15u)) return 0;
  if (a.cols % 16 != 0 || (a.cols * esz) % 16 != 0 || a.out_bytes % 16 != 0) return 0;
  if (env_row_path() && launch_row<IN, KIND, 4>(a, s, st)) return 1;
  *st = launch_warp<IN, KIND, 4>(a, s);
  return 1;
}

template <int IN, int KIND, bool LIFT>
int launch_act(ActArgs& a, int esz, cudaStream_t s) {
  {
    int st = SLSP_OK;
    if constexpr (LIFT) {
      if (try_warp_path<IN, KIND>(a, s, &st)) return st;
    } else if constexpr (KIND != K_NONE) {
      if (try_warp_identity<IN, KIND>(a, s, &st)) return st;
    }
  }
  if (a.rows == 0) return SLSP_OK;
  const size_t smem = ((a.in_cols_pad * esz + 15) & ~static_cast<int64_t>(15)) + (KIND != K_NONE ? a.in_cols_pad : 0);
  if (smem > 200 * 1024) return SLSP_ERR_UNSUPPORTED;
  auto k = act_kernel<IN, KIND, LIFT>;
  // Launch configuration is cached per device, kernel instance and smem size
  // so the entry point stays cheap and CUDA-graph capturable (no per-call
  // queries on the common path).
  struct Occ {
    size_t smem;
    int per_sm;
  };
  static slsp_host::PerDevice<Occ> occ_cache;
  Occ occ{};
  int st = occ_cache.get(&occ, [&](Occ& v) -> int {
    SLSP_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    v.smem = 0;
    return SLSP_OK;
  });
  if (st) return st;
  int per_sm = occ.per_sm;
  if (occ.smem != smem) {  // rare (the row length changed): query and refresh this device's entry
    SLSP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kThreads, smem));
    int dev = 0;
    SLSP_CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(occ_cache.mu);
    occ_cache.val[dev] = Occ{smem, per_sm};
  }
  const int64_t cap = static_cast<int64_t>(slsp_host::num_sms()) * (per_sm > 0 ? per_sm : 1);
  const unsigned grid = static_cast<unsigned>(a.rows < cap ? a.rows : cap);
  k<<<grid, kThreads, smem, s>>>(a);
  SLSP_LAUNCH_CHECK();
  return SLSP_OK;
}

// Double-precision rows (the drop-in's quantize_row<double> /
// fused_quant_slide<double>): quantize.hpp:52-68 / :122-174 with T = double —
// |x|max in double, r = qmax/absmax and codes = quantize_value(x*r) in double,
// exactly the reference's arithmetic. One CTA per row, the row read from
// global (L1/L2) in each pass; not a hot path.
template <int KIND, bool LIFT>
__global__ void __launch_bounds__(256) act_f64_kernel(ActArgs a) {
  __shared__ double s_max[8];
  __shared__ int s_bad[8];
  const int tid = threadIdx.x;
  for (int64_t row = blockIdx.x; row < a.rows; row += gridDim.x) {
    const double* x = reinterpret_cast<const double*>(a.x) + row * a.cols;
    double amax = 0.0;
    int bad = 0;
    for (int64_t k = tid; k < a.cols; k += 256) {
      const double d = x[k];
      bad |= !isfinite(d);
      amax = fmax(amax, fabs(d));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if ((tid & 31) == 0) {
      s_max[tid >> 5] = amax;
      s_bad[tid >> 5] = bad;
    }
    __syncthreads();
    amax = 0.0;
    bad = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      amax = fmax(amax, s_max[w]);
      bad |= s_bad[w];
    }
    __syncthreads();  // s_max / s_bad reused by the next row
    if (bad && tid == 0 && a.status) atomicMin(a.status, static_cast<unsigned long long>(row) << 32);
    const double qmax = KIND == K_INT8 ? 127.0 : 448.0;
    const double r = amax == 0.0 ? 0.0 : qmax / amax;
    if (tid == 0) a.scales[row] = amax == 0.0 ? 1.0f : __double2float_rn(amax / qmax);
    uint8_t* dst = a.out + row * a.out_ld;
    if constexpr (LIFT) {
      for (int64_t j = tid; j < a.out_bytes / 4; j += 256) {  // word j = window j (quantize.hpp:155-166)
        uint32_t word = 0;
        if (j < a.words_real) {
          const int64_t g = j / a.wc;
          const int64_t b = g * a.l + 2 * (j - g * a.wc);
#pragma unroll
          for (int d = 0; d < 4; ++d) {
            const int64_t k = b + d;
            const double v = k < a.cols ? x[k] : 0.0;
            word |= static_cast<uint32_t>(quantize_value(v * r, KIND)) << (8 * d);
          }
        }
        reinterpret_cast<uint32_t*>(dst)[j] = word;
      }
    } else {
      for (int64_t k = tid; k < a.out_bytes; k += 256)
        dst[k] = k < a.cols ? static_cast<uint8_t>(quantize_value(x[k] * r, KIND)) : 0;
    }
  }
}

template <bool LIFT>
int dispatch_quant(int in_dtype, int kind, ActArgs& a, cudaStream_t s) {
  if (in_dtype == SLSP_DT_F64) {
    if (a.rows == 0) return SLSP_OK;
    const unsigned grid = static_cast<unsigned>(a.rows < 148 * 16 ? a.rows : 148 * 16);
    if (kind == SLSP_QUANT_INT8) act_f64_kernel<K_INT8, LIFT><<<grid, 256, 0, s>>>(a);
    else act_f64_kernel<K_FP8, LIFT><<<grid, 256, 0, s>>>(a);
    SLSP_LAUNCH_CHECK();
    return SLSP_OK;
  }
  const int esz = in_dtype == SLSP_DT_F32 ? 4 : 2;
  if (in_dtype == SLSP_DT_F32) {
    return kind == SLSP_QUANT_INT8 ? launch_act<IN_F32, K_INT8, LIFT>(a, esz, s)
                                   : launch_act<IN_F32, K_FP8, LIFT>(a, esz, s);
  }
  return kind == SLSP_QUANT_INT8 ? launch_act<IN_BF16, K_INT8, LIFT>(a, esz, s)
                                 : launch_act<IN_BF16, K_FP8, LIFT>(a, esz, s);
}

// Per-row |x|max (NaN propagates): the partial |x|max of a rank's K-slice in
// the sharded lift (all-reduced with MAX across ranks, then fed to
// slsp_fused_quant_slide_scaled_multi). One warp per row, 16-byte loads
// where the row is aligned.
template <int IN>
__global__ void __launch_bounds__(256) row_absmax_kernel(const uint8_t* x, int64_t rows, int64_t cols, float* out) {
  constexpr int ESZ = IN == IN_F32 ? 4 : 2;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t row = w0; row < rows; row += nw) {
    const uint8_t* src = x + row * cols * ESZ;
    float m = 0.f;
    bool nan = false;
    int64_t done = 0;
    if ((reinterpret_cast<uintptr_t>(src) & 15u) == 0) {
      const int64_t nvec = cols * ESZ / 16;
      for (int64_t i = lane; i < nvec; i += 32) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(src) + i);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if constexpr (IN == IN_F32) {
            const float f = __uint_as_float(w[j]);
            nan |= isnan(f);
            m = fmaxf(m, fabsf(f));
          } else {
            const float f0 = __uint_as_float(w[j] << 16), f1 = __uint_as_float(w[j] & 0xFFFF0000u);
            nan |= isnan(f0) | isnan(f1);
            m = fmaxf(m, fmaxf(fabsf(f0), fabsf(f1)));
          }
        }
      }
      done = nvec * 16 / ESZ;
    }
    for (int64_t i = done + lane; i < cols; i += 32) {
      const float f = in_value<IN>(src, i);
      nan |= isnan(f);
      m = fmaxf(m, fabsf(f));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      nan |= __shfl_xor_sync(0xffffffffu, nan ? 1 : 0, o) != 0;
    }
    if (lane == 0) out[row] = nan ? __int_as_float(0x7fc00000) : m;
  }
}

// Status word: the caller's scratch when checking, else none (kernels skip
// the report; the hot path stays asynchronous and graph-capturable).
struct StatusScope {
  unsigned long long* ptr = nullptr;
  int init(void* ws, cudaStream_t st) {
    if (!ws) return SLSP_OK;
    ptr = static_cast<unsigned long long*>(ws);
    return slsp_host::status_reset(ws, st);
  }
};

}  // namespace

extern "C" {

int slsp_fused_quant_slide(int in_dtype, const void* x, int64_t rows, int64_t cols, int z, int l, int kind,
                           int64_t kp, uint32_t* payload, float* scales, void* status_ws, int64_t* bad_row,
                           slsp_stream_t stream) {
  using namespace slsp_host;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int wc = 0;
  int st = plan(z, l, &wc);  // pattern.hpp plan; hw_n == 4 by construction (quantize.hpp:125)
  if (st) return st;
  if ((in_dtype != SLSP_DT_F32 && in_dtype != SLSP_DT_BF16 && in_dtype != SLSP_DT_F64) || (kind != 0 && kind != 1))
    return SLSP_ERR_INVALID;
  if (rows < 0 || cols < 0) return SLSP_ERR_INVALID;
  const int64_t groups = (cols + l - 1) / l;
  const int64_t words = groups * wc;
  if (kp < words * 4 || kp % 16 != 0) return SLSP_ERR_DIMENSION;
  if ((st = require_sm100())) return st;
  StatusScope ss;
  if ((st = ss.init(status_ws, s))) return st;
  ActArgs a{};
  a.x = static_cast<const uint8_t*>(x);
  a.rows = rows;
  a.cols = cols;
  a.l = l;
  a.wc = wc;
  a.kind = kind;
  a.in_cols_pad = groups * l;
  a.words_real = words;
  a.out_bytes = kp;
  a.out_ld = kp;
  a.out = reinterpret_cast<uint8_t*>(payload);
  a.scales = scales;
  a.status = ss.ptr;
  if ((st = dispatch_quant<true>(in_dtype, kind, a, s))) return st;
  return status_collect(status_ws, s, SLSP_ERR_NON_FINITE, bad_row, nullptr);
}

int slsp_fused_quant_slide_scaled(int in_dtype, const void* x, int64_t rows, int64_t cols, int z, int l, int kind,
                                  int64_t kp, const float* tok_amax, uint32_t* payload, float* scales, void* status_ws,
                                  int64_t* bad_row, slsp_stream_t stream) {
  using namespace slsp_host;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int wc = 0;
  int st = plan(z, l, &wc);
  if (st) return st;
  if ((in_dtype != SLSP_DT_F32 && in_dtype != SLSP_DT_BF16) || (kind != 0 && kind != 1)) return SLSP_ERR_INVALID;
  if (rows < 0 || cols < 0 || (rows > 0 && !tok_amax)) return SLSP_ERR_INVALID;
  const int64_t groups = (cols + l - 1) / l;
  const int64_t words = groups * wc;
  if (kp < words * 4 || kp % 16 != 0) return SLSP_ERR_DIMENSION;
  if ((st = require_sm100())) return st;
  StatusScope ss;
  if ((st = ss.init(status_ws, s))) return st;
  ActArgs a{};
  a.x = static_cast<const uint8_t*>(x);
  a.rows = rows;
  a.cols = cols;
  a.l = l;
  a.wc = wc;
  a.kind = kind;
  a.in_cols_pad = groups * l;
  a.words_real = words;
  a.out_bytes = kp;
  a.out_ld = kp;
  a.out = reinterpret_cast<uint8_t*>(payload);
  a.scales = scales;
  a.status = ss.ptr;
  a.amax_in = tok_amax;
  if ((st = dispatch_quant<true>(in_dtype, kind, a, s))) return st;
  return status_collect(status_ws, s, SLSP_ERR_NON_FINITE, bad_row, nullptr);
}

int slsp_fused_quant_slide_scaled_multi(int in_dtype, const void* x, int64_t rows, int64_t cols, int z, int l,
                                        int kind, const float* tok_amax, void* const* dsts, int ndst, int64_t dst_ld,
                                        int64_t dst_col, float* scales, void* status_ws, int64_t* bad_row,
                                        slsp_stream_t stream) {
  using namespace slsp_host;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int wc = 0;
  int st = plan(z, l, &wc);
  if (st) return st;
  if ((in_dtype != SLSP_DT_F32 && in_dtype != SLSP_DT_BF16) || (kind != 0 && kind != 1)) return SLSP_ERR_INVALID;
  if (rows < 0 || cols < 0 || ndst < 1 || ndst > 8 || !dsts || (rows > 0 && !tok_amax)) return SLSP_ERR_INVALID;
  const int esz = in_dtype == SLSP_DT_F32 ? 4 : 2;
  // the slice is whole quads (4 blocks) so every rank's windows are its own
  // and its lifted bytes are whole 16-byte vectors at a 16-byte column
  if (cols % (4 * l) != 0 || (cols * esz) % 16 != 0) return SLSP_ERR_DIMENSION;
  const int64_t bytes = cols / l * wc * 4;
  if (dst_col < 0 || dst_col % 16 != 0 || dst_ld % 16 != 0 || dst_col + bytes > dst_ld) return SLSP_ERR_DIMENSION;
  for (int d = 0; d < ndst; ++d)
    if (!dsts[d] || (reinterpret_cast<uintptr_t>(dsts[d]) & 15u)) return SLSP_ERR_INVALID;
  if ((st = require_sm100())) return st;
  StatusScope ss;
  if ((st = ss.init(status_ws, s))) return st;
  ActArgs a{};
  a.x = static_cast<const uint8_t*>(x);
  a.rows = rows;
  a.cols = cols;
  a.l = l;
  a.wc = wc;
  a.kind = kind;
  a.in_cols_pad = cols;
  a.words_real = cols / l * wc;
  a.out_bytes = bytes;
  a.out_ld = dst_ld;
  a.out = static_cast<uint8_t*>(dsts[0]) + dst_col;
  a.ndst = ndst - 1;
  for (int d = 1; d < ndst; ++d) a.dst[d - 1] = static_cast<uint8_t*>(dsts[d]) + dst_col;
  a.scales = scales;
  a.status = ss.ptr;
  a.amax_in = tok_amax;
  if (rows > 0) {
    int launched = 0;
    st = SLSP_OK;
    if (in_dtype == SLSP_DT_BF16)
      launched = kind == SLSP_QUANT_INT8 ? try_warp_path<IN_BF16, K_INT8>(a, s, &st)
                                         : try_warp_path<IN_BF16, K_FP8>(a, s, &st);
    else
      launched = kind == SLSP_QUANT_INT8 ? try_warp_path<IN_F32, K_INT8>(a, s, &st)
                                         : try_warp_path<IN_F32, K_FP8>(a, s, &st);
    if (!launched) return SLSP_ERR_UNSUPPORTED;  // (no smem-path fallback for sliced writes)
    if (st) return st;
  }
  return status_collect(status_ws, s, SLSP_ERR_NON_FINITE, bad_row, nullptr);
}

int slsp_row_absmax(int in_dtype, const void* x, int64_t rows, int64_t cols, float* amax, slsp_stream_t stream) {
  using namespace slsp_host;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if ((in_dtype != SLSP_DT_F32 && in_dtype != SLSP_DT_BF16) || rows < 0 || cols < 0) return SLSP_ERR_INVALID;
  int st;
  if ((st = require_sm100())) return st;
  if (rows == 0) return SLSP_OK;
  const int64_t blocks = (rows + 7) / 8;
  const unsigned grid = static_cast<unsigned>(blocks < 65535 * 32 ? blocks : 65535 * 32);
  if (in_dtype == SLSP_DT_BF16) row_absmax_kernel<IN_BF16><<<grid, 256, 0, s>>>(static_cast<const uint8_t*>(x), rows, cols, amax);
  else row_absmax_kernel<IN_F32><<<grid, 256, 0, s>>>(static_cast<const uint8_t*>(x), rows, cols, amax);
  SLSP_LAUNCH_CHECK();
  return SLSP_OK;
}

int slsp_quantize_rows(int in_dtype, const void* x, int64_t rows, int64_t cols, int kind, int64_t kpad, uint8_t* out,
                       float* scales, void* status_ws, int64_t* bad_row, slsp_stream_t stream) {
  using namespace slsp_host;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if ((in_dtype != SLSP_DT_F32 && in_dtype != SLSP_DT_BF16 && in_dtype != SLSP_DT_F64) || (kind != 0 && kind != 1))
    return SLSP_ERR_INVALID;
  if (rows < 0 || cols < 0) return SLSP_ERR_INVALID;
  if (kpad < cols || kpad % 16 != 0) return SLSP_ERR_DIMENSION;
  int st;
  if ((st = require_sm100())) return st;
  StatusScope ss;
  if ((st = ss.init(status_ws, s))) return st;
  ActArgs a{};
  a.x = static_cast<const uint8_t*>(x);
  a.rows = rows;
  a.cols = cols;
  a.l = 1;
  a.wc = 1;
  a.kind = kind;
  a.in_cols_pad = cols;
  a.words_real = 0;
  a.out_bytes = kpad;
  a.out_ld = kpad;
  a.out = out;
  a.scales = scales;
  a.status = ss.ptr;
  if ((st = dispatch_quant<false>(in_dtype, kind, a, s))) return st;
  return status_collect(status_ws, s, SLSP_ERR_NON_FINITE, bad_row, nullptr);
}

int slsp_lift_rows(int dtype, const void* x, int64_t rows, int64_t cols, int z, int l, int64_t kp, void* out,
                   slsp_stream_t stream) {
  using namespace slsp_host;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int wc = 0;
  int st = plan(z, l, &wc);
  if (st) return st;
  if (dtype != SLSP_DT_BF16 && dtype != SLSP_DT_F32) return SLSP_ERR_UNSUPPORTED;
  if (rows < 0 || cols < 0) return SLSP_ERR_INVALID;
  if (cols % l != 0) return SLSP_ERR_DIMENSION;  // quantize.hpp:78-81
  const int esz = elem_size(dtype);
  const int64_t words = cols / l * wc;
  if (kp < words * 4 || (kp * esz) % 16 != 0) return SLSP_ERR_DIMENSION;
  if ((st = require_sm100())) return st;
  StatusScope ss;
  if ((st = ss.init(nullptr, s))) return st;
  ActArgs a{};
  a.x = static_cast<const uint8_t*>(x);
  a.rows = rows;
  a.cols = cols;
  a.l = l;
  a.wc = wc;
  a.in_cols_pad = cols;
  a.words_real = words;
  a.out_bytes = kp * esz;
  a.out_ld = kp * esz;
  a.out = static_cast<uint8_t*>(out);
  a.status = ss.ptr;
  return dtype == SLSP_DT_BF16 ? launch_act<IN_BF16, K_NONE, true>(a, esz, s)
                               : launch_act<IN_F32, K_NONE, true>(a, esz, s);
}

}  // extern "C"
