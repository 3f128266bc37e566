// C bridge over the UNMODIFIED reference headers — TEST INFRASTRUCTURE ONLY.
//
// Compiled by oracle/Makefile straight from /root/reference/proj/include (with
// the local boost::rational stand-in in oracle/shim/) into
// oracle/_ref/libslsp_ref.so. It exposes the reference's own pack_matrix,
// compress, fused_quant_slide, quantize_row, lift_row, sparse_gemm,
// dense_gemm, magnitude_prune and the fp8 codec behind the ref_* C
// interface of oracle/slsp_oracle.h, so tests can (a) pin the plain-C
// restatement in oracle/slsp_oracle.c and (b) generate tests/golden/ fixtures,
// and bench.py --impl reference can time the reference's own CPU path.
// No reference source is copied into this repository.
#include "slsp/container.hpp"
#include "slsp/fp8.hpp"
#include "slsp/gemm.hpp"
#include "slsp/pack.hpp"
#include "slsp/pattern.hpp"
#include "slsp/quantize.hpp"

#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "slsp_oracle.h"

using namespace slsp;

namespace {

// bf16 / e4m3 weight elements. The reference is templated on the element type
// and only needs T{}, copy and operator!= (matrix.hpp:63-67); these wrappers
// give both types "compare by decoded value" semantics, so -0 is zero.
struct Bf16 {
  std::uint16_t bits = 0;
  float value() const {
    std::uint32_t u = static_cast<std::uint32_t>(bits) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
  }
  explicit operator double() const { return value(); }
  friend bool operator!=(const Bf16& a, const Bf16& b) { return a.value() != b.value(); }
  friend bool operator==(const Bf16& a, const Bf16& b) { return a.value() == b.value(); }
};
struct E4m3 {
  std::uint8_t code = 0;
  explicit operator double() const { return fp8_e4m3_decode(code); }
  friend bool operator!=(const E4m3& a, const E4m3& b) {
    return fp8_e4m3_decode(a.code) != fp8_e4m3_decode(b.code);
  }
  friend bool operator==(const E4m3& a, const E4m3& b) { return !(a != b); }
};

enum { ST_OK = 0, ST_NOT_COMPLIANT = 1, ST_DIM = 2, ST_PLAN = 3, ST_NONFINITE = 4,
       ST_INVALID = 5, ST_MALFORMED = 6, ST_UNSUPPORTED = 7 };

// Maps the reference's exception hierarchy (pattern.hpp:24-57) to a status.
template <typename Fn>
int guarded(Fn&& fn, std::string* msg = nullptr) {
  try {
    fn();
    return ST_OK;
  } catch (const NotCompliantError& e) {
    if (msg) *msg = e.what();
    return ST_NOT_COMPLIANT;
  } catch (const DimensionMismatchError& e) {
    if (msg) *msg = e.what();
    return ST_DIM;
  } catch (const AlreadyCompliantError&) {
    return ST_PLAN;
  } catch (const NonIntegralWindowCountError&) {
    return ST_PLAN;
  } catch (const InsufficientCapacityError&) {
    return ST_PLAN;
  } catch (const NonFiniteInputError& e) {
    if (msg) *msg = e.what();
    return ST_NONFINITE;
  } catch (const MalformedMetadataError&) {
    return ST_MALFORMED;
  } catch (const std::invalid_argument&) {
    return ST_INVALID;
  } catch (const std::overflow_error&) {
    return ST_INVALID;
  }
}

template <typename T>
Matrix<T> load(const void* p, std::int64_t rows, std::int64_t cols) {
  Matrix<T> m(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols));
  std::memcpy(m.data.data(), p, sizeof(T) * m.data.size());
  return m;
}

template <typename T>
int pack_t(const void* w, std::int64_t rows, std::int64_t cols, int z, int l, void* out,
           std::int64_t* err_row, std::int64_t* err_block, int threads) {
  std::string msg;
  int st = guarded(
      [&] {
        const auto s = pack_matrix(load<T>(w, rows, cols), SparsityPattern(z, l), threads);
        std::memcpy(out, s.data.data(), sizeof(T) * s.data.size());
      },
      &msg);
  if (st == ST_NOT_COMPLIANT) {  // "row R, block B violates pattern" (pack.hpp:198-200)
    long long r = -1, b = -1;
    std::sscanf(msg.c_str(), "row %lld, block %lld", &r, &b);
    if (err_row) *err_row = r;
    if (err_block) *err_block = b;
  }
  return st;
}

template <typename T>
int compress_t(const void* slided, std::int64_t rows, std::int64_t cols_exp, void* values,
               std::uint8_t* codes, std::int64_t* err_row, std::int64_t* err_window) {
  std::string msg;
  int st = guarded(
      [&] {
        SlidedMatrix<T> s;
        s.rows = static_cast<std::size_t>(rows);
        s.cols_expanded = static_cast<std::size_t>(cols_exp);
        s.pattern = SparsityPattern(2, 4);
        s.data.resize(s.rows * s.cols_expanded);
        std::memcpy(s.data.data(), slided, sizeof(T) * s.data.size());
        const auto c = compress(s);
        std::memcpy(values, c.values.data(), sizeof(T) * c.values.size());
        std::memcpy(codes, c.metadata.data(), c.metadata.size());
      },
      &msg);
  if (st == ST_NOT_COMPLIANT) {  // "window (r, w) holds more than" (gemm.hpp:96-97)
    long long r = -1, w = -1;
    std::sscanf(msg.c_str(), "window (%lld, %lld)", &r, &w);
    if (err_row) *err_row = r;
    if (err_window) *err_window = w;
  }
  return st;
}

template <typename T>
int prune_t(const void* w, std::int64_t rows, std::int64_t cols, int z, int l, void* out) {
  return guarded([&] {
    const auto p = magnitude_prune(load<T>(w, rows, cols), SparsityPattern(z, l));
    std::memcpy(out, p.data.data(), sizeof(T) * p.data.size());
  });
}

template <typename T>
int lift_t(const void* x, std::int64_t rows, std::int64_t cols, int z, int l, void* out) {
  return guarded([&] {
    const WindowPlan plan = plan_decomposition(SparsityPattern(z, l));
    const T* src = static_cast<const T*>(x);
    T* dst = static_cast<T*>(out);
    for (std::int64_t i = 0; i < rows; ++i) {
      const auto lifted = lift_row<T>(std::span<const T>(src + i * cols, cols), plan);
      std::memcpy(dst + i * lifted.size(), lifted.data(), sizeof(T) * lifted.size());
    }
  });
}

QuantKind to_kind(int kind) { return kind == 0 ? QuantKind::int8 : QuantKind::fp8e4m3; }

template <typename T>
int fqs_t(const Matrix<T>& x, int z, int l, int kind, std::uint32_t* payload, float* scales,
          std::int64_t* bad_row, int threads) {
  std::string msg;
  int st = guarded(
      [&] {
        const auto a = fused_quant_slide(x, SparsityPattern(z, l), to_kind(kind), threads);
        std::memcpy(payload, a.payload.data(), 4 * a.payload.size());
        std::memcpy(scales, a.scales.data(), 4 * a.scales.size());
      },
      &msg);
  if (st == ST_NONFINITE) {  // "non-finite activation value in row i" (quantize.hpp:170)
    const auto pos = msg.rfind("row ");
    if (bad_row && pos != std::string::npos) *bad_row = std::stoll(msg.substr(pos + 4));
  }
  return st;
}

Matrix<float> bf16_matrix(const void* x, std::int64_t rows, std::int64_t cols) {
  Matrix<float> m(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols));
  const std::uint16_t* b = static_cast<const std::uint16_t*>(x);
  for (std::size_t i = 0; i < m.data.size(); ++i) m.data[i] = Bf16{b[i]}.value();
  return m;
}

}  // namespace

extern "C" {

int ref_plan(int z, int l, int hw_m, int hw_n, int* window_count, int* starts, int cap) {
  return guarded([&] {
    const auto plan = plan_decomposition(SparsityPattern(z, l, hw_m, hw_n));
    if (plan.window_count > cap) throw std::invalid_argument("cap");
    *window_count = plan.window_count;
    for (int j = 0; j < plan.window_count; ++j) starts[j] = plan.window_starts[j];
  });
}

int ref_pack_matrix(int dtype, const void* w, std::int64_t rows, std::int64_t cols, int z, int l,
                    void* slided, std::int64_t* err_row, std::int64_t* err_block, int threads) {
  switch (dtype) {
    case 0: return pack_t<std::int8_t>(w, rows, cols, z, l, slided, err_row, err_block, threads);
    case 1: return pack_t<Bf16>(w, rows, cols, z, l, slided, err_row, err_block, threads);
    case 2: return pack_t<E4m3>(w, rows, cols, z, l, slided, err_row, err_block, threads);
    case 3: return pack_t<float>(w, rows, cols, z, l, slided, err_row, err_block, threads);
    case 4: return pack_t<double>(w, rows, cols, z, l, slided, err_row, err_block, threads);
  }
  return ST_INVALID;
}

int ref_compress(int dtype, const void* slided, std::int64_t rows, std::int64_t cols_exp,
                 void* values, std::uint8_t* codes, std::int64_t* err_row, std::int64_t* err_window) {
  switch (dtype) {
    case 0: return compress_t<std::int8_t>(slided, rows, cols_exp, values, codes, err_row, err_window);
    case 1: return compress_t<Bf16>(slided, rows, cols_exp, values, codes, err_row, err_window);
    case 2: return compress_t<E4m3>(slided, rows, cols_exp, values, codes, err_row, err_window);
    case 3: return compress_t<float>(slided, rows, cols_exp, values, codes, err_row, err_window);
    case 4: return compress_t<double>(slided, rows, cols_exp, values, codes, err_row, err_window);
  }
  return ST_INVALID;
}

int ref_fused_quant_slide(int in_dtype, const void* x, std::int64_t rows, std::int64_t cols, int z,
                          int l, int kind, std::uint32_t* payload, float* scales,
                          std::int64_t* bad_row, int threads) {
  switch (in_dtype) {
    case 1: return fqs_t(bf16_matrix(x, rows, cols), z, l, kind, payload, scales, bad_row, threads);
    case 3: return fqs_t(load<float>(x, rows, cols), z, l, kind, payload, scales, bad_row, threads);
    case 4: return fqs_t(load<double>(x, rows, cols), z, l, kind, payload, scales, bad_row, threads);
  }
  return ST_INVALID;
}

int ref_quantize_rows(int in_dtype, const void* x, std::int64_t rows, std::int64_t cols, int kind,
                      std::uint8_t* bytes, float* scales, std::int64_t* bad_row) {
  Matrix<double> m(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols));
  if (in_dtype == 1) {
    const auto f = bf16_matrix(x, rows, cols);
    for (std::size_t i = 0; i < m.data.size(); ++i) m.data[i] = f.data[i];
  } else if (in_dtype == 3) {
    const float* f = static_cast<const float*>(x);
    for (std::size_t i = 0; i < m.data.size(); ++i) m.data[i] = f[i];
  } else if (in_dtype == 4) {
    std::memcpy(m.data.data(), x, 8 * m.data.size());
  } else {
    return ST_INVALID;
  }
  std::int64_t current = 0;
  int st = guarded([&] {
    for (std::int64_t i = 0; i < rows; ++i) {
      current = i;
      const auto q = quantize_row<double>(m.row(static_cast<std::size_t>(i)), to_kind(kind));
      std::memcpy(bytes + i * cols, q.bytes.data(), q.bytes.size());
      scales[i] = q.scale;
    }
  });
  if (st == ST_NONFINITE && bad_row) *bad_row = current;
  return st;
}

int ref_lift_rows(int dtype, const void* x, std::int64_t rows, std::int64_t cols, int z, int l,
                  void* out) {
  switch (dtype) {
    case 0: case 2: return lift_t<std::uint8_t>(x, rows, cols, z, l, out);
    case 1: return lift_t<std::uint16_t>(x, rows, cols, z, l, out);
    case 3: return lift_t<float>(x, rows, cols, z, l, out);
    case 4: return lift_t<double>(x, rows, cols, z, l, out);
  }
  return ST_INVALID;
}

int ref_sparse_gemm_words(const std::int8_t* values, const std::uint8_t* codes, std::int64_t rows,
                          std::int64_t wpr, const std::uint32_t* payload, std::int64_t tokens,
                          std::int32_t* y, int threads) {
  return guarded([&] {
    const SparsityPattern p(6, 8);
    CompressedSparseMatrix<std::int8_t> c;
    c.rows = static_cast<std::size_t>(rows);
    c.windows_per_row = static_cast<std::size_t>(wpr);
    c.pattern = p;
    c.values.assign(values, values + rows * wpr * 2);
    c.metadata.assign(codes, codes + rows * wpr * 2);
    QuantizedLiftedActivation a;
    a.rows = static_cast<std::size_t>(tokens);
    a.words_per_row = static_cast<std::size_t>(wpr);
    a.pattern = p;
    a.kind = QuantKind::int8;
    a.payload.assign(payload, payload + tokens * wpr);
    a.scales.assign(static_cast<std::size_t>(tokens), 1.0f);
    const auto out = sparse_gemm(c, a, threads);
    std::memcpy(y, out.data.data(), 4 * out.data.size());
  });
}

int ref_sparse_gemm_f64(const double* values, const std::uint8_t* codes, std::int64_t rows,
                        std::int64_t wpr, const double* lifted, std::int64_t tokens, double* y,
                        int threads) {
  // Inputs are float-representable (decoded e4m3 / bf16 values times
  // float scales), so the reference's float path with double accumulation
  // (accum_type<float>, gemm.hpp:39-42) is exact in its products.
  return guarded([&] {
    CompressedSparseMatrix<float> c;
    c.rows = static_cast<std::size_t>(rows);
    c.windows_per_row = static_cast<std::size_t>(wpr);
    c.pattern = SparsityPattern(6, 8);
    c.values.assign(values, values + rows * wpr * 2);
    c.metadata.assign(codes, codes + rows * wpr * 2);
    Matrix<float> act(static_cast<std::size_t>(tokens), static_cast<std::size_t>(wpr * 4));
    for (std::size_t i = 0; i < act.data.size(); ++i) act.data[i] = static_cast<float>(lifted[i]);
    const auto out = sparse_gemm(c, act, threads);
    for (std::size_t i = 0; i < out.data.size(); ++i) y[i] = out.data[i];
  });
}

int ref_dense_gemm_i8(const std::int8_t* w, std::int64_t n, std::int64_t k, const std::int8_t* x,
                      std::int64_t m, std::int32_t* y, int threads) {
  return guarded([&] {
    const auto out = dense_gemm(load<std::int8_t>(w, n, k), load<std::int8_t>(x, k, m), threads);
    std::memcpy(y, out.data.data(), 4 * out.data.size());
  });
}

int ref_magnitude_prune(int dtype, const void* w, std::int64_t rows, std::int64_t cols, int z, int l,
                        void* out) {
  switch (dtype) {
    case 0: return prune_t<std::int8_t>(w, rows, cols, z, l, out);
    case 1: return prune_t<Bf16>(w, rows, cols, z, l, out);
    case 2: return prune_t<E4m3>(w, rows, cols, z, l, out);
    case 3: return prune_t<float>(w, rows, cols, z, l, out);
    case 4: return prune_t<double>(w, rows, cols, z, l, out);
  }
  return ST_INVALID;
}

std::uint8_t ref_fp8_encode(double x) { return fp8_e4m3_encode(x); }
float ref_fp8_decode(std::uint8_t code) { return fp8_e4m3_decode(code); }
std::uint8_t ref_quantize_value(double scaled, int kind) { return quantize_value(scaled, to_kind(kind)); }

// container.hpp:330-336 pack_codes (the on-disk 2-bit metadata stream).
void ref_pack_codes(const std::uint8_t* codes, std::int64_t count, std::uint8_t* out) {
  const auto packed = slsp::detail::pack_codes(std::vector<std::uint8_t>(codes, codes + count));
  std::memcpy(out, packed.data(), packed.size());
}

// container.hpp serialize(to_container(CompressedSparseMatrix<int8_t>)) — the
// reference's kind-2 file bytes (pinning the loader). codes
// are one 2-bit position per byte (the in-memory format); returns the byte
// count written, or -needed when cap is too small.
std::int64_t ref_serialize_compressed_i8(const std::int8_t* values, const std::uint8_t* codes, std::int64_t rows,
                                         std::int64_t windows, int z, int l, std::uint8_t* out, std::int64_t cap) {
  CompressedSparseMatrix<std::int8_t> cm;
  cm.rows = static_cast<std::size_t>(rows);
  cm.windows_per_row = static_cast<std::size_t>(windows);
  cm.pattern = SparsityPattern(z, l);
  cm.values.assign(values, values + rows * windows * 2);
  cm.metadata.assign(codes, codes + rows * windows * 2);
  const auto bytes = slsp::serialize(slsp::to_container(cm));
  if (static_cast<std::int64_t>(bytes.size()) > cap) return -static_cast<std::int64_t>(bytes.size());
  std::memcpy(out, bytes.data(), bytes.size());
  return static_cast<std::int64_t>(bytes.size());
}

// serialize(to_container(QuantizedLiftedActivation)) — a kind-3 file.
std::int64_t ref_serialize_quantized(const std::uint32_t* payload, const float* scales, std::int64_t rows,
                                     std::int64_t words, int z, int l, int kind, std::uint8_t* out, std::int64_t cap) {
  QuantizedLiftedActivation a;
  a.rows = static_cast<std::size_t>(rows);
  a.words_per_row = static_cast<std::size_t>(words);
  a.pattern = SparsityPattern(z, l);
  a.kind = to_kind(kind);
  a.payload.assign(payload, payload + rows * words);
  a.scales.assign(scales, scales + rows);
  const auto bytes = slsp::serialize(slsp::to_container(a));
  if (static_cast<std::int64_t>(bytes.size()) > cap) return -static_cast<std::int64_t>(bytes.size());
  std::memcpy(out, bytes.data(), bytes.size());
  return static_cast<std::int64_t>(bytes.size());
}

}  // extern "C"
