#pragma once
// Drop-in slsp/quantize.hpp: per-token quantization and Activation Lifting.
// fused_quant_slide / quantize_row run on the B200 kernels through the C ABI
// (slsp_fused_quant_slide / slsp_quantize_rows); the scalar helpers are host
// inline restatements of reference quantize.hpp:26-116.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <span>
#include <string>
#include <vector>

#include "slsp/detail/device.hpp"
#include "slsp/fp8.hpp"
#include "slsp/matrix.hpp"
#include "slsp/pattern.hpp"

namespace slsp {

enum class QuantKind : std::uint8_t { int8, fp8e4m3 };

inline double quant_max(QuantKind kind) { return kind == QuantKind::int8 ? 127.0 : 448.0; }

inline std::uint8_t quantize_value(double scaled, QuantKind kind) {
  if (kind == QuantKind::int8)
    return static_cast<std::uint8_t>(static_cast<std::int8_t>(std::clamp(std::nearbyint(scaled), -127.0, 127.0)));
  return scaled == 0.0 ? std::uint8_t{0} : fp8_e4m3_encode(std::clamp(scaled, -448.0, 448.0));
}

inline double dequant_value(std::uint8_t byte, QuantKind kind) {
  return kind == QuantKind::int8 ? static_cast<double>(static_cast<std::int8_t>(byte))
                                 : static_cast<double>(fp8_e4m3_decode(byte));
}

struct QuantizedRow {
  std::vector<std::uint8_t> bytes;
  float scale = 1.0f;
};

inline std::uint32_t pack_word(std::uint8_t q0, std::uint8_t q1, std::uint8_t q2, std::uint8_t q3) {
  return std::uint32_t{q0} | (std::uint32_t{q1} << 8) | (std::uint32_t{q2} << 16) | (std::uint32_t{q3} << 24);
}
inline std::uint8_t unpack_byte(std::uint32_t word, int pos) { return static_cast<std::uint8_t>(word >> (8 * pos)); }

struct QuantizedLiftedActivation {
  std::size_t rows = 0;
  std::size_t words_per_row = 0;
  SparsityPattern pattern;
  QuantKind kind = QuantKind::int8;
  std::vector<std::uint32_t> payload;
  std::vector<float> scales;

  double qmax() const { return quant_max(kind); }
  std::size_t lifted_cols() const { return words_per_row * 4; }
  std::uint8_t byte_at(std::size_t row, std::size_t lifted_index) const {
    return unpack_byte(payload[row * words_per_row + lifted_index / 4], static_cast<int>(lifted_index % 4));
  }
};

namespace detail {
template <typename T>
constexpr int act_dtype() {
  static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>,
                "the B200 activation kernels take float or double (or bf16 via the C ABI)");
  return std::is_same_v<T, double> ? SLSP_DT_F64 : SLSP_DT_F32;
}
inline std::string nonfinite_message(std::int64_t row) {
  return "non-finite activation value in row " + std::to_string(row);
}
}  // namespace detail

// quantize.hpp:52-68 — one row on the device (slsp_quantize_rows).
template <typename T>
QuantizedRow quantize_row(std::span<const T> x, QuantKind kind) {
  const std::size_t n = x.size();
  const std::int64_t kpad = static_cast<std::int64_t>((n + 15) / 16 * 16);
  detail::DeviceBuffer<T> dx(std::vector<T>(x.begin(), x.end()));
  detail::DeviceBuffer<std::uint8_t> dq(static_cast<std::size_t>(kpad ? kpad : 16));
  detail::DeviceBuffer<float> ds(1);
  detail::StatusScratch ws;
  std::int64_t bad = -1;
  const int st = slsp_quantize_rows(detail::act_dtype<T>(), dx.get(), 1, static_cast<std::int64_t>(n),
                                    static_cast<int>(kind), kpad ? kpad : 16, dq.get(), ds.get(), ws.get(), &bad,
                                    nullptr);
  if (st == SLSP_ERR_NON_FINITE) throw NonFiniteInputError("non-finite activation value");
  detail::raise(st, "quantize_row");
  QuantizedRow out;
  out.bytes = dq.download(n);
  out.scale = ds.download(1)[0];
  return out;
}

// quantize.hpp:72-89 — pure index remapping (host; not on the hot path).
template <typename T>
std::vector<T> lift_row(std::span<const T> x, const WindowPlan& plan) {
  const auto& p = plan.pattern;
  if (x.size() % static_cast<std::size_t>(p.l) != 0)
    throw DimensionMismatchError("row length " + std::to_string(x.size()) + " not divisible by block length " +
                                 std::to_string(p.l));
  std::vector<T> out;
  out.reserve(x.size() / p.l * plan.window_count * p.hw_n);
  for (std::size_t g = 0; g < x.size() / p.l; ++g)
    for (const int s : plan.window_starts)
      for (int d = 0; d < p.hw_n; ++d) out.push_back(x[g * p.l + s + d]);
  return out;
}

// quantize.hpp:122-174 — the fused per-token quantize + lift on the B200.
template <typename T>
QuantizedLiftedActivation fused_quant_slide(const Matrix<T>& x, const SparsityPattern& pattern,
                                            QuantKind kind = QuantKind::int8, int /*threads*/ = 1) {
  if (pattern.hw_n != 4) throw std::invalid_argument("word packing requires hardware window length 4");
  const WindowPlan plan = plan_decomposition(pattern);
  const std::size_t groups = (x.cols + pattern.l - 1) / pattern.l;
  QuantizedLiftedActivation out;
  out.rows = x.rows;
  out.words_per_row = groups * static_cast<std::size_t>(plan.window_count);
  out.pattern = pattern;
  out.kind = kind;
  const std::int64_t kprime = static_cast<std::int64_t>(out.words_per_row * 4);
  const std::int64_t kp = (kprime + 15) / 16 * 16;
  detail::DeviceBuffer<T> dx(x.data);
  detail::DeviceBuffer<std::uint32_t> dp(std::max<std::size_t>(1, x.rows * static_cast<std::size_t>(kp / 4)));
  detail::DeviceBuffer<float> ds(std::max<std::size_t>(1, x.rows));
  detail::StatusScratch ws;
  std::int64_t bad = -1;
  const int st = slsp_fused_quant_slide(detail::act_dtype<T>(), dx.get(), static_cast<std::int64_t>(x.rows),
                                        static_cast<std::int64_t>(x.cols), pattern.z, pattern.l,
                                        static_cast<int>(kind), kp, dp.get(), ds.get(), ws.get(), &bad, nullptr);
  if (st == SLSP_ERR_NON_FINITE) throw NonFiniteInputError(detail::nonfinite_message(bad));
  detail::raise(st, "fused_quant_slide");
  const auto all = dp.download(x.rows * static_cast<std::size_t>(kp / 4));
  out.payload.resize(x.rows * out.words_per_row);
  for (std::size_t i = 0; i < x.rows; ++i)
    std::copy_n(all.begin() + static_cast<std::ptrdiff_t>(i * (kp / 4)), out.words_per_row,
                out.payload.begin() + static_cast<std::ptrdiff_t>(i * out.words_per_row));
  out.scales = ds.download(x.rows);
  return out;
}

}  // namespace slsp
