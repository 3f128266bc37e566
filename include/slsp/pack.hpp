#pragma once
// Drop-in slsp/pack.hpp: the weight transform Φ. pack_matrix and
// magnitude_prune run on the B200 (slsp_pack_matrix, slsp_magnitude_prune);
// verify_compliance and unslide are host utilities (reference pack.hpp:37-72,
// :209-233), not on the hot path.

#include <algorithm>
#include <cstdint>
#include <functional>
#include <optional>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "slsp/detail/device.hpp"
#include "slsp/matrix.hpp"
#include "slsp/pattern.hpp"

namespace slsp {

struct ComplianceReport {
  bool compliant = true;
  std::optional<std::pair<std::size_t, std::size_t>> first_violation;  // (row, window)
  std::vector<std::size_t> nonzero_histogram;                          // [k] = windows holding k nonzeros
};

template <typename T>
ComplianceReport verify_compliance(std::size_t rows, std::size_t cols, std::span<const T> data, int m, int n) {
  if (n <= 0 || m <= 0) throw std::invalid_argument("verify_compliance: need 0 < m, 0 < n");
  if (cols % static_cast<std::size_t>(n) != 0)
    throw DimensionMismatchError("column count " + std::to_string(cols) + " not divisible by window length " +
                                 std::to_string(n));
  if (data.size() != rows * cols) throw DimensionMismatchError("buffer size does not match shape");
  ComplianceReport rep;
  rep.nonzero_histogram.assign(static_cast<std::size_t>(n) + 1, 0);
  for (std::size_t i = 0; i < rows * (cols / n); ++i) {
    int nnz = 0;
    for (int d = 0; d < n; ++d) nnz += is_nonzero(data[i * n + d]);
    ++rep.nonzero_histogram[static_cast<std::size_t>(nnz)];
    if (nnz > m && rep.compliant) {
      rep.compliant = false;
      rep.first_violation = std::make_pair(i / (cols / n), i % (cols / n));
    }
  }
  return rep;
}
template <typename T>
ComplianceReport verify_compliance(const Matrix<T>& mx, int m, int n) {
  return verify_compliance<T>(mx.rows, mx.cols, std::span<const T>(mx.data), m, n);
}
template <typename T>
ComplianceReport verify_compliance(const SlidedMatrix<T>& mx, int m, int n) {
  return verify_compliance<T>(mx.rows, mx.cols_expanded, std::span<const T>(mx.data), m, n);
}

// pack.hpp:171-204 on the B200. Errors carry the reference's message
// ("row R, block B violates pattern Z:L"), lowest offending row first.
template <typename T>
SlidedMatrix<T> pack_matrix(const Matrix<T>& w, const SparsityPattern& pattern, int /*threads*/ = 1) {
  static_assert(detail::dtype_code<T>() >= 0, "element type not supported by the B200 packer");
  const WindowPlan plan = plan_decomposition(pattern);
  if (w.cols % static_cast<std::size_t>(pattern.l) != 0)
    throw DimensionMismatchError("matrix cols " + std::to_string(w.cols) + " not divisible by block length " +
                                 std::to_string(pattern.l));
  SlidedMatrix<T> out;
  out.rows = w.rows;
  out.cols_expanded = w.cols / pattern.l * plan.window_count * pattern.hw_n;
  out.pattern = pattern;
  if (w.rows == 0 || w.cols == 0) {
    out.data.assign(out.rows * out.cols_expanded, T{});
    return out;
  }
  detail::DeviceBuffer<T> dw(w.data);
  detail::DeviceBuffer<T> ds(out.rows * out.cols_expanded);
  detail::StatusScratch ws;
  std::int64_t er = -1, eb = -1;
  const int st = slsp_pack_matrix(detail::dtype_code<T>(), dw.get(), static_cast<std::int64_t>(w.rows),
                                  static_cast<std::int64_t>(w.cols), pattern.z, pattern.l, ds.get(), ws.get(), &er, &eb,
                                  nullptr);
  if (st == SLSP_ERR_NOT_COMPLIANT)
    throw NotCompliantError("row " + std::to_string(er) + ", block " + std::to_string(eb) + " violates pattern " +
                            pattern.label());
  detail::raise(st, "pack_matrix");
  out.data = ds.download();
  return out;
}

namespace detail {

// The reference's test-only packer hooks (pack.hpp:74-122): a per-rejection
// callback and the greedy placement with a capped window count, used to probe
// the capacity argument. Host code: the hook observes individual placement
// decisions, which the B200 packer (one thread per block, table-driven for
// 6:8) does not expose. pack_row with an observer runs this; without one it
// runs on the device like pack_matrix.
using RejectionObserver = std::function<void(std::size_t group, int window, std::size_t src_index)>;

template <typename T>
std::optional<std::size_t> greedy_pack_row(std::span<const T> src, const WindowPlan& plan, std::span<T> dst,
                                           int window_limit, const RejectionObserver* observer = nullptr) {
  const SparsityPattern& p = plan.pattern;
  const std::size_t l = static_cast<std::size_t>(p.l), n = static_cast<std::size_t>(p.hw_n);
  const std::size_t span_out = static_cast<std::size_t>(plan.window_count) * n;
  std::fill(dst.begin(), dst.end(), T{});
  std::optional<std::size_t> first_left;
  for (std::size_t g = 0; g < src.size() / l; ++g) {
    std::uint64_t taken = 0;  // bit k: source position k of this block already placed
    for (int w = 0; w < window_limit; ++w) {
      int placed = 0;
      for (std::size_t d = 0; d < n; ++d) {
        const std::size_t k = static_cast<std::size_t>(plan.window_starts[w]) + d;
        const T v = src[g * l + k];
        if (!is_nonzero(v) || ((taken >> k) & 1u)) continue;
        if (placed == p.hw_m) {  // window full: the value waits for a later window
          if (observer) (*observer)(g, w, g * l + k);
          continue;
        }
        dst[g * span_out + static_cast<std::size_t>(w) * n + d] = v;
        taken |= std::uint64_t{1} << k;
        ++placed;
      }
    }
    for (std::size_t k = 0; k < l && !first_left; ++k)
      if (is_nonzero(src[g * l + k]) && !((taken >> k) & 1u)) first_left = g * l + k;
  }
  return first_left;
}

}  // namespace detail

// pack.hpp:148-167: one row (on the device; with an observer, the host hook above).
template <typename T>
std::vector<T> pack_row(std::span<const T> src, const WindowPlan& plan,
                        const detail::RejectionObserver* observer = nullptr) {
  const auto& p = plan.pattern;
  if (src.size() % static_cast<std::size_t>(p.l) != 0)
    throw DimensionMismatchError("row length " + std::to_string(src.size()) + " not divisible by block length " +
                                 std::to_string(p.l));
  if (observer) {
    for (std::size_t g = 0; g < src.size() / p.l; ++g) {
      int nnz = 0;
      for (int k = 0; k < p.l; ++k) nnz += is_nonzero(src[g * p.l + k]) ? 1 : 0;
      if (nnz > p.z)
        throw NotCompliantError("block " + std::to_string(g) + " exceeds " + std::to_string(p.z) + " nonzeros");
    }
    std::vector<T> dst(src.size() / p.l * plan.window_count * p.hw_n);
    if (auto left = detail::greedy_pack_row<T>(src, plan, dst, plan.window_count, observer))
      throw NotCompliantError("nonzero at index " + std::to_string(*left) + " left unassigned after the last window");
    return dst;
  }
  Matrix<T> one(1, src.size(), std::vector<T>(src.begin(), src.end()));
  try {
    return pack_matrix(one, p).data;
  } catch (const NotCompliantError& e) {
    const std::string msg = e.what();
    const auto b = msg.find("block ");
    throw NotCompliantError("block " + msg.substr(b + 6, msg.find(' ', b + 6) - b - 6) + " exceeds " +
                            std::to_string(p.z) + " nonzeros");
  }
}

// pack.hpp:209-233 inverse (host).
template <typename T>
Matrix<T> unslide(const SlidedMatrix<T>& s) {
  const WindowPlan plan = plan_decomposition(s.pattern);
  const auto& p = s.pattern;
  const std::size_t out_group = static_cast<std::size_t>(plan.window_count) * p.hw_n;
  if (s.cols_expanded % out_group != 0)
    throw DimensionMismatchError("slided width inconsistent with pattern window geometry");
  const std::size_t groups = s.cols_expanded / out_group;
  Matrix<T> w(s.rows, groups * p.l);
  for (std::size_t r = 0; r < s.rows; ++r)
    for (std::size_t g = 0; g < groups; ++g)
      for (int j = 0; j < plan.window_count; ++j)
        for (int d = 0; d < p.hw_n; ++d) {
          const T v = s.data[r * s.cols_expanded + g * out_group + static_cast<std::size_t>(j) * p.hw_n + d];
          if (is_nonzero(v)) w(r, g * p.l + plan.window_starts[j] + d) = v;
        }
  return w;
}

// pack.hpp:238-261 on the B200.
template <typename T>
Matrix<T> magnitude_prune(const Matrix<T>& w, const SparsityPattern& pattern) {
  static_assert(detail::dtype_code<T>() >= 0, "element type not supported by the B200 pruner");
  if (w.cols % static_cast<std::size_t>(pattern.l) != 0)
    throw DimensionMismatchError("matrix cols " + std::to_string(w.cols) + " not divisible by block length " +
                                 std::to_string(pattern.l));
  if (w.data.empty()) return w;
  detail::DeviceBuffer<T> dw(w.data);
  detail::DeviceBuffer<T> dout(w.data.size());
  detail::raise(slsp_magnitude_prune(detail::dtype_code<T>(), dw.get(), static_cast<std::int64_t>(w.rows),
                                     static_cast<std::int64_t>(w.cols), pattern.z, pattern.l, dout.get(), nullptr),
                "magnitude_prune");
  return Matrix<T>(w.rows, w.cols, dout.download());
}

}  // namespace slsp
