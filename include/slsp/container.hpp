#pragma once
// Drop-in slsp/container.hpp: the SLSP tensor file of reference
// container.hpp:1-19 (magic "SLSP", u16 version 1, u8 kind, u8 dtype, four
// u16 pattern fields, u64 rows, u64 cols, u64-length sections — values, then
// the 2-bit code stream for kind 2 or fp32 scales for kind 3 — and a CRC-32
// tail), with the same validation and ContainerError messages, plus the typed
// conversions. Host-side, as in the reference; the device load of a kind-2
// payload into the MMA layout is slsp_load_compressed (include/slsp_b200.h)
// or b200::upload_compressed below.

#include <array>
#include <cstdint>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <unistd.h>
#include <iterator>
#include <span>
#include <string>
#include <vector>

#include "slsp/gemm.hpp"
#include "slsp/matrix.hpp"
#include "slsp/pattern.hpp"
#include "slsp/quantize.hpp"

namespace slsp {

enum class Kind : std::uint8_t { dense = 0, slided = 1, compressed = 2, quantized_lifted = 3 };
enum class Dtype : std::uint8_t { int8 = 0, int32 = 1, fp32 = 2, fp64 = 3, fp8e4m3 = 4 };

inline std::size_t dtype_size(Dtype d) {
  switch (d) {
    case Dtype::int8:
    case Dtype::fp8e4m3: return 1;
    case Dtype::int32:
    case Dtype::fp32: return 4;
    case Dtype::fp64: return 8;
  }
  throw ContainerError("unknown dtype");
}

struct Container {
  Kind kind = Kind::dense;
  Dtype dtype = Dtype::int8;
  std::uint16_t z = 0, l = 0, hw_m = 0, hw_n = 0;
  std::uint64_t rows = 0, cols = 0;
  std::vector<std::uint8_t> values, metadata;
  std::vector<float> scales;
  SparsityPattern pattern() const {
    if (kind == Kind::dense) throw ContainerError("dense container carries no pattern");
    return SparsityPattern(z, l, hw_m, hw_n);
  }
};

namespace detail {

// CRC-32 (IEEE 802.3, reflected polynomial 0xEDB88320; zlib's crc32).
inline std::uint32_t crc32(std::span<const std::uint8_t> bytes) {
  static const std::array<std::uint32_t, 256> table = [] {
    std::array<std::uint32_t, 256> t{};
    for (std::uint32_t i = 0; i < 256; ++i) {
      std::uint32_t c = i;
      for (int b = 0; b < 8; ++b) c = (c & 1u) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      t[i] = c;
    }
    return t;
  }();
  std::uint32_t c = 0xFFFFFFFFu;
  for (const std::uint8_t v : bytes) c = table[(c ^ v) & 0xFFu] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}

template <typename U>
void put_le(std::vector<std::uint8_t>& out, U v) {
  for (std::size_t i = 0; i < sizeof(U); ++i) out.push_back(static_cast<std::uint8_t>(v >> (8 * i)));
}

// Little-endian cursor over a byte span; running past the end is truncation.
class Cursor {
 public:
  explicit Cursor(std::span<const std::uint8_t> b) : b_(b) {}
  template <typename U>
  U get() {
    need(sizeof(U));
    U v = 0;
    for (std::size_t i = 0; i < sizeof(U); ++i) v |= static_cast<U>(static_cast<U>(b_[at_ + i]) << (8 * i));
    at_ += sizeof(U);
    return v;
  }
  std::vector<std::uint8_t> section() {
    const auto n = get<std::uint64_t>();
    need(n);
    std::vector<std::uint8_t> out(b_.begin() + static_cast<std::ptrdiff_t>(at_),
                                  b_.begin() + static_cast<std::ptrdiff_t>(at_ + n));
    at_ += n;
    return out;
  }
  void skip(std::size_t n) { need(n), at_ += n; }
  std::size_t offset() const { return at_; }

 private:
  void need(std::uint64_t n) const {
    if (n > b_.size() - at_) throw ContainerError("container truncated");
  }
  std::span<const std::uint8_t> b_;
  std::size_t at_ = 0;
};

// 2-bit codes, four per byte, low bits first (the on-disk metadata stream).
inline std::vector<std::uint8_t> pack_codes(const std::vector<std::uint8_t>& codes) {
  std::vector<std::uint8_t> out((codes.size() + 3) / 4, 0);
  for (std::size_t i = 0; i < codes.size(); ++i) out[i / 4] |= static_cast<std::uint8_t>((codes[i] & 3u) << (2 * (i % 4)));
  return out;
}

inline std::vector<std::uint8_t> unpack_codes(const std::vector<std::uint8_t>& bytes, std::size_t count) {
  if (bytes.size() < (count + 3) / 4) throw ContainerError("metadata payload does not match shape");
  std::vector<std::uint8_t> out(count);
  for (std::size_t i = 0; i < count; ++i) out[i] = static_cast<std::uint8_t>((bytes[i / 4] >> (2 * (i % 4))) & 3u);
  return out;
}

template <typename T>
constexpr Dtype dtype_of() {
  if constexpr (std::is_same_v<T, std::int8_t>) return Dtype::int8;
  else if constexpr (std::is_same_v<T, std::int32_t>) return Dtype::int32;
  else if constexpr (std::is_same_v<T, float>) return Dtype::fp32;
  else if constexpr (std::is_same_v<T, double>) return Dtype::fp64;
  else static_assert(sizeof(T) == 0, "no container dtype for this element type");
}

template <typename T>
std::vector<std::uint8_t> to_bytes(const std::vector<T>& v) {
  std::vector<std::uint8_t> out(v.size() * sizeof(T));
  if (!v.empty()) std::memcpy(out.data(), v.data(), out.size());  // little-endian host
  return out;
}

template <typename T>
std::vector<T> from_bytes(const std::vector<std::uint8_t>& raw) {
  std::vector<T> out(raw.size() / sizeof(T));
  if (!out.empty()) std::memcpy(out.data(), raw.data(), out.size() * sizeof(T));
  return out;
}

inline void set_pattern(Container& c, const SparsityPattern& p) {
  c.z = static_cast<std::uint16_t>(p.z);
  c.l = static_cast<std::uint16_t>(p.l);
  c.hw_m = static_cast<std::uint16_t>(p.hw_m);
  c.hw_n = static_cast<std::uint16_t>(p.hw_n);
}

}  // namespace detail

// Shape checks of a container's sections (reference validate_payload).
inline void validate_payload(const Container& c) {
  const std::size_t elem = dtype_size(c.dtype);
  if (c.kind == Kind::dense || c.kind == Kind::slided) {
    if (c.values.size() != c.rows * c.cols * elem) throw ContainerError("values payload does not match shape");
  } else if (c.kind == Kind::compressed) {
    if (c.hw_m == 0 || c.hw_n == 0) throw ContainerError("compressed container needs a pattern");
    const std::uint64_t codes = c.rows * c.cols * c.hw_m;
    if (c.values.size() != codes * elem) throw ContainerError("values payload does not match shape");
    if (c.metadata.size() != (codes + 3) / 4) throw ContainerError("metadata payload does not match shape");
  } else {
    if (c.values.size() != c.rows * c.cols * 4) throw ContainerError("word payload does not match shape");
    if (c.scales.size() != c.rows) throw ContainerError("scale count does not match rows");
    if (c.dtype != Dtype::int8 && c.dtype != Dtype::fp8e4m3)
      throw ContainerError("quantized container must be int8 or fp8e4m3");
  }
  const bool zero_pattern = !c.z && !c.l && !c.hw_m && !c.hw_n;
  if (c.kind == Kind::dense && !zero_pattern) throw ContainerError("dense container must zero pattern");
  if (c.kind != Kind::dense && (!c.z || !c.l || !c.hw_m || !c.hw_n))
    throw ContainerError("transformed container needs a pattern");
}

inline std::vector<std::uint8_t> serialize(const Container& c) {
  validate_payload(c);
  std::vector<std::uint8_t> out = {'S', 'L', 'S', 'P'};
  detail::put_le<std::uint16_t>(out, 1);
  out.push_back(static_cast<std::uint8_t>(c.kind));
  out.push_back(static_cast<std::uint8_t>(c.dtype));
  for (const std::uint16_t v : {c.z, c.l, c.hw_m, c.hw_n}) detail::put_le(out, v);
  detail::put_le(out, c.rows);
  detail::put_le(out, c.cols);
  auto section = [&out](const std::vector<std::uint8_t>& s) {
    detail::put_le<std::uint64_t>(out, s.size());
    out.insert(out.end(), s.begin(), s.end());
  };
  section(c.values);
  if (c.kind == Kind::compressed) section(c.metadata);
  if (c.kind == Kind::quantized_lifted) section(detail::to_bytes(c.scales));
  detail::put_le(out, detail::crc32(out));
  return out;
}

inline Container deserialize(std::span<const std::uint8_t> bytes) {
  if (bytes.size() < 36) throw ContainerError("container truncated");
  if (std::memcmp(bytes.data(), "SLSP", 4) != 0) throw ContainerError("bad magic; not a tensor container");
  const auto body = bytes.first(bytes.size() - 4);
  if (detail::crc32(body) != detail::Cursor(bytes.last(4)).get<std::uint32_t>())
    throw ContainerError("checksum mismatch");
  detail::Cursor cur(body);
  cur.skip(4);
  const auto version = cur.get<std::uint16_t>();
  if (version != 1) throw ContainerError("unsupported container version " + std::to_string(version));
  Container c;
  const auto kind = cur.get<std::uint8_t>();
  if (kind > 3) throw ContainerError("unknown kind");
  c.kind = static_cast<Kind>(kind);
  const auto dtype = cur.get<std::uint8_t>();
  if (dtype > 4) throw ContainerError("unknown dtype");
  c.dtype = static_cast<Dtype>(dtype);
  c.z = cur.get<std::uint16_t>();
  c.l = cur.get<std::uint16_t>();
  c.hw_m = cur.get<std::uint16_t>();
  c.hw_n = cur.get<std::uint16_t>();
  c.rows = cur.get<std::uint64_t>();
  c.cols = cur.get<std::uint64_t>();
  c.values = cur.section();
  if (c.kind == Kind::compressed) c.metadata = cur.section();
  if (c.kind == Kind::quantized_lifted) {
    const auto raw = cur.section();
    if (raw.size() % 4 != 0) throw ContainerError("scale payload not a multiple of 4 bytes");
    c.scales = detail::from_bytes<float>(raw);
  }
  if (cur.offset() != body.size()) throw ContainerError("trailing bytes after payload");
  validate_payload(c);
  return c;
}

// Atomic replace (container.hpp:249-262 contract): serialize into
// <path>.tmp<pid> in the destination directory, check the write, then rename
// it over the destination — a failed write leaves the old file intact.
inline void save_container(const std::filesystem::path& path, const Container& c) {
  const auto bytes = serialize(c);
  auto tmp = path;
  tmp += ".tmp" + std::to_string(static_cast<long long>(::getpid()));
  {
    std::ofstream f(tmp, std::ios::binary | std::ios::trunc);
    if (!f) throw ContainerError("cannot open " + tmp.string() + " for writing");
    f.write(reinterpret_cast<const char*>(bytes.data()), static_cast<std::streamsize>(bytes.size()));
    f.flush();
    if (!f) {
      f.close();
      std::error_code ec;
      std::filesystem::remove(tmp, ec);
      throw ContainerError("write failed: " + tmp.string());
    }
  }
  std::error_code ec;
  std::filesystem::rename(tmp, path, ec);
  if (ec) {
    std::filesystem::remove(tmp, ec);
    throw ContainerError("cannot rename " + tmp.string() + " to " + path.string());
  }
}

inline Container load_container(const std::filesystem::path& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw ContainerError("cannot open " + path.string());
  const std::vector<std::uint8_t> bytes((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  return deserialize(bytes);
}

// ---- typed conversions -------------------------------------------------------------
template <typename T>
Container to_container(const Matrix<T>& m) {
  Container c;
  c.dtype = detail::dtype_of<T>();
  c.rows = m.rows;
  c.cols = m.cols;
  c.values = detail::to_bytes(m.data);
  return c;
}

template <typename T>
Container to_container(const SlidedMatrix<T>& s) {
  Container c;
  c.kind = Kind::slided;
  c.dtype = detail::dtype_of<T>();
  detail::set_pattern(c, s.pattern);
  c.rows = s.rows;
  c.cols = s.cols_expanded;
  c.values = detail::to_bytes(s.data);
  return c;
}

template <typename T>
Container to_container(const CompressedSparseMatrix<T>& cm) {
  Container c;
  c.kind = Kind::compressed;
  c.dtype = detail::dtype_of<T>();
  detail::set_pattern(c, cm.pattern);
  c.rows = cm.rows;
  c.cols = cm.windows_per_row;
  c.values = detail::to_bytes(cm.values);
  c.metadata = detail::pack_codes(cm.metadata);
  return c;
}

inline Container to_container(const QuantizedLiftedActivation& a) {
  Container c;
  c.kind = Kind::quantized_lifted;
  c.dtype = a.kind == QuantKind::int8 ? Dtype::int8 : Dtype::fp8e4m3;
  detail::set_pattern(c, a.pattern);
  c.rows = a.rows;
  c.cols = a.words_per_row;
  c.values = detail::to_bytes(a.payload);
  c.scales = a.scales;
  return c;
}

template <typename T>
Matrix<T> dense_from(const Container& c) {
  if (c.kind != Kind::dense) throw ContainerError("expected a dense container");
  if (c.dtype != detail::dtype_of<T>()) throw ContainerError("container dtype mismatch");
  return Matrix<T>(c.rows, c.cols, detail::from_bytes<T>(c.values));
}

template <typename T>
SlidedMatrix<T> slided_from(const Container& c) {
  if (c.kind != Kind::slided) throw ContainerError("expected a slided container");
  if (c.dtype != detail::dtype_of<T>()) throw ContainerError("container dtype mismatch");
  SlidedMatrix<T> s;
  s.rows = c.rows;
  s.cols_expanded = c.cols;
  s.pattern = c.pattern();
  s.data = detail::from_bytes<T>(c.values);
  return s;
}

template <typename T>
CompressedSparseMatrix<T> compressed_from(const Container& c) {
  if (c.kind != Kind::compressed) throw ContainerError("expected a compressed container");
  if (c.dtype != detail::dtype_of<T>()) throw ContainerError("container dtype mismatch");
  CompressedSparseMatrix<T> cm;
  cm.rows = c.rows;
  cm.windows_per_row = c.cols;
  cm.pattern = c.pattern();
  cm.values = detail::from_bytes<T>(c.values);
  cm.metadata = detail::unpack_codes(c.metadata, c.rows * c.cols * c.hw_m);
  return cm;
}

inline QuantizedLiftedActivation quantized_from(const Container& c) {
  if (c.kind != Kind::quantized_lifted) throw ContainerError("expected a quantized container");
  QuantizedLiftedActivation a;
  a.rows = c.rows;
  a.words_per_row = c.cols;
  a.pattern = c.pattern();
  a.kind = c.dtype == Dtype::int8 ? QuantKind::int8 : QuantKind::fp8e4m3;
  a.payload = detail::from_bytes<std::uint32_t>(c.values);
  a.scales = c.scales;
  return a;
}

}  // namespace slsp
