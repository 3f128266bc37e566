// C++ drop-in parity program: the reference's own test scenarios
// (proj/tests/test_pack.cpp, test_quantize.cpp, test_gemm.cpp) written against
// the B200 drop-in headers in include/slsp/ — same API, same expectations —
// executed on the GPU through libslsp_b200.so. Exit code = number of failures.
// Built by tests/cpp/Makefile; run by tests/test_gpu_dropin.py.
#include <cstdio>
#include <fstream>
#include <functional>
#include <iterator>
#include <limits>
#include <random>
#include <string>
#include <vector>

#include "slsp/slsp.hpp"

using namespace slsp;

static int failures = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static Matrix<std::int8_t> compliant(std::mt19937_64& rng, const SparsityPattern& p, std::size_t rows,
                                     std::size_t groups) {
  Matrix<std::int8_t> w(rows, groups * p.l);
  std::uniform_int_distribution<int> nnz_d(0, p.z), val(-127, 126);
  std::vector<int> pos(p.l);
  for (std::size_t r = 0; r < rows; ++r)
    for (std::size_t g = 0; g < groups; ++g) {
      for (int k = 0; k < p.l; ++k) pos[k] = k;
      std::shuffle(pos.begin(), pos.end(), rng);
      const int nnz = nnz_d(rng);
      for (int k = 0; k < nnz; ++k) {
        const int v = val(rng);
        w(r, g * p.l + pos[k]) = static_cast<std::int8_t>(v >= 0 ? v + 1 : v);
      }
    }
  return w;
}

int main() {
  const SparsityPattern p68(6, 8);
  // test_pattern.cpp:24-30
  {
    const auto plan = plan_decomposition(p68);
    CHECK(plan.window_count == 3 && plan.window_starts == (std::vector<int>{0, 2, 4}));
    CHECK(plan.expansion == Ratio(3, 2));
    CHECK((throws<AlreadyCompliantError>([] { plan_decomposition(SparsityPattern(1, 4)); })));
  }
  // test_pack.cpp:48-59, test_gemm.cpp:114-127 (worked example = 112)
  {
    Matrix<std::int8_t> w(1, 8, {1, 2, 3, 0, 4, 5, 0, 6});
    const auto s = pack_matrix(w, p68);
    CHECK(s.data == (std::vector<std::int8_t>{1, 2, 0, 0, 3, 0, 4, 0, 0, 5, 0, 6}));
    Matrix<std::int8_t> x(8, 1);
    for (int k = 0; k < 8; ++k) x(k, 0) = static_cast<std::int8_t>(k + 1);
    const auto c = compress(s);
    CHECK(c.values == (std::vector<std::int8_t>{1, 2, 3, 4, 5, 6}));
    CHECK(c.metadata == (std::vector<std::uint8_t>{0, 1, 0, 2, 1, 3}));
    const auto y = sparse_gemm(c, lift_activations(x, plan_decomposition(p68)));
    CHECK(y(0, 0) == 112);
    CHECK(dense_gemm(w, x)(0, 0) == 112);
  }
  // test_pack.cpp:225-237
  {
    Matrix<std::int8_t> w(2, 16);
    for (int k = 0; k < 7; ++k) w(1, 8 + k) = 1;
    try {
      pack_matrix(w, p68);
      CHECK(false);
    } catch (const NotCompliantError& e) {
      const std::string msg = e.what();
      CHECK(msg.find("row 1") != std::string::npos && msg.find("block 1") != std::string::npos);
    }
  }
  // test_quantize.cpp:265-276 and :241-263 (fused == composition)
  {
    Matrix<float> x(1, 8, {1, 2, 3, 4, 5, 6, 7, 8});
    const auto a = fused_quant_slide(x, p68, QuantKind::int8);
    CHECK(a.words_per_row == 3 && a.lifted_cols() == 12);
    const auto q = quantize_row<float>(x.row(0), QuantKind::int8);
    const auto lifted = lift_row<std::uint8_t>(q.bytes, plan_decomposition(p68));
    for (std::size_t k = 0; k < 12; ++k) CHECK(a.byte_at(0, k) == lifted[k]);
    Matrix<float> bad(2, 8);
    bad(1, 3) = std::numeric_limits<float>::infinity();
    CHECK((throws<NonFiniteInputError>([&] { fused_quant_slide(bad, p68); })));
  }
  // test_gemm.cpp:299-323: packed-word sparse path == dense on quantized X
  {
    std::mt19937_64 rng(13);
    const auto w = compliant(rng, p68, 12, 3);
    Matrix<float> xr(5, w.cols);
    std::uniform_real_distribution<float> d(-2.0f, 2.0f);
    for (auto& v : xr.data) v = d(rng);
    const auto sparse = sparse_gemm(compress(pack_matrix(w, p68)), fused_quant_slide(xr, p68, QuantKind::int8));
    Matrix<std::int8_t> q(w.cols, xr.rows);
    for (std::size_t t = 0; t < xr.rows; ++t) {
      const auto qr = quantize_row<float>(xr.row(t), QuantKind::int8);
      for (std::size_t k = 0; k < w.cols; ++k) q(k, t) = static_cast<std::int8_t>(qr.bytes[k]);
    }
    CHECK(dense_gemm(w, q).data == sparse.data);
  }
  // acceptance.cpp:45-71 in miniature: random W/X pairs exact, all patterns
  {
    std::mt19937_64 rng(1001);
    for (const auto& p : {SparsityPattern(4, 6), SparsityPattern(6, 8), SparsityPattern(8, 10), SparsityPattern(14, 16)}) {
      for (int trial = 0; trial < 4; ++trial) {
        const auto w = compliant(rng, p, 1 + rng() % 64, 1 + rng() % (256 / p.l));
        Matrix<std::int8_t> x(w.cols, 1 + rng() % 16);
        std::uniform_int_distribution<int> dv(-127, 127);
        for (auto& v : x.data) v = static_cast<std::int8_t>(dv(rng));
        const auto rep = check_equivalence(w, x, p);
        CHECK(rep.exact && rep.max_abs_diff == 0.0);
      }
    }
  }
  // magnitude_prune -> compliant, unslide(pack) round trip (test_pack.cpp:204-212)
  {
    std::mt19937_64 rng(22);
    Matrix<std::int8_t> w(64, 512);
    std::uniform_int_distribution<int> dv(-127, 127);
    for (auto& v : w.data) v = static_cast<std::int8_t>(dv(rng));
    const auto pruned = magnitude_prune(w, p68);
    CHECK(verify_compliance(pruned, 6, 8).compliant);
    const auto s = pack_matrix(pruned, p68);
    CHECK(verify_compliance(s, 2, 4).compliant);
    CHECK(unslide(s).data == pruned.data);
    CHECK(decompress(compress(s)).data == s.data);
  }
  // container.hpp: files the REFERENCE wrote (tests/golden, gen_golden.py) —
  // parse, typed conversion, byte-exact re-serialization, the GEMM on the
  // loaded weights == the GEMM on weights packed here (test_container.cpp)
  {
    const std::string gold = std::string(SLSP_GOLDEN_DIR) + "/";
    for (const char* tag : {"even", "odd"}) {
      const auto path = gold + "container_6_8_" + tag + ".slsp";
      const auto c = load_container(path);
      CHECK(c.kind == Kind::compressed && c.z == 6 && c.l == 8);
      const auto cm = compressed_from<std::int8_t>(c);
      std::ifstream f(path, std::ios::binary);
      const std::vector<std::uint8_t> bytes((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
      CHECK(serialize(to_container(cm)) == bytes);
      // the same weights through this library's packer give the same operands
      const auto w = unslide(decompress(cm));
      const auto mine = compress(pack_matrix(w, SparsityPattern(6, 8)));
      CHECK(mine.values == cm.values && mine.metadata == cm.metadata);
      std::mt19937_64 rng(5);
      Matrix<float> x(7, w.cols);
      std::uniform_real_distribution<float> dx(-1.0f, 1.0f);
      for (auto& v : x.data) v = dx(rng);
      const auto act = fused_quant_slide(x, SparsityPattern(6, 8), QuantKind::int8);
      CHECK(sparse_gemm(cm, act).data == sparse_gemm(mine, act).data);
    }
    const auto q = quantized_from(load_container(gold + "container_fqs_6_8.slsp"));
    CHECK(q.rows == 9 && q.words_per_row * 4 == 144 && q.kind == QuantKind::int8);
    auto bad = serialize(to_container(q));
    bad[40] ^= 0x5A;
    CHECK(throws<ContainerError>([&] { deserialize(bad); }));
    CHECK(throws<ContainerError>([&] { deserialize(std::vector<std::uint8_t>(10, 0)); }));
  }
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "OK", failures);
  return failures;
}
