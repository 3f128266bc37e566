// Minimal stand-in for <boost/rational.hpp> (Boost is not installed in this
// image). TEST INFRASTRUCTURE ONLY: it exists so that the reference headers in
// /root/reference/proj/include/slsp can be compiled unmodified into the
// oracle/_ref bridge. Only the operations the hot-path headers use are
// provided (pattern.hpp:22-185): construction, + - * /, comparisons,
// numerator/denominator and rational_cast.
#pragma once
#include <cstdint>
#include <numeric>
#include <stdexcept>

namespace boost {

template <typename I>
class rational {
 public:
  rational() : n_(0), d_(1) {}
  rational(I n) : n_(n), d_(1) {}  // NOLINT(implicit)
  rational(I n, I d) : n_(n), d_(d) { normalize(); }
  I numerator() const { return n_; }
  I denominator() const { return d_; }

  friend rational operator+(const rational& a, const rational& b) {
    return rational(a.n_ * b.d_ + b.n_ * a.d_, a.d_ * b.d_);
  }
  friend rational operator-(const rational& a, const rational& b) {
    return rational(a.n_ * b.d_ - b.n_ * a.d_, a.d_ * b.d_);
  }
  friend rational operator*(const rational& a, const rational& b) {
    return rational(a.n_ * b.n_, a.d_ * b.d_);
  }
  friend rational operator/(const rational& a, const rational& b) {
    return rational(a.n_ * b.d_, a.d_ * b.n_);
  }
  friend bool operator==(const rational& a, const rational& b) { return a.n_ == b.n_ && a.d_ == b.d_; }
  friend bool operator!=(const rational& a, const rational& b) { return !(a == b); }
  friend bool operator<(const rational& a, const rational& b) { return a.n_ * b.d_ < b.n_ * a.d_; }
  friend bool operator>(const rational& a, const rational& b) { return b < a; }
  friend bool operator<=(const rational& a, const rational& b) { return !(b < a); }
  friend bool operator>=(const rational& a, const rational& b) { return !(a < b); }

 private:
  void normalize() {
    if (d_ == 0) throw std::domain_error("rational: zero denominator");
    if (d_ < 0) { n_ = -n_; d_ = -d_; }
    const I g = std::gcd(n_ < 0 ? -n_ : n_, d_);
    if (g > 1) { n_ /= g; d_ /= g; }
  }
  I n_, d_;
};

template <typename T, typename I>
T rational_cast(const rational<I>& r) {
  return static_cast<T>(r.numerator()) / static_cast<T>(r.denominator());
}

}  // namespace boost
