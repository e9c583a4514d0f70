// ORACLE TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// Minimal stand-in for the subset of Boost.Multiprecision that the read-only
// reference (/root/reference/proj) uses: `cpp_int` (signed arbitrary
// precision integer) and `cpp_rational` (normalised exact rational), plus the
// free functions msb / powm / numerator / denominator / export_bits /
// import_bits.  The reference's `vendor/` directory (which held Boost) is
// absent (proj/.gitignore:2, proj/README.md:41-43) and Boost is not installed
// in this image, so this header restates the published Boost semantics the
// reference relies on:
//   * truncating division, remainder takes the sign of the dividend
//     (cpp_int follows built-in integer semantics);
//   * cpp_rational is always kept in lowest terms with a positive denominator;
//   * export_bits/import_bits default to most-significant-chunk first and
//     export a single zero chunk for the value 0;
//   * conversion of a rational to double is correctly rounded.
// Boost version: unpinned by the reference (README says only "Boost.
// Multiprecision headers"); only exact integer/rational semantics matter for
// residues, so any correct big-integer gives identical tables.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <iterator>
#include <ostream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace boost {
namespace multiprecision {

class cpp_int {
 public:
  cpp_int() = default;
  template <class T, class = std::enable_if_t<std::is_integral_v<T>>>
  cpp_int(T v) {  // NOLINT(implicit)
    if constexpr (std::is_signed_v<T>) {
      if (v < 0) {
        neg_ = true;
        set_u64(static_cast<uint64_t>(0) - static_cast<uint64_t>(static_cast<int64_t>(v)));
        normalize();
        return;
      }
    }
    set_u64(static_cast<uint64_t>(v));
    normalize();
  }

  // --- observers -----------------------------------------------------------
  bool is_zero() const { return mag_.empty(); }
  bool is_neg() const { return neg_; }
  const std::vector<uint32_t>& limbs() const { return mag_; }
  int sign() const { return is_zero() ? 0 : (neg_ ? -1 : 1); }
  explicit operator bool() const { return !is_zero(); }

  size_t bit_length() const {
    if (mag_.empty()) return 0;
    uint32_t top = mag_.back();
    size_t b = 0;
    while (top) { ++b; top >>= 1; }
    return (mag_.size() - 1) * 32 + b;
  }

  template <class T, class = std::enable_if_t<std::is_integral_v<T>>>
  explicit operator T() const {
    // modular wrap like Boost's conversion of in-range values; the
    // reference only converts values that fit.
    uint64_t lo = 0;
    if (!mag_.empty()) lo = mag_[0];
    if (mag_.size() > 1) lo |= static_cast<uint64_t>(mag_[1]) << 32;
    if (neg_) lo = static_cast<uint64_t>(0) - lo;
    return static_cast<T>(lo);
  }
  explicit operator double() const { return to_ld<double>(); }
  explicit operator long double() const { return to_ld<long double>(); }

  // --- arithmetic ----------------------------------------------------------
  cpp_int operator-() const {
    cpp_int r = *this;
    if (!r.is_zero()) r.neg_ = !r.neg_;
    return r;
  }
  cpp_int& operator+=(const cpp_int& o) { return add_signed(o, false); }
  cpp_int& operator-=(const cpp_int& o) { return add_signed(o, true); }
  cpp_int& operator*=(const cpp_int& o) {
    if (is_zero() || o.is_zero()) { *this = cpp_int(); return *this; }
    std::vector<uint32_t> r(mag_.size() + o.mag_.size(), 0);
    for (size_t i = 0; i < mag_.size(); ++i) {
      uint64_t carry = 0;
      const uint64_t a = mag_[i];
      for (size_t j = 0; j < o.mag_.size(); ++j) {
        uint64_t t = a * o.mag_[j] + r[i + j] + carry;
        r[i + j] = static_cast<uint32_t>(t);
        carry = t >> 32;
      }
      size_t k = i + o.mag_.size();
      while (carry) {
        uint64_t t = static_cast<uint64_t>(r[k]) + carry;
        r[k] = static_cast<uint32_t>(t);
        carry = t >> 32;
        ++k;
      }
    }
    neg_ = neg_ != o.neg_;
    mag_ = std::move(r);
    normalize();
    return *this;
  }
  cpp_int& operator/=(const cpp_int& o) {
    cpp_int q, r;
    divmod(*this, o, q, r);
    *this = std::move(q);
    return *this;
  }
  cpp_int& operator%=(const cpp_int& o) {
    cpp_int q, r;
    divmod(*this, o, q, r);
    *this = std::move(r);
    return *this;
  }
  cpp_int& operator<<=(unsigned s) {
    if (is_zero()) return *this;
    const size_t w = s / 32, b = s % 32;
    std::vector<uint32_t> r(mag_.size() + w + 1, 0);
    for (size_t i = 0; i < mag_.size(); ++i) {
      const uint64_t v = static_cast<uint64_t>(mag_[i]) << b;
      r[i + w] |= static_cast<uint32_t>(v);
      r[i + w + 1] |= static_cast<uint32_t>(v >> 32);
    }
    mag_ = std::move(r);
    normalize();
    return *this;
  }
  cpp_int& operator>>=(unsigned s) {
    // Boost: right shift of a negative value rounds toward -inf (like
    // arithmetic shift); the reference only shifts non-negative values.
    if (is_zero()) return *this;
    const bool was_neg = neg_;
    bool lost = false;
    const size_t w = s / 32, b = s % 32;
    if (w >= mag_.size()) {
      lost = true;
      mag_.clear();
    } else {
      for (size_t i = 0; i < w; ++i) lost |= mag_[i] != 0;
      if (b) lost |= (mag_[w] & ((1u << b) - 1)) != 0;
      std::vector<uint32_t> r(mag_.size() - w, 0);
      for (size_t i = 0; i < r.size(); ++i) {
        uint64_t v = mag_[i + w];
        if (i + w + 1 < mag_.size()) v |= static_cast<uint64_t>(mag_[i + w + 1]) << 32;
        r[i] = static_cast<uint32_t>(v >> b);
      }
      mag_ = std::move(r);
    }
    normalize();
    if (was_neg) {
      neg_ = !is_zero();
      if (lost) *this -= cpp_int(1);
    }
    return *this;
  }
  cpp_int& operator|=(const cpp_int& o) {
    // only used on non-negative values by the reference
    if (neg_ || o.neg_) throw std::domain_error("shim: bitwise or on negative");
    if (o.mag_.size() > mag_.size()) mag_.resize(o.mag_.size(), 0);
    for (size_t i = 0; i < o.mag_.size(); ++i) mag_[i] |= o.mag_[i];
    normalize();
    return *this;
  }

  // --- comparisons ---------------------------------------------------------
  static int cmp_mag(const std::vector<uint32_t>& a, const std::vector<uint32_t>& b) {
    if (a.size() != b.size()) return a.size() < b.size() ? -1 : 1;
    for (size_t i = a.size(); i-- > 0;)
      if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
  }
  static int cmp(const cpp_int& a, const cpp_int& b) {
    if (a.neg_ != b.neg_) return a.neg_ ? -1 : 1;
    const int c = cmp_mag(a.mag_, b.mag_);
    return a.neg_ ? -c : c;
  }

  // Truncating division: q = trunc(a/b), r = a - q*b (sign of a).
  static void divmod(const cpp_int& a, const cpp_int& b, cpp_int& q, cpp_int& r) {
    if (b.is_zero()) throw std::overflow_error("shim: division by zero");
    std::vector<uint32_t> qm, rm;
    divmod_mag(a.mag_, b.mag_, qm, rm);
    q.mag_ = std::move(qm);
    q.neg_ = a.neg_ != b.neg_;
    q.normalize();
    r.mag_ = std::move(rm);
    r.neg_ = a.neg_;
    r.normalize();
  }

  std::string str() const {
    if (is_zero()) return "0";
    std::string s;
    cpp_int v = *this;
    v.neg_ = false;
    const cpp_int ten9(1000000000u);
    while (!v.is_zero()) {
      cpp_int q, r;
      divmod(v, ten9, q, r);
      uint32_t chunk = static_cast<uint32_t>(r);
      for (int i = 0; i < 9; ++i) {
        s.push_back(static_cast<char>('0' + chunk % 10));
        chunk /= 10;
        if (q.is_zero() && chunk == 0) break;
      }
      v = std::move(q);
    }
    while (s.size() > 1 && s.back() == '0') s.pop_back();
    if (neg_) s.push_back('-');
    std::reverse(s.begin(), s.end());
    return s;
  }

  // raw access for import/export
  std::vector<uint32_t>& raw_mag() { return mag_; }
  void set_neg(bool n) { neg_ = n; normalize(); }
  void normalize() {
    while (!mag_.empty() && mag_.back() == 0) mag_.pop_back();
    if (mag_.empty()) neg_ = false;
  }

 private:
  void set_u64(uint64_t v) {
    mag_.clear();
    if (v) {
      mag_.push_back(static_cast<uint32_t>(v));
      if (v >> 32) mag_.push_back(static_cast<uint32_t>(v >> 32));
    }
  }

  template <class F>
  F to_ld() const {
    F r = 0;
    for (size_t i = mag_.size(); i-- > 0;) r = r * F(4294967296.0) + F(mag_[i]);
    // exact when the value has <= mantissa bits (the reference only
    // converts after shifting to <= 53 bits, ckks.cpp:147-155)
    return neg_ ? -r : r;
  }

  static void add_mag(std::vector<uint32_t>& a, const std::vector<uint32_t>& b) {
    if (b.size() > a.size()) a.resize(b.size(), 0);
    uint64_t carry = 0;
    for (size_t i = 0; i < a.size(); ++i) {
      uint64_t t = static_cast<uint64_t>(a[i]) + (i < b.size() ? b[i] : 0) + carry;
      a[i] = static_cast<uint32_t>(t);
      carry = t >> 32;
      if (!carry && i >= b.size()) break;
    }
    if (carry) a.push_back(static_cast<uint32_t>(carry));
  }
  // a -= b, requires |a| >= |b|
  static void sub_mag(std::vector<uint32_t>& a, const std::vector<uint32_t>& b) {
    int64_t borrow = 0;
    for (size_t i = 0; i < a.size(); ++i) {
      int64_t t = static_cast<int64_t>(a[i]) - (i < b.size() ? b[i] : 0) - borrow;
      borrow = t < 0;
      if (t < 0) t += (static_cast<int64_t>(1) << 32);
      a[i] = static_cast<uint32_t>(t);
      if (!borrow && i >= b.size()) break;
    }
  }
  cpp_int& add_signed(const cpp_int& o, bool negate_o) {
    const bool on = negate_o ? !o.neg_ && !o.is_zero() : o.neg_;
    if (neg_ == on) {
      add_mag(mag_, o.mag_);
    } else if (cmp_mag(mag_, o.mag_) >= 0) {
      sub_mag(mag_, o.mag_);
    } else {
      std::vector<uint32_t> t = o.mag_;
      sub_mag(t, mag_);
      mag_ = std::move(t);
      neg_ = on;
    }
    normalize();
    return *this;
  }

  // Knuth algorithm D on 32-bit limbs.
  static void divmod_mag(const std::vector<uint32_t>& a, const std::vector<uint32_t>& b,
                         std::vector<uint32_t>& q, std::vector<uint32_t>& r) {
    q.clear();
    r.clear();
    if (cmp_mag(a, b) < 0) { r = a; return; }
    if (b.size() == 1) {
      const uint64_t d = b[0];
      q.assign(a.size(), 0);
      uint64_t rem = 0;
      for (size_t i = a.size(); i-- > 0;) {
        const uint64_t cur = (rem << 32) | a[i];
        q[i] = static_cast<uint32_t>(cur / d);
        rem = cur % d;
      }
      if (rem) r.push_back(static_cast<uint32_t>(rem));
      while (!q.empty() && q.back() == 0) q.pop_back();
      return;
    }
    const size_t n = b.size(), m = a.size() - b.size();
    int s = 0;
    for (uint32_t top = b.back(); !(top & 0x80000000u); top <<= 1) ++s;
    std::vector<uint32_t> bn(n), an(a.size() + 1);
    for (size_t i = n; i-- > 0;)
      bn[i] = (b[i] << s) | (s && i ? static_cast<uint32_t>(static_cast<uint64_t>(b[i - 1]) >> (32 - s)) : 0);
    an[a.size()] = s ? static_cast<uint32_t>(static_cast<uint64_t>(a.back()) >> (32 - s)) : 0;
    for (size_t i = a.size(); i-- > 0;)
      an[i] = (a[i] << s) | (s && i ? static_cast<uint32_t>(static_cast<uint64_t>(a[i - 1]) >> (32 - s)) : 0);
    q.assign(m + 1, 0);
    const uint64_t B = static_cast<uint64_t>(1) << 32;
    for (size_t j = m + 1; j-- > 0;) {
      const uint64_t num = (static_cast<uint64_t>(an[j + n]) << 32) | an[j + n - 1];
      uint64_t qhat = num / bn[n - 1];
      uint64_t rhat = num % bn[n - 1];
      while (qhat >= B || qhat * bn[n - 2] > ((rhat << 32) | an[j + n - 2])) {
        --qhat;
        rhat += bn[n - 1];
        if (rhat >= B) break;
      }
      int64_t borrow = 0;
      uint64_t carry = 0;
      for (size_t i = 0; i < n; ++i) {
        const uint64_t p = qhat * bn[i] + carry;
        carry = p >> 32;
        const int64_t t = static_cast<int64_t>(an[i + j]) - static_cast<int64_t>(p & 0xffffffffu) - borrow;
        an[i + j] = static_cast<uint32_t>(t);
        borrow = t < 0;
      }
      const int64_t t = static_cast<int64_t>(an[j + n]) - static_cast<int64_t>(carry) - borrow;
      an[j + n] = static_cast<uint32_t>(t);
      if (t < 0) {
        --qhat;
        uint64_t c = 0;
        for (size_t i = 0; i < n; ++i) {
          const uint64_t s2 = static_cast<uint64_t>(an[i + j]) + bn[i] + c;
          an[i + j] = static_cast<uint32_t>(s2);
          c = s2 >> 32;
        }
        an[j + n] = static_cast<uint32_t>(static_cast<uint64_t>(an[j + n]) + c);
      }
      q[j] = static_cast<uint32_t>(qhat);
    }
    r.assign(n, 0);
    for (size_t i = 0; i < n; ++i)
      r[i] = (an[i] >> s) | (s ? static_cast<uint32_t>(static_cast<uint64_t>(an[i + 1]) << (32 - s)) : 0);
    while (!q.empty() && q.back() == 0) q.pop_back();
    while (!r.empty() && r.back() == 0) r.pop_back();
  }

  bool neg_ = false;
  std::vector<uint32_t> mag_;  // little-endian 32-bit limbs, no leading zeros
};

// --- free operators (cpp_int with cpp_int or integral) ----------------------
#define CK_SHIM_BINOP(op, cop)                                                  \
  inline cpp_int operator op(cpp_int a, const cpp_int& b) { a cop b; return a; } \
  template <class T, class = std::enable_if_t<std::is_integral_v<T>>>          \
  inline cpp_int operator op(cpp_int a, T b) { a cop cpp_int(b); return a; }  \
  template <class T, class = std::enable_if_t<std::is_integral_v<T>>>          \
  inline cpp_int operator op(T a, const cpp_int& b) { cpp_int r(a); r cop b; return r; }
CK_SHIM_BINOP(+, +=)
CK_SHIM_BINOP(-, -=)
CK_SHIM_BINOP(*, *=)
CK_SHIM_BINOP(/, /=)
CK_SHIM_BINOP(%, %=)
CK_SHIM_BINOP(|, |=)
#undef CK_SHIM_BINOP

inline cpp_int operator<<(cpp_int a, unsigned s) { a <<= s; return a; }
inline cpp_int operator>>(cpp_int a, unsigned s) { a >>= s; return a; }
inline cpp_int operator<<(cpp_int a, int s) { a <<= static_cast<unsigned>(s); return a; }
inline cpp_int operator>>(cpp_int a, int s) { a >>= static_cast<unsigned>(s); return a; }
template <class T, class = std::enable_if_t<std::is_integral_v<T> && !std::is_same_v<T, int> && !std::is_same_v<T, unsigned>>>
inline cpp_int operator<<(cpp_int a, T s) { a <<= static_cast<unsigned>(s); return a; }
template <class T, class = std::enable_if_t<std::is_integral_v<T> && !std::is_same_v<T, int> && !std::is_same_v<T, unsigned>>>
inline cpp_int operator>>(cpp_int a, T s) { a >>= static_cast<unsigned>(s); return a; }

#define CK_SHIM_CMP(op)                                                                     \
  inline bool operator op(const cpp_int& a, const cpp_int& b) { return cpp_int::cmp(a, b) op 0; } \
  template <class T, class = std::enable_if_t<std::is_integral_v<T>>>                      \
  inline bool operator op(const cpp_int& a, T b) { return cpp_int::cmp(a, cpp_int(b)) op 0; } \
  template <class T, class = std::enable_if_t<std::is_integral_v<T>>>                      \
  inline bool operator op(T a, const cpp_int& b) { return cpp_int::cmp(cpp_int(a), b) op 0; }
CK_SHIM_CMP(==)
CK_SHIM_CMP(!=)
CK_SHIM_CMP(<)
CK_SHIM_CMP(>)
CK_SHIM_CMP(<=)
CK_SHIM_CMP(>=)
#undef CK_SHIM_CMP

inline std::ostream& operator<<(std::ostream& os, const cpp_int& v) { return os << v.str(); }

// Index of the most significant set bit (Boost: undefined for <= 0; throws).
inline unsigned msb(const cpp_int& v) {
  if (v <= 0) throw std::domain_error("shim: msb of non-positive value");
  return static_cast<unsigned>(v.bit_length() - 1);
}

inline cpp_int abs(const cpp_int& v) { return v < 0 ? -v : v; }

inline cpp_int gcd(cpp_int a, cpp_int b) {
  a = abs(a);
  b = abs(b);
  while (!b.is_zero()) {
    cpp_int r = a % b;
    a = std::move(b);
    b = std::move(r);
  }
  return a;
}

inline cpp_int powm(const cpp_int& base, const cpp_int& exp, const cpp_int& mod) {
  cpp_int result = cpp_int(1) % mod;
  cpp_int b = base % mod;
  if (b < 0) b += mod;
  const size_t bits = exp.bit_length();
  for (size_t i = bits; i-- > 0;) {
    result = result * result % mod;
    const auto& l = exp.limbs();
    if ((l[i / 32] >> (i % 32)) & 1u) result = result * b % mod;
  }
  return result;
}

// export_bits: chunks of `chunk_size` bits, most-significant first by default.
template <class OutputIterator>
OutputIterator export_bits(const cpp_int& val, OutputIterator out, unsigned chunk_size,
                           bool msv_first = true) {
  if (chunk_size != 8) throw std::invalid_argument("shim: only 8-bit chunks");
  cpp_int v = abs(val);
  if (v.is_zero()) {
    *out = 0;
    ++out;
    return out;
  }
  std::vector<uint8_t> bytes;
  const auto& l = v.limbs();
  const size_t nbytes = (v.bit_length() + 7) / 8;
  for (size_t i = 0; i < nbytes; ++i) bytes.push_back(static_cast<uint8_t>(l[i / 4] >> (8 * (i % 4))));
  if (msv_first) std::reverse(bytes.begin(), bytes.end());
  for (uint8_t b : bytes) {
    *out = b;
    ++out;
  }
  return out;
}

template <class Iterator>
cpp_int& import_bits(cpp_int& val, Iterator i, Iterator j, unsigned chunk_size = 0,
                     bool msv_first = true) {
  if (chunk_size != 8) throw std::invalid_argument("shim: only 8-bit chunks");
  std::vector<uint8_t> bytes(i, j);
  if (msv_first) std::reverse(bytes.begin(), bytes.end());
  auto& m = val.raw_mag();
  m.assign((bytes.size() + 3) / 4, 0);
  for (size_t k = 0; k < bytes.size(); ++k) m[k / 4] |= static_cast<uint32_t>(bytes[k]) << (8 * (k % 4));
  val.set_neg(false);
  return val;
}

// ---------------------------------------------------------------------------
class cpp_rational {
 public:
  cpp_rational() : num_(0), den_(1) {}
  cpp_rational(const cpp_int& v) : num_(v), den_(1) {}  // NOLINT
  template <class T, class = std::enable_if_t<std::is_integral_v<T>>>
  cpp_rational(T v) : num_(v), den_(1) {}  // NOLINT
  cpp_rational(const cpp_int& n, const cpp_int& d) : num_(n), den_(d) { norm(); }
  template <class A, class B,
            class = std::enable_if_t<std::is_integral_v<A> && std::is_integral_v<B>>>
  cpp_rational(A n, B d) : num_(n), den_(d) { norm(); }

  const cpp_int& num() const { return num_; }
  const cpp_int& den() const { return den_; }

  cpp_rational& operator+=(const cpp_rational& o) {
    num_ = num_ * o.den_ + o.num_ * den_;
    den_ *= o.den_;
    norm();
    return *this;
  }
  cpp_rational& operator-=(const cpp_rational& o) {
    num_ = num_ * o.den_ - o.num_ * den_;
    den_ *= o.den_;
    norm();
    return *this;
  }
  cpp_rational& operator*=(const cpp_rational& o) {
    num_ *= o.num_;
    den_ *= o.den_;
    norm();
    return *this;
  }
  cpp_rational& operator/=(const cpp_rational& o) {
    if (o.num_.is_zero()) throw std::overflow_error("shim: rational division by zero");
    cpp_int n = num_ * o.den_;
    cpp_int d = den_ * o.num_;
    num_ = std::move(n);
    den_ = std::move(d);
    norm();
    return *this;
  }
  cpp_rational operator-() const { return cpp_rational(-num_, den_); }

  static int cmp(const cpp_rational& a, const cpp_rational& b) {
    return cpp_int::cmp(a.num_ * b.den_, b.num_ * a.den_);
  }

  // Correctly rounded (round-to-nearest-even) conversion.
  explicit operator double() const {
    if (num_.is_zero()) return 0.0;
    const bool neg = num_ < 0;
    cpp_int n = abs(num_);
    const long nb = static_cast<long>(n.bit_length());
    const long db = static_cast<long>(den_.bit_length());
    // scale so the integer quotient has at least 55 significant bits
    long shift = 55 - (nb - db);
    if (shift > 0) n <<= static_cast<unsigned>(shift);
    cpp_int d = den_;
    if (shift < 0) d <<= static_cast<unsigned>(-shift);
    cpp_int q, r;
    cpp_int::divmod(n, d, q, r);
    // q has 55 or 56 bits; keep 53, round with guard + sticky
    long extra = static_cast<long>(q.bit_length()) - 53;
    bool sticky = !r.is_zero();
    uint64_t qv = static_cast<uint64_t>(q);
    uint64_t mant = qv >> extra;
    const uint64_t rem = qv & ((static_cast<uint64_t>(1) << extra) - 1);
    const uint64_t half = static_cast<uint64_t>(1) << (extra - 1);
    if (rem > half || (rem == half && (sticky || (mant & 1)))) ++mant;
    double out = std::ldexp(static_cast<double>(mant), static_cast<int>(extra - shift));
    return neg ? -out : out;
  }

 private:
  void norm() {
    if (den_.is_zero()) throw std::overflow_error("shim: zero denominator");
    if (den_ < 0) {
      num_ = -num_;
      den_ = -den_;
    }
    cpp_int g = gcd(num_, den_);
    if (g > 1) {
      num_ /= g;
      den_ /= g;
    }
    if (num_.is_zero()) den_ = 1;
  }
  cpp_int num_, den_;
};

inline cpp_int numerator(const cpp_rational& r) { return r.num(); }
inline cpp_int denominator(const cpp_rational& r) { return r.den(); }

#define CK_SHIM_RBINOP(op, cop)                                                              \
  inline cpp_rational operator op(cpp_rational a, const cpp_rational& b) { a cop b; return a; } \
  inline cpp_rational operator op(cpp_rational a, const cpp_int& b) { a cop cpp_rational(b); return a; } \
  inline cpp_rational operator op(const cpp_int& a, const cpp_rational& b) { cpp_rational r(a); r cop b; return r; } \
  template <class T, class = std::enable_if_t<std::is_integral_v<T>>>                        \
  inline cpp_rational operator op(cpp_rational a, T b) { a cop cpp_rational(b); return a; } \
  template <class T, class = std::enable_if_t<std::is_integral_v<T>>>                        \
  inline cpp_rational operator op(T a, const cpp_rational& b) { cpp_rational r(a); r cop b; return r; }
CK_SHIM_RBINOP(+, +=)
CK_SHIM_RBINOP(-, -=)
CK_SHIM_RBINOP(*, *=)
CK_SHIM_RBINOP(/, /=)
#undef CK_SHIM_RBINOP

#define CK_SHIM_RCMP(op)                                                                        \
  inline bool operator op(const cpp_rational& a, const cpp_rational& b) { return cpp_rational::cmp(a, b) op 0; } \
  inline bool operator op(const cpp_rational& a, const cpp_int& b) { return cpp_rational::cmp(a, cpp_rational(b)) op 0; } \
  template <class T, class = std::enable_if_t<std::is_integral_v<T>>>                           \
  inline bool operator op(const cpp_rational& a, T b) { return cpp_rational::cmp(a, cpp_rational(b)) op 0; }
CK_SHIM_RCMP(==)
CK_SHIM_RCMP(!=)
CK_SHIM_RCMP(<)
CK_SHIM_RCMP(>)
CK_SHIM_RCMP(<=)
CK_SHIM_RCMP(>=)
#undef CK_SHIM_RCMP

inline std::ostream& operator<<(std::ostream& os, const cpp_rational& v) {
  return os << v.num() << '/' << v.den();
}

}  // namespace multiprecision
}  // namespace boost
