// ckks32_b200.hpp — header-only C++ mirror of the reference evaluator API
// (/root/reference/proj/include/ckks32/ckks.hpp:102-219) over the C ABI of
// include/ck32_b200.h.
//
// Same names, argument meaning, level/scale ledger and exception types as
// the reference (std::invalid_argument / std::runtime_error); residues live in
// device memory as canonical uint32 (the reference's correct_lazy() view).
// The scale ledger is an exact rational over 64-bit limbs products; the
// reference uses Boost cpp_rational (ckks.hpp:30) — here the numerator and
// denominator are kept as explicit prime-product lists, so equality and
// division by q_{l-2} q_{l-1} are exact without a big-integer library.
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/ck32_b200.h"

namespace ckks32::b200 {

inline void check(ck_status s) {
  if (s == CK_OK) return;
  const std::string msg = ck_last_error();
  if (s == CK_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// Exact scale ledger: value = 2^pow2 * prod(num) / prod(den) (all factors are
// basis primes or powers of two, which is all the hot path produces).
struct Scale {
  int pow2 = 0;
  std::vector<uint32_t> num, den;
  static Scale two_pow(int b) { return Scale{b, {}, {}}; }
  // 2^p2 * prod(n) / prod(d) for arbitrary positive integer factors, reduced
  static Scale rational(int p2, std::vector<uint32_t> n, std::vector<uint32_t> d) {
    Scale r{p2, std::move(n), std::move(d)};
    r.normalize();
    return r;
  }
  Scale operator*(const Scale& o) const {
    Scale r{pow2 + o.pow2, num, den};
    r.num.insert(r.num.end(), o.num.begin(), o.num.end());
    r.den.insert(r.den.end(), o.den.begin(), o.den.end());
    r.normalize();
    return r;
  }
  Scale divided_by(uint32_t a, uint32_t b) const {
    Scale r = *this;
    r.den.push_back(a);
    r.den.push_back(b);
    r.normalize();
    return r;
  }
  // canonical form (the reference's Rational is always reduced): factors of
  // two folded into pow2, every other factor split into primes, common primes
  // cancelled -- equal values compare equal and log2_rational sees the reduced
  // fraction.  Basis primes pass the primality test at once.
  static bool is_prime32(uint32_t n) {  // deterministic Miller-Rabin for 32-bit n
    if (n < 2) return false;
    for (uint32_t p : {2u, 3u, 5u, 7u, 11u, 13u})
      if (n % p == 0) return n == p;
    uint32_t d = n - 1;
    int r = 0;
    while (!(d & 1)) d >>= 1, ++r;
    for (uint64_t a : {2ull, 7ull, 61ull}) {
      uint64_t x = 1, b = a % n, e = d;
      for (; e; e >>= 1, b = b * b % n)
        if (e & 1) x = x * b % n;
      if (x == 1 || x == n - 1) continue;
      bool comp = true;
      for (int i = 1; i < r && comp; ++i) {
        x = x * x % n;
        if (x == n - 1) comp = false;
      }
      if (comp) return false;
    }
    return true;
  }
  static void split(std::vector<uint32_t>& v, int& twos) {
    std::vector<uint32_t> out;
    for (uint32_t f : v) {
      if (f == 0) throw std::invalid_argument("zero scale factor");
      while (!(f & 1)) f >>= 1, ++twos;
      if (f == 1) continue;
      if (is_prime32(f)) {
        out.push_back(f);
        continue;
      }
      for (uint32_t p = 3; (uint64_t)p * p <= f; p += 2)
        while (f % p == 0) out.push_back(p), f /= p;
      if (f > 1) out.push_back(f);
    }
    v = std::move(out);
  }
  void normalize() {
    int tn = 0, td = 0;
    split(num, tn);
    split(den, td);
    pow2 += tn - td;
    std::sort(num.begin(), num.end());
    std::sort(den.begin(), den.end());
    std::vector<uint32_t> n2, d2;
    std::set_difference(num.begin(), num.end(), den.begin(), den.end(), std::back_inserter(n2));
    std::set_difference(den.begin(), den.end(), num.begin(), num.end(), std::back_inserter(d2));
    num = std::move(n2);
    den = std::move(d2);
  }
  bool operator==(const Scale& o) const { return pow2 == o.pow2 && num == o.num && den == o.den; }
};

namespace detail {
// little-endian 32-bit-limb naturals: just enough arithmetic for the ledger
// comparisons (the reference uses Boost cpp_rational, ckks.hpp:30)
using Nat = std::vector<uint32_t>;
inline void nat_trim(Nat& a) {
  while (a.size() > 1 && a.back() == 0) a.pop_back();
}
inline Nat nat_mul(const Nat& a, const Nat& b) {
  Nat r(a.size() + b.size(), 0);
  for (size_t i = 0; i < a.size(); ++i) {
    uint64_t carry = 0;
    for (size_t j = 0; j < b.size(); ++j) {
      const uint64_t t = (uint64_t)a[i] * b[j] + r[i + j] + carry;
      r[i + j] = (uint32_t)t;
      carry = t >> 32;
    }
    r[i + b.size()] += (uint32_t)carry;
  }
  nat_trim(r);
  return r;
}
inline Nat nat_shl(Nat a, int bits) {
  const int words = bits / 32, b = bits % 32;
  if (b) {
    uint32_t carry = 0;
    for (auto& x : a) {
      const uint32_t nx = (x << b) | carry;
      carry = x >> (32 - b);
      x = nx;
    }
    if (carry) a.push_back(carry);
  }
  a.insert(a.begin(), (size_t)words, 0u);
  nat_trim(a);
  return a;
}
inline int nat_cmp(const Nat& a, const Nat& b) {
  if (a.size() != b.size()) return a.size() < b.size() ? -1 : 1;
  for (size_t i = a.size(); i-- > 0;)
    if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
  return 0;
}
inline Nat nat_sub(const Nat& a, const Nat& b) {  // a >= b
  Nat r = a;
  int64_t borrow = 0;
  for (size_t i = 0; i < r.size(); ++i) {
    int64_t t = (int64_t)r[i] - (i < b.size() ? b[i] : 0) - borrow;
    borrow = t < 0;
    r[i] = (uint32_t)(t + (borrow << 32));
  }
  nat_trim(r);
  return r;
}
inline Nat nat_of(const std::vector<uint32_t>& factors, int twos) {
  Nat r{1};
  for (uint32_t f : factors) r = nat_mul(r, Nat{f});
  return nat_shl(r, twos);
}
}  // namespace detail

// check_same_scale (ckks.cpp:131-136): scales must agree within 2^-40
// relative, |a - b| 2^40 <= a, evaluated exactly on cross products
inline void check_same_scale(const Scale& a, const Scale& b) {
  using namespace detail;
  const Nat an = nat_of(a.num, std::max(a.pow2, 0)), ad = nat_of(a.den, std::max(-a.pow2, 0));
  const Nat bn = nat_of(b.num, std::max(b.pow2, 0)), bd = nat_of(b.den, std::max(-b.pow2, 0));
  const Nat x = nat_mul(an, bd), y = nat_mul(bn, ad);  // a = x / (ad bd), b = y / (ad bd)
  const Nat diff = nat_cmp(x, y) >= 0 ? nat_sub(x, y) : nat_sub(y, x);
  if (nat_cmp(nat_shl(diff, 40), x) > 0) throw std::invalid_argument("scale mismatch beyond tolerance");
}

struct CkksParams {  // ckks.hpp:46-54
  uint32_t n = 1u << 16, l = 54, alpha = 14, delta_bits = 48;
  uint32_t hamming = 256;  // secret Hamming weight (host-side sampling)
  double sigma = 3.2;      // error standard deviation
  bool lazy_rescale = false;
};

// Device buffer of uint32 residues.  Ownership is shared so that a result
// the library writes as one block ([v0; v1], [c0; c1], [count][2][level])
// can be handed out as separate objects without device-to-device copies:
// slice() returns a view that keeps the whole allocation alive.
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  DeviceBuffer(ck_context* ctx, size_t words) : ctx_(ctx), words_(words) {
    void* p = nullptr;
    check(ck_malloc(ctx, std::max<size_t>(words, 1) * 4, &p));
    base_ = std::shared_ptr<uint32_t>(static_cast<uint32_t*>(p), [ctx](uint32_t* q) { ck_free(ctx, q); });
    ptr_ = base_.get();
  }
  DeviceBuffer(DeviceBuffer&&) noexcept = default;
  DeviceBuffer& operator=(DeviceBuffer&&) noexcept = default;
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  // a view of words [off, off + words) sharing this allocation
  DeviceBuffer slice(size_t off, size_t words) const {
    if (off + words > words_) throw std::invalid_argument("slice out of range");
    DeviceBuffer v;
    v.ctx_ = ctx_;
    v.base_ = base_;
    v.ptr_ = ptr_ + off;
    v.words_ = words;
    return v;
  }
  uint32_t* data() const { return ptr_; }
  size_t words() const { return words_; }
  ck_context* context() const { return ctx_; }
  void upload(const uint32_t* host, size_t words, ck_stream st = nullptr) {
    check(ck_memcpy_h2d(ctx_, ptr_, host, words * 4, st));
    check(ck_stream_sync(ctx_, st));
  }
  std::vector<uint32_t> download(ck_stream st = nullptr) const {
    std::vector<uint32_t> h(words_);
    check(ck_memcpy_d2h(ctx_, h.data(), ptr_, words_ * 4, st));
    check(ck_stream_sync(ctx_, st));
    return h;
  }

 private:
  ck_context* ctx_ = nullptr;
  std::shared_ptr<uint32_t> base_;
  uint32_t* ptr_ = nullptr;
  size_t words_ = 0;
};

class CkksContext {  // ckks.cpp:160-176
 public:
  explicit CkksContext(CkksParams p, int device = 0, const std::vector<uint32_t>* primes = nullptr) : p_(p) {
    ck_params cp{p.n, p.l, p.alpha, p.delta_bits, p.lazy_rescale ? 1 : 0};
    ck_context* c = nullptr;
    check(ck_context_create(&cp, primes ? primes->data() : nullptr, device, &c));
    ctx_.reset(c);
    primes_.resize(p.l + p.alpha);
    check(ck_context_primes(c, primes_.data()));
  }
  const CkksParams& params() const { return p_; }
  ck_context* raw() const { return ctx_.get(); }
  // every call through this context is issued on this CUDA stream
  // (cudaStream_t; NULL = the legacy default stream).  Calls are asynchronous
  // on it; results are valid once the stream is synchronised (sync()).
  void set_stream(ck_stream st) { st_ = st; }
  ck_stream stream() const { return st_; }
  void sync() const { check(ck_stream_sync(ctx_.get(), st_)); }
  const std::vector<uint32_t>& primes() const { return primes_; }
  uint32_t num_digits(uint32_t level) const { return (level + p_.alpha - 1) / p_.alpha; }
  Scale default_scale() const { return Scale::two_pow((int)p_.delta_bits); }
  std::vector<uint64_t> counters() const {
    std::vector<uint64_t> c(7);
    check(ck_context_counters(ctx_.get(), c.data()));
    return c;
  }

 private:
  struct Del {
    void operator()(ck_context* c) const { ck_context_destroy(c); }
  };
  CkksParams p_;
  ck_stream st_ = nullptr;
  std::unique_ptr<ck_context, Del> ctx_;
  std::vector<uint32_t> primes_;
};

struct Ciphertext {  // ckks.hpp:61-66; data = [2][level][n]
  DeviceBuffer data;
  Scale scale;
  uint32_t level = 0;
  bool pending_rescale = false;
};

enum class KeyKind : uint8_t { Relin = 0, Rotation = 1 };
struct EvaluationKey {  // ckks.hpp:79-84; data = [D][2][L+alpha][n]
  DeviceBuffer data;
  KeyKind kind = KeyKind::Relin;
  int64_t rotation = 0;
};

inline Ciphertext make_ciphertext(CkksContext& ctx, uint32_t level, Scale s) {
  return Ciphertext{DeviceBuffer(ctx.raw(), 2ull * level * ctx.params().n), std::move(s), level, false};
}

inline Ciphertext rescale(CkksContext& ctx, const Ciphertext& ct) {  // ckks.cpp:789-802
  if (ct.level < 4) throw std::invalid_argument("level exhausted");
  Ciphertext out = make_ciphertext(ctx, ct.level - 2,
                                   ct.scale.divided_by(ctx.primes()[ct.level - 2], ctx.primes()[ct.level - 1]));
  check(ck_rescale(ctx.raw(), ct.level, 1, ct.data.data(), out.data.data(), ctx.stream()));
  return out;
}

inline Ciphertext hmult(CkksContext& ctx, const Ciphertext& x_in, const Ciphertext& y_in,
                        const EvaluationKey& relin) {  // ckks.cpp:804-865
  if (relin.kind != KeyKind::Relin) throw std::invalid_argument("hmult needs a relinearization key");
  Ciphertext fx, fy;
  const Ciphertext* x = &x_in;
  const Ciphertext* y = &y_in;
  if (x_in.pending_rescale) fx = rescale(ctx, x_in), x = &fx;  // Flushed (ckks.cpp:664-676)
  if (y_in.pending_rescale) fy = rescale(ctx, y_in), y = &fy;
  if (x->level != y->level) throw std::invalid_argument("level mismatch");
  const uint32_t l = x->level;
  if (l < 4) throw std::invalid_argument("level exhausted");
  const bool lazy = ctx.params().lazy_rescale;
  Scale s = x->scale * y->scale;
  if (!lazy) s = s.divided_by(ctx.primes()[l - 2], ctx.primes()[l - 1]);
  Ciphertext out = make_ciphertext(ctx, lazy ? l : l - 2, s);
  out.pending_rescale = lazy;
  check(ck_hmult(ctx.raw(), l, 1, x->data.data(), y->data.data(), relin.data.data(), out.data.data(), ctx.stream()));
  return out;
}

inline Ciphertext hrot(CkksContext& ctx, const Ciphertext& ct_in, int64_t r,
                       const EvaluationKey& evk) {  // ckks.cpp:890-897
  Ciphertext f;
  const Ciphertext* ct = &ct_in;
  if (ct_in.pending_rescale) f = rescale(ctx, ct_in), ct = &f;
  if (evk.kind != KeyKind::Rotation || evk.rotation != r) throw std::invalid_argument("rotation key mismatch");
  Ciphertext out = make_ciphertext(ctx, ct->level, ct->scale);
  check(ck_hrot(ctx.raw(), ct->level, 1, ct->data.data(), r, evk.data.data(), out.data.data(), ctx.stream()));
  return out;
}

inline Ciphertext hadd(CkksContext& ctx, const Ciphertext& x, const Ciphertext& y) {  // ckks.cpp:557-571
  if (x.level != y.level) throw std::invalid_argument("level mismatch");
  if (x.pending_rescale != y.pending_rescale) throw std::invalid_argument("pending-rescale state mismatch");
  check_same_scale(x.scale, y.scale);
  Ciphertext out = make_ciphertext(ctx, x.level, x.scale);
  out.pending_rescale = x.pending_rescale;
  check(ck_hadd(ctx.raw(), x.level, 1, x.data.data(), y.data.data(), out.data.data(), ctx.stream()));
  return out;
}

struct Plaintext {  // ckks.hpp:56-59; data = [level (+alpha)][n], evaluation domain, Montgomery
  DeviceBuffer data;
  Scale scale;
  uint32_t level = 0;
  uint32_t p_count = 0;
};

// log2_rational (ckks.cpp:140-158) of the ledger value, operation for
// operation: numerator and denominator as exact big integers (the prime
// products times the power of two), each cut to its top 53 bits, then
// shift + log2(num / den).  encode feeds this to the same powl / x87
// rounding as the reference, so plaintexts are bit-identical at any scale.
namespace detail {
struct BigU {  // little-endian 32-bit limbs
  std::vector<uint32_t> w{1};
  void mul(uint32_t m) {
    uint64_t carry = 0;
    for (auto& x : w) {
      const uint64_t t = (uint64_t)x * m + carry;
      x = (uint32_t)t;
      carry = t >> 32;
    }
    if (carry) w.push_back((uint32_t)carry);
  }
  void shl(int b) {
    for (; b >= 31; b -= 31) mul(1u << 31);
    if (b > 0) mul(1u << b);
  }
  int msb() const { return 32 * ((int)w.size() - 1) + 31 - __builtin_clz(w.back()); }
  uint64_t bits(int lo) const {  // floor(value / 2^lo), < 2^53 when lo = msb - 52
    uint64_t v = 0;
    for (int i = 52; i >= 0; --i) {
      const int b = lo + i;
      if (b >= 0 && b / 32 < (int)w.size() && (w[b / 32] >> (b % 32) & 1u)) v |= 1ull << i;
    }
    return v;
  }
};
}  // namespace detail
inline double scale_log2(const Scale& s) {
  detail::BigU num, den;
  for (uint32_t a : s.num) num.mul(a);
  for (uint32_t b : s.den) den.mul(b);
  if (s.pow2 >= 0) num.shl(s.pow2);
  else den.shl(-s.pow2);
  const int bn = num.msb(), bd = den.msb();
  int64_t shift = 0;
  double n = 0, d = 0;
  if (bn > 52) {
    n = (double)num.bits(bn - 52);
    shift += bn - 52;
  } else {
    n = (double)num.bits(0);
  }
  if (bd > 52) {
    d = (double)den.bits(bd - 52);
    shift -= bd - 52;
  } else {
    d = (double)den.bits(0);
  }
  return static_cast<double>(shift) + std::log2(n / d);
}

// encode (ckks.cpp:278-319): host slots -> device plaintext
inline Plaintext encode(CkksContext& ctx, const std::vector<std::complex<double>>& slots, const Scale& scale,
                        uint32_t level, bool p_extend = false) {
  const uint32_t n = ctx.params().n;
  if (slots.size() > n / 2) throw std::invalid_argument("too many slots");
  if (level < 1 || level > ctx.params().l) throw std::invalid_argument("level out of range");
  const uint32_t pc = p_extend ? ctx.params().alpha : 0;
  Plaintext pt{DeviceBuffer(ctx.raw(), (size_t)(level + pc) * n), scale, level, pc};
  void* dz = nullptr;
  const size_t bytes = std::max<size_t>(slots.size(), 1) * 16;
  check(ck_malloc(ctx.raw(), bytes, &dz));
  try {
    if (!slots.empty()) check(ck_memcpy_h2d(ctx.raw(), dz, slots.data(), slots.size() * 16, ctx.stream()));
    check(ck_encode(ctx.raw(), static_cast<const double*>(dz), (uint32_t)slots.size(), scale_log2(scale), level,
                    p_extend ? 1 : 0, pt.data.data(), ctx.stream()));
    check(ck_stream_sync(ctx.raw(), ctx.stream()));
  } catch (...) {
    ck_free(ctx.raw(), dz);
    throw;
  }
  check(ck_free(ctx.raw(), dz));
  return pt;
}

// decode (ckks.cpp:321-362): device plaintext -> n/2 host slots
inline std::vector<std::complex<double>> decode(CkksContext& ctx, const Plaintext& pt) {
  const uint32_t n = ctx.params().n;
  void* dz = nullptr;
  check(ck_malloc(ctx.raw(), (size_t)n / 2 * 16, &dz));
  std::vector<std::complex<double>> out(n / 2);
  try {
    // the exact rational scale: slots bit-identical to the reference's decode (ckks.cpp:353)
    detail::BigU num, den;
    for (uint32_t f : pt.scale.num) num.mul(f);
    for (uint32_t f : pt.scale.den) den.mul(f);
    if (pt.scale.pow2 >= 0) num.shl(pt.scale.pow2);
    else den.shl(-pt.scale.pow2);
    if (num.w.size() <= 8 && den.w.size() <= 8)
      check(ck_decode_rational(ctx.raw(), pt.data.data(), pt.level, scale_log2(pt.scale), num.w.data(),
                               (uint32_t)num.w.size(), den.w.data(), (uint32_t)den.w.size(), static_cast<double*>(dz),
                               ctx.stream()));
    else
      check(ck_decode(ctx.raw(), pt.data.data(), pt.level, scale_log2(pt.scale), static_cast<double*>(dz),
                      ctx.stream()));
    check(ck_memcpy_d2h(ctx.raw(), out.data(), dz, out.size() * 16, ctx.stream()));
    check(ck_stream_sync(ctx.raw(), ctx.stream()));
  } catch (...) {
    ck_free(ctx.raw(), dz);
    throw;
  }
  check(ck_free(ctx.raw(), dz));
  return out;
}

inline Ciphertext pmult(CkksContext& ctx, const Ciphertext& ct, const Plaintext& pt) {  // ckks.cpp:586-600
  if (ct.level != pt.level || pt.p_count != 0) throw std::invalid_argument("level mismatch");
  Ciphertext out = make_ciphertext(ctx, ct.level, ct.scale * pt.scale);
  out.pending_rescale = ct.pending_rescale;
  check(ck_pmult(ctx.raw(), ct.level, 1, ct.data.data(), pt.data.data(), out.data.data(), ctx.stream()));
  return out;
}

inline Ciphertext padd(CkksContext& ctx, const Ciphertext& ct, const Plaintext& pt) {  // ckks.cpp:573-584
  if (ct.level != pt.level || pt.p_count != 0) throw std::invalid_argument("level mismatch");
  check_same_scale(ct.scale, pt.scale);
  Ciphertext out = make_ciphertext(ctx, ct.level, ct.scale);
  out.pending_rescale = ct.pending_rescale;
  check(ck_padd(ctx.raw(), ct.level, 1, ct.data.data(), pt.data.data(), out.data.data(), ctx.stream()));
  return out;
}

// --- key switching building blocks (ckks.hpp:179-189) -----------------------
enum class Domain : uint8_t { Coefficient = 0, Evaluation = 1 };  // poly.hpp:17

// poly.hpp:74-119: device rows, Q prefix then P rows.  row(i) works on a host
// mirror with explicit synchronisation (pull(): device -> host, push():
// host -> device), the GPU counterpart of the reference's host row pointers
// (poly.hpp:94-97).
struct Polynomial {
  DeviceBuffer data;
  uint32_t q_count = 0, p_count = 0;
  Domain domain = Domain::Evaluation;
  bool mont = true;
  std::vector<uint32_t> host;

  uint32_t rows() const { return q_count + p_count; }
  size_t n() const { return rows() ? data.words() / rows() : 0; }
  void pull(ck_stream st = nullptr) { host = data.download(st); }
  void push(ck_stream st = nullptr) {
    if (host.size() != data.words()) throw std::invalid_argument("host mirror not pulled");
    data.upload(host.data(), host.size(), st);
  }
  uint32_t* row(uint32_t i) {
    if (host.size() != data.words()) throw std::invalid_argument("host mirror not pulled (call pull())");
    return host.data() + (size_t)i * n();
  }
  const uint32_t* row(uint32_t i) const {
    if (host.size() != data.words()) throw std::invalid_argument("host mirror not pulled (call pull())");
    return host.data() + (size_t)i * n();
  }
};
struct HoistState {  // ckks.hpp:88-91: D x (level + alpha) rows
  DeviceBuffer digits;
  uint32_t level = 0, D = 0;
};

inline HoistState mod_up(CkksContext& ctx, const Polynomial& d) {  // ckks.cpp:680-731
  if (d.p_count != 0) throw std::invalid_argument("mod_up input must be Q-only");
  const uint32_t l = d.q_count, D = ctx.num_digits(l), n = ctx.params().n;
  HoistState h{DeviceBuffer(ctx.raw(), (size_t)D * (l + ctx.params().alpha) * n), l, D};
  check(ck_mod_up(ctx.raw(), l, d.data.data(), h.digits.data(), ctx.stream()));
  return h;
}

inline std::pair<Polynomial, Polynomial> key_mult(CkksContext& ctx, const HoistState& h,
                                                  const EvaluationKey& evk) {  // ckks.cpp:733-770
  const uint32_t rows = h.level + ctx.params().alpha, n = ctx.params().n;
  if (evk.data.words() < (size_t)h.D * 2 * (ctx.params().l + ctx.params().alpha) * n)
    throw std::invalid_argument("evaluation key has too few digits");
  DeviceBuffer v(ctx.raw(), 2ull * rows * n);
  check(ck_key_mult(ctx.raw(), h.level, h.digits.data(), evk.data.data(), v.data(), ctx.stream()));
  // v0 and v1 are the two halves of the one block the kernel wrote (no copies)
  return {Polynomial{v.slice(0, (size_t)rows * n), h.level, ctx.params().alpha},
          Polynomial{v.slice((size_t)rows * n, (size_t)rows * n), h.level, ctx.params().alpha}};
}

inline Polynomial mod_down(CkksContext& ctx, const Polynomial& v) {  // ckks.cpp:772-776
  if (v.p_count != ctx.params().alpha) throw std::invalid_argument("mod_down expects a P-extended polynomial");
  Polynomial out{DeviceBuffer(ctx.raw(), (size_t)v.q_count * ctx.params().n), v.q_count, 0};
  check(ck_mod_down(ctx.raw(), v.q_count, v.data.data(), out.data.data(), ctx.stream()));
  return out;
}

inline std::pair<Polynomial, Polynomial> key_switch(CkksContext& ctx, const Polynomial& d,
                                                    const EvaluationKey& evk) {  // ckks.cpp:778-787
  if (d.p_count != 0) throw std::invalid_argument("mod_up input must be Q-only");
  const uint32_t l = d.q_count, n = ctx.params().n;
  DeviceBuffer out(ctx.raw(), 2ull * l * n);
  check(ck_key_switch(ctx.raw(), l, d.data.data(), evk.data.data(), out.data(), ctx.stream()));
  return {Polynomial{out.slice(0, (size_t)l * n), l, 0}, Polynomial{out.slice((size_t)l * n, (size_t)l * n), l, 0}};
}

// hoisted_rotations (ckks.cpp:899-925): one ModUp shared by every rotation
inline std::vector<Ciphertext> hoisted_rotations(CkksContext& ctx, const Ciphertext& ct,
                                                 const std::vector<int64_t>& rots,
                                                 const std::vector<const EvaluationKey*>& evks) {
  if (rots.size() != evks.size()) throw std::invalid_argument("rotation/key count mismatch");
  std::vector<const uint32_t*> kp(rots.size());
  for (size_t i = 0; i < rots.size(); ++i) {
    if (rots[i] != 0 && (!evks[i] || evks[i]->kind != KeyKind::Rotation || evks[i]->rotation != rots[i]))
      throw std::invalid_argument("rotation key mismatch");
    kp[i] = rots[i] != 0 ? evks[i]->data.data() : nullptr;
  }
  const size_t w = 2ull * ct.level * ctx.params().n;
  DeviceBuffer all(ctx.raw(), std::max<size_t>(1, rots.size()) * w);
  check(ck_hoisted_rotations(ctx.raw(), ct.level, ct.data.data(), (uint32_t)rots.size(), rots.data(), kp.data(),
                             all.data(), ctx.stream()));
  std::vector<Ciphertext> out;
  for (size_t i = 0; i < rots.size(); ++i) out.push_back(Ciphertext{all.slice(i * w, w), ct.scale, ct.level, false});
  return out;
}

// hoisted_rotate_accumulate (ckks.cpp:945-1012): sum_i pt_i * rot_{r_i}(ct) with
// one ModUp and one ModDown; plaintexts P-extended at the ciphertext level
// (rotation 0 needs no key: pass nullptr)
inline Ciphertext hoisted_rotate_accumulate(CkksContext& ctx, const Ciphertext& ct_in,
                                            const std::vector<int64_t>& rots,
                                            const std::vector<const Plaintext*>& pts,
                                            const std::vector<const EvaluationKey*>& evks) {
  if (rots.empty() || rots.size() != pts.size() || rots.size() != evks.size())
    throw std::invalid_argument("rotation/plaintext/key count mismatch");
  Ciphertext f;
  const Ciphertext* ct = &ct_in;
  if (ct_in.pending_rescale) f = rescale(ctx, ct_in), ct = &f;  // Flushed (ckks.cpp:664-676)
  std::vector<const uint32_t*> pp(rots.size()), kp(rots.size(), nullptr);
  for (size_t i = 0; i < rots.size(); ++i) {
    if (!pts[i]) throw std::invalid_argument("missing plaintext");
    if (pts[i]->level != ct->level || pts[i]->p_count != ctx.params().alpha)
      throw std::invalid_argument("plaintexts must be P-extended at the ciphertext level");
    check_same_scale(pts[0]->scale, pts[i]->scale);
    pp[i] = pts[i]->data.data();
    if (rots[i] == 0) continue;
    if (!evks[i] || evks[i]->kind != KeyKind::Rotation || evks[i]->rotation != rots[i])
      throw std::invalid_argument("rotation key mismatch");
    kp[i] = evks[i]->data.data();
  }
  Ciphertext out = make_ciphertext(ctx, ct->level, ct->scale * pts[0]->scale);
  check(ck_hoisted_rotate_accumulate(ctx.raw(), ct->level, ct->data.data(), (uint32_t)rots.size(), rots.data(),
                                     pp.data(), kp.data(), out.data.data(), ctx.stream()));
  return out;
}

// --- kernel level (ntt.hpp:90-91, bconv.hpp:53-54, automorphism.hpp:51-52, poly.hpp:123-130)
namespace detail {
inline std::vector<uint32_t> gidx(const CkksContext& ctx, const Polynomial& p) {  // poly.hpp:103-106
  std::vector<uint32_t> g(p.rows());
  for (uint32_t i = 0; i < p.rows(); ++i) g[i] = i < p.q_count ? i : ctx.params().l + (i - p.q_count);
  return g;
}
inline void check_binary(const Polynomial& a, const Polynomial& b) {  // poly.cpp:115-119
  if (a.q_count != b.q_count || a.p_count != b.p_count) throw std::invalid_argument("basis prefix mismatch");
  if (a.domain != b.domain) throw std::invalid_argument("domain mismatch");
  if (a.mont != b.mont) throw std::invalid_argument("Montgomery flag mismatch");
}
}  // namespace detail

inline void ntt_forward(CkksContext& ctx, Polynomial& p) {  // ntt.cpp:288-299
  if (p.domain != Domain::Coefficient) throw std::invalid_argument("ntt_forward expects coefficient domain");
  if (p.mont) throw std::invalid_argument("ntt_forward expects plain form (entry merge)");
  const auto g = detail::gidx(ctx, p);
  check(ck_ntt_forward(ctx.raw(), p.data.data(), p.rows(), g.data(), ctx.stream()));
  p.domain = Domain::Evaluation;
  p.mont = true;
}

// intt_inverse (ntt.cpp:301-312); epilogue_mont (one canonical Montgomery
// constant per row) = NttPlan::inverse_row's fused part-1 epilogue (ntt.hpp:72-73)
inline void intt_inverse(CkksContext& ctx, Polynomial& p, const uint32_t* epilogue_mont = nullptr) {
  if (p.domain != Domain::Evaluation) throw std::invalid_argument("intt_inverse expects evaluation domain");
  if (!p.mont) throw std::invalid_argument("intt_inverse expects Montgomery form");
  const auto g = detail::gidx(ctx, p);
  check(ck_intt_inverse(ctx.raw(), p.data.data(), p.rows(), g.data(), epilogue_mont, ctx.stream()));
  p.domain = Domain::Coefficient;
  p.mont = false;
}

// BConvTable (bconv.hpp:17-30) by global prime index; c (centred Montgomery
// (P/P_j) mod q_i, [dst][src]) may be supplied, else the library derives it
struct BConvTable {
  std::vector<uint32_t> src, dst;
  std::vector<int32_t> c;
};
inline BConvTable make_bconv_table(std::vector<uint32_t> src_gidx, std::vector<uint32_t> dst_gidx) {
  return BConvTable{std::move(src_gidx), std::move(dst_gidx), {}};
}
// bconv_part2 (bconv.cpp:96-174): src = src.size() contiguous canonical rows,
// dst = dst.size() contiguous rows
inline void bconv_part2(CkksContext& ctx, const uint32_t* src, const BConvTable& t, uint32_t* dst) {
  if (t.c.empty())
    check(ck_bconv(ctx.raw(), src, (uint32_t)t.src.size(), t.src.data(), dst, (uint32_t)t.dst.size(), t.dst.data(),
                   ctx.stream()));
  else
    check(ck_bconv_table(ctx.raw(), src, (uint32_t)t.src.size(), t.src.data(), dst, (uint32_t)t.dst.size(),
                         t.dst.data(), t.c.data(), ctx.stream()));
}

// mod_switch (bconv.cpp:176-213): evaluation rows over src_gidx -> Q_[0, dst_q) + P_[0, dst_p)
inline Polynomial mod_switch(CkksContext& ctx, const Polynomial& a, const std::vector<uint32_t>& src_gidx,
                             uint32_t dst_q, uint32_t dst_p) {
  if (a.domain != Domain::Evaluation || !a.mont)
    throw std::invalid_argument("mod_switch expects evaluation-domain Montgomery input");
  if (a.rows() != src_gidx.size()) throw std::invalid_argument("input rows do not match table source");
  Polynomial out{DeviceBuffer(ctx.raw(), (size_t)(dst_q + dst_p) * ctx.params().n), dst_q, dst_p};
  check(ck_mod_switch(ctx.raw(), a.data.data(), a.rows(), src_gidx.data(), out.data.data(), dst_q, dst_p,
                      ctx.stream()));
  return out;
}

// AutomorphismMap (automorphism.hpp:18-49) by its Galois element
struct AutomorphismMap {
  uint32_t n = 0;
  int64_t r = 0;
  uint64_t galois = 1;
  static AutomorphismMap rotation(uint32_t n, int64_t r) {  // 5^-r mod 2n (automorphism.cpp:11-23)
    const int64_t half = n / 2;
    int64_t e = (-r) % half;
    if (e < 0) e += half;
    uint64_t g = 1;
    for (int64_t i = 0; i < e; ++i) g = g * 5 % (2ull * n);
    return {n, r, g};
  }
  static AutomorphismMap conjugation(uint32_t n) { return {n, 0, 2ull * n - 1}; }
};
// apply_automorphism (automorphism.cpp:76-100), either domain
inline Polynomial apply_automorphism(CkksContext& ctx, const Polynomial& p, const AutomorphismMap& map) {
  if (map.n != ctx.params().n) throw std::invalid_argument("ring degree mismatch");
  Polynomial out{DeviceBuffer(ctx.raw(), p.data.words()), p.q_count, p.p_count, p.domain, p.mont};
  check(ck_automorphism_galois(ctx.raw(), p.data.data(), out.data.data(), p.q_count, p.p_count, map.galois,
                               p.domain == Domain::Coefficient, ctx.stream()));
  return out;
}

// element-wise (poly.cpp:121-205), Q-prefix or P-extended
namespace detail {
inline Polynomial ew(CkksContext& ctx, int op, const Polynomial& a, const Polynomial& b, bool mont_out) {
  check_binary(a, b);
  Polynomial out{DeviceBuffer(ctx.raw(), a.data.words()), a.q_count, a.p_count, a.domain, mont_out};
  check(ck_ew_binary(ctx.raw(), op, a.data.data(), b.data.data(), out.data.data(), a.q_count, a.p_count,
                     ctx.stream()));
  return out;
}
}  // namespace detail
inline Polynomial ew_add(CkksContext& ctx, const Polynomial& a, const Polynomial& b) {
  return detail::ew(ctx, 0, a, b, a.mont);
}
inline Polynomial ew_sub(CkksContext& ctx, const Polynomial& a, const Polynomial& b) {
  return detail::ew(ctx, 1, a, b, a.mont);
}
inline Polynomial ew_mul(CkksContext& ctx, const Polynomial& a, const Polynomial& b) {
  if (!a.mont || !b.mont) throw std::invalid_argument("ew_mul expects Montgomery-form operands");
  return detail::ew(ctx, 2, a, b, true);
}
inline Polynomial ew_mul_const(CkksContext& ctx, const Polynomial& a, const std::vector<uint32_t>& consts_mont) {
  if (consts_mont.size() != a.rows()) throw std::invalid_argument("constant count mismatch");
  Polynomial out{DeviceBuffer(ctx.raw(), a.data.words()), a.q_count, a.p_count, a.domain, a.mont};
  check(ck_ew_mul_const(ctx.raw(), a.data.data(), consts_mont.data(), out.data.data(), a.q_count, a.p_count,
                        ctx.stream()));
  return out;
}
inline void ew_add_inplace(CkksContext& ctx, Polynomial& a, const Polynomial& b) {
  detail::check_binary(a, b);
  check(ck_ew_binary(ctx.raw(), 0, a.data.data(), b.data.data(), a.data.data(), a.q_count, a.p_count, ctx.stream()));
}
inline void ew_sub_inplace(CkksContext& ctx, Polynomial& a, const Polynomial& b) {
  detail::check_binary(a, b);
  check(ck_ew_binary(ctx.raw(), 1, a.data.data(), b.data.data(), a.data.data(), a.q_count, a.p_count, ctx.stream()));
}

// --- batches: B independent ciphertexts [B][2][level][n] sharing one key, one
// launch sequence per mechanism (the throughput path bench.py measures) ------
struct CiphertextBatch {
  DeviceBuffer data;
  Scale scale;
  uint32_t level = 0, batch = 0;
  bool pending_rescale = false;
  // element i as a Ciphertext view (no copy)
  Ciphertext operator[](uint32_t i) const {
    const size_t w = data.words() / std::max<uint32_t>(batch, 1);
    return Ciphertext{data.slice(i * w, w), scale, level, pending_rescale};
  }
};
inline CiphertextBatch make_batch(CkksContext& ctx, uint32_t batch, uint32_t level, Scale s) {
  return CiphertextBatch{DeviceBuffer(ctx.raw(), 2ull * batch * level * ctx.params().n), std::move(s), level, batch,
                         false};
}
inline CiphertextBatch rescale(CkksContext& ctx, const CiphertextBatch& x) {  // ckks.cpp:789-802
  if (x.level < 4) throw std::invalid_argument("level exhausted");
  CiphertextBatch out = make_batch(ctx, x.batch, x.level - 2,
                                   x.scale.divided_by(ctx.primes()[x.level - 2], ctx.primes()[x.level - 1]));
  check(ck_rescale(ctx.raw(), x.level, x.batch, x.data.data(), out.data.data(), ctx.stream()));
  return out;
}
inline CiphertextBatch hmult(CkksContext& ctx, const CiphertextBatch& x_in, const CiphertextBatch& y_in,
                             const EvaluationKey& relin) {  // ckks.cpp:804-865, batched
  if (relin.kind != KeyKind::Relin) throw std::invalid_argument("hmult needs a relinearization key");
  CiphertextBatch fx, fy;
  const CiphertextBatch* x = &x_in;
  const CiphertextBatch* y = &y_in;
  if (x_in.pending_rescale) fx = rescale(ctx, x_in), x = &fx;
  if (y_in.pending_rescale) fy = rescale(ctx, y_in), y = &fy;
  if (x->level != y->level || x->batch != y->batch) throw std::invalid_argument("level mismatch");
  const uint32_t l = x->level;
  if (l < 4) throw std::invalid_argument("level exhausted");
  const bool lazy = ctx.params().lazy_rescale;
  Scale s = x->scale * y->scale;
  if (!lazy) s = s.divided_by(ctx.primes()[l - 2], ctx.primes()[l - 1]);
  CiphertextBatch out = make_batch(ctx, x->batch, lazy ? l : l - 2, s);
  out.pending_rescale = lazy;
  check(ck_hmult(ctx.raw(), l, x->batch, x->data.data(), y->data.data(), relin.data.data(), out.data.data(),
                 ctx.stream()));
  return out;
}
inline CiphertextBatch hrot(CkksContext& ctx, const CiphertextBatch& x_in, int64_t r,
                            const EvaluationKey& evk) {  // ckks.cpp:890-897, batched
  CiphertextBatch f;
  const CiphertextBatch* x = &x_in;
  if (x_in.pending_rescale) f = rescale(ctx, x_in), x = &f;
  if (evk.kind != KeyKind::Rotation || evk.rotation != r) throw std::invalid_argument("rotation key mismatch");
  CiphertextBatch out = make_batch(ctx, x->batch, x->level, x->scale);
  check(ck_hrot(ctx.raw(), x->level, x->batch, x->data.data(), r, evk.data.data(), out.data.data(), ctx.stream()));
  return out;
}
inline CiphertextBatch hadd(CkksContext& ctx, const CiphertextBatch& x, const CiphertextBatch& y) {
  if (x.level != y.level || x.batch != y.batch) throw std::invalid_argument("level mismatch");
  if (x.pending_rescale != y.pending_rescale) throw std::invalid_argument("pending-rescale state mismatch");
  check_same_scale(x.scale, y.scale);
  CiphertextBatch out = make_batch(ctx, x.batch, x.level, x.scale);
  out.pending_rescale = x.pending_rescale;
  check(ck_hadd(ctx.raw(), x.level, x.batch, x.data.data(), y.data.data(), out.data.data(), ctx.stream()));
  return out;
}
inline CiphertextBatch pmult(CkksContext& ctx, const CiphertextBatch& x, const Plaintext& pt) {
  if (x.level != pt.level || pt.p_count != 0) throw std::invalid_argument("level mismatch");
  CiphertextBatch out = make_batch(ctx, x.batch, x.level, x.scale * pt.scale);
  out.pending_rescale = x.pending_rescale;
  check(ck_pmult(ctx.raw(), x.level, x.batch, x.data.data(), pt.data.data(), out.data.data(), ctx.stream()));
  return out;
}

// decrypt (ckks.cpp:541-553): m = b + a s; `s` = the secret's evaluation rows (>= level)
inline Plaintext decrypt(CkksContext& ctx, const Ciphertext& ct, const DeviceBuffer& s) {
  Plaintext pt{DeviceBuffer(ctx.raw(), (size_t)ct.level * ctx.params().n), ct.scale, ct.level, 0};
  check(ck_decrypt(ctx.raw(), ct.level, 1, ct.data.data(), s.data(), pt.data.data(), ctx.stream()));
  return pt;
}

// ---- keys and encryption with the caller's std::mt19937_64 (ckks.hpp:155-167) ----
// The randomness is drawn on the host from the caller's generator in the
// reference's order and with its formulas (Box-Muller on two 53-bit draws,
// Fisher-Yates ternary positions, rng() % q residues: ckks.cpp:33-60,
// 383-395), so a generator state yields the reference's keys and ciphertexts
// bit for bit; the arithmetic (coeffs_to_eval NTTs, the products) is on the GPU.
namespace detail {
inline std::vector<int64_t> gaussian(std::mt19937_64& rng, uint32_t n, double sigma) {
  std::vector<int64_t> out(n);
  for (auto& v : out) {
    const double u1 = (static_cast<double>(rng() >> 11) + 0.5) * 0x1p-53;
    const double u2 = static_cast<double>(rng() >> 11) * 0x1p-53;
    const double r = std::sqrt(-2.0 * std::log(u1));
    v = std::llround(r * std::cos(2.0 * 3.141592653589793238462643383279502884 * u2) * sigma);
  }
  return out;
}
inline std::vector<int64_t> ternary(std::mt19937_64& rng, uint32_t n, uint32_t h) {
  if (h > n) throw std::invalid_argument("hamming weight exceeds n");
  std::vector<uint32_t> pos(n);
  for (uint32_t i = 0; i < n; ++i) pos[i] = i;
  std::vector<int64_t> out(n, 0);
  for (uint32_t i = 0; i < h; ++i) {  // partial Fisher-Yates: position i picks from [i, n)
    std::swap(pos[i], pos[i + static_cast<uint32_t>(rng() % (n - i))]);
    out[pos[i]] = (rng() & 1) ? 1 : -1;
  }
  return out;
}
// coeffs_to_eval (ckks.cpp:366-380) on the GPU: [level + pc][n]
inline DeviceBuffer coeffs_to_eval(CkksContext& ctx, const std::vector<int64_t>& c, uint32_t level, uint32_t pc) {
  const uint32_t n = ctx.params().n;
  DeviceBuffer dc(ctx.raw(), 2ull * n);
  dc.upload(reinterpret_cast<const uint32_t*>(c.data()), 2ull * n);
  DeviceBuffer out(ctx.raw(), (size_t)(level + pc) * n);
  check(ck_coeffs_to_eval(ctx.raw(), reinterpret_cast<const int64_t*>(dc.data()), level, pc, out.data(), ctx.stream()));
  check(ck_stream_sync(ctx.raw(), ctx.stream()));
  return out;
}
// uniform_eval (ckks.cpp:383-395): Q rows [0, qc) then P rows [0, pc), rng() % q
inline DeviceBuffer uniform_eval(CkksContext& ctx, std::mt19937_64& rng, uint32_t qc, uint32_t pc) {
  const uint32_t n = ctx.params().n, L = ctx.params().l;
  std::vector<uint32_t> h((size_t)(qc + pc) * n);
  for (uint32_t i = 0; i < qc + pc; ++i) {
    const uint64_t q = ctx.primes()[i < qc ? i : L + (i - qc)];
    for (uint32_t k = 0; k < n; ++k) h[(size_t)i * n + k] = static_cast<uint32_t>(rng() % q);
  }
  DeviceBuffer out(ctx.raw(), h.size());
  out.upload(h.data(), h.size());
  return out;
}
}  // namespace detail

struct SecretKey {  // ckks.hpp:68-71: coefficients and evaluation rows over L + alpha
  std::vector<int64_t> coeffs;
  DeviceBuffer s;
};
struct PublicKey {  // ckks.hpp:73-77: (b, a) at level L, data = [2][L][n]
  DeviceBuffer data;
};

inline SecretKey keygen(CkksContext& ctx, std::mt19937_64& rng) {  // ckks.cpp:399-405
  SecretKey sk;
  sk.coeffs = detail::ternary(rng, ctx.params().n, ctx.params().hamming);
  sk.s = detail::coeffs_to_eval(ctx, sk.coeffs, ctx.params().l, ctx.params().alpha);
  return sk;
}

namespace detail {
inline void encrypt_sk_into(CkksContext& ctx, uint32_t l, const uint32_t* m, const SecretKey& sk,
                            std::mt19937_64& rng, uint32_t* out) {
  DeviceBuffer a = uniform_eval(ctx, rng, l, 0);
  DeviceBuffer e = coeffs_to_eval(ctx, gaussian(rng, ctx.params().n, ctx.params().sigma), l, 0);
  check(ck_encrypt_sk(ctx.raw(), l, m, a.data(), e.data(), sk.s.data(), out, ctx.stream()));
  check(ck_stream_sync(ctx.raw(), ctx.stream()));
}
}  // namespace detail

inline PublicKey pubkey_gen(CkksContext& ctx, const SecretKey& sk, std::mt19937_64& rng) {  // ckks.cpp:407-424
  const uint32_t l = ctx.params().l, n = ctx.params().n;
  DeviceBuffer zero(ctx.raw(), (size_t)l * n);
  std::vector<uint32_t> z((size_t)l * n, 0);
  zero.upload(z.data(), z.size());
  PublicKey pk{DeviceBuffer(ctx.raw(), 2ull * l * n)};
  detail::encrypt_sk_into(ctx, l, zero.data(), sk, rng, pk.data.data());
  return pk;
}

// evk_gen (ckks.cpp:426-477): digit k = (b_k, a_k) with b_k = e_k + g_k s_src - a_k s_dst
// over the full L + alpha rows; relinearisation s_src = s^2, s_dst = s;
// rotation r s_src = s, s_dst = phi_{-r}(s).  The gadget factor
// g_k = P dhat_k (dhat_k^-1 mod d_k) needs no big integers here: it is
// P mod q for the primes q of digit k and 0 mod every other prime.
inline EvaluationKey evk_gen(CkksContext& ctx, const SecretKey& sk, KeyKind kind, int64_t rotation,
                             std::mt19937_64& rng) {
  const uint32_t L = ctx.params().l, A = ctx.params().alpha, n = ctx.params().n, rows = L + A;
  const uint32_t D = ctx.num_digits(L);
  const size_t poly = (size_t)rows * n;
  EvaluationKey evk{DeviceBuffer(ctx.raw(), (size_t)D * 2 * poly), kind, kind == KeyKind::Rotation ? rotation : 0};
  const uint32_t* s = sk.s.data();
  DeviceBuffer rot;
  const uint32_t* s_dst = s;
  if (kind == KeyKind::Rotation) {
    rot = DeviceBuffer(ctx.raw(), poly);
    check(ck_automorphism(ctx.raw(), s, rot.data(), rows, -rotation, ctx.stream()));
    s_dst = rot.data();
  }
  const auto& pr = ctx.primes();
  for (uint32_t k = 0; k < D; ++k) {
    std::vector<uint32_t> gm(rows, 0u);
    for (uint32_t i = k * A; i < std::min((k + 1) * A, L); ++i) {
      const uint64_t q = pr[i];
      uint64_t pm = 1;
      for (uint32_t j = 0; j < A; ++j) pm = pm * (pr[L + j] % q) % q;
      gm[i] = (uint32_t)((pm << 32) % q);  // Montgomery form
    }
    DeviceBuffer a = detail::uniform_eval(ctx, rng, L, A);
    DeviceBuffer e = detail::coeffs_to_eval(ctx, detail::gaussian(rng, n, ctx.params().sigma), L, A);
    uint32_t* bk = evk.data.data() + (size_t)k * 2 * poly;
    check(ck_memcpy_d2d(ctx.raw(), bk + poly, a.data(), poly * 4, ctx.stream()));
    check(ck_evk_digit(ctx.raw(), s, s_dst, a.data(), e.data(), gm.data(), kind == KeyKind::Relin ? 1 : 0, bk,
                       ctx.stream()));
  }
  check(ck_stream_sync(ctx.raw(), ctx.stream()));
  return evk;
}

// encrypt (ckks.cpp:497-539): (m + e - a s, a) / (v pk.b + e0 + m, v pk.a + e1)
inline Ciphertext encrypt(CkksContext& ctx, const Plaintext& pt, const SecretKey& sk, std::mt19937_64& rng) {
  if (pt.p_count != 0) throw std::invalid_argument("cannot encrypt a P-extended plaintext");
  Ciphertext ct = make_ciphertext(ctx, pt.level, pt.scale);
  detail::encrypt_sk_into(ctx, pt.level, pt.data.data(), sk, rng, ct.data.data());
  return ct;
}
inline Ciphertext encrypt(CkksContext& ctx, const Plaintext& pt, const PublicKey& pk, std::mt19937_64& rng) {
  if (pt.p_count != 0) throw std::invalid_argument("cannot encrypt a P-extended plaintext");
  const uint32_t l = pt.level, n = ctx.params().n, L = ctx.params().l;
  DeviceBuffer v = detail::coeffs_to_eval(ctx, detail::ternary(rng, n, ctx.params().hamming), l, 0);
  DeviceBuffer e0 = detail::coeffs_to_eval(ctx, detail::gaussian(rng, n, ctx.params().sigma), l, 0);
  DeviceBuffer e1 = detail::coeffs_to_eval(ctx, detail::gaussian(rng, n, ctx.params().sigma), l, 0);
  DeviceBuffer pkl(ctx.raw(), 2ull * l * n);  // the level-l prefix of both halves
  check(ck_memcpy_d2d(ctx.raw(), pkl.data(), pk.data.data(), (size_t)l * n * 4, ctx.stream()));
  check(ck_memcpy_d2d(ctx.raw(), pkl.data() + (size_t)l * n, pk.data.data() + (size_t)L * n, (size_t)l * n * 4,
                      ctx.stream()));
  Ciphertext ct = make_ciphertext(ctx, l, pt.scale);
  check(ck_encrypt_pk(ctx.raw(), l, pt.data.data(), v.data(), e0.data(), e1.data(), pkl.data(), ct.data.data(),
                      ctx.stream()));
  check(ck_stream_sync(ctx.raw(), ctx.stream()));
  return ct;
}

}  // namespace ckks32::b200
