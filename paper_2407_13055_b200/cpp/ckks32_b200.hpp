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

struct CkksParams {  // ckks.hpp:46-54
  uint32_t n = 1u << 16, l = 54, alpha = 14, delta_bits = 48;
  uint32_t hamming = 256;  // secret Hamming weight (host-side sampling)
  double sigma = 3.2;      // error standard deviation
  bool lazy_rescale = false;
};

// Owning device buffer of uint32 residues.
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  DeviceBuffer(ck_context* ctx, size_t words) : ctx_(ctx), words_(words) {
    void* p = nullptr;
    check(ck_malloc(ctx, words * 4, &p));
    ptr_ = static_cast<uint32_t*>(p);
  }
  DeviceBuffer(DeviceBuffer&& o) noexcept { *this = std::move(o); }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    std::swap(ctx_, o.ctx_);
    std::swap(ptr_, o.ptr_);
    std::swap(words_, o.words_);
    return *this;
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  ~DeviceBuffer() {
    if (ptr_) ck_free(ctx_, ptr_);
  }
  uint32_t* data() const { return ptr_; }
  size_t words() const { return words_; }
  void upload(const uint32_t* host, size_t words) {
    check(ck_memcpy_h2d(ctx_, ptr_, host, words * 4, nullptr));
    check(ck_stream_sync(ctx_, nullptr));
  }
  std::vector<uint32_t> download() const {
    std::vector<uint32_t> h(words_);
    check(ck_memcpy_d2h(ctx_, h.data(), ptr_, words_ * 4, nullptr));
    check(ck_stream_sync(ctx_, nullptr));
    return h;
  }

 private:
  ck_context* ctx_ = nullptr;
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
  check(ck_rescale(ctx.raw(), ct.level, 1, ct.data.data(), out.data.data(), nullptr));
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
  check(ck_hmult(ctx.raw(), l, 1, x->data.data(), y->data.data(), relin.data.data(), out.data.data(), nullptr));
  return out;
}

inline Ciphertext hrot(CkksContext& ctx, const Ciphertext& ct_in, int64_t r,
                       const EvaluationKey& evk) {  // ckks.cpp:890-897
  Ciphertext f;
  const Ciphertext* ct = &ct_in;
  if (ct_in.pending_rescale) f = rescale(ctx, ct_in), ct = &f;
  if (evk.kind != KeyKind::Rotation || evk.rotation != r) throw std::invalid_argument("rotation key mismatch");
  Ciphertext out = make_ciphertext(ctx, ct->level, ct->scale);
  check(ck_hrot(ctx.raw(), ct->level, 1, ct->data.data(), r, evk.data.data(), out.data.data(), nullptr));
  return out;
}

inline Ciphertext hadd(CkksContext& ctx, const Ciphertext& x, const Ciphertext& y) {  // ckks.cpp:557-571
  if (x.level != y.level) throw std::invalid_argument("level mismatch");
  if (x.pending_rescale != y.pending_rescale) throw std::invalid_argument("pending-rescale state mismatch");
  if (!(x.scale == y.scale)) throw std::invalid_argument("scale mismatch beyond tolerance");
  Ciphertext out = make_ciphertext(ctx, x.level, x.scale);
  out.pending_rescale = x.pending_rescale;
  check(ck_hadd(ctx.raw(), x.level, 1, x.data.data(), y.data.data(), out.data.data(), nullptr));
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
    if (!slots.empty()) check(ck_memcpy_h2d(ctx.raw(), dz, slots.data(), slots.size() * 16, nullptr));
    check(ck_encode(ctx.raw(), static_cast<const double*>(dz), (uint32_t)slots.size(), scale_log2(scale), level,
                    p_extend ? 1 : 0, pt.data.data(), nullptr));
    check(ck_stream_sync(ctx.raw(), nullptr));
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
    check(ck_decode(ctx.raw(), pt.data.data(), pt.level, scale_log2(pt.scale), static_cast<double*>(dz), nullptr));
    check(ck_memcpy_d2h(ctx.raw(), out.data(), dz, out.size() * 16, nullptr));
    check(ck_stream_sync(ctx.raw(), nullptr));
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
  check(ck_pmult(ctx.raw(), ct.level, 1, ct.data.data(), pt.data.data(), out.data.data(), nullptr));
  return out;
}

inline Ciphertext padd(CkksContext& ctx, const Ciphertext& ct, const Plaintext& pt) {  // ckks.cpp:573-584
  if (ct.level != pt.level || pt.p_count != 0) throw std::invalid_argument("level mismatch");
  if (!(ct.scale == pt.scale)) throw std::invalid_argument("scale mismatch beyond tolerance");
  Ciphertext out = make_ciphertext(ctx, ct.level, ct.scale);
  out.pending_rescale = ct.pending_rescale;
  check(ck_padd(ctx.raw(), ct.level, 1, ct.data.data(), pt.data.data(), out.data.data(), nullptr));
  return out;
}

// --- key switching building blocks (ckks.hpp:179-189) -----------------------
struct Polynomial {  // poly.hpp:74-119 (device rows, Q prefix then P rows; evaluation domain, Montgomery)
  DeviceBuffer data;
  uint32_t q_count = 0, p_count = 0;
};
struct HoistState {  // ckks.hpp:88-91: D x (level + alpha) rows
  DeviceBuffer digits;
  uint32_t level = 0, D = 0;
};

inline HoistState mod_up(CkksContext& ctx, const Polynomial& d) {  // ckks.cpp:680-731
  if (d.p_count != 0) throw std::invalid_argument("mod_up input must be Q-only");
  const uint32_t l = d.q_count, D = ctx.num_digits(l), n = ctx.params().n;
  HoistState h{DeviceBuffer(ctx.raw(), (size_t)D * (l + ctx.params().alpha) * n), l, D};
  check(ck_mod_up(ctx.raw(), l, d.data.data(), h.digits.data(), nullptr));
  return h;
}

inline std::pair<Polynomial, Polynomial> key_mult(CkksContext& ctx, const HoistState& h,
                                                  const EvaluationKey& evk) {  // ckks.cpp:733-770
  const uint32_t rows = h.level + ctx.params().alpha, n = ctx.params().n;
  DeviceBuffer v(ctx.raw(), 2ull * rows * n);
  check(ck_key_mult(ctx.raw(), h.level, h.digits.data(), evk.data.data(), v.data(), nullptr));
  Polynomial v0{DeviceBuffer(ctx.raw(), (size_t)rows * n), h.level, ctx.params().alpha};
  Polynomial v1{DeviceBuffer(ctx.raw(), (size_t)rows * n), h.level, ctx.params().alpha};
  check(ck_memcpy_d2d(ctx.raw(), v0.data.data(), v.data(), (size_t)rows * n * 4, nullptr));
  check(ck_memcpy_d2d(ctx.raw(), v1.data.data(), v.data() + (size_t)rows * n, (size_t)rows * n * 4, nullptr));
  return {std::move(v0), std::move(v1)};
}

inline Polynomial mod_down(CkksContext& ctx, const Polynomial& v) {  // ckks.cpp:772-776
  if (v.p_count != ctx.params().alpha) throw std::invalid_argument("mod_down expects a P-extended polynomial");
  Polynomial out{DeviceBuffer(ctx.raw(), (size_t)v.q_count * ctx.params().n), v.q_count, 0};
  check(ck_mod_down(ctx.raw(), v.q_count, v.data.data(), out.data.data(), nullptr));
  return out;
}

inline std::pair<Polynomial, Polynomial> key_switch(CkksContext& ctx, const Polynomial& d,
                                                    const EvaluationKey& evk) {  // ckks.cpp:778-787
  if (d.p_count != 0) throw std::invalid_argument("mod_up input must be Q-only");
  const uint32_t l = d.q_count, n = ctx.params().n;
  DeviceBuffer out(ctx.raw(), 2ull * l * n);
  check(ck_key_switch(ctx.raw(), l, d.data.data(), evk.data.data(), out.data(), nullptr));
  Polynomial c0{DeviceBuffer(ctx.raw(), (size_t)l * n), l, 0}, c1{DeviceBuffer(ctx.raw(), (size_t)l * n), l, 0};
  check(ck_memcpy_d2d(ctx.raw(), c0.data.data(), out.data(), (size_t)l * n * 4, nullptr));
  check(ck_memcpy_d2d(ctx.raw(), c1.data.data(), out.data() + (size_t)l * n, (size_t)l * n * 4, nullptr));
  return {std::move(c0), std::move(c1)};
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
                             all.data(), nullptr));
  std::vector<Ciphertext> out;
  for (size_t i = 0; i < rots.size(); ++i) {
    Ciphertext c = make_ciphertext(ctx, ct.level, ct.scale);
    check(ck_memcpy_d2d(ctx.raw(), c.data.data(), all.data() + i * w, w * 4, nullptr));
    out.push_back(std::move(c));
  }
  return out;
}

// decrypt (ckks.cpp:541-553): m = b + a s; `s` = the secret's evaluation rows (>= level)
inline Plaintext decrypt(CkksContext& ctx, const Ciphertext& ct, const DeviceBuffer& s) {
  Plaintext pt{DeviceBuffer(ctx.raw(), (size_t)ct.level * ctx.params().n), ct.scale, ct.level, 0};
  check(ck_decrypt(ctx.raw(), ct.level, 1, ct.data.data(), s.data(), pt.data.data(), nullptr));
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
  check(ck_coeffs_to_eval(ctx.raw(), reinterpret_cast<const int64_t*>(dc.data()), level, pc, out.data(), nullptr));
  check(ck_stream_sync(ctx.raw(), nullptr));
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
  check(ck_encrypt_sk(ctx.raw(), l, m, a.data(), e.data(), sk.s.data(), out, nullptr));
  check(ck_stream_sync(ctx.raw(), nullptr));
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
    check(ck_automorphism(ctx.raw(), s, rot.data(), rows, -rotation, nullptr));
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
    check(ck_memcpy_d2d(ctx.raw(), bk + poly, a.data(), poly * 4, nullptr));
    check(ck_evk_digit(ctx.raw(), s, s_dst, a.data(), e.data(), gm.data(), kind == KeyKind::Relin ? 1 : 0, bk,
                       nullptr));
  }
  check(ck_stream_sync(ctx.raw(), nullptr));
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
  check(ck_memcpy_d2d(ctx.raw(), pkl.data(), pk.data.data(), (size_t)l * n * 4, nullptr));
  check(ck_memcpy_d2d(ctx.raw(), pkl.data() + (size_t)l * n, pk.data.data() + (size_t)L * n, (size_t)l * n * 4,
                      nullptr));
  Ciphertext ct = make_ciphertext(ctx, l, pt.scale);
  check(ck_encrypt_pk(ctx.raw(), l, pt.data.data(), v.data(), e0.data(), e1.data(), pkl.data(), ct.data.data(),
                      nullptr));
  check(ck_stream_sync(ctx.raw(), nullptr));
  return ct;
}

}  // namespace ckks32::b200
