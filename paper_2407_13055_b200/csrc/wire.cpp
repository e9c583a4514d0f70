// Wire formats of the reference, byte-compatible, as a
// pure client of the C ABI: rows move with ck_memcpy_d2h / ck_memcpy_h2d
// straight between device memory and the blob (device rows are canonical
// residues, so a blob is written without any per-word conversion).
//
//   basis       "RBS1"  serialize_basis / deserialize_basis   rns.cpp:168-216
//   polynomial  "PLS1"  serialize_poly / deserialize_poly     poly.cpp:293-352
//   ciphertext  "CTS1"  serialize_ciphertext / deserialize_*  ckks.cpp:1090-1121
//   eval key    "EVK1"  serialize_evk / deserialize_evk       ckks.cpp:1123-1154
//
// Error classes follow the reference: the polynomial and basis readers throw
// std::runtime_error (CK_RUNTIME_ERROR), the ciphertext / key headers and
// their length fields std::invalid_argument (CK_INVALID_ARGUMENT).
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ck32_b200.h"

namespace ck {
void set_last_error(const char* msg);  // ck_context.cu: the message ck_last_error() returns
}

namespace {

struct RtErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ArgErr : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

template <class F>
ck_status guard(F&& f) {
  try {
    f();
    return CK_OK;
  } catch (const ArgErr& e) {
    ck::set_last_error(e.what());
    return CK_INVALID_ARGUMENT;
  } catch (const RtErr& e) {
    ck::set_last_error(e.what());
    return CK_RUNTIME_ERROR;
  } catch (const std::exception& e) {
    ck::set_last_error(e.what());
    return CK_RUNTIME_ERROR;
  }
}

void ok(ck_status s) {
  if (s == CK_INVALID_ARGUMENT) throw ArgErr(ck_last_error());
  if (s != CK_OK) throw RtErr(ck_last_error());
}

struct Info {
  ck_params p{};
  std::vector<uint32_t> primes;
};
Info info(const ck_context* ctx) {
  Info i;
  ok(ck_context_params(ctx, &i.p));
  i.primes.resize(i.p.l + i.p.alpha);
  ok(ck_context_primes(ctx, i.primes.data()));
  return i;
}

// RnsBasis::hash (rns.cpp:119-133): FNV-1a over little-endian u64 words
uint64_t basis_hash(const Info& I) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&h](uint64_t v) {
    for (int b = 0; b < 8; ++b) {
      h ^= (v >> (8 * b)) & 0xff;
      h *= 1099511628211ull;
    }
  };
  mix(I.p.n);
  mix(I.p.delta_bits);
  for (uint32_t i = 0; i < I.p.l; ++i) mix(I.primes[i]);
  mix(~0ull);
  for (uint32_t i = 0; i < I.p.alpha; ++i) mix(I.primes[I.p.l + i]);
  return h;
}

struct Writer {
  uint8_t* out;
  size_t cap, pos = 0;
  bool measure;  // out == NULL: only count
  void raw(const void* p, size_t k) {
    if (!measure) {
      if (pos + k > cap) throw ArgErr("output buffer too small");
      std::memcpy(out + pos, p, k);
    }
    pos += k;
  }
  void u8(uint8_t v) { raw(&v, 1); }
  void u32(uint32_t v) {
    const uint8_t b[4] = {(uint8_t)v, (uint8_t)(v >> 8), (uint8_t)(v >> 16), (uint8_t)(v >> 24)};
    raw(b, 4);
  }
  void u64(uint64_t v) {
    u32((uint32_t)v);
    u32((uint32_t)(v >> 32));
  }
  uint8_t* reserve(size_t k) {  // space for rows copied straight from the device
    uint8_t* p = measure ? nullptr : out + pos;
    if (!measure && pos + k > cap) throw ArgErr("output buffer too small");
    pos += k;
    return p;
  }
};

template <class E>
struct Reader {
  const uint8_t* in;
  size_t len, pos = 0;
  const char* trunc;
  uint32_t u32() {
    if (pos + 4 > len) throw E(trunc);
    const uint32_t v = (uint32_t)in[pos] | (uint32_t)in[pos + 1] << 8 | (uint32_t)in[pos + 2] << 16 |
                       (uint32_t)in[pos + 3] << 24;
    pos += 4;
    return v;
  }
  uint64_t u64() {
    const uint64_t lo = u32();
    return lo | (uint64_t)u32() << 32;
  }
};

constexpr uint32_t kPolyMagic = 0x31534c50u, kBasisMagic = 0x31534252u, kCtMagic = 0x31535443u,
                   kEvkMagic = 0x314b5645u;

// serialize_poly (poly.cpp:297-320); rows on the device, canonical
void put_poly(Writer& w, ck_context* ctx, const Info& I, const uint32_t* rows, uint32_t qc, uint32_t pc, int domain,
              int mont, ck_stream st) {
  w.u32(kPolyMagic);
  w.u32(I.p.n);
  w.u32(qc);
  w.u32(pc);
  w.u32((uint32_t)domain);
  w.u32(mont ? 1 : 0);
  const uint64_t h = basis_hash(I);
  w.u32((uint32_t)h);
  w.u32((uint32_t)(h >> 32));
  const size_t bytes = (size_t)(qc + pc) * I.p.n * 4;
  uint8_t* dst = w.reserve(bytes);
  if (dst && bytes) {
    ok(ck_memcpy_d2h(ctx, dst, rows, bytes, st));
    ok(ck_stream_sync(ctx, st));
  }
}

// deserialize_poly (poly.cpp:322-352) into device rows; returns {qc, pc, domain, mont}
void get_poly(const uint8_t* in, size_t len, ck_context* ctx, const Info& I, uint32_t* rows, uint32_t cap_rows,
              uint32_t meta[4], ck_stream st) {
  Reader<RtErr> r{in, len, 0, "truncated polynomial blob"};
  if (r.u32() != kPolyMagic) throw RtErr("bad polynomial magic");
  if (r.u32() != I.p.n) throw RtErr("ring degree mismatch");
  const uint32_t qc = r.u32(), pc = r.u32(), dom = r.u32(), mont = r.u32() != 0;
  uint64_t h = r.u32();
  h |= (uint64_t)r.u32() << 32;
  if (h != basis_hash(I)) throw RtErr("basis hash mismatch");
  if (qc > I.p.l || pc > I.p.alpha) throw RtErr("polynomial rows exceed the basis");
  const size_t words = (size_t)(qc + pc) * I.p.n;
  if (r.pos + words * 4 > len) throw RtErr("truncated polynomial blob");
  if (qc + pc > cap_rows) throw ArgErr("device buffer too small for the polynomial");
  // the device keeps canonical residues (every kernel relies on it); a blob
  // written by the reference always is (poly.cpp:316 writes correct(row[j], q))
  for (uint32_t i = 0; i < qc + pc; ++i) {
    const uint32_t q = I.primes[i < qc ? i : I.p.l + (i - qc)];
    const uint8_t* row = in + r.pos + (size_t)i * I.p.n * 4;
    for (uint32_t j = 0; j < I.p.n; ++j) {
      uint32_t v;
      std::memcpy(&v, row + 4 * j, 4);
      if (v >= q) throw RtErr("residue out of range for its prime");
    }
  }
  if (words) {
    ok(ck_memcpy_h2d(ctx, rows, in + r.pos, words * 4, st));
    ok(ck_stream_sync(ctx, st));
  }
  meta[0] = qc;
  meta[1] = pc;
  meta[2] = dom;
  meta[3] = mont;
}

// put_bigint (ckks.cpp:1042-1049): u32 length, sign byte, export_bits
// magnitude (most significant byte first; zero exports as one zero byte)
void put_big(Writer& w, const uint8_t* be, size_t n) {
  while (n > 1 && be[0] == 0) {
    ++be;
    --n;
  }
  static const uint8_t zero = 0;
  if (n == 0) {
    be = &zero;
    n = 1;
  }
  w.u32((uint32_t)n);
  w.u8(0);
  w.raw(be, n);
}

// get_bigint (ckks.cpp:1051-1061); returns whether the value is zero
bool get_big(Reader<ArgErr>& r, uint8_t* out, size_t cap, size_t* n_out) {
  const uint32_t n = r.u32();
  if (r.pos + 1 + n > r.len) throw ArgErr("truncated input");
  if (r.in[r.pos] != 0) throw ArgErr("negative scale");
  r.pos += 1;
  if (n > cap || !out) throw ArgErr("scale buffer too small");
  bool zero = true;
  for (uint32_t i = 0; i < n; ++i) zero &= r.in[r.pos + i] == 0;
  std::memcpy(out, r.in + r.pos, n);
  *n_out = n;
  r.pos += n;
  return zero;
}

// put_poly / get_poly (ckks.cpp:1075-1088): u64 length + poly blob
void put_sized_poly(Writer& w, ck_context* ctx, const Info& I, const uint32_t* rows, uint32_t qc, uint32_t pc,
                    ck_stream st) {
  w.u64(32 + (uint64_t)(qc + pc) * I.p.n * 4);
  put_poly(w, ctx, I, rows, qc, pc, 1, 1, st);
}
void get_sized_poly(Reader<ArgErr>& r, ck_context* ctx, const Info& I, uint32_t* rows, uint32_t want_q,
                    uint32_t want_p, ck_stream st) {
  const uint64_t n = r.u64();
  if (r.pos + n > r.len) throw ArgErr("truncated input");
  uint32_t meta[4];
  get_poly(r.in + r.pos, (size_t)n, ctx, I, rows, want_q + want_p, meta, st);
  if (meta[0] != want_q || meta[1] != want_p)
    throw ArgErr("polynomial shape does not match the container (" + std::to_string(meta[0]) + "+" +
                 std::to_string(meta[1]) + " rows)");
  if (meta[2] != 1 || meta[3] != 1) throw ArgErr("expected evaluation-domain Montgomery polynomial");
  r.pos += n;
}

}  // namespace

extern "C" {

ck_status ck_serialize_basis(const ck_context* ctx, uint8_t* out, size_t cap, size_t* len) {
  return guard([&] {
    const Info I = info(ctx);
    Writer w{out, cap, 0, out == nullptr};
    w.u32(kBasisMagic);
    w.u32(1);
    w.u32(I.p.n);
    w.u32(I.p.l);
    w.u32(I.p.alpha);
    w.u32(I.p.delta_bits);
    for (uint32_t q : I.primes) w.u32(q);
    if (len) *len = w.pos;
  });
}

ck_status ck_deserialize_basis(const uint8_t* in, size_t len, ck_params* params, uint32_t* primes, uint32_t cap) {
  return guard([&] {
    Reader<RtErr> r{in, len, 0, "truncated basis blob"};
    if (r.u32() != kBasisMagic) throw RtErr("bad basis magic");
    if (r.u32() != 1) throw RtErr("bad basis version");
    ck_params p{};
    p.n = r.u32();
    p.l = r.u32();
    p.alpha = r.u32();
    p.delta_bits = r.u32();
    if (p.l + p.alpha > cap) throw ArgErr("prime buffer too small");
    for (uint32_t i = 0; i < p.l + p.alpha; ++i) primes[i] = r.u32();
    if (params) *params = p;
  });
}

ck_status ck_serialize_poly(ck_context* ctx, const uint32_t* rows_dev, uint32_t q_count, uint32_t p_count, int domain,
                            int mont, uint8_t* out, size_t cap, size_t* len, ck_stream stream) {
  return guard([&] {
    const Info I = info(ctx);
    if (q_count > I.p.l || p_count > I.p.alpha) throw ArgErr("rows exceed the basis");
    Writer w{out, cap, 0, out == nullptr};
    put_poly(w, ctx, I, rows_dev, q_count, p_count, domain, mont, stream);
    if (len) *len = w.pos;
  });
}

ck_status ck_deserialize_poly(ck_context* ctx, const uint8_t* in, size_t len, uint32_t* rows_dev, uint32_t cap_rows,
                              uint32_t meta[4], ck_stream stream) {
  return guard([&] {
    const Info I = info(ctx);
    uint32_t m[4];
    get_poly(in, len, ctx, I, rows_dev, cap_rows, m, stream);
    if (meta) std::memcpy(meta, m, sizeof m);
  });
}

ck_status ck_serialize_ciphertext(ck_context* ctx, const uint32_t* ct_dev, uint32_t level, int pending_rescale,
                                  const uint8_t* scale_num, size_t num_len, const uint8_t* scale_den, size_t den_len,
                                  uint8_t* out, size_t cap, size_t* len, ck_stream stream) {
  return guard([&] {
    const Info I = info(ctx);
    if (level > I.p.l) throw ArgErr("level out of range");
    Writer w{out, cap, 0, out == nullptr};
    w.u32(kCtMagic);
    w.u32(1);
    w.u32(level);
    w.u8(pending_rescale ? 1 : 0);
    put_big(w, scale_num, num_len);
    put_big(w, scale_den, den_len);
    put_sized_poly(w, ctx, I, ct_dev, level, 0, stream);
    put_sized_poly(w, ctx, I, ct_dev + (size_t)level * I.p.n, level, 0, stream);
    if (len) *len = w.pos;
  });
}

ck_status ck_deserialize_ciphertext(ck_context* ctx, const uint8_t* in, size_t len, uint32_t* ct_dev,
                                    uint32_t cap_level, uint32_t* level, int* pending_rescale, uint8_t* scale_num,
                                    size_t num_cap, size_t* num_len, uint8_t* scale_den, size_t den_cap,
                                    size_t* den_len, ck_stream stream) {
  return guard([&] {
    const Info I = info(ctx);
    Reader<ArgErr> r{in, len, 0, "truncated input"};
    if (r.u32() != kCtMagic || r.u32() != 1) throw ArgErr("bad ciphertext header");
    const uint32_t lv = r.u32();
    if (r.pos >= len) throw ArgErr("truncated input");
    const int pend = in[r.pos++] != 0;
    size_t nl = 0, dl = 0;
    get_big(r, scale_num, num_cap, &nl);
    if (get_big(r, scale_den, den_cap, &dl)) throw ArgErr("zero denominator");
    if (lv > cap_level) throw ArgErr("device buffer too small for the ciphertext");
    get_sized_poly(r, ctx, I, ct_dev, lv, 0, stream);
    get_sized_poly(r, ctx, I, ct_dev + (size_t)lv * I.p.n, lv, 0, stream);
    *level = lv;
    *pending_rescale = pend;
    *num_len = nl;
    *den_len = dl;
  });
}

ck_status ck_serialize_evk(ck_context* ctx, const uint32_t* evk_dev, uint32_t digits, int kind, int64_t rotation,
                           uint8_t* out, size_t cap, size_t* len, ck_stream stream) {
  return guard([&] {
    const Info I = info(ctx);
    const uint32_t rows = I.p.l + I.p.alpha;
    Writer w{out, cap, 0, out == nullptr};
    w.u32(kEvkMagic);
    w.u32(1);
    w.u32((uint32_t)kind);
    w.u64((uint64_t)rotation);
    w.u32(digits);
    for (uint32_t k = 0; k < 2 * digits; ++k)
      put_sized_poly(w, ctx, I, evk_dev + (size_t)k * rows * I.p.n, I.p.l, I.p.alpha, stream);
    if (len) *len = w.pos;
  });
}

ck_status ck_deserialize_evk(ck_context* ctx, const uint8_t* in, size_t len, uint32_t* evk_dev, uint32_t cap_digits,
                             int* kind, int64_t* rotation, uint32_t* digits, ck_stream stream) {
  return guard([&] {
    const Info I = info(ctx);
    const uint32_t rows = I.p.l + I.p.alpha;
    Reader<ArgErr> r{in, len, 0, "truncated input"};
    if (r.u32() != kEvkMagic || r.u32() != 1) throw ArgErr("bad key header");
    const int kd = (int)r.u32();
    const int64_t rot = (int64_t)r.u64();
    const uint32_t d = r.u32();
    if (d > cap_digits) throw ArgErr("device buffer too small for the key");
    for (uint32_t k = 0; k < 2 * d; ++k)
      get_sized_poly(r, ctx, I, evk_dev + (size_t)k * rows * I.p.n, I.p.l, I.p.alpha, stream);
    *kind = kd;
    *rotation = rot;
    *digits = d;
  });
}

}  // extern "C"
