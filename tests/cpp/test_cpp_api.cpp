// C++ drop-in check: drives the header-only mirror (paper_2407_13055_b200/cpp/
// ckks32_b200.hpp) the way the reference's own tests drive ckks.hpp
// (test_ckks.cpp:293-380): hmult + hrot on ciphertexts read from raw files,
// results written back for the Python side to compare with the oracle, plus
// the exception contract (std::invalid_argument on level / key misuse).
//
//   test_cpp_api <dir> <n> <l> <alpha> <level>
// <dir>/x.bin, y.bin: [2][level][n] u32; evk.bin: [D][2][L+alpha][n] u32
// writes <dir>/out_hmult.bin, out_hrot.bin
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <random>
#include <string>
#include <stdexcept>
#include <vector>

#include "../../paper_2407_13055_b200/cpp/ckks32_b200.hpp"

using namespace ckks32::b200;

static std::vector<uint32_t> read_file(const std::string& p, size_t words) {
  std::vector<uint32_t> v(words);
  std::ifstream f(p, std::ios::binary);
  if (!f.read(reinterpret_cast<char*>(v.data()), words * 4)) throw std::runtime_error("short read " + p);
  return v;
}
static void write_file(const std::string& p, const std::vector<uint32_t>& v) {
  std::ofstream f(p, std::ios::binary);
  f.write(reinterpret_cast<const char*>(v.data()), v.size() * 4);
}

// keys mode: keygen + encode + secret-key encrypt with the reference's own
// generator type, in the fixture driver's order (oracle/ref_driver.cpp
// ref_gen_fixtures: keygen, relin / rot 1 / rot 3 evk_gen, slots u, v)
//   test_cpp_api keys <dir> <seed> <n> <l> <alpha> <delta_bits>
// writes <dir>/sk_rows.bin [L+alpha][n], evk_*.bin [D][2][L+alpha][n], ct_u.bin, ct_v.bin [2][l][n]
static int keys_mode(char** argv) {
  const std::string dir = argv[2];
  std::mt19937_64 rng(std::strtoull(argv[3], nullptr, 10));
  CkksParams p;
  p.n = std::atoi(argv[4]);
  p.l = std::atoi(argv[5]);
  p.alpha = std::atoi(argv[6]);
  p.delta_bits = std::atoi(argv[7]);
  p.hamming = std::min<uint32_t>(p.hamming, p.n / 4);  // bench.cpp:337
  CkksContext ctx(p);
  SecretKey sk = keygen(ctx, rng);
  write_file(dir + "/sk_rows.bin", sk.s.download());
  write_file(dir + "/evk_relin.bin", evk_gen(ctx, sk, KeyKind::Relin, 0, rng).data.download());
  write_file(dir + "/evk_rot1.bin", evk_gen(ctx, sk, KeyKind::Rotation, 1, rng).data.download());
  write_file(dir + "/evk_rot3.bin", evk_gen(ctx, sk, KeyKind::Rotation, 3, rng).data.download());
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  std::vector<std::complex<double>> z[2];  // slots u, v drawn before either encryption
  for (auto& zz : z) {
    zz.resize(p.n / 2);
    for (auto& v : zz) {
      const double re = dist(rng);
      v = {re, dist(rng)};
    }
  }
  for (int i = 0; i < 2; ++i) {
    Plaintext pt = encode(ctx, z[i], ctx.default_scale(), p.l);
    if (i == 1) write_file(dir + "/pt_v.bin", pt.data.download());
    Ciphertext ct = encrypt(ctx, pt, sk, rng);
    write_file(dir + (i ? "/ct_v.bin" : "/ct_u.bin"), ct.data.download());
  }
  std::printf("cpp keys ok\n");
  return 0;
}

int main(int argc, char** argv) {
  if (argc >= 8 && std::string(argv[1]) == "keys") return keys_mode(argv);
  if (argc < 6) {
    std::fprintf(stderr, "usage: %s dir n l alpha level\n", argv[0]);
    return 2;
  }
  const std::string dir = argv[1];
  CkksParams p;
  p.n = std::atoi(argv[2]);
  p.l = std::atoi(argv[3]);
  p.alpha = std::atoi(argv[4]);
  p.delta_bits = 55;
  const uint32_t level = std::atoi(argv[5]);
  CkksContext ctx(p);
  const size_t ctw = 2ull * level * p.n;
  const size_t evw = (size_t)ctx.num_digits(p.l) * 2 * (p.l + p.alpha) * p.n;

  Ciphertext x = make_ciphertext(ctx, level, ctx.default_scale());
  Ciphertext y = make_ciphertext(ctx, level, ctx.default_scale());
  x.data.upload(read_file(dir + "/x.bin", ctw).data(), ctw);
  y.data.upload(read_file(dir + "/y.bin", ctw).data(), ctw);
  EvaluationKey relin{DeviceBuffer(ctx.raw(), evw), KeyKind::Relin, 0};
  relin.data.upload(read_file(dir + "/evk.bin", evw).data(), evw);
  EvaluationKey rot{DeviceBuffer(ctx.raw(), evw), KeyKind::Rotation, 1};
  rot.data.upload(read_file(dir + "/evk.bin", evw).data(), evw);

  Ciphertext m = hmult(ctx, x, y, relin);
  if (m.level != level - 2) throw std::runtime_error("hmult level ledger");
  Ciphertext expect_scale = make_ciphertext(ctx, 2, ctx.default_scale() * ctx.default_scale());
  if (!(m.scale == expect_scale.scale.divided_by(ctx.primes()[level - 2], ctx.primes()[level - 1])))
    throw std::runtime_error("hmult scale ledger");
  write_file(dir + "/out_hmult.bin", m.data.download());
  Ciphertext r = hrot(ctx, x, 1, rot);
  write_file(dir + "/out_hrot.bin", r.data.download());

  int errors = 0;
  try {  // rotation key passed to hmult (ckks.cpp:806-807)
    hmult(ctx, x, y, rot);
    ++errors;
  } catch (const std::invalid_argument&) {
  }
  try {  // wrong rotation amount (ckks.cpp:872-873)
    hrot(ctx, x, 2, rot);
    ++errors;
  } catch (const std::invalid_argument&) {
  }
  {  // encode -> decode round trip through the mirror (ckks.cpp:278-362)
    std::vector<std::complex<double>> z(p.n / 2);
    for (size_t t = 0; t < z.size(); ++t) z[t] = {std::sin(0.1 * t), std::cos(0.37 * t)};
    Plaintext pt = encode(ctx, z, ctx.default_scale(), level);
    const auto back = decode(ctx, pt);
    double err = 0;
    for (size_t t = 0; t < z.size(); ++t) err = std::max(err, std::abs(back[t] - z[t]));
    if (!(err < 1e-9)) throw std::runtime_error("encode/decode round trip error " + std::to_string(err));
    try {  // too many slots (ckks.cpp:281)
      z.resize(p.n / 2 + 1);
      encode(ctx, z, ctx.default_scale(), level);
      ++errors;
    } catch (const std::invalid_argument&) {
    }
  }
  {  // key-switching building blocks: key_switch == mod_down(key_mult(mod_up(d))) (ckks.cpp:778-787)
    Polynomial d{DeviceBuffer(ctx.raw(), (size_t)level * p.n), level, 0};
    check(ck_memcpy_d2d(ctx.raw(), d.data.data(), x.data.data() + (size_t)level * p.n, (size_t)level * p.n * 4,
                        nullptr));
    auto ks = key_switch(ctx, d, relin);
    HoistState h = mod_up(ctx, d);
    auto v = key_mult(ctx, h, relin);
    Polynomial c0 = mod_down(ctx, v.first), c1 = mod_down(ctx, v.second);
    if (ks.first.data.download() != c0.data.download() || ks.second.data.download() != c1.data.download())
      throw std::runtime_error("key_switch != mod_down(key_mult(mod_up))");
    // hoisted rotation by 1 == hrot by 1 (ckks.cpp:899-925)
    auto hr = hoisted_rotations(ctx, x, {1}, {&rot});
    if (hr[0].data.download() != r.data.download()) throw std::runtime_error("hoisted rotation != hrot");
  }
  {  // batched overloads on a non-default stream: element i of the batch == the single-ciphertext result
    ck_stream st = nullptr;
    check(ck_stream_create(ctx.raw(), &st));
    ctx.set_stream(st);
    CiphertextBatch X = make_batch(ctx, 3, level, ctx.default_scale()), Y = make_batch(ctx, 3, level, ctx.default_scale());
    for (uint32_t i = 0; i < 3; ++i) {
      check(ck_memcpy_d2d(ctx.raw(), X[i].data.data(), x.data.data(), ctw * 4, st));
      check(ck_memcpy_d2d(ctx.raw(), Y[i].data.data(), y.data.data(), ctw * 4, st));
    }
    CiphertextBatch M = hmult(ctx, X, Y, relin), R = hrot(ctx, X, 1, rot);
    ctx.sync();
    for (uint32_t i = 0; i < 3; ++i)
      if (M[i].data.download(st) != m.data.download() || R[i].data.download(st) != r.data.download())
        throw std::runtime_error("batched hmult/hrot != single");
    if (!(M.scale == m.scale) || M.level != m.level) throw std::runtime_error("batched ledger");
    ctx.set_stream(nullptr);
    check(ck_stream_destroy(ctx.raw(), st));
  }
  {  // hoisted_rotate_accumulate with the Montgomery one R mod q as plaintext
    const uint32_t rows = level + p.alpha;
    std::vector<uint32_t> one((size_t)rows * p.n);
    for (uint32_t i = 0; i < rows; ++i) {
      const uint64_t q = ctx.primes()[i < level ? i : p.l + (i - level)];
      for (uint32_t k = 0; k < p.n; ++k) one[(size_t)i * p.n + k] = (uint32_t)((1ull << 32) % q);
    }
    Plaintext pt1{DeviceBuffer(ctx.raw(), one.size()), Scale::two_pow(0), level, p.alpha};
    pt1.data.upload(one.data(), one.size());
    Ciphertext id = hoisted_rotate_accumulate(ctx, x, {0}, {&pt1}, {nullptr});  // r = 0: pt * ct, no key switch
    if (id.data.download() != x.data.download()) throw std::runtime_error("hoisted accumulate(r = 0, pt = 1) != ct");
    // r = 1 (ModDown after the automorphism: equal to hrot only up to the BConv error, so the
    // Python side compares it with the oracle's hoisted_rotate_accumulate)
    Ciphertext acc = hoisted_rotate_accumulate(ctx, x, {1}, {&pt1}, {&rot});
    write_file(dir + "/out_acc.bin", acc.data.download());
  }
  {  // kernel level: NTT round trip on the host row mirror, automorphism group law, ew identities
    Polynomial c{DeviceBuffer(ctx.raw(), (size_t)3 * p.n), 2, 1, Domain::Coefficient, false};
    c.host.assign((size_t)3 * p.n, 0);
    for (uint32_t i = 0; i < 3; ++i) {
      const uint32_t q = ctx.primes()[i < 2 ? i : p.l];
      for (uint32_t k = 0; k < p.n; ++k) c.row(i)[k] = (uint32_t)((k * 2654435761ull + i) % q);
    }
    c.push();
    const auto orig = c.host;
    ntt_forward(ctx, c);
    try {  // domain discipline (ntt.cpp:288-291)
      ntt_forward(ctx, c);
      ++errors;
    } catch (const std::invalid_argument&) {
    }
    auto rot3 = apply_automorphism(ctx, c, AutomorphismMap::rotation(p.n, 3));
    auto back = apply_automorphism(ctx, rot3, AutomorphismMap::rotation(p.n, -3));
    if (back.data.download() != c.data.download()) throw std::runtime_error("rot 3 then rot -3 != identity");
    auto sum = ew_add(ctx, c, rot3);
    ew_sub_inplace(ctx, sum, rot3);
    if (sum.data.download() != c.data.download()) throw std::runtime_error("ew_add then ew_sub_inplace");
    intt_inverse(ctx, c);
    c.pull();
    if (c.host != orig) throw std::runtime_error("ntt round trip on the host mirror");
    if (c.row(1)[5] != orig[p.n + 5]) throw std::runtime_error("row() view");
  }
  {  // scale tolerance (ckks.cpp:131-136): 2^-41 relative passes, 2^-39 fails
    Ciphertext xs = make_ciphertext(ctx, level, Scale::rational(0, {(1u << 31) + 1u}, {}));
    Ciphertext ys = make_ciphertext(ctx, level, Scale::rational(0, {(1u << 31) + 1u}, {}));
    check(ck_memcpy_d2d(ctx.raw(), xs.data.data(), x.data.data(), ctw * 4, nullptr));
    check(ck_memcpy_d2d(ctx.raw(), ys.data.data(), y.data.data(), ctw * 4, nullptr));
    ys.scale = Scale::rational(-1, {(1u << 31) + 1u, (1u << 30) + 1u, 2u}, {(1u << 30) + 1u});  // equal
    (void)hadd(ctx, xs, ys);
    xs.scale = Scale::two_pow(48);
    ys.scale = Scale::rational(0, {193u, 65537u, 22253377u}, {});  // 2^48 + 1: 2^-48 relative
    (void)hadd(ctx, xs, ys);
    xs.scale = ys.scale = Scale::rational(0, {(1u << 31) + 1u}, {});
    ys.scale = Scale::rational(0, {(1u << 31) + 2u}, {});  // 2^-31 relative: beyond 2^-40
    try {
      hadd(ctx, xs, ys);
      ++errors;
    } catch (const std::invalid_argument&) {
    }
  }
  const uint64_t n_launch = ck_launch_count(ctx.raw());
  std::printf("cpp api ok: hmult level %u -> %u, hrot level %u, %llu kernel launches, %d contract errors\n", level,
              m.level, r.level, (unsigned long long)n_launch, errors);
  return errors ? 1 : 0;
}
