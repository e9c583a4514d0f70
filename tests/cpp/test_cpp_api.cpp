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
  const uint64_t n_launch = ck_launch_count(ctx.raw());
  std::printf("cpp api ok: hmult level %u -> %u, hrot level %u, %llu kernel launches, %d contract errors\n", level,
              m.level, r.level, (unsigned long long)n_launch, errors);
  return errors ? 1 : 0;
}
