// ORACLE TEST INFRASTRUCTURE ONLY — links the read-only reference library
// (oracle/_ref/libckks32_ref.so, built from /root/reference/proj/src by
// oracle/Makefile).  Exposes a small extern "C" surface so Python can
//   * dump golden fixtures through the reference's own serialisers
//     (serialize_poly / serialize_ciphertext / serialize_evk / serialize_basis,
//      poly.cpp:295-352, ckks.cpp:1090-1154, rns.cpp:168-216),
//   * run one mechanism on seeded synthetic inputs at full size and return the
//     canonical output residues (hashed on the Python side),
//   * time the reference CPU path with its own harness
//     (bench::run_mechanism_bench, bench.cpp:332-389).
// Never imported by the product path.

#include <cstdio>
#include <cstring>
#include <fstream>
#include <random>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "ckks32/bench.hpp"
#include "ckks32/ckks.hpp"

using namespace ckks32;

namespace {

std::string g_err;

void write_blob(const std::string& path, const std::vector<uint8_t>& b) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot open " + path);
  f.write(reinterpret_cast<const char*>(b.data()), static_cast<std::streamsize>(b.size()));
}

CkksParams make_params(uint32_t n, uint32_t l, uint32_t alpha, uint32_t db, bool lazy) {
  CkksParams p;
  p.n = n;
  p.l = l;
  p.alpha = alpha;
  p.delta_bits = db;
  p.hamming = std::min<uint32_t>(p.hamming, n / 4);  // same rule as bench.cpp:337
  p.lazy_rescale = lazy;
  return p;
}

std::vector<std::complex<double>> unit_slots(std::mt19937_64& rng, uint32_t count) {
  std::uniform_real_distribution<double> dist(-1.0, 1.0);  // bench.cpp:305-311
  std::vector<std::complex<double>> u(count);
  for (auto& v : u) v = {dist(rng), dist(rng)};
  return u;
}

// random_poly of bench.cpp:121-129: rng() % q, row-major.
Polynomial random_poly(CkksContext& ctx, uint32_t qc, uint32_t pc, std::mt19937_64& rng,
                       Domain dom, bool mont) {
  Polynomial p(ctx.basis(), qc, pc, dom, mont, &ctx.pool());
  for (uint32_t i = 0; i < p.rows(); ++i)
    for (uint32_t k = 0; k < p.n(); ++k) p.row(i)[k] = static_cast<int32_t>(rng() % p.prime_at(i).q);
  return p;
}

size_t put_canonical(const Polynomial& p, uint32_t* out, size_t off, size_t cap) {
  const size_t need = static_cast<size_t>(p.rows()) * p.n();
  if (off + need > cap) throw std::runtime_error("output buffer too small");
  for (uint32_t i = 0; i < p.rows(); ++i) {
    const uint32_t q = p.prime_at(i).q;
    for (uint32_t k = 0; k < p.n(); ++k) out[off + static_cast<size_t>(i) * p.n() + k] = correct(p.row(i)[k], q);
  }
  return off + need;
}

// Synthetic evaluation key: D digits of (b, a) over the full PQ basis,
// uniform residues.
EvaluationKey synthetic_evk(CkksContext& ctx, KeyKind kind, int64_t rot, std::mt19937_64& rng) {
  EvaluationKey evk;
  evk.kind = kind;
  evk.rotation = rot;
  const uint32_t l = ctx.params().l, alpha = ctx.params().alpha;
  for (uint32_t k = 0; k < ctx.num_digits(l); ++k) {
    auto b = random_poly(ctx, l, alpha, rng, Domain::Evaluation, true);
    auto a = random_poly(ctx, l, alpha, rng, Domain::Evaluation, true);
    evk.digits.emplace_back(std::move(b), std::move(a));
  }
  return evk;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_basis(uint32_t n, uint32_t l, uint32_t alpha, uint32_t db, uint32_t* primes_out) {
  try {
    auto b = generate_basis(n, l, alpha, db);
    for (uint32_t i = 0; i < l; ++i) primes_out[i] = b->q_primes[i].q;
    for (uint32_t i = 0; i < alpha; ++i) primes_out[l + i] = b->p_primes[i].q;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Twiddle-table export (ntt.cpp:100-135) for pinning the restatement.
int ref_twiddles(uint32_t n, uint32_t l, uint32_t alpha, uint32_t db, uint32_t gidx,
                 uint32_t* fwd, uint32_t* inv, uint32_t* scalars /* psi,fwd1_r2,exit_x,exit_y */) {
  try {
    auto b = generate_basis(n, l, alpha, db);
    auto tw = build_twiddles(b);
    const auto& T = tw->per_prime.at(gidx);
    std::memcpy(fwd, T.fwd.data(), sizeof(uint32_t) * n);
    std::memcpy(inv, T.inv.data(), sizeof(uint32_t) * n);
    scalars[0] = T.psi;
    scalars[1] = T.fwd1_r2;
    scalars[2] = T.exit_x;
    scalars[3] = T.exit_y;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Raw (lazy, signed) row transforms exactly as the reference's default plan
// computes them: forward_row / inverse_row (ntt.cpp:176-272).
int ref_ntt_rows(uint32_t n, uint32_t l, uint32_t alpha, uint32_t db, int inverse, uint32_t rows,
                 const uint32_t* gidx, int32_t* data, const uint32_t* epilogue) {
  try {
    CkksContext ctx(make_params(n, l, alpha, db, false));
    for (uint32_t r = 0; r < rows; ++r) {
      int32_t* row = data + static_cast<size_t>(r) * n;
      if (inverse)
        ctx.plan().inverse_row(row, gidx[r], epilogue ? &epilogue[r] : nullptr);
      else
        ctx.plan().forward_row(row, gidx[r]);
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Golden fixtures with real keys: every blob uses the reference serialisers.
int ref_gen_fixtures(uint32_t n, uint32_t l, uint32_t alpha, uint32_t db, uint64_t seed,
                     const char* outdir_c) {
  try {
    const std::string od(outdir_c);
    CkksContext ctx(make_params(n, l, alpha, db, false));
    auto W = [&](const std::string& name, const std::vector<uint8_t>& b) { write_blob(od + "/" + name, b); };
    W("basis.bin", serialize_basis(*ctx.basis()));

    std::mt19937_64 rng(seed);
    auto sk = keygen(ctx, rng);
    auto relin = evk_gen(ctx, sk, KeyKind::Relin, 0, rng);
    auto rot1 = evk_gen(ctx, sk, KeyKind::Rotation, 1, rng);
    auto rot3 = evk_gen(ctx, sk, KeyKind::Rotation, 3, rng);
    W("sk.bin", serialize_poly(sk.s));
    W("evk_relin.bin", serialize_evk(relin));
    W("evk_rot1.bin", serialize_evk(rot1));
    W("evk_rot3.bin", serialize_evk(rot3));

    auto u = unit_slots(rng, ctx.slots());
    auto v = unit_slots(rng, ctx.slots());
    auto Wz = [&](const std::string& name, const std::vector<std::complex<double>>& z) {
      std::vector<uint8_t> b(z.size() * 16);
      std::memcpy(b.data(), z.data(), b.size());
      W(name, b);
    };
    Wz("slots_u.f64", u);  // complex<double> (re, im) little-endian
    Wz("slots_v.f64", v);
    auto pt_u = encode(ctx, u, ctx.default_scale(), l);
    auto pt_v = encode(ctx, v, ctx.default_scale(), l);
    auto ct_u = encrypt(ctx, pt_u, sk, rng);
    auto ct_v = encrypt(ctx, pt_v, sk, rng);
    W("pt_v.bin", serialize_poly(pt_v.poly));
    W("ct_u.bin", serialize_ciphertext(ct_u));
    W("ct_v.bin", serialize_ciphertext(ct_v));

    // mechanisms
    W("out_hmult.bin", serialize_ciphertext(hmult(ctx, ct_u, ct_v, relin)));
    W("out_decrypt_u.bin", serialize_poly(decrypt(ctx, ct_u, sk).poly));
    W("out_decrypt_hmult.bin", serialize_poly(decrypt(ctx, hmult(ctx, ct_u, ct_v, relin), sk).poly));
    W("out_hrot1.bin", serialize_ciphertext(hrot(ctx, ct_u, 1, rot1)));
    W("out_hrot3.bin", serialize_ciphertext(hrot(ctx, ct_u, 3, rot3)));
    W("out_rescale.bin", serialize_ciphertext(rescale(ctx, ct_u)));
    W("out_hadd.bin", serialize_ciphertext(hadd(ctx, ct_u, ct_v)));
    W("out_padd.bin", serialize_ciphertext(padd(ctx, ct_u, pt_v)));
    W("out_pmult.bin", serialize_ciphertext(pmult(ctx, ct_u, pt_v)));

    // key-switching pieces on d = ct_u.a
    auto hoist = mod_up(ctx, ct_u.a);
    for (size_t k = 0; k < hoist.digits.size(); ++k)
      W("out_modup_d" + std::to_string(k) + ".bin", serialize_poly(hoist.digits[k]));
    auto [v0, v1] = key_mult(ctx, hoist, relin);
    W("out_keymult_v0.bin", serialize_poly(v0));
    W("out_keymult_v1.bin", serialize_poly(v1));
    W("out_moddown_v0.bin", serialize_poly(mod_down(ctx, v0)));
    auto [c0, c1] = key_switch(ctx, ct_u.a, relin);
    W("out_keyswitch_c0.bin", serialize_poly(c0));
    W("out_keyswitch_c1.bin", serialize_poly(c1));

    // hoisting (ckks.cpp:899-1012)
    std::vector<int64_t> rots = {1, 3};
    std::vector<const EvaluationKey*> kp = {&rot1, &rot3};
    auto hr = hoisted_rotations(ctx, ct_u, rots, kp);
    W("out_hoisted_r1.bin", serialize_ciphertext(hr[0]));
    W("out_hoisted_r3.bin", serialize_ciphertext(hr[1]));
    std::vector<int64_t> arots = {0, 1, 3};
    std::vector<Plaintext> pts;
    pts.reserve(3);
    std::vector<const Plaintext*> pp;
    for (int i = 0; i < 3; ++i) {
      auto w = unit_slots(rng, ctx.slots());
      pts.push_back(encode(ctx, w, ctx.default_scale(), l, /*p_extend=*/true));
    }
    for (int i = 0; i < 3; ++i) {
      pp.push_back(&pts[i]);
      W("pt_acc" + std::to_string(i) + ".bin", serialize_poly(pts[i].poly));
    }
    std::vector<const EvaluationKey*> akp = {nullptr, &rot1, &rot3};
    W("out_hoisted_acc.bin", serialize_ciphertext(hoisted_rotate_accumulate(ctx, ct_u, arots, pp, akp)));

    // lazy-rescale HMult (ckks.cpp:853-863): separate context, keys regenerated
    // from the same seed (test_ckks.cpp:320-362 does the same)
    {
      CkksContext lctx(make_params(n, l, alpha, db, true));
      std::mt19937_64 lrng(seed);
      auto lsk = keygen(lctx, lrng);
      auto lrelin = evk_gen(lctx, lsk, KeyKind::Relin, 0, lrng);
      auto lct_u = deserialize_ciphertext(serialize_ciphertext(ct_u), lctx.basis(), &lctx.pool());
      auto lct_v = deserialize_ciphertext(serialize_ciphertext(ct_v), lctx.basis(), &lctx.pool());
      W("out_hmult_lazy.bin", serialize_ciphertext(hmult(lctx, lct_u, lct_v, lrelin)));
    }

    // plain transforms of ct_u.b (evaluation -> coefficient -> evaluation)
    {
      Polynomial t = ct_u.b.clone(&ctx.pool());
      intt_inverse(t, ctx.plan());
      W("out_intt_ctub.bin", serialize_poly(t));
      Polynomial coeff = random_poly(ctx, l, alpha, rng, Domain::Coefficient, false);
      W("in_ntt_coeff.bin", serialize_poly(coeff));
      ntt_forward(coeff, ctx.plan());
      W("out_ntt_coeff.bin", serialize_poly(coeff));
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// One mechanism on seeded synthetic inputs: rng = mt19937_64(seed);
// x.b, x.a, y.b, y.a = random_poly(level rows, evaluation, Montgomery) in that
// order; then the evk digits k = 0..D(L)-1, each b_k then a_k over the full
// L+alpha rows.  Output: canonical residues of the result (b rows then a rows).
int ref_synthetic_op(uint32_t n, uint32_t l, uint32_t alpha, uint32_t db, uint32_t level,
                     const char* op_c, uint64_t seed, int64_t rot, uint32_t* out, size_t cap,
                     size_t* written) {
  try {
    const std::string op(op_c);
    const bool lazy = op == "hmult_lazy";
    CkksContext ctx(make_params(n, l, alpha, db, lazy));
    std::mt19937_64 rng(seed);
    Ciphertext x, y;
    x.b = random_poly(ctx, level, 0, rng, Domain::Evaluation, true);
    x.a = random_poly(ctx, level, 0, rng, Domain::Evaluation, true);
    y.b = random_poly(ctx, level, 0, rng, Domain::Evaluation, true);
    y.a = random_poly(ctx, level, 0, rng, Domain::Evaluation, true);
    x.level = y.level = level;
    x.scale = y.scale = ctx.default_scale();
    const bool is_rot = op == "hrot" || op == "hoisted";
    auto evk = synthetic_evk(ctx, is_rot ? KeyKind::Rotation : KeyKind::Relin, is_rot ? rot : 0, rng);
    size_t off = 0;
    if (op == "hmult" || op == "hmult_lazy") {
      auto o = hmult(ctx, x, y, evk);
      off = put_canonical(o.b, out, off, cap);
      off = put_canonical(o.a, out, off, cap);
    } else if (op == "hrot") {
      auto o = hrot(ctx, x, rot, evk);
      off = put_canonical(o.b, out, off, cap);
      off = put_canonical(o.a, out, off, cap);
    } else if (op == "rescale") {
      auto o = rescale(ctx, x);
      off = put_canonical(o.b, out, off, cap);
      off = put_canonical(o.a, out, off, cap);
    } else if (op == "key_switch") {
      auto [c0, c1] = key_switch(ctx, x.a, evk);
      off = put_canonical(c0, out, off, cap);
      off = put_canonical(c1, out, off, cap);
    } else if (op == "mod_up") {
      auto h = mod_up(ctx, x.a);
      for (auto& d : h.digits) off = put_canonical(d, out, off, cap);
    } else if (op == "ntt") {
      // forward NTT of x.b's rows reinterpreted as coefficient-domain input
      Polynomial c = x.b.clone(&ctx.pool());
      c.set_domain(Domain::Coefficient);
      c.set_mont(false);
      ntt_forward(c, ctx.plan());
      off = put_canonical(c, out, off, cap);
    } else if (op == "intt") {
      Polynomial c = x.b.clone(&ctx.pool());
      intt_inverse(c, ctx.plan());
      off = put_canonical(c, out, off, cap);
    } else {
      throw std::invalid_argument("unknown op " + op);
    }
    *written = off;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// CPU baseline: the reference's own mechanism benchmark (bench.cpp:332-389).
int ref_mechanism_bench(const char* op, uint32_t n, uint32_t l, uint32_t alpha, uint32_t db,
                        uint32_t level, uint32_t reps, uint32_t warmup, uint64_t seed,
                        double* median_ns, double* min_ns, int* omp_threads, uint64_t* counters7) {
  try {
    bench::SweepSpec spec;
    spec.op = op;
    spec.n = n;
    spec.l = l;
    spec.alpha = alpha;
    spec.delta_bits = db;
    spec.level = level;
    spec.reps = reps;
    spec.warmup = warmup;
    spec.seed = seed;
    auto rep = bench::run_mechanism_bench(spec);
    const auto& row = rep.rows.at(0);
    *median_ns = row.median_ns;
    *min_ns = row.min_ns;
#ifdef _OPENMP
    *omp_threads = omp_get_max_threads();
#else
    *omp_threads = 1;
#endif
    for (size_t i = 0; i < row.counters.size() && i < 7; ++i) counters7[i] = row.counters[i].second;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// encode (ckks.cpp:278-319) of `count` complex slots (re, im interleaved) at
// scale num/den; writes the plaintext rows as canonical residues.
int ref_encode(uint32_t n, uint32_t l, uint32_t alpha, uint32_t db, const double* slots, uint32_t count,
               uint64_t num, uint64_t den, uint32_t level, int p_extend, uint32_t* out, size_t cap) {
  try {
    CkksContext ctx(make_params(n, l, alpha, db, false));
    std::vector<std::complex<double>> z(count);
    for (uint32_t t = 0; t < count; ++t) z[t] = {slots[2 * t], slots[2 * t + 1]};
    const Rational scale = Rational(BigInt(num)) / Rational(BigInt(den));
    Plaintext pt = encode(ctx, z, scale, level, p_extend != 0);
    put_canonical(pt.poly, out, 0, cap);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// decode (ckks.cpp:321-362) of plaintext rows given as canonical residues
// (evaluation domain, Montgomery); writes n/2 complex slots.  The scale is
// num / den given as little-endian 32-bit limbs (ref_decode: 64-bit values).
static BigInt from_limbs(const uint32_t* w, uint32_t nw) {
  BigInt x = 0;
  for (uint32_t i = nw; i-- > 0;) {
    x <<= 32;
    x += BigInt(w[i]);
  }
  return x;
}
int ref_decode_big(uint32_t n, uint32_t l, uint32_t alpha, uint32_t db, const uint32_t* rows, uint32_t level,
                   const uint32_t* num, uint32_t nnum, const uint32_t* den, uint32_t nden, double* out) {
  try {
    CkksContext ctx(make_params(n, l, alpha, db, false));
    Plaintext pt;
    pt.scale = Rational(from_limbs(num, nnum)) / Rational(from_limbs(den, nden));
    pt.level = level;
    pt.poly = Polynomial(ctx.basis(), level, 0, Domain::Evaluation, true, &ctx.pool());
    for (uint32_t i = 0; i < level; ++i)
      for (uint32_t k = 0; k < n; ++k) pt.poly.row(i)[k] = static_cast<int32_t>(rows[static_cast<size_t>(i) * n + k]);
    const auto z = decode(ctx, pt);
    for (uint32_t t = 0; t < n / 2; ++t) {
      out[2 * t] = z[t].real();
      out[2 * t + 1] = z[t].imag();
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

int ref_decode(uint32_t n, uint32_t l, uint32_t alpha, uint32_t db, const uint32_t* rows, uint32_t level,
               uint64_t num, uint64_t den, double* out) {
  try {
    CkksContext ctx(make_params(n, l, alpha, db, false));
    Plaintext pt;
    pt.scale = Rational(BigInt(num)) / Rational(BigInt(den));
    pt.level = level;
    pt.poly = Polynomial(ctx.basis(), level, 0, Domain::Evaluation, true, &ctx.pool());
    for (uint32_t i = 0; i < level; ++i)
      for (uint32_t k = 0; k < n; ++k) pt.poly.row(i)[k] = static_cast<int32_t>(rows[static_cast<size_t>(i) * n + k]);
    const auto z = decode(ctx, pt);
    for (uint32_t t = 0; t < n / 2; ++t) {
      out[2 * t] = z[t].real();
      out[2 * t + 1] = z[t].imag();
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

}  // extern "C"
