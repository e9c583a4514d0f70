// GPU backend for the reference's own C++ API.
//
// This translation unit is compiled against the reference's public headers
// (proj/include/ckks32/*.hpp, read-only) and defines the hot-path functions
// they declare -- NTT / INTT, base conversion, ModSwitch, automorphism, the
// element-wise operations, ModUp / KeyMult / ModDown / key switching,
// rescale, HMult, HRot, hoisting, HAdd / PAdd / PMult and the element-wise
// part of decrypt, encode / decode -- as calls into the sm_100a library through its C ABI
// (include/ck32_b200.h).  Linked in front of the reference's objects (whose
// definitions of exactly these symbols are weakened, see Makefile), it turns
// any reference caller into a GPU caller without touching the caller: the
// reference's own unit tests and acceptance suite are linked this way and run
// on the B200 (tests/test_ref_suite_gpu.py).
//
// What stays the reference's: the data types (Polynomial with host rows,
// BufferPool, RnsBasis, the Rational scale ledger), basis generation, table
// construction and key / randomness sampling (host-side in the reference
// too; their NTTs and element-wise products run here).  Every residue this backend hands back is canonical
// in [0, q) -- the reference's correct() view of its lazy values, which every
// reference consumer accepts; raw int32 equality with the CPU's lazy schedule
// is not part of the contract.
//
// Argument checks and exception types restate the reference's (the cited
// lines); the counters (OpCounters) advance by the GPU library's counts,
// which follow the reference's profile.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "ck32_b200.h"
#include "ckks32/automorphism.hpp"
#include "ckks32/bconv.hpp"
#include "ckks32/ckks.hpp"
#include "ckks32/ntt.hpp"
#include "ckks32/poly.hpp"

namespace ck32gpu {
using namespace ckks32;

void check(ck_status s) {
  if (s == CK_OK) return;
  const std::string msg = ck_last_error();
  if (s == CK_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error("ck32-b200: " + msg);
}

// One GPU context per (basis primes, lazy policy); kernel-level calls that
// only know primes (bconv_part2) reuse any context that holds them.
struct Gpu {
  ck_context* h = nullptr;
  uint32_t n = 0, l = 0, alpha = 0;
  std::vector<uint32_t> primes;  // Q then P
  std::map<uint32_t, uint32_t> index;  // prime -> global index in this context
  uint32_t gidx(uint32_t q) const {
    auto it = index.find(q);
    if (it == index.end()) throw std::invalid_argument("prime not in the GPU context");
    return it->second;
  }
};

std::map<std::vector<uint32_t>, std::unique_ptr<Gpu>>& registry() {
  static std::map<std::vector<uint32_t>, std::unique_ptr<Gpu>> r;
  return r;
}

Gpu& make(uint32_t n, uint32_t l, uint32_t alpha, uint32_t delta_bits, bool lazy, std::vector<uint32_t> primes) {
  std::vector<uint32_t> key = {n, l, alpha, delta_bits, lazy ? 1u : 0u};
  key.insert(key.end(), primes.begin(), primes.end());
  auto& slot = registry()[key];
  if (!slot) {
    auto g = std::make_unique<Gpu>();
    ck_params p{n, l, alpha, delta_bits, lazy ? 1 : 0};
    check(ck_context_create(&p, primes.data(), 0, &g->h));
    g->n = n;
    g->l = l;
    g->alpha = alpha;
    g->primes = std::move(primes);
    for (uint32_t i = 0; i < g->primes.size(); ++i) g->index.emplace(g->primes[i], i);
    slot = std::move(g);
  }
  return *slot;
}

Gpu& for_basis(const RnsBasis& b, bool lazy = false) {
  std::vector<uint32_t> pr;
  for (const auto& c : b.q_primes) pr.push_back(c.q);
  for (const auto& c : b.p_primes) pr.push_back(c.q);
  return make(b.n, (uint32_t)b.l(), (uint32_t)b.alpha(), b.delta_bits, lazy, std::move(pr));
}

Gpu& for_ctx(CkksContext& ctx) { return for_basis(*ctx.basis(), ctx.params().lazy_rescale); }

Gpu& for_primes(uint32_t n, const std::vector<uint32_t>& need) {
  for (auto& kv : registry()) {
    Gpu& g = *kv.second;
    if (g.n != n) continue;
    bool all = true;
    for (uint32_t q : need) all &= g.index.count(q) != 0;
    if (all) return g;
  }
  std::vector<uint32_t> u;  // an ad-hoc context over exactly these primes
  for (uint32_t q : need)
    if (std::find(u.begin(), u.end(), q) == u.end()) u.push_back(q);
  return make(n, (uint32_t)u.size(), 0, 0, false, u);
}

// Device buffer (the library's allocator).
struct Dev {
  ck_context* c = nullptr;
  void* p = nullptr;
  Dev(ck_context* ctx, size_t words) : c(ctx) {
    if (words) check(ck_malloc(c, words * 4, &p));
  }
  Dev(const Dev&) = delete;
  Dev(Dev&& o) noexcept : c(o.c), p(o.p) { o.p = nullptr; }
  ~Dev() {
    if (p) ck_free(c, p);
  }
  uint32_t* u() const { return static_cast<uint32_t*>(p); }
};

inline uint32_t canon(int64_t v, uint32_t q) {
  int64_t r = v % (int64_t)q;
  return (uint32_t)(r < 0 ? r + q : r);
}

// rows of p (canonicalised) -> device at dst
void put_rows(const Gpu& g, const Polynomial& p, uint32_t first, uint32_t count, uint32_t* dst) {
  const size_t n = p.n();
  std::vector<uint32_t> tmp((size_t)count * n);
  for (uint32_t i = 0; i < count; ++i) {
    const uint32_t q = p.prime_at(first + i).q;
    const int32_t* r = p.row(first + i);
    uint32_t* t = tmp.data() + (size_t)i * n;
    for (size_t j = 0; j < n; ++j) t[j] = canon(r[j], q);
  }
  if (!tmp.empty()) {
    check(ck_memcpy_h2d(g.h, dst, tmp.data(), tmp.size() * 4, nullptr));
    check(ck_stream_sync(g.h, nullptr));
  }
}
Dev up(const Gpu& g, const Polynomial& p) {
  Dev d(g.h, (size_t)p.rows() * p.n());
  put_rows(g, p, 0, p.rows(), d.u());
  return d;
}
// The element-wise ops keep the reference's raw representation (ops 4-6 of
// ck_ew_binary: its signed lazy int32 values and formulas, bit for bit), so
// callers that compare raw rows (test_poly.cpp:41, :112) see what the CPU
// code would have produced.
Dev up_raw(const Gpu& g, const Polynomial& p) {
  Dev d(g.h, (size_t)p.rows() * p.n());
  if (p.rows()) {
    check(ck_memcpy_h2d(g.h, d.u(), p.row(0), (size_t)p.rows() * p.n() * 4, nullptr));
    check(ck_stream_sync(g.h, nullptr));
  }
  return d;
}
// device rows -> p (rows are contiguous in the pool buffer)
void get_rows(const Gpu& g, const uint32_t* src, Polynomial& p, uint32_t first, uint32_t count) {
  if (!count) return;
  check(ck_memcpy_d2h(g.h, p.row(first), src, (size_t)count * p.n() * 4, nullptr));
  check(ck_stream_sync(g.h, nullptr));
}
Polynomial down(const Gpu& g, const uint32_t* src, std::shared_ptr<const RnsBasis> basis, uint32_t qc, uint32_t pc,
                Domain dom, bool mont, BufferPool* pool) {
  Polynomial p(std::move(basis), qc, pc, dom, mont, pool);
  get_rows(g, src, p, 0, qc + pc);
  return p;
}

// ciphertext -> device [2][level]
Dev up_ct(const Gpu& g, const Ciphertext& ct) {
  const size_t ln = (size_t)ct.level * g.n;
  Dev d(g.h, 2 * ln);
  put_rows(g, ct.b, 0, ct.level, d.u());
  put_rows(g, ct.a, 0, ct.level, d.u() + ln);
  return d;
}
Ciphertext down_ct(const Gpu& g, const uint32_t* src, CkksContext& ctx, uint32_t level) {
  Ciphertext ct;
  ct.level = level;
  ct.b = down(g, src, ctx.basis(), level, 0, Domain::Evaluation, true, &ctx.pool());
  ct.a = down(g, src + (size_t)level * g.n, ctx.basis(), level, 0, Domain::Evaluation, true, &ctx.pool());
  return ct;
}

// Evaluation keys stay resident: [D][2][L+alpha][n], re-uploaded only when the
// key object's contents change (full 64-bit fingerprint of its residues).
struct KeyEntry {
  uint64_t fp = 0;
  size_t digits = 0;
  std::unique_ptr<Dev> dev;
};
std::map<std::pair<const Gpu*, const EvaluationKey*>, KeyEntry>& key_cache() {
  static std::map<std::pair<const Gpu*, const EvaluationKey*>, KeyEntry> m;
  return m;
}
uint64_t fingerprint(const EvaluationKey& evk) {
  uint64_t h = 0x9e3779b97f4a7c15ull ^ evk.digits.size();
  for (const auto& [b, a] : evk.digits)
    for (const Polynomial* p : {&b, &a}) {
      const size_t words = (size_t)p->rows() * p->n();
      const int32_t* w = p->row(0);
      uint64_t acc = 0;
      for (size_t i = 0; i < words; ++i) acc = (acc ^ (uint32_t)w[i]) * 0x100000001b3ull;
      h = (h ^ acc) * 0xff51afd7ed558ccdull;
    }
  return h;
}
const uint32_t* key_dev(Gpu& g, const EvaluationKey& evk) {
  const uint32_t rows = g.l + g.alpha;
  for (const auto& [b, a] : evk.digits)
    if (b.q_count() != g.l || b.p_count() != g.alpha || a.q_count() != g.l || a.p_count() != g.alpha)
      throw std::invalid_argument("evaluation key digits must span the full PQ basis");
  KeyEntry& e = key_cache()[{&g, &evk}];
  const uint64_t fp = fingerprint(evk);
  if (!e.dev || e.fp != fp || e.digits != evk.digits.size()) {
    e.dev = std::make_unique<Dev>(g.h, evk.digits.size() * 2ull * rows * g.n);
    for (size_t k = 0; k < evk.digits.size(); ++k) {
      put_rows(g, evk.digits[k].first, 0, rows, e.dev->u() + (2 * k) * (size_t)rows * g.n);
      put_rows(g, evk.digits[k].second, 0, rows, e.dev->u() + (2 * k + 1) * (size_t)rows * g.n);
    }
    e.fp = fp;
    e.digits = evk.digits.size();
  }
  return e.dev->u();
}

// OpCounters advance by what the GPU library counted for the call.
struct Counted {
  const Gpu& g;
  CkksContext& ctx;
  uint64_t before[7];
  Counted(const Gpu& g_, CkksContext& c) : g(g_), ctx(c) { check(ck_context_counters(g.h, before)); }
  void commit() {
    uint64_t after[7];
    check(ck_context_counters(g.h, after));
    OpCounters& o = ctx.counters();
    o.modup += after[0] - before[0];
    o.moddown += after[1] - before[1];
    o.ntt += after[2] - before[2];
    o.intt += after[3] - before[3];
    o.keymult += after[4] - before[4];
    o.bconv += after[5] - before[5];
    o.rescale += after[6] - before[6];
  }
};

// --- the reference's argument checks (ckks.cpp:115-136, poly.cpp:115-119) ---
void check_eval_mont(const Polynomial& p, const char* what) {
  if (p.domain() != Domain::Evaluation || !p.mont())
    throw std::invalid_argument(std::string(what) + ": expected evaluation-domain Montgomery form");
}
void check_pair(const Ciphertext& ct) {
  if (!ct.b.shape_matches(ct.a) || ct.b.domain() != ct.a.domain() || ct.b.mont() != ct.a.mont())
    throw std::invalid_argument("ciphertext halves out of sync");
  check_eval_mont(ct.b, "ciphertext");
  if (ct.b.q_count() != ct.level || ct.b.p_count() != 0)
    throw std::invalid_argument("ciphertext level/shape mismatch");
}
void check_same_scale(const Rational& a, const Rational& b) {
  const Rational diff = a >= b ? a - b : b - a;
  if (diff * (BigInt(1) << 40) > a) throw std::invalid_argument("scale mismatch beyond tolerance");
}
void check_binary(const Polynomial& a, const Polynomial& b) {
  if (!a.shape_matches(b)) throw std::invalid_argument("basis prefix mismatch");
  if (a.domain() != b.domain()) throw std::invalid_argument("domain mismatch");
  if (a.mont() != b.mont()) throw std::invalid_argument("Montgomery flag mismatch");
}

uint32_t log2u(uint32_t n) {
  uint32_t b = 0;
  while ((1u << b) < n) ++b;
  return b;
}

}  // namespace ck32gpu

namespace ckks32 {
using namespace ck32gpu;

// ============================================================ kernel level ==
// NttPlan::forward_row / inverse_row (ntt.hpp:71-73): one row through the GPU.
void NttPlan::forward_row(int32_t* row, uint32_t gidx) const {
  // the reference's raw representation end to end (ck_ntt_forward_raw: its
  // signed lazy butterflies, bit for bit -- test_ntt.cpp:203-227 compares
  // raw rows with forward_row_serial)
  Gpu& g = for_basis(*tables().basis);
  Dev d(g.h, g.n);
  check(ck_memcpy_h2d(g.h, d.u(), row, g.n * 4, nullptr));
  check(ck_ntt_forward_raw(g.h, reinterpret_cast<int32_t*>(d.u()), 1, &gidx, nullptr));
  check(ck_memcpy_d2h(g.h, row, d.u(), g.n * 4, nullptr));
  check(ck_stream_sync(g.h, nullptr));
}

void NttPlan::inverse_row(int32_t* row, uint32_t gidx, const uint32_t* epilogue_mont) const {
  Gpu& g = for_basis(*tables().basis);
  Dev d(g.h, g.n);
  check(ck_memcpy_h2d(g.h, d.u(), row, g.n * 4, nullptr));
  check(ck_intt_inverse_raw(g.h, reinterpret_cast<int32_t*>(d.u()), 1, &gidx, epilogue_mont, nullptr));
  check(ck_memcpy_d2h(g.h, row, d.u(), g.n * 4, nullptr));
  check(ck_stream_sync(g.h, nullptr));
}

// ntt_forward / intt_inverse (ntt.cpp:288-312): whole polynomial, raw representation
void ntt_forward(Polynomial& p, const NttPlan& plan) {
  if (p.domain() != Domain::Coefficient) throw std::invalid_argument("ntt_forward expects coefficient domain");
  if (p.mont()) throw std::invalid_argument("ntt_forward expects plain form (entry merge)");
  Gpu& g = for_basis(*plan.tables().basis);
  Dev d = up_raw(g, p);
  std::vector<uint32_t> gi(p.rows());
  for (uint32_t i = 0; i < p.rows(); ++i) gi[i] = p.global_prime_index(i);
  check(ck_ntt_forward_raw(g.h, reinterpret_cast<int32_t*>(d.u()), p.rows(), gi.data(), nullptr));
  get_rows(g, d.u(), p, 0, p.rows());
  p.set_domain(Domain::Evaluation);
  p.set_mont(true);
}

void intt_inverse(Polynomial& p, const NttPlan& plan) {
  if (p.domain() != Domain::Evaluation) throw std::invalid_argument("intt_inverse expects evaluation domain");
  if (!p.mont()) throw std::invalid_argument("intt_inverse expects Montgomery form");
  Gpu& g = for_basis(*plan.tables().basis);
  Dev d = up_raw(g, p);
  std::vector<uint32_t> gi(p.rows());
  for (uint32_t i = 0; i < p.rows(); ++i) gi[i] = p.global_prime_index(i);
  check(ck_intt_inverse_raw(g.h, reinterpret_cast<int32_t*>(d.u()), p.rows(), gi.data(), nullptr, nullptr));
  get_rows(g, d.u(), p, 0, p.rows());
  p.set_domain(Domain::Coefficient);
  p.set_mont(false);
}

// bconv_part1 (bconv.cpp:64-80): row j times part1_mont[j], canonical
void bconv_part1(Polynomial& t, const BConvTable& table) {
  if (t.domain() != Domain::Coefficient) throw std::invalid_argument("part1 expects coefficient domain");
  if (t.rows() != table.src_count()) throw std::invalid_argument("row count does not match table source");
  for (uint32_t j = 0; j < t.rows(); ++j)
    if (t.prime_at(j).q != table.src[j].q) throw std::invalid_argument("source prime mismatch");
  Gpu& g = for_basis(*t.basis());
  Dev d = up(g, t);
  check(ck_ew_mul_const(g.h, d.u(), table.part1_mont.data(), d.u(), t.q_count(), t.p_count(), nullptr));
  get_rows(g, d.u(), t, 0, t.rows());
}

// bconv_part2 (bconv.cpp:96-174) with the caller's table
void bconv_part2(const int32_t* src, uint32_t n, const BConvTable& table, const BConvTiling& tiling,
                 int32_t* const* dst_rows) {
  const uint32_t rows = (uint32_t)table.dst_count(), sc = (uint32_t)table.src_count();
  validate_tiling(tiling, rows, n);  // the reference's own validation and errors
  if (rows == 0) return;
  std::vector<uint32_t> need;
  for (const auto& c : table.src) need.push_back(c.q);
  for (const auto& c : table.dst) need.push_back(c.q);
  Gpu& g = for_primes(n, need);
  std::vector<uint32_t> sg(sc), dg(rows), tmp((size_t)sc * n);
  for (uint32_t j = 0; j < sc; ++j) {
    sg[j] = g.gidx(table.src[j].q);
    for (uint32_t x = 0; x < n; ++x) tmp[(size_t)j * n + x] = canon(src[(size_t)j * n + x], table.src[j].q);
  }
  for (uint32_t i = 0; i < rows; ++i) dg[i] = g.gidx(table.dst[i].q);
  Dev s(g.h, (size_t)sc * n), o(g.h, (size_t)rows * n);
  check(ck_memcpy_h2d(g.h, s.u(), tmp.data(), tmp.size() * 4, nullptr));
  check(ck_bconv_table(g.h, s.u(), sc, sg.data(), o.u(), rows, dg.data(), table.c.data(), nullptr));
  std::vector<uint32_t> out((size_t)rows * n);
  check(ck_memcpy_d2h(g.h, out.data(), o.u(), out.size() * 4, nullptr));
  check(ck_stream_sync(g.h, nullptr));
  for (uint32_t i = 0; i < rows; ++i) std::memcpy(dst_rows[i], out.data() + (size_t)i * n, (size_t)n * 4);
}

// mod_switch (bconv.cpp:176-213): INTT with the table's part 1, the table's
// part 2, NTT -- all on the GPU, one upload and one download
Polynomial mod_switch(const Polynomial& a, uint32_t dst_q_count, uint32_t dst_p_count, const BConvTable& table,
                      const NttPlan& plan, const BConvTiling& tiling, BufferPool* pool) {
  if (a.domain() != Domain::Evaluation || !a.mont())
    throw std::invalid_argument("mod_switch expects evaluation-domain Montgomery input");
  if (a.rows() != table.src_count()) throw std::invalid_argument("input rows do not match table source");
  for (uint32_t j = 0; j < a.rows(); ++j)
    if (a.prime_at(j).q != table.src[j].q) throw std::invalid_argument("source prime mismatch");
  Polynomial out(a.basis(), dst_q_count, dst_p_count, Domain::Coefficient, false, pool);
  if (out.rows() != table.dst_count()) throw std::invalid_argument("output rows do not match table destination");
  for (uint32_t i = 0; i < out.rows(); ++i)
    if (out.prime_at(i).q != table.dst[i].q) throw std::invalid_argument("destination prime mismatch");
  validate_tiling(tiling, out.rows(), a.n());
  Gpu& g = for_basis(*plan.tables().basis);
  Dev w = up(g, a), o(g.h, (size_t)out.rows() * a.n());
  std::vector<uint32_t> sg(a.rows()), dg(out.rows());
  for (uint32_t j = 0; j < a.rows(); ++j) sg[j] = a.global_prime_index(j);
  for (uint32_t i = 0; i < out.rows(); ++i) dg[i] = out.global_prime_index(i);
  check(ck_intt_inverse(g.h, w.u(), a.rows(), sg.data(), table.part1_mont.data(), nullptr));
  check(ck_bconv_table(g.h, w.u(), a.rows(), sg.data(), o.u(), out.rows(), dg.data(), table.c.data(), nullptr));
  check(ck_ntt_forward(g.h, o.u(), out.rows(), dg.data(), nullptr));
  get_rows(g, o.u(), out, 0, out.rows());
  out.set_domain(Domain::Evaluation);
  out.set_mont(true);
  return out;
}

// apply_automorphism (automorphism.cpp:76-100): the map's Galois element is
// recovered from its own table (dest(0) = brev((g - 1) / 2)); the GPU
// computes both domains' index rules from it
namespace {
uint64_t galois_of(const AutomorphismMap& map) {
  const uint32_t bits = log2u(map.n());
  return 2ull * bit_reverse(map.dest(0), bits) + 1;
}
}  // namespace

Polynomial apply_automorphism(const Polynomial& p, const AutomorphismMap& map, BufferPool* pool) {
  if (p.n() != map.n()) throw std::invalid_argument("ring degree mismatch");
  Gpu& g = for_basis(*p.basis());
  Dev in = up(g, p), out(g.h, (size_t)p.rows() * p.n());
  check(ck_automorphism_galois(g.h, in.u(), out.u(), p.q_count(), p.p_count(), galois_of(map),
                               p.domain() == Domain::Coefficient, nullptr));
  return down(g, out.u(), p.basis(), p.q_count(), p.p_count(), p.domain(), p.mont(), pool);
}

void apply_automorphism_inplace(Polynomial& p, const AutomorphismMap& map) {
  if (p.domain() != Domain::Evaluation) throw std::invalid_argument("in-place variant is evaluation-domain only");
  if (p.n() != map.n()) throw std::invalid_argument("ring degree mismatch");
  Gpu& g = for_basis(*p.basis());
  Dev in = up(g, p), out(g.h, (size_t)p.rows() * p.n());
  check(ck_automorphism_galois(g.h, in.u(), out.u(), p.q_count(), p.p_count(), galois_of(map), 0, nullptr));
  get_rows(g, out.u(), p, 0, p.rows());
}

// element-wise (poly.cpp:121-205)
namespace {
Polynomial ew(int op, const Polynomial& a, const Polynomial& b, BufferPool* pool, bool mont_out) {
  check_binary(a, b);
  Gpu& g = for_basis(*a.basis());
  Dev x = up_raw(g, a), y = up_raw(g, b);
  check(ck_ew_binary(g.h, op + 4, x.u(), y.u(), x.u(), a.q_count(), a.p_count(), nullptr));
  return down(g, x.u(), a.basis(), a.q_count(), a.p_count(), a.domain(), mont_out, pool);
}
void ew_inplace(int op, Polynomial& a, const Polynomial& b) {
  check_binary(a, b);
  Gpu& g = for_basis(*a.basis());
  Dev x = up_raw(g, a), y = up_raw(g, b);
  check(ck_ew_binary(g.h, op + 4, x.u(), y.u(), x.u(), a.q_count(), a.p_count(), nullptr));
  get_rows(g, x.u(), a, 0, a.rows());
}
}  // namespace

Polynomial ew_add(const Polynomial& a, const Polynomial& b, BufferPool* pool) { return ew(0, a, b, pool, a.mont()); }
Polynomial ew_sub(const Polynomial& a, const Polynomial& b, BufferPool* pool) { return ew(1, a, b, pool, a.mont()); }
Polynomial ew_mul(const Polynomial& a, const Polynomial& b, BufferPool* pool) {
  if (!a.mont() || !b.mont()) throw std::invalid_argument("ew_mul expects Montgomery-form operands");
  return ew(2, a, b, pool, true);
}
Polynomial ew_mul_const(const Polynomial& a, std::span<const uint32_t> consts_mont, BufferPool* pool) {
  if (consts_mont.size() != a.rows()) throw std::invalid_argument("constant count mismatch");
  Gpu& g = for_basis(*a.basis());
  Dev x = up_raw(g, a);
  check(ck_ew_mul_const_raw(g.h, x.u(), consts_mont.data(), x.u(), a.q_count(), a.p_count(), nullptr));
  return down(g, x.u(), a.basis(), a.q_count(), a.p_count(), a.domain(), a.mont(), pool);
}
void ew_add_inplace(Polynomial& a, const Polynomial& b) { ew_inplace(0, a, b); }
void ew_sub_inplace(Polynomial& a, const Polynomial& b) { ew_inplace(1, a, b); }

// ============================================================== mechanisms ==
HoistState mod_up(CkksContext& ctx, const Polynomial& d) {  // ckks.cpp:680-731
  check_eval_mont(d, "mod_up");
  if (d.p_count() != 0) throw std::invalid_argument("mod_up input must be Q-only");
  Gpu& g = for_ctx(ctx);
  const uint32_t l = d.q_count(), rows = l + g.alpha, D = ctx.num_digits(l);
  Dev x = up(g, d), h(g.h, (size_t)D * rows * g.n);
  Counted cnt(g, ctx);
  check(ck_mod_up(g.h, l, x.u(), h.u(), nullptr));
  cnt.commit();
  HoistState hs;
  hs.level = l;
  for (uint32_t k = 0; k < D; ++k)
    hs.digits.push_back(down(g, h.u() + (size_t)k * rows * g.n, ctx.basis(), l, g.alpha, Domain::Evaluation, true,
                             &ctx.pool()));
  return hs;
}

std::pair<Polynomial, Polynomial> key_mult(CkksContext& ctx, const HoistState& hoist,
                                           const EvaluationKey& evk) {  // ckks.cpp:733-770
  const uint32_t l = hoist.level, D = (uint32_t)hoist.digits.size();
  if (evk.digits.size() < D) throw std::invalid_argument("evaluation key has too few digits");
  Gpu& g = for_ctx(ctx);
  const uint32_t rows = l + g.alpha;
  if (D != ctx.num_digits(l)) throw std::invalid_argument("hoist state does not match its level");
  Dev h(g.h, (size_t)D * rows * g.n), v(g.h, 2ull * rows * g.n);
  for (uint32_t k = 0; k < D; ++k) {
    if (hoist.digits[k].q_count() != l || hoist.digits[k].p_count() != g.alpha)
      throw std::invalid_argument("hoist digit shape mismatch");
    put_rows(g, hoist.digits[k], 0, rows, h.u() + (size_t)k * rows * g.n);
  }
  const uint32_t* k = key_dev(g, evk);
  Counted cnt(g, ctx);
  check(ck_key_mult(g.h, l, h.u(), k, v.u(), nullptr));
  cnt.commit();
  return {down(g, v.u(), ctx.basis(), l, g.alpha, Domain::Evaluation, true, &ctx.pool()),
          down(g, v.u() + (size_t)rows * g.n, ctx.basis(), l, g.alpha, Domain::Evaluation, true, &ctx.pool())};
}

Polynomial mod_down(CkksContext& ctx, const Polynomial& v) {  // ckks.cpp:772-776
  if (v.p_count() != ctx.params().alpha) throw std::invalid_argument("mod_down expects a P-extended polynomial");
  Gpu& g = for_ctx(ctx);
  const uint32_t l = v.q_count();
  Dev x = up(g, v), o(g.h, (size_t)l * g.n);
  Counted cnt(g, ctx);
  check(ck_mod_down(g.h, l, x.u(), o.u(), nullptr));
  cnt.commit();
  return down(g, o.u(), ctx.basis(), l, 0, Domain::Evaluation, true, &ctx.pool());
}

std::pair<Polynomial, Polynomial> key_switch(CkksContext& ctx, const Polynomial& d,
                                             const EvaluationKey& evk) {  // ckks.cpp:778-787
  check_eval_mont(d, "mod_up");
  if (d.p_count() != 0) throw std::invalid_argument("mod_up input must be Q-only");
  Gpu& g = for_ctx(ctx);
  const uint32_t l = d.q_count();
  if (evk.digits.size() < ctx.num_digits(l)) throw std::invalid_argument("evaluation key has too few digits");
  Dev x = up(g, d), o(g.h, 2ull * l * g.n);
  const uint32_t* k = key_dev(g, evk);
  Counted cnt(g, ctx);
  check(ck_key_switch(g.h, l, x.u(), k, o.u(), nullptr));
  cnt.commit();
  return {down(g, o.u(), ctx.basis(), l, 0, Domain::Evaluation, true, &ctx.pool()),
          down(g, o.u() + (size_t)l * g.n, ctx.basis(), l, 0, Domain::Evaluation, true, &ctx.pool())};
}

Ciphertext rescale(CkksContext& ctx, const Ciphertext& ct) {  // ckks.cpp:789-802
  check_pair(ct);
  const uint32_t l = ct.level;
  if (l < 4) throw std::invalid_argument("level exhausted");
  Gpu& g = for_ctx(ctx);
  Dev x = up_ct(g, ct), o(g.h, 2ull * (l - 2) * g.n);
  Counted cnt(g, ctx);
  check(ck_rescale(g.h, l, 1, x.u(), o.u(), nullptr));
  cnt.commit();
  Ciphertext out = down_ct(g, o.u(), ctx, l - 2);
  out.scale = ct.scale / Rational(BigInt(ctx.basis()->q_primes[l - 2].q) * ctx.basis()->q_primes[l - 1].q);
  out.pending_rescale = false;
  return out;
}

namespace {
// applies a deferred rescale first (ckks.cpp:663-676)
struct Flushed {
  Ciphertext storage;
  const Ciphertext* ct = nullptr;
  Flushed(CkksContext& ctx, const Ciphertext& in) {
    if (in.pending_rescale) {
      storage = rescale(ctx, in);
      ct = &storage;
    } else {
      ct = &in;
    }
  }
  const Ciphertext& operator*() const { return *ct; }
};
}  // namespace

Ciphertext hmult(CkksContext& ctx, const Ciphertext& x_in, const Ciphertext& y_in,
                 const EvaluationKey& relin) {  // ckks.cpp:804-865
  if (relin.kind != KeyKind::Relin) throw std::invalid_argument("hmult needs a relinearization key");
  Flushed fx(ctx, x_in), fy(ctx, y_in);
  const Ciphertext& x = *fx;
  const Ciphertext& y = *fy;
  check_pair(x);
  check_pair(y);
  if (x.level != y.level) throw std::invalid_argument("level mismatch");
  const uint32_t l = x.level;
  if (l < 4) throw std::invalid_argument("level exhausted");
  if (relin.digits.size() < ctx.num_digits(l)) throw std::invalid_argument("evaluation key has too few digits");
  Gpu& g = for_ctx(ctx);
  const bool lazy = ctx.params().lazy_rescale;
  const uint32_t lo = lazy ? l : l - 2;
  Dev dx = up_ct(g, x), dy = up_ct(g, y), o(g.h, 2ull * lo * g.n);
  const uint32_t* k = key_dev(g, relin);
  Counted cnt(g, ctx);
  check(ck_hmult(g.h, l, 1, dx.u(), dy.u(), k, o.u(), nullptr));
  cnt.commit();
  Ciphertext out = down_ct(g, o.u(), ctx, lo);
  if (!lazy) {
    out.scale = x.scale * y.scale /
                Rational(BigInt(ctx.basis()->q_primes[l - 2].q) * ctx.basis()->q_primes[l - 1].q);
    out.pending_rescale = false;
  } else {
    out.scale = x.scale * y.scale;
    out.pending_rescale = true;
  }
  return out;
}

Ciphertext hrot(CkksContext& ctx, const Ciphertext& ct_in, int64_t r,
                const EvaluationKey& evk) {  // ckks.cpp:869-897
  Flushed f(ctx, ct_in);
  const Ciphertext& ct = *f;
  check_pair(ct);
  if (evk.kind != KeyKind::Rotation || evk.rotation != r) throw std::invalid_argument("rotation key mismatch");
  if (evk.digits.size() < ctx.num_digits(ct.level)) throw std::invalid_argument("evaluation key has too few digits");
  Gpu& g = for_ctx(ctx);
  Dev x = up_ct(g, ct), o(g.h, 2ull * ct.level * g.n);
  const uint32_t* k = key_dev(g, evk);
  Counted cnt(g, ctx);
  check(ck_hrot(g.h, ct.level, 1, x.u(), r, k, o.u(), nullptr));
  cnt.commit();
  Ciphertext out = down_ct(g, o.u(), ctx, ct.level);
  out.scale = ct.scale;
  return out;
}

std::vector<Ciphertext> hoisted_rotations(CkksContext& ctx, const Ciphertext& ct_in,
                                          std::span<const int64_t> rotations,
                                          std::span<const EvaluationKey* const> evks) {  // ckks.cpp:899-925
  if (rotations.size() != evks.size()) throw std::invalid_argument("rotation/key count mismatch");
  Flushed f(ctx, ct_in);
  const Ciphertext& ct = *f;
  check_pair(ct);
  Gpu& g = for_ctx(ctx);
  std::vector<const uint32_t*> keys(rotations.size(), nullptr);
  for (size_t i = 0; i < rotations.size(); ++i) {
    if (rotations[i] == 0) continue;
    if (!evks[i]) throw std::invalid_argument("missing rotation key");
    if (evks[i]->kind != KeyKind::Rotation || evks[i]->rotation != rotations[i])
      throw std::invalid_argument("rotation key mismatch");
    keys[i] = key_dev(g, *evks[i]);
  }
  const size_t cw = 2ull * ct.level * g.n;
  Dev x = up_ct(g, ct), o(g.h, cw * rotations.size());
  Counted cnt(g, ctx);
  check(ck_hoisted_rotations(g.h, ct.level, x.u(), (uint32_t)rotations.size(), rotations.data(), keys.data(), o.u(),
                             nullptr));
  cnt.commit();
  std::vector<Ciphertext> out;
  for (size_t i = 0; i < rotations.size(); ++i) {
    out.push_back(down_ct(g, o.u() + i * cw, ctx, ct.level));
    out.back().scale = ct.scale;
  }
  return out;
}

Ciphertext hoisted_rotate_accumulate(CkksContext& ctx, const Ciphertext& ct_in, std::span<const int64_t> rotations,
                                     std::span<const Plaintext* const> pts,
                                     std::span<const EvaluationKey* const> evks) {  // ckks.cpp:945-1012
  if (rotations.empty() || rotations.size() != pts.size() || rotations.size() != evks.size())
    throw std::invalid_argument("rotation/plaintext/key count mismatch");
  Flushed f(ctx, ct_in);
  const Ciphertext& ct = *f;
  check_pair(ct);
  const uint32_t l = ct.level, alpha = ctx.params().alpha;
  for (const Plaintext* pt : pts) {
    if (!pt) throw std::invalid_argument("missing plaintext");
    check_eval_mont(pt->poly, "hoisted accumulate");
    if (pt->level != l || pt->poly.p_count() != alpha)
      throw std::invalid_argument("plaintexts must be P-extended at the ciphertext level");
    check_same_scale(pts[0]->scale, pt->scale);
  }
  Gpu& g = for_ctx(ctx);
  std::vector<const uint32_t*> keys(rotations.size(), nullptr);
  for (size_t i = 0; i < rotations.size(); ++i) {
    if (rotations[i] == 0) continue;
    if (!evks[i] || evks[i]->kind != KeyKind::Rotation || evks[i]->rotation != rotations[i])
      throw std::invalid_argument("rotation key mismatch");
    keys[i] = key_dev(g, *evks[i]);
  }
  std::vector<Dev> pdev;
  std::vector<const uint32_t*> pp;
  for (const Plaintext* pt : pts) {
    pdev.push_back(up(g, pt->poly));
    pp.push_back(pdev.back().u());
  }
  Dev x = up_ct(g, ct), o(g.h, 2ull * l * g.n);
  Counted cnt(g, ctx);
  check(ck_hoisted_rotate_accumulate(g.h, l, x.u(), (uint32_t)rotations.size(), rotations.data(), pp.data(),
                                     keys.data(), o.u(), nullptr));
  cnt.commit();
  Ciphertext out = down_ct(g, o.u(), ctx, l);
  out.scale = ct.scale * pts[0]->scale;
  return out;
}

// element-wise mechanisms (ckks.cpp:557-600)
Ciphertext hadd(CkksContext& ctx, const Ciphertext& x, const Ciphertext& y) {
  check_pair(x);
  check_pair(y);
  if (x.level != y.level) throw std::invalid_argument("level mismatch");
  if (x.pending_rescale != y.pending_rescale) throw std::invalid_argument("pending-rescale state mismatch");
  check_same_scale(x.scale, y.scale);
  Gpu& g = for_ctx(ctx);
  Dev dx = up_ct(g, x), dy = up_ct(g, y), o(g.h, 2ull * x.level * g.n);
  check(ck_hadd(g.h, x.level, 1, dx.u(), dy.u(), o.u(), nullptr));
  Ciphertext out = down_ct(g, o.u(), ctx, x.level);
  out.scale = x.scale;
  out.pending_rescale = x.pending_rescale;
  return out;
}

Ciphertext padd(CkksContext& ctx, const Ciphertext& ct, const Plaintext& pt) {
  check_pair(ct);
  check_eval_mont(pt.poly, "padd");
  if (ct.level != pt.level || pt.poly.p_count() != 0) throw std::invalid_argument("level mismatch");
  check_same_scale(ct.scale, pt.scale);
  Gpu& g = for_ctx(ctx);
  Dev dx = up_ct(g, ct), dp = up(g, pt.poly), o(g.h, 2ull * ct.level * g.n);
  check(ck_padd(g.h, ct.level, 1, dx.u(), dp.u(), o.u(), nullptr));
  Ciphertext out = down_ct(g, o.u(), ctx, ct.level);
  out.scale = ct.scale;
  out.pending_rescale = ct.pending_rescale;
  return out;
}

Ciphertext pmult(CkksContext& ctx, const Ciphertext& ct, const Plaintext& pt) {
  check_pair(ct);
  check_eval_mont(pt.poly, "pmult");
  if (ct.level != pt.level || pt.poly.p_count() != 0) throw std::invalid_argument("level mismatch");
  Gpu& g = for_ctx(ctx);
  Dev dx = up_ct(g, ct), dp = up(g, pt.poly), o(g.h, 2ull * ct.level * g.n);
  check(ck_pmult(g.h, ct.level, 1, dx.u(), dp.u(), o.u(), nullptr));
  Ciphertext out = down_ct(g, o.u(), ctx, ct.level);
  out.scale = ct.scale * pt.scale;
  out.pending_rescale = ct.pending_rescale;
  return out;
}

// encode (ckks.cpp:278-319): the GPU encoder replays the reference's FFT and
// its x87 long-double scaling, so the residues are the reference's bit for bit
Plaintext encode(CkksContext& ctx, std::span<const std::complex<double>> slots, const Rational& scale, uint32_t level,
                 bool p_extend) {
  const uint32_t n = ctx.params().n;
  if (slots.size() > n / 2) throw std::invalid_argument("too many slots");
  if (level < 1 || level > ctx.params().l) throw std::invalid_argument("level out of range");
  if (scale <= 0 || log2_rational(scale) > 60.0) throw std::invalid_argument("scale out of the representable range");
  Gpu& g = for_ctx(ctx);
  const uint32_t pc = p_extend ? ctx.params().alpha : 0;
  Dev z(g.h, std::max<size_t>(1, 4 * slots.size())), o(g.h, (size_t)(level + pc) * n);
  if (!slots.empty()) check(ck_memcpy_h2d(g.h, z.u(), slots.data(), slots.size() * 16, nullptr));
  check(ck_encode(g.h, reinterpret_cast<const double*>(z.u()), (uint32_t)slots.size(), log2_rational(scale), level,
                  p_extend ? 1 : 0, o.u(), nullptr));
  Plaintext pt;
  pt.scale = scale;
  pt.level = level;
  pt.poly = down(g, o.u(), ctx.basis(), level, pc, Domain::Evaluation, true, &ctx.pool());
  ctx.counters().ntt += level + pc;  // as the reference's encode counts it (ckks.cpp:317)
  return pt;
}

// decode (ckks.cpp:321-362): the exact rational scale goes to the GPU, which
// rounds Rational(v) / scale to double once, as the reference: bit-identical slots
std::vector<std::complex<double>> decode(CkksContext& ctx, const Plaintext& pt) {
  check_eval_mont(pt.poly, "decode");
  const uint32_t n = ctx.params().n;
  const double need_bits = log2_rational(pt.scale) + 40.0;  // the reference's prefix rule (ckks.cpp:326-333)
  uint32_t c = 1;
  double bits = std::log2((double)ctx.basis()->q_primes[0].q);
  while (c < pt.level && bits < need_bits) bits += std::log2((double)ctx.basis()->q_primes[c++].q);
  Gpu& g = for_ctx(ctx);
  Dev x(g.h, (size_t)pt.level * n), z(g.h, (size_t)n / 2 * 4);
  put_rows(g, pt.poly, 0, pt.level, x.u());
  {  // the exact rational scale (the shim's limbs): slots bit-identical to the reference's
    const BigInt sn = boost::multiprecision::numerator(pt.scale), sd = boost::multiprecision::denominator(pt.scale);
    const auto& nl = sn.limbs();
    const auto& dl = sd.limbs();
    if (!nl.empty() && !dl.empty() && nl.size() <= 8 && dl.size() <= 8)
      check(ck_decode_rational(g.h, x.u(), pt.level, log2_rational(pt.scale), nl.data(), (uint32_t)nl.size(), dl.data(),
                               (uint32_t)dl.size(), reinterpret_cast<double*>(z.u()), nullptr));
    else
      check(ck_decode(g.h, x.u(), pt.level, log2_rational(pt.scale), reinterpret_cast<double*>(z.u()), nullptr));
  }
  std::vector<std::complex<double>> out(n / 2);
  check(ck_memcpy_d2h(g.h, out.data(), z.u(), out.size() * 16, nullptr));
  check(ck_stream_sync(g.h, nullptr));
  ctx.counters().intt += c;
  return out;
}

Plaintext decrypt(CkksContext& ctx, const Ciphertext& ct, const SecretKey& sk) {  // ckks.cpp:541-555
  check_pair(ct);
  Gpu& g = for_ctx(ctx);
  Dev dx = up_ct(g, ct), ds(g.h, (size_t)ct.level * g.n), o(g.h, (size_t)ct.level * g.n);
  put_rows(g, sk.s, 0, ct.level, ds.u());
  check(ck_decrypt(g.h, ct.level, 1, dx.u(), ds.u(), o.u(), nullptr));
  Plaintext pt;
  pt.scale = ct.scale;
  pt.level = ct.level;
  pt.poly = down(g, o.u(), ctx.basis(), ct.level, 0, Domain::Evaluation, true, &ctx.pool());
  return pt;
}

}  // namespace ckks32
