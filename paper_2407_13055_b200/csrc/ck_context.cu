// Host runtime of ck32-b200: basis and table generation, per-level plans,
// mechanism orchestration and the extern "C" ABI declared in
// include/ck32_b200.h.
//
// Host-side table math restates the reference (rns.cpp:63-117 basis,
// modarith.cpp:30-54 roots/Montgomery constants, ntt.cpp:100-135 twiddles,
// bconv.cpp:13-46 conversion tables, ckks.cpp:188-265 per-level tables) with
// machine-word modular arithmetic: (P/P_j) mod q is the product of the other
// source primes reduced mod q, so no big integers are needed.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/ck32_b200.h"
#include "ck_common.cuh"
#include "ck_kernels.h"

// NVTX range per C-ABI mechanism call (tracing), visible in Nsight
// timelines; a no-op (one pointer test) when no tool is attached.
namespace {
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace
#define CK_RANGE(name) NvtxRange ck_nvtx_range_(name)

namespace ck {
namespace {
thread_local std::string g_err;
}  // namespace
// the message ck_last_error() returns, for ABI entry points in other files (wire.cpp)
void set_last_error(const char* msg) { g_err = msg; }
namespace {

struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define CK_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) throw CudaError(std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ------------------------------------------------------------ modular math --
uint64_t pow_mod(uint64_t b, uint64_t e, uint64_t m) {
  unsigned __int128 acc = 1 % m;
  b %= m;
  while (e) {
    if (e & 1) acc = acc * b % m;
    b = (uint64_t)((unsigned __int128)b * b % m);
    e >>= 1;
  }
  return (uint64_t)acc;
}
uint32_t mulm(uint32_t a, uint32_t b, uint32_t q) { return (uint32_t)((uint64_t)a * b % q); }
uint32_t invm(uint32_t a, uint32_t q) { return (uint32_t)pow_mod(a, q - 2, q); }
uint32_t shoup(uint32_t w, uint32_t q) { return (uint32_t)(((uint64_t)w << 32) / q); }
uint32_t r_mod(uint32_t q) { return (uint32_t)((1ull << 32) % q); }
uint32_t to_mont(uint32_t a, uint32_t q) { return (uint32_t)(((uint64_t)a << 32) % q); }
uint32_t bit_reverse(uint32_t x, uint32_t bits) {
  uint32_t r = 0;
  for (uint32_t i = 0; i < bits; ++i) r |= ((x >> i) & 1u) << (bits - 1 - i);
  return r;
}

// Deterministic Miller-Rabin (modarith.cpp:7-28).
bool is_prime(uint64_t v) {
  static const uint64_t bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (v < 2) return false;
  for (uint64_t p : bases)
    if (v % p == 0) return v == p;
  uint64_t d = v - 1;
  int s = 0;
  while ((d & 1) == 0) d >>= 1, ++s;
  for (uint64_t a : bases) {
    uint64_t x = pow_mod(a, d, v);
    if (x == 1 || x == v - 1) continue;
    bool composite = true;
    for (int i = 1; i < s; ++i) {
      x = (uint64_t)((unsigned __int128)x * x % v);
      if (x == v - 1) {
        composite = false;
        break;
      }
    }
    if (composite) return false;
  }
  return true;
}

// First g >= 2 whose (q-1)/2N power has order 2N (modarith.cpp:30-40): the
// exact root choice fixes the evaluation-point order, so it is parity-critical.
uint32_t find_root_2n(uint32_t q, uint32_t n) {
  const uint64_t order = 2ull * n;
  if ((q - 1) % order != 0) throw InvalidArgument("q not NTT-friendly for n");
  const uint64_t cof = (q - 1) / order;
  for (uint64_t g = 2; g < q; ++g) {
    const uint64_t cand = pow_mod(g, cof, q);
    if (pow_mod(cand, n, q) == q - 1) return (uint32_t)cand;
  }
  throw std::runtime_error("no primitive 2N-th root found");
}

// Largest primes = 1 mod 2n below `top`, descending (rns.cpp:10-20).
std::vector<uint32_t> scan_down(uint64_t top, uint64_t two_n, size_t count, uint64_t stop_at = 0) {
  std::vector<uint32_t> out;
  uint64_t k = (top - 1) / two_n * two_n + 1;
  if (k >= top) k -= two_n;
  for (; k > two_n && k > stop_at && out.size() < count; k -= two_n)
    if (is_prime(k)) out.push_back((uint32_t)k);
  return out;
}

// generate_basis (rns.cpp:63-117): Q primes in delta groups, worst-matched
// groups first; P primes the largest admissible below the cap.
std::vector<uint32_t> generate_basis(uint32_t n, uint32_t l, uint32_t alpha, uint32_t db) {
  if (n == 0 || (n & (n - 1)) != 0) throw InvalidArgument("n must be a power of two");
  if (l == 0 || l % 2 != 0) throw InvalidArgument("l must be positive and even");
  const uint64_t two_n = 2ull * n;
  const uint64_t cap = std::min<uint64_t>(1ull << 29, (1ull << 32) / std::max<uint32_t>(alpha + 2, 3));
  const uint64_t slots = cap > two_n ? (cap - two_n) / two_n : 0;
  if (slots < l + alpha) throw std::runtime_error("prime window smaller than requested prime count");
  auto p_list = scan_down(cap, two_n, alpha);
  if (p_list.size() < alpha) throw std::runtime_error("too few auxiliary primes");
  const uint64_t p_min = alpha ? p_list.back() : cap;
  uint64_t q_top = std::min<uint64_t>(cap, (uint64_t)std::sqrt(std::ldexp(1.0, (int)db + 1)));
  q_top = std::min(q_top, p_min);
  auto cands = scan_down(q_top, two_n, l);
  if (cands.size() < l) {
    auto extra = scan_down(p_min, two_n, (size_t)-1, q_top - 1);
    cands.insert(cands.end(), extra.begin(), extra.end());
  }
  std::sort(cands.begin(), cands.end());
  cands.erase(std::unique(cands.begin(), cands.end()), cands.end());
  if (cands.size() < l) throw std::runtime_error("too few main primes");
  struct Group {
    uint32_t a, b;
    double lg() const { return std::log2((double)a) + std::log2((double)b); }
  };
  std::vector<Group> groups;
  double lo = std::ldexp(1.0, (int)db - 1), hi = std::ldexp(1.0, (int)db + 1);
  for (int widen = 0; groups.size() < l / 2 && widen <= 12; ++widen) {
    size_t i = 0;
    while (i < cands.size() && groups.size() < l / 2) {
      const double a = (double)cands[i];
      size_t j = cands.size() - 1;
      while (j > i && a * (double)cands[j] >= hi) --j;
      if (j > i && a * (double)cands[j] >= lo) {
        groups.push_back({std::max(cands[i], cands[j]), std::min(cands[i], cands[j])});
        cands.erase(cands.begin() + j);
        cands.erase(cands.begin() + i);
      } else {
        ++i;
      }
    }
    lo /= 2;
    hi *= 2;
  }
  if (groups.size() < l / 2) throw std::runtime_error("cannot form enough delta groups in the prime window");
  std::stable_sort(groups.begin(), groups.end(), [&](const Group& x, const Group& y) {
    return std::abs(x.lg() - db) > std::abs(y.lg() - db);
  });
  std::vector<uint32_t> primes;
  for (const auto& g : groups) {
    primes.push_back(g.a);
    primes.push_back(g.b);
  }
  primes.insert(primes.end(), p_list.begin(), p_list.end());
  return primes;
}

// ---------------------------------------------------------------- device blob
// One cudaMalloc holding a plan's small tables (job lists, constants, maps).
class Blob {
 public:
  Blob() = default;
  Blob(const Blob&) = delete;  // owns a device allocation
  Blob& operator=(const Blob&) = delete;
  Blob(Blob&& o) noexcept : host_(std::move(o.host_)), dev_(o.dev_) { o.dev_ = nullptr; }
  Blob& operator=(Blob&& o) noexcept {
    if (this != &o) {
      if (dev_) cudaFree(dev_);
      host_ = std::move(o.host_);
      dev_ = o.dev_;
      o.dev_ = nullptr;
    }
    return *this;
  }
  template <class T>
  size_t add(const std::vector<T>& v) {
    const size_t off = (host_.size() + 15) / 16 * 16;
    host_.resize(off + v.size() * sizeof(T));
    if (!v.empty()) std::memcpy(host_.data() + off, v.data(), v.size() * sizeof(T));
    return off;
  }
  void upload() {
    if (dev_) cudaFree(dev_);
    CK_CUDA(cudaMalloc(&dev_, std::max<size_t>(host_.size(), 16)));
    CK_CUDA(cudaMemcpy(dev_, host_.data(), host_.size(), cudaMemcpyHostToDevice));
  }
  template <class T>
  T* at(size_t off) const {
    return reinterpret_cast<T*>(static_cast<char*>(dev_) + off);
  }
  ~Blob() {
    if (dev_) cudaFree(dev_);
  }

 private:
  std::vector<char> host_;
  void* dev_ = nullptr;
};

struct NttPlan {  // one batched transform
  Blob blob;
  size_t jobs_off = 0, exits_off = 0;
  int njobs = 0;
};
struct BconvPlan {
  Blob blob;
  size_t groups_off = 0, cmat_off = 0, row_off = 0, prime_off = 0;
  int ngroups = 0, max_sc = 1;
  uint64_t src_rows = 0, dst_rows = 0;  // algorithmic rows read / written per batch item
  // tensor-core path (bconv_tc.cu): per-group split-word B tables
  bool tc_ok = false;
  size_t tc_tab_off = 0, tc_boff_off = 0;
  int tc_max_npad = 0, tc_max_dc = 0;
};

// Split-word B tables of the tcgen05 BConv (bconv_tc.cu) for every group of a
// plan: row n = 4 i + a (destination i, byte a), column k = 4 j + b (source j,
// byte b) holds byte a of (C[i][j] * 2^(8b) mod q_i), laid out in the UMMA
// canonical K-major no-swizzle layout (8-row x 16-byte core matrices).
template <class QF>
void add_bconv_tc(BconvPlan& bp, const std::vector<BconvGroup>& groups, const std::vector<uint32_t>& cmat,
                  const std::vector<uint16_t>& dprime, QF qf, uint32_t n) {
  int max_sc = 0, max_dc = 0;
  for (const auto& G : groups) {
    max_sc = std::max(max_sc, (int)G.sc);
    max_dc = std::max(max_dc, (int)G.dc);
  }
  bp.tc_ok = !groups.empty() && bconv_tc_supported((int)n, max_sc, max_dc);
  if (!bp.tc_ok) return;
  const int KB = max_sc > 8 ? 64 : 32, sbo = (KB / 16) * 128;
  std::vector<uint8_t> tab;
  std::vector<uint32_t> offs;
  for (const auto& G : groups) {
    const int npad = (4 * (int)G.dc + 15) / 16 * 16;
    bp.tc_max_npad = std::max(bp.tc_max_npad, npad);
    const size_t off = tab.size();
    offs.push_back((uint32_t)off);
    tab.resize(off + (size_t)npad * KB, 0);
    for (uint32_t i = 0; i < G.dc; ++i) {
      const uint32_t qi = qf(dprime[G.map_off + i]);
      for (uint32_t j = 0; j < G.sc; ++j) {
        const uint64_t c = cmat[G.cmat_off + i * G.sc + j];
        for (int b = 0; b < 4; ++b) {
          const uint32_t cp = (uint32_t)((c << (8 * b)) % qi);
          for (int a = 0; a < 4; ++a) {
            const int nr = 4 * (int)i + a, kc = 4 * (int)j + b;
            tab[off + (nr / 8) * sbo + (kc / 16) * 128 + (nr % 8) * 16 + (kc % 16)] = (uint8_t)(cp >> (8 * a));
          }
        }
      }
    }
  }
  bp.tc_max_dc = max_dc;
  bp.tc_boff_off = bp.blob.add(offs);
  bp.tc_tab_off = bp.blob.add(tab);
}
// ModUp at one level: INTT(+part1) of the level rows, per-digit BConv, NTT.
// Tables of the fused INTT-B -> BConv -> NTT-1 kernel (ntt256.cu k_conv_mid).
struct ConvMidPlan {
  Blob blob;
  size_t groups_off = 0, cmat_off = 0, row_off = 0, prime_off = 0, sprime_off = 0, sexit_off = 0;
  int ngroups = 0, max_sc = 1;
};
struct ModUpPlan {
  uint32_t level = 0, D = 0;
  NttPlan intt, ntt;
  BconvPlan bc;
  ConvMidPlan cm;
  uint64_t ntt_rows = 0;
};
// drop_and_divide for npoly polynomials of (out_q + sc) rows each.
struct SwitchPlan {
  uint32_t out_q = 0, sc = 0, npoly = 0;
  NttPlan intt, ntt;
  BconvPlan bc;
  ConvMidPlan cm;
  Blob consts;  // div_inv_mont [out_q]
};

}  // namespace

// ================================================================ context ==
struct Context {
  ck_params p{};
  int device = 0;
  uint32_t n = 0, logn = 0, L = 0, alpha = 0;
  std::vector<uint32_t> primes;  // Q then P
  std::vector<uint32_t> psi;
  std::vector<PrimeDev> pdev_host;
  PrimeDev* d_primes = nullptr;
  uint2* d_fwd = nullptr;
  uint2* d_inv = nullptr;
  uint32_t* d_pmont = nullptr;  // P mod q_i (Montgomery), i < L
  uint2* d_tw2f = nullptr;      // N = 2^16 row-pass tables (ntt256.cu), per-row permuted
  uint2* d_tw2i = nullptr;
  bool use_ntt256 = true;
  bool use_cluster = false;  // CK32_NTT_CLUSTER=1: single-pass 8-CTA cluster/DSMEM NTT (slower today)
  bool use_row_km = true;
  bool use_fused_combine = true;  // CK32_NO_FUSED_COMBINE=1: separate k_combine after the ModDown NTT
  bool use_hrot_tail = false;     // CK32_FUSED_TAIL=1: HRot tail fused into the ModDown forward row pass (measured
                                  // neutral: 16.82k vs 16.86k ops/s, profiles/r2/README.md), else k_hrot_tail
  bool use_tc = true;  // tcgen05 split-word BConv (bconv_tc.cu; CK32_TC=0: the CUDA-core k_bconv)  // CK32_NO_ROW_KEYMULT=1: separate NTT row pass and KeyMult kernels
  bool tail_gather = false;  // CK32_TAIL_GATHER=1: the gather HRot tail (one coefficient per thread), else k_hrot_tail4
  int tc_var = 2;       // tcgen05 BConv kernel: 1 = k_bconv_tc, 2 = k_bconv_tc2 (slimmer epilogue; default)
  int bconv_fp64 = 0;   // CK32_BCONV_FP64=1|2|3: exact BConv dot products on the FP64 pipe for all / 1 of 2 / 2 of 3 rows
  bool use_fused = false;  // CK32_FUSED=1: INTT-B + BConv + NTT-1 in one kernel (k_conv_mid; slower today)
  int ntt_chunk_limbs = 1 << 30;  // limbs per pass-1/pass-2 launch pair (CK32_NTT_CHUNK; measured: no gain)
  std::map<uint32_t, std::unique_ptr<ModUpPlan>> modup;
  std::map<std::tuple<int, uint32_t, uint32_t>, std::unique_ptr<SwitchPlan>> switches;
  std::map<int64_t, uint32_t*> rot_maps;
  std::map<std::string, std::unique_ptr<NttPlan>> adhoc_ntt;
  std::map<std::string, std::unique_ptr<BconvPlan>> adhoc_bc;
  std::map<uint32_t, std::unique_ptr<Blob>> row_primes;  // (level+alpha)-row prime maps
  std::map<std::pair<uint32_t, uint32_t>, std::unique_ptr<Blob>> poly_maps;  // (q_rows, p_rows) -> row prime map
  // row -> global prime of a Polynomial with q_rows Q-prefix rows then p_rows
  // P rows (poly.hpp:103-106), cached on the device
  const uint16_t* poly_row_primes(uint32_t q_rows, uint32_t p_rows) {
    if (q_rows > L || p_rows > alpha || q_rows + p_rows == 0) throw InvalidArgument("rows exceed the basis");
    auto& b = poly_maps[{q_rows, p_rows}];
    if (!b) {
      std::vector<uint16_t> rp(q_rows + p_rows);
      for (uint32_t i = 0; i < q_rows + p_rows; ++i) rp[i] = (uint16_t)(i < q_rows ? i : L + (i - q_rows));
      b = std::make_unique<Blob>();
      b->add(rp);
      b->upload();
    }
    return b->at<uint16_t>(0);
  }
  struct Scratch {
    void* ptr = nullptr;
    size_t bytes = 0;
  };
  std::map<cudaStream_t, Scratch> scratch;  // one arena per stream: mechanisms on different streams run concurrently
  uint64_t counters[7] = {0, 0, 0, 0, 0, 0, 0};  // modup moddown ntt intt keymult bconv rescale
  std::atomic<uint64_t> launches{0};

  // Optional per-kernel-class CUDA-event timing (ck_profile): each launch
  // group is bracketed by events on its own stream; algorithmic bytes per
  // launch follow SURVEY.md §8(d).
  struct ProfRec {
    int cls;
    cudaEvent_t a, b;
    double bytes;
    uint64_t launches;
  };
  bool prof = false;
  std::vector<ProfRec> prof_recs;
  std::vector<cudaEvent_t> ev_pool;
  cudaEvent_t ev_get() {
    if (ev_pool.empty()) {
      cudaEvent_t e;
      CK_CUDA(cudaEventCreate(&e));
      return e;
    }
    cudaEvent_t e = ev_pool.back();
    ev_pool.pop_back();
    return e;
  }
  struct ProfScope {
    Context* c;
    cudaStream_t st;
    int cls;
    double bytes;
    uint64_t nl;
    cudaEvent_t a = nullptr;
    ProfScope(Context* c_, int cls_, double bytes_, uint64_t nl_, cudaStream_t st_)
        : c(c_), st(st_), cls(cls_), bytes(bytes_), nl(nl_) {
      if (c->prof) {
        a = c->ev_get();
        cudaEventRecord(a, st);
      }
    }
    ~ProfScope() {
      if (a) {
        cudaEvent_t b = c->ev_get();
        cudaEventRecord(b, st);
        c->prof_recs.push_back({cls, a, b, bytes, nl});
      }
    }
  };

  // encode / decode tables (encode.cu), built on first use
  double2 *d_fft_fwd = nullptr, *d_fft_inv = nullptr, *d_twist_enc = nullptr, *d_twist_dec = nullptr;
  uint32_t* d_jidx = nullptr;
  std::map<uint32_t, Blob> crt_consts;  // prefix length -> device CRT constants

  // Host tables restating ckks.cpp:63-99 and :301-303, :346: per-stage FFT
  // twiddles with the reference's recurrence (w *= wl, std::complex<double>,
  // host-compiled like the reference so every value is bit-identical), the
  // encode twist psi^-k, the decode twist psi^k, and the slot order 5^t.
  void enc_tables() {
    if (d_jidx) return;
    const uint32_t nn = n;
    std::vector<double2> tw[2] = {std::vector<double2>(nn - 1), std::vector<double2>(nn - 1)};
    for (int inv = 0; inv < 2; ++inv)
      for (uint32_t len = 2; len <= nn; len <<= 1) {
        const double ang = (inv ? -2.0 : 2.0) * M_PI / static_cast<double>(len);
        const std::complex<double> wl(std::cos(ang), std::sin(ang));
        std::complex<double> w(1.0, 0.0);
        for (uint32_t j = 0; j < len / 2; ++j) {
          tw[inv][len / 2 - 1 + j] = make_double2(w.real(), w.imag());
          w *= wl;
        }
      }
    std::vector<double2> te(nn), td(nn);
    const double ange = -M_PI / static_cast<double>(nn);
    for (uint32_t k = 0; k < nn; ++k) {
      te[k] = make_double2(std::cos(ange * k), std::sin(ange * k));
      const double angd = M_PI * k / static_cast<double>(nn);
      td[k] = make_double2(std::cos(angd), std::sin(angd));
    }
    std::vector<uint32_t> jidx(nn / 2);
    uint64_t g = 1;
    for (uint32_t t = 0; t < nn / 2; ++t) {
      jidx[t] = static_cast<uint32_t>((g - 1) / 2);
      g = g * 5 % (2ull * nn);
    }
    auto up = [](auto& v, auto*& d) {
      CK_CUDA(cudaMalloc(&d, sizeof(v[0]) * std::max<size_t>(v.size(), 1)));
      CK_CUDA(cudaMemcpy(d, v.data(), sizeof(v[0]) * v.size(), cudaMemcpyHostToDevice));
    };
    up(tw[0], d_fft_fwd);
    up(tw[1], d_fft_inv);
    up(te, d_twist_enc);
    up(td, d_twist_dec);
    up(jidx, d_jidx);
  }
  // NttPrimeTable constants of every prime for the raw-representation NTT
  // (ntt.cpp:124-131: r2 = 2^64, fwd1_r2 = psi^{n/2} R^2, exit_x = n^-1,
  // exit_y = psi^{-n/2} n^-1), uploaded on first use
  Blob raw_consts;
  bool raw_ready = false;
  const RawNttConst* raw_const() {
    if (!raw_ready) {
      std::vector<RawNttConst> v(primes.size());
      for (size_t g = 0; g < primes.size(); ++g) {
        const uint32_t qq = primes[g], R = r_mod(qq), r2 = mulm(R, R, qq);
        const uint32_t ph = (uint32_t)pow_mod(psi[g], n / 2, qq), ninv = invm(n % qq, qq);
        v[g].r2 = (int32_t)r2;
        v[g].fwd1_r2 = (int32_t)mulm(ph, r2, qq);
        v[g].exit_x = (int32_t)ninv;
        v[g].exit_y = (int32_t)mulm(invm(ph, qq), ninv, qq);
      }
      raw_consts.add(v);
      raw_consts.upload();
      raw_ready = true;
    }
    return raw_consts.at<RawNttConst>(0);
  }
  // CRT constants of the first cnt primes (multi-precision, ckks.cpp:337-346),
  // uploaded once per prefix length
  const CrtConst* crt_const(uint32_t cnt) {
    auto it = crt_consts.find(cnt);
    if (it != crt_consts.end()) return it->second.at<CrtConst>(0);
    if (cnt > (uint32_t)kMaxCrt) throw InvalidArgument("decode: CRT lift over more than 16 primes is not supported");
    auto mul = [](std::vector<uint32_t>& v, uint32_t m) {  // v *= m (little-endian limbs)
      uint64_t carry = 0;
      for (auto& x : v) {
        const uint64_t t = (uint64_t)x * m + carry;
        x = (uint32_t)t;
        carry = t >> 32;
      }
      if (carry) v.push_back((uint32_t)carry);
    };
    CrtConst cc;
    cc.c = (int)cnt;
    std::vector<uint32_t> M{1};
    for (uint32_t i = 0; i < cnt; ++i) mul(M, q(i));
    for (size_t j = 0; j < M.size() && j < (size_t)kMaxCrt + 1; ++j) cc.m[j] = M[j];
    for (uint32_t i = 0; i < cnt; ++i) {
      std::vector<uint32_t> Mi{1};
      uint64_t mi_mod_qi = 1;  // (M / q_i) mod q_i
      for (uint32_t k = 0; k < cnt; ++k)
        if (k != i) {
          mul(Mi, q(k));
          mi_mod_qi = mi_mod_qi * (q(k) % q(i)) % q(i);
        }
      cc.q[i] = q(i);
      cc.y[i] = invm((uint32_t)mi_mod_qi, q(i));
      for (size_t j = 0; j < Mi.size() && j < (size_t)kMaxCrt; ++j) cc.mi[i][j] = Mi[j];
    }
    Blob b;
    b.add(std::vector<CrtConst>{cc});
    b.upload();
    return crt_consts.emplace(cnt, std::move(b)).first->second.at<CrtConst>(0);
  }

  ~Context() {
    cudaSetDevice(device);
    cudaDeviceSynchronize();
    for (auto* d : {d_fft_fwd, d_fft_inv, d_twist_enc, d_twist_dec})
      if (d) cudaFree(d);
    if (d_jidx) cudaFree(d_jidx);
    for (auto& kv : rot_maps) cudaFree(kv.second);
    for (auto& kv : rot_dest) cudaFree(kv.second);
    if (d_primes) cudaFree(d_primes);
    if (d_fwd) cudaFree(d_fwd);
    if (d_inv) cudaFree(d_inv);
    if (d_pmont) cudaFree(d_pmont);
    if (d_tw2f) cudaFree(d_tw2f);
    if (d_tw2i) cudaFree(d_tw2i);
    for (auto& kv : scratch)
      if (kv.second.ptr) cudaFree(kv.second.ptr);
  }

  uint32_t q(uint32_t g) const { return primes[g]; }
  uint32_t gidx(uint32_t level, uint32_t row) const { return row < level ? row : L + (row - level); }
  uint32_t digits(uint32_t level) const {
    if (alpha == 0) throw InvalidArgument("key switching needs P primes (alpha = 0)");
    return (level + alpha - 1) / alpha;
  }
  size_t rowsz() const { return (size_t)n; }

  void* scratch_get(size_t bytes, cudaStream_t st) {
    Scratch& sc = scratch[st];
    if (bytes > sc.bytes) {
      CK_CUDA(cudaStreamSynchronize(st));
      if (sc.ptr) cudaFree(sc.ptr);
      sc.ptr = nullptr;
      const size_t want = bytes + bytes / 8;
      CK_CUDA(cudaMalloc(&sc.ptr, want));
      sc.bytes = want;
    }
    return sc.ptr;
  }

  // Inverse exit constants for prime g with plain epilogue factor e (ntt.cpp:76-84).
  ExitConst exit_const(uint32_t g, uint32_t e) const {
    const uint32_t qq = q(g);
    const uint32_t rinv = invm(r_mod(qq), qq);
    const uint32_t ninv = invm(n % qq, qq);
    const uint32_t psih_inv = invm((uint32_t)pow_mod(psi[g], n / 2, qq), qq);
    const uint32_t cx = mulm(mulm(ninv, rinv, qq), e, qq);
    const uint32_t cy = mulm(mulm(mulm(psih_inv, ninv, qq), rinv, qq), e, qq);
    return make_uint4(cx, shoup(cx, qq), cy, shoup(cy, qq));
  }

  // make_bconv_table (bconv.cpp:13-46): (P/P_j) mod q_i in Montgomery form,
  // and part1 = (P/P_j)^-1 mod p_j (plain; folded into the INTT exit).
  void bconv_consts(const std::vector<uint32_t>& sg, const std::vector<uint32_t>& dg, std::vector<uint32_t>& cmat,
                    std::vector<uint32_t>& part1) const {
    part1.resize(sg.size());
    for (size_t j = 0; j < sg.size(); ++j) {
      const uint32_t pj = q(sg[j]);
      uint32_t ph = 1 % pj;
      for (size_t k = 0; k < sg.size(); ++k)
        if (k != j) ph = mulm(ph, q(sg[k]) % pj, pj);
      part1[j] = invm(ph, pj);
    }
    for (size_t i = 0; i < dg.size(); ++i) {
      const uint32_t qi = q(dg[i]);
      for (size_t j = 0; j < sg.size(); ++j) {
        uint32_t ph = 1 % qi;
        for (size_t k = 0; k < sg.size(); ++k)
          if (k != j) ph = mulm(ph, q(sg[k]) % qi, qi);
        cmat.push_back(to_mont(ph, qi));
      }
    }
  }

  // One k_conv_mid group: sources (global prime sg[j], rows src_off + j with
  // part-1 exits), destinations (global prime dg[i], row drow[i]).
  void add_conv_group(std::vector<ConvMidGroup>& groups, std::vector<uint32_t>& cmat, std::vector<uint32_t>& drow_all,
                      std::vector<uint16_t>& dprime, std::vector<uint16_t>& sprime, std::vector<ExitConst>& sexit,
                      uint32_t src_off, const std::vector<uint32_t>& sg, const std::vector<uint32_t>& dg,
                      const std::vector<uint32_t>& drow) const {
    std::vector<uint32_t> cm, part1;
    bconv_consts(sg, dg, cm, part1);
    ConvMidGroup G;
    G.src_off = src_off;
    G.sc = (uint32_t)sg.size();
    G.dc = (uint32_t)dg.size();
    G.cmat_off = (uint32_t)cmat.size();
    G.map_off = (uint32_t)drow_all.size();
    G.src_map_off = (uint32_t)sprime.size();
    for (size_t i = 0; i < dg.size(); ++i)
      for (size_t j = 0; j < sg.size(); ++j) {  // x R folded in: the NTT skips the entry merge
        const uint32_t qi = q(dg[i]);
        cmat.push_back(mulm(cm[i * sg.size() + j], r_mod(qi), qi));
      }
    for (size_t i = 0; i < dg.size(); ++i) {
      drow_all.push_back(drow[i]);
      dprime.push_back((uint16_t)dg[i]);
    }
    for (size_t j = 0; j < sg.size(); ++j) {
      sprime.push_back((uint16_t)sg[j]);
      sexit.push_back(exit_const(sg[j], part1[j]));
    }
    groups.push_back(G);
  }
  static void upload_conv(ConvMidPlan& cm, const std::vector<ConvMidGroup>& groups, const std::vector<uint32_t>& cmat,
                          const std::vector<uint32_t>& drow, const std::vector<uint16_t>& dprime,
                          const std::vector<uint16_t>& sprime, const std::vector<ExitConst>& sexit) {
    cm.groups_off = cm.blob.add(groups);
    cm.cmat_off = cm.blob.add(cmat);
    cm.row_off = cm.blob.add(drow);
    cm.prime_off = cm.blob.add(dprime);
    cm.sprime_off = cm.blob.add(sprime);
    cm.sexit_off = cm.blob.add(sexit);
    cm.ngroups = (int)groups.size();
    cm.max_sc = 1;
    for (const auto& g : groups) cm.max_sc = std::max<int>(cm.max_sc, (int)g.sc);
    cm.blob.upload();
  }

  void check_bconv_width(const std::vector<uint32_t>& sg) const {
    // unsigned int64 accumulation is exact while sc * max(p) < 2^32 (the
    // reference's cap makes (alpha+2) * p < 2^32, rns.cpp:69-72)
    uint64_t pmax = 0;
    for (uint32_t g : sg) pmax = std::max<uint64_t>(pmax, q(g));
    if (sg.size() > 16 || (uint64_t)sg.size() * pmax >= (1ull << 32))
      throw InvalidArgument("base-conversion source too wide");
  }

  const ModUpPlan& modup_plan(uint32_t level) {
    auto it = modup.find(level);
    if (it != modup.end()) return *it->second;
    auto pl = std::make_unique<ModUpPlan>();
    pl->level = level;
    pl->D = digits(level);
    const uint32_t rows = level + alpha;
    std::vector<RowJob> ijobs, njobs;
    std::vector<ExitConst> exits;
    std::vector<BconvGroup> groups;
    std::vector<uint32_t> cmat, drow;
    std::vector<uint16_t> dprime;
    int max_sc = 1;
    std::vector<ConvMidGroup> cgroups;
    std::vector<uint32_t> ccmat, cdrow;
    std::vector<uint16_t> cdprime, csprime;
    std::vector<ExitConst> csexit;
    for (uint32_t k = 0; k < pl->D; ++k) {  // modup_table (ckks.cpp:188-202)
      const uint32_t b = k * alpha, e = std::min((k + 1) * alpha, level);
      std::vector<uint32_t> sg, dg;
      for (uint32_t j = b; j < e; ++j) sg.push_back(j);
      for (uint32_t i = 0; i < rows; ++i)
        if (i < b || i >= e) dg.push_back(gidx(level, i));
      check_bconv_width(sg);
      std::vector<uint32_t> part1;
      BconvGroup G;
      G.src_off = b;
      G.sc = (uint32_t)sg.size();
      G.dc = (uint32_t)dg.size();
      G.cmat_off = (uint32_t)cmat.size();
      G.map_off = (uint32_t)drow.size();
      bconv_consts(sg, dg, cmat, part1);
      for (size_t i = 0; i < dg.size(); ++i)  // x R: the forward NTT then skips its entry merge
        for (size_t j = 0; j < sg.size(); ++j) {
          uint32_t& cij = cmat[G.cmat_off + i * sg.size() + j];
          cij = mulm(cij, r_mod(q(dg[i])), q(dg[i]));
        }
      max_sc = std::max<int>(max_sc, (int)sg.size());
      for (uint32_t i = 0; i < rows; ++i)
        if (i < b || i >= e) {
          drow.push_back(k * rows + i);
          dprime.push_back((uint16_t)gidx(level, i));
          njobs.push_back({k * rows + i, k * rows + i, (uint16_t)gidx(level, i), 0});
        }
      groups.push_back(G);
      for (uint32_t j = 0; j < sg.size(); ++j) {
        ijobs.push_back({b + j, b + j, (uint16_t)(b + j), (uint16_t)exits.size()});
        exits.push_back(exit_const(b + j, part1[j]));
      }
      std::vector<uint32_t> dr;
      for (uint32_t i = 0; i < rows; ++i)
        if (i < b || i >= e) dr.push_back(k * rows + i);
      add_conv_group(cgroups, ccmat, cdrow, cdprime, csprime, csexit, b, sg, dg, dr);
    }
    upload_conv(pl->cm, cgroups, ccmat, cdrow, cdprime, csprime, csexit);
    pl->intt.jobs_off = pl->intt.blob.add(ijobs);
    pl->intt.exits_off = pl->intt.blob.add(exits);
    pl->intt.njobs = (int)ijobs.size();
    pl->intt.blob.upload();
    pl->ntt.jobs_off = pl->ntt.blob.add(njobs);
    pl->ntt.njobs = (int)njobs.size();
    pl->ntt.blob.upload();
    pl->ntt_rows = njobs.size();
    pl->bc.groups_off = pl->bc.blob.add(groups);
    pl->bc.cmat_off = pl->bc.blob.add(cmat);
    pl->bc.row_off = pl->bc.blob.add(drow);
    pl->bc.prime_off = pl->bc.blob.add(dprime);
    pl->bc.ngroups = (int)groups.size();
    pl->bc.max_sc = max_sc;
    pl->bc.src_rows = level;
    pl->bc.dst_rows = drow.size();
    add_bconv_tc(pl->bc, groups, cmat, dprime, [&](uint32_t g) { return q(g); }, n);
    pl->bc.blob.upload();
    auto& ref = *pl;
    modup[level] = std::move(pl);
    return ref;
  }

  // kind 0 = ModDown (src P, out level), 1 = rescale (src 2 tail Q, out level-2),
  // 2 = merged (src 2 tail Q + P, out level-2)  (ckks.cpp:206-258)
  const SwitchPlan& switch_plan(int kind, uint32_t level, uint32_t npoly) {
    auto key = std::make_tuple(kind, level, npoly);
    auto it = switches.find(key);
    if (it != switches.end()) return *it->second;
    auto pl = std::make_unique<SwitchPlan>();
    std::vector<uint32_t> sg;
    uint32_t out_q = level;
    if (kind == 0) {
      for (uint32_t j = 0; j < alpha; ++j) sg.push_back(L + j);
    } else {
      if (level < 4) throw InvalidArgument("level exhausted");
      out_q = level - 2;
      sg = {level - 2, level - 1};
      if (kind == 2)
        for (uint32_t j = 0; j < alpha; ++j) sg.push_back(L + j);
    }
    check_bconv_width(sg);
    const uint32_t sc = (uint32_t)sg.size();
    pl->out_q = out_q;
    pl->sc = sc;
    pl->npoly = npoly;
    std::vector<uint32_t> dg(out_q);
    for (uint32_t i = 0; i < out_q; ++i) dg[i] = i;
    std::vector<uint32_t> cmat, part1;
    bconv_consts(sg, dg, cmat, part1);
    for (uint32_t i = 0; i < out_q; ++i)  // x R: the forward NTT then skips its entry merge
      for (uint32_t j = 0; j < sc; ++j) cmat[i * sc + j] = mulm(cmat[i * sc + j], r_mod(q(dg[i])), q(dg[i]));
    std::vector<RowJob> ijobs, njobs;
    std::vector<ExitConst> exits;
    std::vector<BconvGroup> groups;
    std::vector<uint32_t> drow;
    std::vector<uint16_t> dprime;
    for (uint32_t j = 0; j < sc; ++j) exits.push_back(exit_const(sg[j], part1[j]));
    for (uint32_t p = 0; p < npoly; ++p) {
      for (uint32_t j = 0; j < sc; ++j)
        ijobs.push_back({p * (out_q + sc) + out_q + j, p * sc + j, (uint16_t)sg[j], (uint16_t)j});
      BconvGroup G;
      G.src_off = p * sc;
      G.sc = sc;
      G.dc = out_q;
      G.cmat_off = 0;
      G.map_off = (uint32_t)drow.size();
      groups.push_back(G);
      for (uint32_t i = 0; i < out_q; ++i) {
        drow.push_back(p * out_q + i);
        dprime.push_back((uint16_t)i);
        njobs.push_back({p * out_q + i, p * out_q + i, (uint16_t)i, 0});
      }
    }
    pl->intt.jobs_off = pl->intt.blob.add(ijobs);
    pl->intt.exits_off = pl->intt.blob.add(exits);
    pl->intt.njobs = (int)ijobs.size();
    pl->intt.blob.upload();
    pl->ntt.jobs_off = pl->ntt.blob.add(njobs);
    pl->ntt.njobs = (int)njobs.size();
    pl->ntt.blob.upload();
    pl->bc.groups_off = pl->bc.blob.add(groups);
    pl->bc.cmat_off = pl->bc.blob.add(cmat);
    pl->bc.row_off = pl->bc.blob.add(drow);
    pl->bc.prime_off = pl->bc.blob.add(dprime);
    pl->bc.ngroups = (int)groups.size();
    pl->bc.max_sc = (int)sc;
    pl->bc.src_rows = (uint64_t)npoly * sc;
    pl->bc.dst_rows = (uint64_t)npoly * out_q;
    add_bconv_tc(pl->bc, groups, cmat, dprime, [&](uint32_t g) { return q(g); }, n);
    pl->bc.blob.upload();
    // divisor = product of the source primes; one Montgomery inverse per row
    std::vector<uint32_t> dinv(out_q);
    for (uint32_t i = 0; i < out_q; ++i) {
      uint32_t d = 1 % q(i);
      for (uint32_t g : sg) d = mulm(d, q(g) % q(i), q(i));
      dinv[i] = to_mont(invm(d, q(i)), q(i));
    }
    pl->consts.add(dinv);
    pl->consts.upload();
    {
      std::vector<ConvMidGroup> cgroups;
      std::vector<uint32_t> ccmat, cdrow;
      std::vector<uint16_t> cdprime, csprime;
      std::vector<ExitConst> csexit;
      for (uint32_t p = 0; p < npoly; ++p) {
        std::vector<uint32_t> dr(out_q);
        for (uint32_t i = 0; i < out_q; ++i) dr[i] = p * out_q + i;
        add_conv_group(cgroups, ccmat, cdrow, cdprime, csprime, csexit, p * sc, sg, dg, dr);
      }
      upload_conv(pl->cm, cgroups, ccmat, cdrow, cdprime, csprime, csexit);
    }
    auto& ref = *pl;
    switches[key] = std::move(pl);
    return ref;
  }

  // dest[i] of the rotation map (AutomorphismMap::dest, automorphism.cpp:40-46): the inverse of rotation_map
  std::map<int64_t, uint32_t*> rot_dest;
  const uint32_t* rotation_dest(int64_t r) {
    auto it = rot_dest.find(r);
    if (it != rot_dest.end()) return it->second;
    const int64_t half = (int64_t)n / 2;
    int64_t e = (-r) % half;
    if (e < 0) e += half;
    uint64_t g = 1;
    const uint64_t mod = 2ull * n;
    for (int64_t i = 0; i < e; ++i) g = g * 5 % mod;
    std::vector<uint32_t> dest(n);
    for (uint32_t i = 0; i < n; ++i) {
      const uint32_t bi = bit_reverse(i, logn);
      const uint32_t phi = (uint32_t)((((2ull * bi + 1) * g) % mod - 1) / 2);
      dest[i] = bit_reverse(phi, logn);
    }
    uint32_t* d = nullptr;
    CK_CUDA(cudaMalloc(&d, n * sizeof(uint32_t)));
    CK_CUDA(cudaMemcpy(d, dest.data(), n * sizeof(uint32_t), cudaMemcpyHostToDevice));
    rot_dest[r] = d;
    return d;
  }
  const uint32_t* rotation_map(int64_t r) {  // AutomorphismMap::rotation (automorphism.cpp:11-69)
    auto it = rot_maps.find(r);
    if (it != rot_maps.end()) return it->second;
    const int64_t half = (int64_t)n / 2;
    int64_t e = (-r) % half;
    if (e < 0) e += half;
    uint64_t g = 1;
    const uint64_t mod = 2ull * n;
    for (int64_t i = 0; i < e; ++i) g = g * 5 % mod;
    std::vector<uint32_t> src(n);
    for (uint32_t i = 0; i < n; ++i) {
      const uint32_t bi = bit_reverse(i, logn);
      const uint32_t phi = (uint32_t)((((2ull * bi + 1) * g) % mod - 1) / 2);
      src[bit_reverse(phi, logn)] = i;
    }
    uint32_t* d = nullptr;
    CK_CUDA(cudaMalloc(&d, n * sizeof(uint32_t)));
    CK_CUDA(cudaMemcpy(d, src.data(), n * sizeof(uint32_t), cudaMemcpyHostToDevice));
    rot_maps[r] = d;
    return d;
  }

  // ------------------------------------------------------------- launches --
  // jobs_override: a device job table to use instead of the plan's (same
  // count) -- the limb-sharded peer exchange selects its parity on the device
  void run_ntt(const NttPlan& pl, bool inverse, int batch, const uint32_t* src, uint64_t src_bs, uint32_t* dst,
               uint64_t dst_bs, int entry, cudaStream_t st, const RowJob* jobs_override = nullptr) {
    if (pl.njobs == 0 || batch == 0) return;
    NttLaunch a;
    a.jobs = jobs_override ? jobs_override : pl.blob.at<RowJob>(pl.jobs_off);
    a.njobs = pl.njobs;
    a.batch = batch;
    a.src = src;
    a.src_bs = src_bs;
    a.dst = dst;
    a.dst_bs = dst_bs;
    a.primes = d_primes;
    a.tw = inverse ? d_inv : d_fwd;
    a.exits = inverse ? pl.blob.at<ExitConst>(pl.exits_off) : nullptr;
    a.entry = entry;
    ProfScope ps(this, inverse ? 1 : 0, 8.0 * n * pl.njobs * batch, 2, st);
    if (logn == 16 && d_tw2f && use_ntt256 && use_cluster && ntt_cluster_available()) {
      if (inverse)
        ntt_cluster_inverse(a, d_tw2i, st);
      else
        ntt_cluster_forward(a, d_tw2f, st);
      launches += 1;
    } else if (logn == 16 && d_tw2f && use_ntt256) {
      // L2-resident chunks: pass 2 of a chunk reads pass 1's output while it
      // is still in the 126 MB L2, so each limb crosses HBM once each way.
      const int chunk = ntt_chunk_limbs;
      const int bchunk = std::max(1, std::min(batch, chunk));
      const int jchunk = std::max(1, chunk / bchunk);
      for (int j0 = 0; j0 < pl.njobs; j0 += jchunk) {
        for (int b0 = 0; b0 < batch; b0 += bchunk) {
          NttLaunch c = a;
          c.jobs = a.jobs + j0;
          c.njobs = std::min(jchunk, pl.njobs - j0);
          c.batch = std::min(bchunk, batch - b0);
          c.src = src + (uint64_t)b0 * src_bs;
          c.dst = dst + (uint64_t)b0 * dst_bs;
          if (inverse)
            ntt256_inverse(c, d_tw2i, st);
          else
            ntt256_forward(c, d_tw2f, st);
          launches += 2;
        }
      }
      launches -= 2;
    } else if (logn == 17 && d_tw2f && use_ntt256) {
      if (inverse)
        ntt131k_inverse(a, d_tw2i, st);
      else
        ntt131k_forward(a, d_tw2f, st);
    } else if (inverse) {
      ntt_inverse((int)logn, a, st);
    } else {
      ntt_forward((int)logn, a, st);
    }
    launches += 2;
  }
  void run_bconv(const BconvPlan& pl, int batch, const uint32_t* src, uint64_t src_bs, uint32_t* dst, uint64_t dst_bs,
                 cudaStream_t st, const uint64_t* src_rows = nullptr) {
    if (batch == 0) return;
    BconvLaunch a;
    a.groups = pl.blob.at<BconvGroup>(pl.groups_off);
    a.ngroups = pl.ngroups;
    a.batch = batch;
    a.max_sc = pl.max_sc;
    a.src = src;
    a.src_bs = src_bs;
    a.dst = dst;
    a.dst_bs = dst_bs;
    a.cmat = pl.blob.at<uint32_t>(pl.cmat_off);
    a.dst_row = pl.blob.at<uint32_t>(pl.row_off);
    a.dst_prime = pl.blob.at<uint16_t>(pl.prime_off);
    a.primes = d_primes;
    a.src_rows = src_rows;
    ProfScope ps(this, 2, 4.0 * n * (pl.src_rows + pl.dst_rows) * batch, 1, st);
    if (use_tc && pl.tc_ok && !src_rows) {
      BconvTc t;
      t.btab = pl.blob.at<unsigned char>(pl.tc_tab_off);
      t.boff = pl.blob.at<uint32_t>(pl.tc_boff_off);
      t.max_npad = pl.tc_max_npad;
      t.max_dc = pl.tc_max_dc;
      t.variant = tc_var;
      bconv_tc((int)n, a, t, st);
    } else {
      bconv((int)n, a, st, bconv_fp64);
    }
    ++launches;
  }

  bool fused() const { return logn == 16 && d_tw2f && use_ntt256 && use_fused; }
  NttLaunch ntt_args(const NttPlan& pl, bool inverse, int batch, const uint32_t* src, uint64_t src_bs, uint32_t* dst,
                     uint64_t dst_bs) const {
    NttLaunch a;
    a.jobs = pl.blob.at<RowJob>(pl.jobs_off);
    a.njobs = pl.njobs;
    a.batch = batch;
    a.src = src;
    a.src_bs = src_bs;
    a.dst = dst;
    a.dst_bs = dst_bs;
    a.primes = d_primes;
    a.tw = inverse ? d_inv : d_fwd;
    a.exits = inverse ? pl.blob.at<ExitConst>(pl.exits_off) : nullptr;
    return a;
  }
  // fused path: INTT pass A -> [INTT pass B + BConv + NTT pass 1] -> NTT pass 2
  void run_convert(const NttPlan& ipl, const ConvMidPlan& cm, const NttPlan& npl, int B, const uint32_t* src,
                   uint64_t src_bs, uint32_t* mid, uint64_t mid_bs, uint32_t* dst, uint64_t dst_bs, double bytes_in,
                   double bytes_out, cudaStream_t st) {
    {
      ProfScope ps(this, 1, 8.0 * n * ipl.njobs * B, 1, st);
      ntt256_pass(2, ntt_args(ipl, true, B, src, src_bs, mid, mid_bs), d_tw2i, st);
    }
    {
      ProfScope ps(this, 7, bytes_in + bytes_out, 1, st);
      ConvMidLaunch a;
      a.groups = cm.blob.at<ConvMidGroup>(cm.groups_off);
      a.ngroups = cm.ngroups;
      a.batch = B;
      a.max_sc = cm.max_sc;
      a.src = mid;
      a.src_bs = mid_bs;
      a.dst = dst;
      a.dst_bs = dst_bs;
      a.cmat = cm.blob.at<uint32_t>(cm.cmat_off);
      a.dst_row = cm.blob.at<uint32_t>(cm.row_off);
      a.dst_prime = cm.blob.at<uint16_t>(cm.prime_off);
      a.src_prime = cm.blob.at<uint16_t>(cm.sprime_off);
      a.src_exit = cm.blob.at<ExitConst>(cm.sexit_off);
      a.primes = d_primes;
      a.fwd_tw = d_fwd;
      a.inv_tw = d_inv;
      conv_mid(a, st);
    }
    {
      ProfScope ps(this, 0, 8.0 * n * npl.njobs * B, 1, st);
      ntt256_pass(1, ntt_args(npl, false, B, dst, dst_bs, dst, dst_bs), d_tw2f, st);
    }
    launches += 3;
  }

  // ModUp (ckks.cpp:680-731) of B polynomials d (level rows, batch stride d_bs)
  // into ext [B][D][level+alpha]; uses `is` [B][level] as INTT scratch.
  // The digit rows of ext are NOT written: key_mult reads them from d.
  void mod_up(uint32_t level, int B, const uint32_t* d, uint64_t d_bs, uint32_t* is, uint32_t* ext,
              cudaStream_t st) {
    const ModUpPlan& pl = modup_plan(level);
    const uint64_t N = n;
    const uint64_t ext_bs = (uint64_t)pl.D * (level + alpha) * N;
    if (fused()) {
      run_convert(pl.intt, pl.cm, pl.ntt, B, d, d_bs, is, level * N, ext, ext_bs, 4.0 * N * level * B,
                  4.0 * N * pl.ntt_rows * B, st);
    } else {
      run_ntt(pl.intt, true, B, d, d_bs, is, level * N, 0, st);
      run_bconv(pl.bc, B, is, level * N, ext, ext_bs, st);
      run_ntt(pl.ntt, false, B, ext, ext_bs, ext, ext_bs, 0, st);  // BConv output already carries R
    }
    counters[0] += B;
    counters[3] += (uint64_t)B * level;
    counters[5] += (uint64_t)B * pl.D;
    counters[2] += (uint64_t)B * pl.ntt_rows;
  }

  // ModUp + KeyMult (+ fold) into v [B][2][level+alpha]. For N = 2^16 the
  // extension's forward row pass is fused into KeyMult (k_row_keymult): ext
  // only ever holds column-pass output.
  // pre (optional): the drop-and-divide that consumes v next; when the fused
  // row pass + KeyMult kernel supports it, that switch's INTT pass A is done
  // in the KeyMult epilogue (its source rows go to ts, row-transformed) and
  // the return value is true -- the caller then runs only pass B.
  bool mod_up_key_mult(uint32_t level, int B, const uint32_t* d, uint64_t d_bs, uint32_t* is, uint32_t* ext,
                       const uint32_t* evk, const uint32_t* fold, uint64_t fold_bs, uint32_t* v, cudaStream_t st,
                       const SwitchPlan* pre = nullptr, uint32_t* ts = nullptr, uint64_t ts_bs = 0) {
    if (!(logn == 16 && d_tw2f && use_ntt256 && use_row_km)) {
      mod_up(level, B, d, d_bs, is, ext, st);
      key_mult_v(level, B, ext, d, d_bs, evk, fold, fold_bs, v, st);
      return false;
    }
    const ModUpPlan& pl = modup_plan(level);
    const uint64_t N = n;
    const uint64_t ext_bs = (uint64_t)pl.D * (level + alpha) * N;
    run_ntt(pl.intt, true, B, d, d_bs, is, level * N, 0, st);
    run_bconv(pl.bc, B, is, level * N, ext, ext_bs, st);
    {
      ProfScope ps(this, 0, 4.0 * n * pl.ntt.njobs * B, 1, st);  // column pass: half of the NTT traffic
      NttLaunch a = ntt_args(pl.ntt, false, B, ext, ext_bs, ext, ext_bs);
      a.entry = 0;  // BConv output already carries R
      ntt256_pass(0, a, d_tw2f, st);
    }
    KeyMultLaunch a;
    a.level = (int)level;
    a.alpha = (int)alpha;
    a.L = (int)L;
    a.D = (int)pl.D;
    a.batch = B;
    a.ext = ext;
    a.ext_bs = ext_bs;
    a.d = d;
    a.d_bs = d_bs;
    a.evk = evk;
    a.fold = fold;
    a.fold_bs = fold_bs;
    a.p_mont = d_pmont;
    a.v = v;
    a.v_bs = 2ull * (level + alpha) * n;
    a.primes = d_primes;
    bool fused_intt = false;
    if (pre && ts && !fused() && pre->out_q + pre->sc == level + alpha && pre->npoly == 2) {
      KeyMultLaunch t = a;
      t.ts = ts;
      t.ts_bs = ts_bs;
      t.ts_sc = (int)pre->sc;
      t.ts_q = (int)(pre->sc - alpha);  // tail Q rows among the sources (2 merged, 0 ModDown)
      t.src_lo = (int)(level - t.ts_q);
      t.inv_full = d_inv;
      if (t.ts_q >= 0 && row_keymult_fuses_intt(t)) {
        a = t;
        fused_intt = true;
      }
    }
    {
      // Per ciphertext: the row pass reads the extension rows' column-pass
      // output (4N B per row; its result never leaves the SM), KeyMult reads
      // the digits' own rows in place from d (4N B x level) and writes v0, v1
      // (2 (level + alpha) rows), the fold reads d0, d1 (2 level rows).  The
      // key (2D (level + alpha) rows) is shared by the whole batch: counted
      // once per launch.
      ProfScope ps(this, 8,
                   4.0 * n * B * (pl.ntt_rows + level + 2.0 * (level + alpha)) + (fold ? 8.0 * n * level * B : 0.0) +
                       4.0 * n * 2.0 * pl.D * (level + alpha),
                   1, st);
      row_keymult(a, d_tw2f, st, d_fwd);
    }
    launches += 2;
    counters[0] += B;
    counters[3] += (uint64_t)B * level;
    counters[5] += (uint64_t)B * pl.D;
    counters[2] += (uint64_t)B * pl.ntt_rows;
    counters[4] += (uint64_t)B * pl.D;
    return fused_intt;
  }

  // key_mult (+ optional fold) into v [B][2][level+alpha]
  void key_mult_v(uint32_t level, int B, const uint32_t* ext, const uint32_t* d, uint64_t d_bs, const uint32_t* evk,
                  const uint32_t* fold, uint64_t fold_bs, uint32_t* v, cudaStream_t st) {
    KeyMultLaunch a;
    a.level = (int)level;
    a.alpha = (int)alpha;
    a.L = (int)L;
    a.D = (int)digits(level);
    a.batch = B;
    a.ext = ext;
    a.ext_bs = (uint64_t)a.D * (level + alpha) * n;
    a.d = d;
    a.d_bs = d_bs;
    a.evk = evk;
    a.fold = fold;
    a.fold_bs = fold_bs;
    a.p_mont = d_pmont;
    a.v = v;
    a.v_bs = 2ull * (level + alpha) * n;
    a.primes = d_primes;
    // per ciphertext: D operand rows per output row (extension rows + the
    // digits' own rows read in place), writes v0, v1 (+ d0, d1 for the folded
    // Q rows); the key's 2D rows per output row are read once per launch
    // (one key for the whole batch)
    ProfScope ps(this, 3,
                 4.0 * n * (level + alpha) * (a.D + 2.0) * B + (fold ? 8.0 * n * level * B : 0.0) +
                     4.0 * n * (level + alpha) * 2.0 * a.D,
                 1, st);
    key_mult((int)n, a, st);
    ++launches;
    counters[4] += (uint64_t)B * a.D;
  }

  // HRot's ModDown (drop_and_divide with the ModDown table, ckks.cpp:611-655)
  // with the rest of rotate_with (ckks.cpp:875-882) fused into the forward
  // NTT's row pass: out = phi_r((v - conv) d^-1 + (b, 0)), written straight
  // into the output ciphertexts.  true when the fused path applies.
  bool drop_divide_hrot(const SwitchPlan& pl, int B, const uint32_t* v, uint64_t v_bs, uint32_t* ts, uint32_t* o,
                        const uint32_t* ct, uint64_t ct_bs, int64_t r, uint32_t* out, cudaStream_t st,
                        bool pre_intt = false) {
    if (!(logn == 16 && d_tw2f && use_ntt256 && !use_cluster && ntt_chunk_limbs >= (1 << 30) && use_fused_combine &&
          use_hrot_tail && !fused()))
      return false;
    const uint64_t N = n;
    const uint64_t ts_bs = (uint64_t)pl.npoly * pl.sc * N, o_bs = (uint64_t)pl.npoly * pl.out_q * N;
    switch_intt(pl, B, v, v_bs, ts, ts_bs, pre_intt, st);
    run_bconv(pl.bc, B, ts, ts_bs, o, o_bs, st);
    {
      // NTT (8N B per row) + the tail's extra reads: v (4N B per row) and b (4N B per Q row of poly 0)
      ProfScope ps(this, 10, 8.0 * n * pl.ntt.njobs * B + 4.0 * n * pl.out_q * pl.npoly * B + 4.0 * n * pl.out_q * B,
                   2, st);
      NttLaunch a = ntt_args(pl.ntt, false, B, o, o_bs, o, o_bs);
      CombineArgs cb;
      cb.v = v;
      cb.v_bs = v_bs;
      cb.prow = pl.out_q + pl.sc;
      cb.out_q = pl.out_q;
      cb.dinv = pl.consts.at<uint32_t>(0);
      cb.add = ct;
      cb.add_bs = ct_bs;
      cb.dest = rotation_dest(r);
      cb.out = out;
      cb.out_bs = ct_bs;
      ntt256_forward_hrot_tail(a, d_tw2f, cb, st);
      launches += 2;
    }
    counters[3] += (uint64_t)B * pl.npoly * pl.sc;
    counters[5] += (uint64_t)B * pl.npoly;
    counters[2] += (uint64_t)B * pl.npoly * pl.out_q;
    return true;
  }

  // drop_and_divide (ckks.cpp:611-655) for B x npoly polynomials v (out_q+sc
  // rows each, poly stride, batch stride) into o [B][npoly][out_q]; ts scratch
  // [B][npoly][sc]. If `combine_now` is false the caller fuses the combine.
  // inverse NTT of a switch's source rows v -> ts, or, when the fused KeyMult
  // already ran pass A into ts (pre_intt), only pass B in place on ts
  void switch_intt(const SwitchPlan& pl, int B, const uint32_t* v, uint64_t v_bs, uint32_t* ts, uint64_t ts_bs,
                   bool pre_intt, cudaStream_t st) {
    if (!pre_intt) {
      run_ntt(pl.intt, true, B, v, v_bs, ts, ts_bs, 0, st);
      return;
    }
    ProfScope ps(this, 1, 8.0 * n * pl.intt.njobs * B, 1, st);
    ntt256_pass(3, ntt_args(pl.intt, true, B, ts, ts_bs, ts, ts_bs), d_tw2i, st);
    launches += 1;
  }

  void drop_divide(const SwitchPlan& pl, int B, const uint32_t* v, uint64_t v_bs, uint32_t* ts, uint32_t* o,
                   bool combine_now, cudaStream_t st, bool pre_intt = false) {
    const uint64_t N = n;
    const uint64_t prow = pl.out_q + pl.sc;
    const uint64_t ts_bs = (uint64_t)pl.npoly * pl.sc * N, o_bs = (uint64_t)pl.npoly * pl.out_q * N;
    if (fused()) {
      if (pre_intt) throw std::logic_error("fused INTT pass A with the k_conv_mid path");
      run_convert(pl.intt, pl.cm, pl.ntt, B, v, v_bs, ts, ts_bs, o, o_bs, 4.0 * N * pl.npoly * pl.sc * B,
                  4.0 * N * pl.npoly * pl.out_q * B, st);
    } else if (combine_now && logn == 16 && d_tw2f && use_ntt256 && !use_cluster && ntt_chunk_limbs >= (1 << 30) &&
               use_fused_combine) {
      switch_intt(pl, B, v, v_bs, ts, ts_bs, pre_intt, st);
      run_bconv(pl.bc, B, ts, ts_bs, o, o_bs, st);
      {  // forward NTT with the combine fused into its row pass
        // NTT (8N B per row) + the combine's extra read of v (4N B per row)
        ProfScope ps(this, 9, 8.0 * n * pl.ntt.njobs * B + 4.0 * n * pl.out_q * pl.npoly * B, 2, st);
        NttLaunch a = ntt_args(pl.ntt, false, B, o, o_bs, o, o_bs);
        CombineArgs cb;
        cb.v = v;
        cb.v_bs = v_bs;
        cb.prow = (uint32_t)prow;
        cb.out_q = pl.out_q;
        cb.dinv = pl.consts.at<uint32_t>(0);
        ntt256_forward_combine(a, d_tw2f, cb, st);
        launches += 2;
      }
      combine_now = false;
    } else {
      switch_intt(pl, B, v, v_bs, ts, ts_bs, pre_intt, st);
      run_bconv(pl.bc, B, ts, ts_bs, o, o_bs, st);
      run_ntt(pl.ntt, false, B, o, o_bs, o, o_bs, 0, st);  // BConv output already carries R
    }
    if (combine_now) {
      ProfScope ps(this, 5, 12.0 * n * pl.out_q * pl.npoly * B, 1, st);
      combine((int)n, (int)pl.out_q, (int)pl.npoly, B, v, prow * N, v_bs, o, pl.out_q * N,
              (uint64_t)pl.npoly * pl.out_q * N, pl.consts.at<uint32_t>(0), d_primes, st);
      ++launches;
    }
    counters[3] += (uint64_t)B * pl.npoly * pl.sc;
    counters[5] += (uint64_t)B * pl.npoly;
    counters[2] += (uint64_t)B * pl.npoly * pl.out_q;
  }
};

// ========================================================= limb sharding ==
// One shard of a limb-sharded ciphertext:
// rank s of G owns Q primes [qlo, qhi) and P primes L + [plo, phi) (balanced
// contiguous blocks). Shard-local polynomials hold the owned rows only: the
// owned Q rows below the level, then (when the polynomial carries them) the
// owned P rows. NTT/INTT, KeyMult, the fold, the combine and the automorphism
// are row-local; the only exchange is before each BConv, where every shard
// needs all source rows (the digit rows in ModUp, the dropped rows in
// ModDown / rescale): the host all-gathers the INTT'd source rows that
// `modup_begin` / `switch_begin` leave in a send buffer.
struct Shard {
  ~Shard() {
    if (xbuf) cudaFree(xbuf);
    if (ctl) cudaFree(ctl);
  }
  Context* c = nullptr;
  uint32_t G = 1, s = 0, qlo = 0, qhi = 0, plo = 0, phi = 0, qmax = 0, pmax = 0;

  static uint32_t block_lo(uint32_t t, uint32_t total, uint32_t G) { return (uint32_t)((uint64_t)t * total / G); }
  uint32_t q_lo(uint32_t t) const { return block_lo(t, c->L, G); }
  uint32_t q_hi(uint32_t t) const { return block_lo(t + 1, c->L, G); }
  uint32_t p_lo(uint32_t t) const { return block_lo(t, c->alpha, G); }
  uint32_t p_hi(uint32_t t) const { return block_lo(t + 1, c->alpha, G); }
  // owned Q rows of rank t below `level`
  uint32_t lq_of(uint32_t t, uint32_t level) const {
    const uint32_t lo = q_lo(t), hi = std::min(q_hi(t), level);
    return hi > lo ? hi - lo : 0;
  }
  uint32_t lq(uint32_t level) const { return lq_of(s, level); }
  uint32_t lp() const { return phi - plo; }
  bool owns_t(uint32_t t, uint32_t g) const {
    return g < c->L ? (g >= q_lo(t) && g < q_hi(t)) : (g - c->L >= p_lo(t) && g - c->L < p_hi(t));
  }
  // row of global prime g in a shard-local polynomial at `level` (Q rows then P rows)
  uint32_t local_row(uint32_t level, uint32_t g) const { return g < c->L ? g - qlo : lq(level) + (g - c->L - plo); }
  uint32_t smax(int kind) const { return kind == 0 ? pmax : kind == 1 ? 2 : pmax + 2; }

  // The phase-1 INTT jobs of the peer exchange for both buffer parities:
  // [2][njobs], dst_off relative to the exchange buffer's base (kind 0: the
  // ModUp send buffers, 1: the switch send buffers), so the parity can be
  // chosen on the device (k_shard_advance) and a captured step replays.
  std::vector<RowJob> parity_jobs(const std::vector<RowJob>& jobs, int kind) const {
    std::vector<RowJob> out;
    for (uint32_t par = 0; par < 2; ++par)
      for (RowJob j : jobs) {
        j.dst_off += kind == 0 ? par * qmax : 2 * qmax + par * 2 * (pmax + 2);
        out.push_back(j);
      }
    return out;
  }
  struct UpPlan {
    NttPlan intt, ntt;
    size_t intt_par_off = 0;
    BconvPlan bc;
    Blob maps;
    size_t digit_off = 0, prime_off = 0, erow_off = 0;
    uint32_t lq = 0, rows = 0, D = 0, ntt_rows = 0;
  };
  struct DownPlan {
    NttPlan intt, ntt;
    size_t intt_par_off = 0;
    BconvPlan bc;
    Blob consts;  // dinv [lqo]
    uint32_t sc = 0, smax = 0, vrows = 0, lqo = 0, out_q = 0, own_sc = 0;
    std::vector<uint32_t> rank_cnt;  // own sources per rank (gathered order = rank order)
  };
  std::map<uint32_t, std::unique_ptr<UpPlan>> up;
  std::map<std::pair<int, uint32_t>, std::unique_ptr<DownPlan>> down;

  const UpPlan& up_plan(uint32_t level) {
    auto it = up.find(level);
    if (it != up.end()) return *it->second;
    auto pl = std::make_unique<UpPlan>();
    const uint32_t alpha = c->alpha, L = c->L;
    pl->lq = lq(level);
    pl->rows = pl->lq + lp();
    pl->D = c->digits(level);
    auto gl = [&](uint32_t r) { return r < pl->lq ? qlo + r : L + plo + (r - pl->lq); };
    std::vector<RowJob> ijobs, njobs;
    std::vector<ExitConst> exits;
    for (uint32_t r = 0; r < pl->lq; ++r) {  // INTT + part 1 of the owned digit rows (ckks.cpp:690-697)
      const uint32_t g = qlo + r, k = g / alpha;
      std::vector<uint32_t> sg, cm, part1;
      for (uint32_t j = k * alpha; j < std::min((k + 1) * alpha, level); ++j) sg.push_back(j);
      c->bconv_consts(sg, {}, cm, part1);
      ijobs.push_back({r, r, (uint16_t)g, (uint16_t)exits.size()});
      exits.push_back(c->exit_const(g, part1[g - k * alpha]));
    }
    std::vector<BconvGroup> groups;
    std::vector<uint32_t> cmat, drow;
    std::vector<uint16_t> dprime;
    int max_sc = 1;
    for (uint32_t k = 0; k < pl->D; ++k) {  // per digit: BConv to the owned rows outside the digit
      const uint32_t b = k * alpha, e = std::min((k + 1) * alpha, level);
      std::vector<uint32_t> sg, dg, part1;
      for (uint32_t j = b; j < e; ++j) sg.push_back(j);
      std::vector<uint32_t> rr;
      for (uint32_t r = 0; r < pl->rows; ++r) {
        const uint32_t g = gl(r);
        if (g < b || g >= e) {
          dg.push_back(g);
          rr.push_back(r);
        }
      }
      if (dg.empty()) continue;
      c->check_bconv_width(sg);
      BconvGroup G0;
      G0.src_off = b;
      G0.sc = (uint32_t)sg.size();
      G0.dc = (uint32_t)dg.size();
      G0.cmat_off = (uint32_t)cmat.size();
      G0.map_off = (uint32_t)drow.size();
      c->bconv_consts(sg, dg, cmat, part1);
      max_sc = std::max<int>(max_sc, (int)sg.size());
      for (size_t i = 0; i < dg.size(); ++i) {
        drow.push_back(k * pl->rows + rr[i]);
        dprime.push_back((uint16_t)dg[i]);
        njobs.push_back({k * pl->rows + rr[i], k * pl->rows + rr[i], (uint16_t)dg[i], 0});
      }
      groups.push_back(G0);
    }
    pl->intt.jobs_off = pl->intt.blob.add(ijobs);
    pl->intt.exits_off = pl->intt.blob.add(exits);
    pl->intt.njobs = (int)ijobs.size();
    pl->intt_par_off = pl->intt.blob.add(parity_jobs(ijobs, 0));
    pl->intt.blob.upload();
    pl->ntt.jobs_off = pl->ntt.blob.add(njobs);
    pl->ntt.njobs = (int)njobs.size();
    pl->ntt.blob.upload();
    pl->ntt_rows = (uint32_t)njobs.size();
    pl->bc.groups_off = pl->bc.blob.add(groups);
    pl->bc.cmat_off = pl->bc.blob.add(cmat);
    pl->bc.row_off = pl->bc.blob.add(drow);
    pl->bc.prime_off = pl->bc.blob.add(dprime);
    pl->bc.ngroups = (int)groups.size();
    pl->bc.max_sc = max_sc;
    pl->bc.src_rows = (uint64_t)alpha * groups.size();
    pl->bc.dst_rows = drow.size();
    add_bconv_tc(pl->bc, groups, cmat, dprime, [&](uint32_t g) { return c->q(g); }, c->n);
    pl->bc.blob.upload();
    std::vector<int16_t> digit(pl->rows);
    std::vector<uint16_t> prime(pl->rows), erow(pl->rows);
    for (uint32_t r = 0; r < pl->rows; ++r) {
      const uint32_t g = gl(r);
      prime[r] = (uint16_t)g;
      digit[r] = r < pl->lq ? (int16_t)(g / alpha) : (int16_t)-1;
      erow[r] = (uint16_t)(r < pl->lq ? r : (qhi - qlo) + (r - pl->lq));  // key rows: owned Q (all levels), owned P
    }
    pl->digit_off = pl->maps.add(digit);
    pl->prime_off = pl->maps.add(prime);
    pl->erow_off = pl->maps.add(erow);
    pl->maps.upload();
    auto& ref = *pl;
    up[level] = std::move(pl);
    return ref;
  }

  // kind 0 ModDown (sources P, out level), 1 rescale (sources 2 tail Q rows,
  // out level-2), 2 merged (tail Q rows + P, out level-2)  (ckks.cpp:206-258)
  const DownPlan& down_plan(int kind, uint32_t level) {
    auto key = std::make_pair(kind, level);
    auto it = down.find(key);
    if (it != down.end()) return *it->second;
    auto pl = std::make_unique<DownPlan>();
    const uint32_t L = c->L, alpha = c->alpha;
    std::vector<uint32_t> sg;
    pl->out_q = level;
    if (kind == 0) {
      for (uint32_t j = 0; j < alpha; ++j) sg.push_back(L + j);
    } else {
      if (level < 4) throw InvalidArgument("level exhausted");
      pl->out_q = level - 2;
      sg = {level - 2, level - 1};
      if (kind == 2)
        for (uint32_t j = 0; j < alpha; ++j) sg.push_back(L + j);
    }
    c->check_bconv_width(sg);
    pl->sc = (uint32_t)sg.size();
    pl->smax = smax(kind);
    pl->vrows = kind == 1 ? lq(level) : lq(level) + lp();
    pl->lqo = lq(pl->out_q);
    std::vector<uint32_t> cm0, part1;  // part 1 depends on the source set only
    c->bconv_consts(sg, {}, cm0, part1);
    std::map<uint32_t, uint32_t> p1;
    for (size_t j = 0; j < sg.size(); ++j) p1[sg[j]] = part1[j];
    std::vector<uint32_t> gathered;  // source order after the all-gather: rank order, then sg order
    for (uint32_t t = 0; t < G; ++t) {
      uint32_t cnt = 0;
      for (uint32_t g : sg)
        if (owns_t(t, g)) {
          gathered.push_back(g);
          ++cnt;
        }
      pl->rank_cnt.push_back(cnt);
    }
    std::vector<RowJob> ijobs, njobs;
    std::vector<ExitConst> exits;
    std::vector<uint32_t> own;
    for (uint32_t g : sg)
      if (owns_t(s, g)) own.push_back(g);
    pl->own_sc = (uint32_t)own.size();
    for (uint32_t u = 0; u < own.size(); ++u) exits.push_back(c->exit_const(own[u], p1[own[u]]));
    for (uint32_t p = 0; p < 2; ++p)
      for (uint32_t u = 0; u < own.size(); ++u)
        ijobs.push_back({p * pl->vrows + local_row(level, own[u]), p * pl->smax + u, (uint16_t)own[u], (uint16_t)u});
    std::vector<uint32_t> dg;
    for (uint32_t r = 0; r < pl->lqo; ++r) dg.push_back(qlo + r);
    std::vector<uint32_t> cmat, part1g;
    if (!dg.empty()) c->bconv_consts(gathered, dg, cmat, part1g);
    std::vector<BconvGroup> groups;
    std::vector<uint32_t> drow;
    std::vector<uint16_t> dprime;
    for (uint32_t p = 0; p < 2 && !dg.empty(); ++p) {
      BconvGroup G0;
      G0.src_off = p * pl->sc;
      G0.sc = pl->sc;
      G0.dc = pl->lqo;
      G0.cmat_off = 0;
      G0.map_off = (uint32_t)drow.size();
      groups.push_back(G0);
      for (uint32_t r = 0; r < pl->lqo; ++r) {
        drow.push_back(p * pl->lqo + r);
        dprime.push_back((uint16_t)(qlo + r));
        njobs.push_back({p * pl->lqo + r, p * pl->lqo + r, (uint16_t)(qlo + r), 0});
      }
    }
    pl->intt.jobs_off = pl->intt.blob.add(ijobs);
    pl->intt.exits_off = pl->intt.blob.add(exits);
    pl->intt.njobs = (int)ijobs.size();
    pl->intt_par_off = pl->intt.blob.add(parity_jobs(ijobs, 1));
    pl->intt.blob.upload();
    pl->ntt.jobs_off = pl->ntt.blob.add(njobs);
    pl->ntt.njobs = (int)njobs.size();
    pl->ntt.blob.upload();
    pl->bc.groups_off = pl->bc.blob.add(groups);
    pl->bc.cmat_off = pl->bc.blob.add(cmat);
    pl->bc.row_off = pl->bc.blob.add(drow);
    pl->bc.prime_off = pl->bc.blob.add(dprime);
    pl->bc.ngroups = (int)groups.size();
    pl->bc.max_sc = (int)pl->sc;
    pl->bc.src_rows = 2ull * pl->sc;
    pl->bc.dst_rows = 2ull * pl->lqo;
    add_bconv_tc(pl->bc, groups, cmat, dprime, [&](uint32_t g) { return c->q(g); }, c->n);
    pl->bc.blob.upload();
    std::vector<uint32_t> dinv(std::max<uint32_t>(pl->lqo, 1), 0);
    for (uint32_t r = 0; r < pl->lqo; ++r) {
      const uint32_t qq = c->q(qlo + r);
      uint32_t d = 1 % qq;
      for (uint32_t g : sg) d = mulm(d, c->q(g) % qq, qq);
      dinv[r] = to_mont(invm(d, qq), qq);
    }
    pl->consts.add(dinv);
    pl->consts.upload();
    auto& ref = *pl;
    down[key] = std::move(pl);
    return ref;
  }

  // ---- peer exchange ("peer-mapped loads inside BConv") ----
  // Every rank owns one exchange allocation, mapped by all peers (CUDA IPC
  // across processes, plain pointers between virtual shards of one process):
  //   [ModUp send x 2][switch send x 2][flags: 2 kinds x G words][error word]
  // Phase 1 writes the rank's INTT rows into its own send buffer (parity =
  // epoch & 1, so a buffer is rewritten only after every peer has signalled
  // the following exchange of that kind, i.e. finished reading it) and
  // publishes the epoch into every peer's flag word; phase 2 waits for all
  // peers' flags, then its BConv reads the source rows straight from the
  // peers' send buffers through a row-address table -- no all-gather buffer,
  // no copy: the NVLink transfer happens inside the BConv loads.
  void* xbuf = nullptr;
  uint64_t up_words = 0, sw_words = 0, xbytes = 0;
  std::vector<uint64_t> peers;  // exchange base of every rank (own included)
  // Device-side exchange state (this rank only, not shared): the epoch of
  // each exchange kind, and what the current epoch's buffer parity selects
  // -- the phase-1 INTT job table and the phase-2 BConv source-row table.
  // Every kernel of a phase takes fixed pointers, so a step that uses the
  // peer exchange can be captured in a CUDA graph and replayed.
  uint32_t* ctl = nullptr;      // [2] epochs
  RowJob* jobs_cur[2] = {nullptr, nullptr};
  uint64_t* rows_cur[2] = {nullptr, nullptr};
  Blob sig_tab;                 // [2 kinds][G] peer flag addresses for this rank
  Blob up_tab;                  // [2 parities][L] ModUp source-row addresses
  std::map<std::pair<int, uint32_t>, std::unique_ptr<Blob>> down_tab;  // [2 parities][2 sc]
  uint64_t timeout_ns = 10ull * 1000 * 1000 * 1000;

  uint64_t up_off(uint32_t par) const { return (uint64_t)par * up_words * 4; }
  uint64_t sw_off(uint32_t par) const { return (2 * up_words + (uint64_t)par * sw_words) * 4; }
  uint64_t flag_off(int kind, uint32_t t) const { return (2 * up_words + 2 * sw_words) * 4 + ((uint64_t)kind * G + t) * 4; }
  uint64_t err_off() const { return flag_off(0, 0) + 2ull * G * 4; }
  uint32_t* own_flags(int kind) const { return reinterpret_cast<uint32_t*>(static_cast<char*>(xbuf) + flag_off(kind, 0)); }
  uint32_t* err_word() const { return reinterpret_cast<uint32_t*>(static_cast<char*>(xbuf) + err_off()); }

  void* exchange_buffer(uint64_t* bytes) {
    if (!xbuf) {
      up_words = (uint64_t)qmax * c->n;
      sw_words = 2ull * (pmax + 2) * c->n;
      xbytes = err_off() + 256;
      CK_CUDA(cudaMalloc(&xbuf, xbytes));
      CK_CUDA(cudaMemset(xbuf, 0, xbytes));
      // [2] epochs | jobs_cur [qmax] + [2 (pmax + 2)] | rows_cur [L] + [2 (alpha + 2)]
      const size_t nj0 = qmax, nj1 = 2ull * (pmax + 2), nr0 = c->L, nr1 = 2ull * (c->alpha + 2);
      const size_t bytes = 16 + (nj0 + nj1) * sizeof(RowJob) + (nr0 + nr1) * 8 + 64;
      CK_CUDA(cudaMalloc(&ctl, bytes));
      CK_CUDA(cudaMemset(ctl, 0, bytes));
      char* p = reinterpret_cast<char*>(ctl) + 16;
      jobs_cur[0] = reinterpret_cast<RowJob*>(p);
      jobs_cur[1] = jobs_cur[0] + nj0;
      p += (nj0 + nj1) * sizeof(RowJob);
      p = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + 7) & ~uintptr_t(7));
      rows_cur[0] = reinterpret_cast<uint64_t*>(p);
      rows_cur[1] = rows_cur[0] + nr0;
    }
    if (bytes) *bytes = xbytes;
    return xbuf;
  }
  void set_peers(const uint64_t* bases, uint32_t world) {
    if (world != G) throw InvalidArgument("peer table size != world");
    exchange_buffer(nullptr);
    peers.assign(bases, bases + G);
    if (peers[s] != reinterpret_cast<uint64_t>(xbuf)) throw InvalidArgument("peer table: own entry is not this shard's buffer");
    std::vector<uint64_t> sig(2ull * G);
    for (int k = 0; k < 2; ++k)
      for (uint32_t t = 0; t < G; ++t) sig[k * G + t] = peers[t] + flag_off(k, s);
    sig_tab = Blob();
    sig_tab.add(sig);
    sig_tab.upload();
    std::vector<uint64_t> ut(2ull * c->L);  // global Q row g -> owner's send buffer row g - q_lo(owner)
    for (uint32_t par = 0; par < 2; ++par)
      for (uint32_t t = 0; t < G; ++t)
        for (uint32_t g = q_lo(t); g < q_hi(t); ++g)
          ut[par * c->L + g] = peers[t] + up_off(par) + (uint64_t)(g - q_lo(t)) * c->n * 4;
    up_tab = Blob();
    up_tab.add(ut);
    up_tab.upload();
    down_tab.clear();
    // A fresh peer set restarts the epochs, so the flag words and the error
    // word must restart too: stale flags from an earlier peer set would
    // satisfy the next wait at once (and let BConv read rows that are not
    // written yet).  Callers barrier after set_peers, so no peer publishes
    // into this buffer before the reset has landed.
    CK_CUDA(cudaMemset(static_cast<char*>(xbuf) + flag_off(0, 0), 0, 2ull * G * 4 + 4));
    CK_CUDA(cudaMemset(ctl, 0, 8));  // epochs restart with the peer set
    CK_CUDA(cudaDeviceSynchronize());
  }
  bool peer_mode() const { return !peers.empty(); }
  // [2 parities][2 sc] source-row addresses of a drop-and-divide exchange
  const uint64_t* down_rows(int kind, uint32_t level) {
    auto key = std::make_pair(kind, level);
    auto it = down_tab.find(key);
    if (it == down_tab.end()) {
      const DownPlan& pl = down_plan(kind, level);
      std::vector<uint64_t> rt(4ull * pl.sc);  // gathered order: rank t's u-th own source, polys p
      for (uint32_t q = 0; q < 2; ++q) {
        uint32_t off = 0;
        for (uint32_t t = 0; t < G; ++t) {
          for (uint32_t u = 0; u < pl.rank_cnt[t]; ++u)
            for (uint32_t p = 0; p < 2; ++p)
              rt[(size_t)q * 2 * pl.sc + p * pl.sc + off + u] =
                  peers[t] + sw_off(q) + ((uint64_t)p * pl.smax + u) * c->n * 4;
          off += pl.rank_cnt[t];
        }
      }
      auto b = std::make_unique<Blob>();
      b->add(rt);
      b->upload();
      it = down_tab.emplace(key, std::move(b)).first;
    }
    return it->second->at<uint64_t>(0);
  }
  // phase 2 head: wait for every peer's flag of this kind's current (device)
  // epoch, then select that epoch's parity of the row table into rows_cur
  void peer_wait(int kind, const uint64_t* rows2, int nrows, cudaStream_t st) {
    if (!peer_mode()) throw InvalidArgument("no recv buffer and no peer exchange set up");
    shard_wait(own_flags(kind), (int)G, ctl + kind, err_word(), timeout_ns, rows2, rows_cur[kind], nrows, st);
    c->launches += 1;
  }
  // phase 1 head: advance this kind's epoch and select the INTT job parity
  void peer_advance(int kind, const NttPlan& intt, size_t par_off, cudaStream_t st) {
    shard_advance(ctl + kind, intt.blob.at<RowJob>(par_off), jobs_cur[kind], intt.njobs, st);
    c->launches += 1;
  }
  uint32_t peer_error() const {
    uint32_t e = 0;
    if (xbuf) CK_CUDA(cudaMemcpy(&e, err_word(), 4, cudaMemcpyDeviceToHost));
    return e;
  }

  // ---- phases ----  (send == nullptr / recv == nullptr: peer exchange)
  void modup_begin(uint32_t level, const uint32_t* d, uint32_t* send, cudaStream_t st) {
    const UpPlan& pl = up_plan(level);
    if (!send) {
      if (!peer_mode()) throw InvalidArgument("no send buffer and no peer exchange set up");
      peer_advance(0, pl.intt, pl.intt_par_off, st);
      c->run_ntt(pl.intt, true, 1, d, 0, static_cast<uint32_t*>(xbuf), 0, 0, st, jobs_cur[0]);
      shard_signal(sig_tab.at<uint64_t>(0), (int)G, ctl + 0, st);
      c->launches += 1;
    } else {
      c->run_ntt(pl.intt, true, 1, d, 0, send, 0, 0, st);
    }
    c->counters[3] += pl.lq;
  }
  void modup_keymult(uint32_t level, const uint32_t* recv, const uint32_t* d, const uint32_t* evk,
                     const uint32_t* fold, uint32_t* v, cudaStream_t st) {
    const UpPlan& pl = up_plan(level);
    const uint64_t N = c->n;
    uint32_t* compact = static_cast<uint32_t*>(c->scratch_get(((size_t)level + (size_t)pl.D * pl.rows) * N * 4, st));
    uint32_t* ext = compact + (size_t)level * N;
    const uint64_t* rows = nullptr;
    if (!recv) {  // peer exchange: wait for every rank's phase 1, read their rows in place
      if (!peer_mode()) throw InvalidArgument("no recv buffer and no peer exchange set up");
      peer_wait(0, up_tab.at<uint64_t>(0), (int)c->L, st);
      rows = rows_cur[0];
    } else {
      for (uint32_t t = 0; t < G; ++t) {  // gathered blocks -> global row order
        const uint32_t cnt = lq_of(t, level);
        if (cnt)
          CK_CUDA(cudaMemcpyAsync(compact + (size_t)q_lo(t) * N, recv + (size_t)t * qmax * N, (size_t)cnt * N * 4,
                                  cudaMemcpyDeviceToDevice, st));
      }
    }
    if (pl.bc.ngroups) {
      c->run_bconv(pl.bc, 1, compact, 0, ext, 0, st, rows);
      c->run_ntt(pl.ntt, false, 1, ext, 0, ext, 0, 1, st);
    }
    ShardKeyMultLaunch a;
    a.rows = (int)pl.rows;
    a.lq = (int)pl.lq;
    a.D = (int)pl.D;
    a.erows = (int)((qhi - qlo) + lp());
    a.ext = ext;
    a.d = d;
    a.evk = evk;
    a.fold = fold;
    a.digit = pl.maps.at<int16_t>(pl.digit_off);
    a.prime = pl.maps.at<uint16_t>(pl.prime_off);
    a.erow = pl.maps.at<uint16_t>(pl.erow_off);
    a.p_mont = c->d_pmont;
    a.v = v;
    a.primes = c->d_primes;
    a.err = recv ? nullptr : err_word();
    {
      Context::ProfScope ps(c, 3, 4.0 * N * pl.rows * (3.0 * pl.D + 2), 1, st);
      shard_key_mult((int)N, a, st);
    }
    c->launches += 1;
    c->counters[0] += 1;
    c->counters[5] += pl.D;
    c->counters[2] += pl.ntt_rows;
    c->counters[4] += pl.D;
  }
  void switch_begin(int kind, uint32_t level, const uint32_t* v, uint32_t* send, cudaStream_t st) {
    const DownPlan& pl = down_plan(kind, level);
    if (!send) {
      if (!peer_mode()) throw InvalidArgument("no send buffer and no peer exchange set up");
      peer_advance(1, pl.intt, pl.intt_par_off, st);
      c->run_ntt(pl.intt, true, 1, v, 0, static_cast<uint32_t*>(xbuf), 0, 0, st, jobs_cur[1]);
      shard_signal(sig_tab.at<uint64_t>(0) + G, (int)G, ctl + 1, st);
      c->launches += 1;
    } else {
      c->run_ntt(pl.intt, true, 1, v, 0, send, 0, 0, st);
    }
    c->counters[3] += 2ull * pl.own_sc;
  }
  void switch_end(int kind, uint32_t level, const uint32_t* recv, const uint32_t* v, const uint32_t* add,
                  uint32_t add_mask, const uint32_t* src_map, uint32_t* out, cudaStream_t st) {
    const DownPlan& pl = down_plan(kind, level);
    const uint64_t N = c->n;
    uint32_t* compact = static_cast<uint32_t*>(c->scratch_get((2ull * pl.sc + 2ull * pl.lqo) * N * 4, st));
    uint32_t* o = compact + 2ull * pl.sc * N;
    const uint64_t* rows = nullptr;
    if (!recv) {  // peer exchange
      if (!peer_mode()) throw InvalidArgument("no recv buffer and no peer exchange set up");
      peer_wait(1, down_rows(kind, level), (int)(2 * pl.sc), st);
      rows = rows_cur[1];
    } else {
      uint32_t off = 0;
      for (uint32_t t = 0; t < G; ++t) {  // [G][2][smax] -> [2][sc] in gathered order
        const uint32_t cnt = pl.rank_cnt[t];
        for (uint32_t p = 0; p < 2 && cnt; ++p)
          CK_CUDA(cudaMemcpyAsync(compact + ((size_t)p * pl.sc + off) * N,
                                  recv + ((size_t)t * 2 * pl.smax + (size_t)p * pl.smax) * N, (size_t)cnt * N * 4,
                                  cudaMemcpyDeviceToDevice, st));
        off += cnt;
      }
    }
    if (pl.lqo) {
      c->run_bconv(pl.bc, 1, compact, 0, o, 0, st, rows);
      c->run_ntt(pl.ntt, false, 1, o, 0, o, 0, 1, st);
      ShardTailLaunch a;
      a.v = v;
      a.v_ps = (uint64_t)pl.vrows * N;
      a.o = o;
      a.o_ps = (uint64_t)pl.lqo * N;
      a.dinv = pl.consts.at<uint32_t>(0);
      a.prime_base = (int)qlo;
      a.add = add;
      a.add_ps = (uint64_t)pl.lqo * N;
      a.add_mask = add_mask;
      a.src_map = src_map;
      a.out = out;
      a.out_ps = (uint64_t)pl.lqo * N;
      a.primes = c->d_primes;
      a.err = recv ? nullptr : err_word();
      {
        Context::ProfScope ps(c, 5, 4.0 * N * pl.lqo * (add ? 7 : 6), 1, st);
        shard_tail((int)N, (int)pl.lqo, a, st);
      }
      c->launches += 1;
    }
    c->counters[5] += 2;
    c->counters[2] += 2ull * pl.lqo;
  }
};

namespace {

void check_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw CudaError(std::string("kernel launch: ") + cudaGetErrorString(e));
}

template <class F>
ck_status guard(F&& f) {
  try {
    f();
    return CK_OK;
  } catch (const InvalidArgument& e) {
    g_err = e.what();
    return CK_INVALID_ARGUMENT;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return CK_INVALID_ARGUMENT;
  } catch (const CudaError& e) {
    g_err = e.what();
    return CK_CUDA_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return CK_RUNTIME_ERROR;
  }
}

Context* C(ck_context* c) {
  if (!c) throw InvalidArgument("null context");
  return reinterpret_cast<Context*>(c);
}
cudaStream_t S(ck_stream s) { return reinterpret_cast<cudaStream_t>(s); }

void check_level(const Context* c, uint32_t level, uint32_t min_level = 1) {
  if (level < min_level || level > c->L) throw InvalidArgument("level out of range");
}
void check_ptr(const void* p) {
  if (!p) throw InvalidArgument("null buffer");
}

}  // namespace
}  // namespace ck

using namespace ck;

extern "C" {

const char* ck_last_error(void) { return ck::g_err.c_str(); }
const char* ck_version(void) { return "ck32-b200 0.1.0 (sm_100a)"; }

// Row-pass twiddle tables of k_rowx (ntt256.cu) for rows of R = 2^LOGR,
// N = 256 R, x = R r + c, in consumption order per row (512 or 256 pairs):
//   forward stage 8 + s uses F[(256 << s) + (r << s) + (c >> (LOGR - s))]:
//     phase A (c = tau + TPR j, s < 5): row-shared, [2^s - 1 + (j >> (5 - s))]
//     phase B (c = 32 tau + j, s >= 5): per thread, [32 + (off(s) + blk) TPR + tau]
//   inverse stage v uses I[(N >> (v + 1)) + (r << (LOGR - 1 - v)) + (c >> (v + 1))]:
//     phase A (c = 32 tau + j, v < LOGR - 5): per thread, [(offI(v) + blk) TPR + tau]
//     phase B (c = tau + TPR j): row-shared, [RS_BASE + offR + blk]
// (same values as the reference tables, ntt.cpp:124-128).
static void build_rowx_tables(const std::vector<uint2>& fwd, const std::vector<uint2>& inv, uint32_t n, int logr,
                              uint32_t np, uint2** d_f, uint2** d_i) {
  const uint32_t R = 1u << logr, TPR = R / 32, PB = logr - 5;
  const uint32_t rs_base = TPR * (32 - (1u << (5 - PB)));
  std::vector<uint2> tf((size_t)np * n), ti((size_t)np * n);
#pragma omp parallel for schedule(static)
  for (int g = 0; g < (int)np; ++g) {
    const uint2* F = fwd.data() + (size_t)g * n;
    const uint2* I = inv.data() + (size_t)g * n;
    for (uint32_t r = 0; r < 256; ++r) {
      uint2* A = tf.data() + ((size_t)g * 256 + r) * R;
      uint2* B = ti.data() + ((size_t)g * 256 + r) * R;
      A[31] = B[R - 1] = make_uint2(0, 0);
      for (uint32_t s = 0; s < 5; ++s)
        for (uint32_t blk = 0; blk < (1u << s); ++blk) A[(1u << s) - 1 + blk] = F[(256u << s) + (r << s) + blk];
      for (uint32_t s = 5; s < (uint32_t)logr; ++s) {
        const uint32_t off = (1u << (s - PB)) - (1u << (5 - PB));
        for (uint32_t blk = 0; blk < (1u << (s - PB)); ++blk)
          for (uint32_t tau = 0; tau < TPR; ++tau)
            A[32 + (off + blk) * TPR + tau] = F[(256u << s) + (r << s) + (tau << (s - PB)) + blk];
      }
      const uint32_t offi[4] = {0, 16, 24, 28}, offr[5] = {0, 16, 24, 28, 30};
      for (uint32_t v = 0; v < PB; ++v)
        for (uint32_t blk = 0; blk < (16u >> v); ++blk)
          for (uint32_t tau = 0; tau < TPR; ++tau)
            B[(offi[v] + blk) * TPR + tau] = I[(n >> (v + 1)) + (r << (logr - 1 - v)) + (tau << (4 - v)) + blk];
      for (uint32_t t = 0; t < 5; ++t) {
        const uint32_t v = PB + t;
        for (uint32_t blk = 0; blk < (16u >> t); ++blk)
          B[rs_base + offr[t] + blk] = I[(n >> (v + 1)) + (r << (logr - 1 - v)) + blk];
      }
    }
  }
  CK_CUDA(cudaMalloc(d_f, tf.size() * sizeof(uint2)));
  CK_CUDA(cudaMemcpy(*d_f, tf.data(), tf.size() * sizeof(uint2), cudaMemcpyHostToDevice));
  CK_CUDA(cudaMalloc(d_i, ti.size() * sizeof(uint2)));
  CK_CUDA(cudaMemcpy(*d_i, ti.data(), ti.size() * sizeof(uint2), cudaMemcpyHostToDevice));
}

ck_status ck_context_create(const ck_params* params, const uint32_t* primes, int device, ck_context** out) {
  return guard([&] {
    if (!params || !out) throw InvalidArgument("null argument");
    const ck_params& p = *params;
    if (p.n < 8 || (p.n & (p.n - 1)) != 0 || p.n > (1u << 17))
      throw InvalidArgument("ring degree must be a power of two in [8, 2^17]");
    // generate_basis needs an even l (double-prime pairs) and alpha >= 1; a
    // caller-supplied basis may be any shape the reference accepts (e.g. the
    // kernel-level tests' generate_basis(n, 2, 0, ...)): mechanisms that need
    // P primes check alpha when they run.
    if (p.l < 1 || (!primes && (p.l % 2 != 0 || p.alpha < 1)))
      throw InvalidArgument("level count must be even and >= 2, alpha >= 1");
    if (p.l + p.alpha > (uint32_t)kMaxRows) throw InvalidArgument("too many primes");
    auto c = std::make_unique<Context>();
    c->p = p;
    c->device = device;
    c->n = p.n;
    while ((1u << c->logn) < p.n) ++c->logn;
    c->L = p.l;
    c->alpha = p.alpha;
    if (primes) {
      c->primes.assign(primes, primes + p.l + p.alpha);
      for (uint32_t q : c->primes)
        if (q >= (1u << 29) || (q % (2 * p.n)) != 1 || !is_prime(q))
          throw InvalidArgument("prime must be < 2^29, = 1 mod 2n");
    } else {
      c->primes = generate_basis(p.n, p.l, p.alpha, p.delta_bits);
    }
    CK_CUDA(cudaSetDevice(device));
    const uint32_t np = p.l + p.alpha, n = p.n;
    c->psi.resize(np);
    c->pdev_host.resize(np);
    std::vector<uint2> fwd((size_t)np * n), inv((size_t)np * n);
#pragma omp parallel for schedule(dynamic)
    for (int g = 0; g < (int)np; ++g) {  // build_twiddles (ntt.cpp:100-135), plain + Shoup
      const uint32_t q = c->primes[g];
      const uint32_t psi = find_root_2n(q, n);
      c->psi[g] = psi;
      const uint32_t psi_inv = invm(psi, q);
      std::vector<uint32_t> pw(n), pwi(n);
      pw[0] = pwi[0] = 1;
      for (uint32_t k = 1; k < n; ++k) {
        pw[k] = mulm(pw[k - 1], psi, q);
        pwi[k] = mulm(pwi[k - 1], psi_inv, q);
      }
      uint2* F = fwd.data() + (size_t)g * n;
      uint2* I = inv.data() + (size_t)g * n;
      F[0] = I[0] = make_uint2(0, 0);
      for (uint32_t i = 1; i < n; ++i) {
        const uint32_t e = bit_reverse(i, c->logn);
        F[i] = make_uint2(pw[e], shoup(pw[e], q));
        I[i] = make_uint2(pwi[e], shoup(pwi[e], q));
      }
      PrimeDev& P = c->pdev_host[g];
      P.q = q;
      P.q2 = 2 * q;
      uint32_t inv32 = q;
      for (int i = 0; i < 5; ++i) inv32 *= 2u - q * inv32;  // modarith.cpp:47-49
      P.qinv_neg = 0u - inv32;
      P.r = r_mod(q);
      P.r_sh = shoup(P.r, q);
      P.w1r = mulm(pw[n / 2], P.r, q);
      P.w1r_sh = shoup(P.w1r, q);
      P.qinv = inv32;
    }
    CK_CUDA(cudaMalloc(&c->d_primes, np * sizeof(PrimeDev)));
    CK_CUDA(cudaMemcpy(c->d_primes, c->pdev_host.data(), np * sizeof(PrimeDev), cudaMemcpyHostToDevice));
    CK_CUDA(cudaMalloc(&c->d_fwd, fwd.size() * sizeof(uint2)));
    CK_CUDA(cudaMemcpy(c->d_fwd, fwd.data(), fwd.size() * sizeof(uint2), cudaMemcpyHostToDevice));
    CK_CUDA(cudaMalloc(&c->d_inv, inv.size() * sizeof(uint2)));
    CK_CUDA(cudaMemcpy(c->d_inv, inv.data(), inv.size() * sizeof(uint2), cudaMemcpyHostToDevice));
    c->use_ntt256 = std::getenv("CK32_GENERIC_NTT") == nullptr;  // A/B switch for parity tests
    if (const char* ch = std::getenv("CK32_NTT_CHUNK")) c->ntt_chunk_limbs = std::max(1, std::atoi(ch));
    c->use_fused = std::getenv("CK32_FUSED") != nullptr;
    c->use_row_km = std::getenv("CK32_NO_ROW_KEYMULT") == nullptr;
    if (const char* f = std::getenv("CK32_BCONV_FP64")) c->bconv_fp64 = std::atoi(f);
    // BConv on tcgen05 by default (whole-step A/B r2ad / r2ae: 16.95-17.01k vs
    // 16.91-16.97k ops/s with the CUDA-core kernel: the IMAD.WIDE work moves
    // to the tensor pipe while the other stream's NTTs hold the IMAD pipe);
    // CK32_TC=0 selects the CUDA-core kernel, as does an FP64-pipe mode
    const char* tc = std::getenv("CK32_TC");
    c->use_tc = (tc ? std::atoi(tc) != 0 : true) && c->bconv_fp64 == 0;
    c->tc_var = tc && std::atoi(tc) == 1 ? 1 : 2;  // CK32_TC=1: the first tcgen05 kernel
    c->tail_gather = std::getenv("CK32_TAIL_GATHER") != nullptr;
    c->use_fused_combine = std::getenv("CK32_NO_FUSED_COMBINE") == nullptr;
    c->use_hrot_tail = std::getenv("CK32_FUSED_TAIL") != nullptr;
    c->use_cluster = std::getenv("CK32_NTT_CLUSTER") != nullptr;
    if (n == 65536) {
      // Row-pass twiddles of ntt256.cu, permuted per row in thread-consumption
      // order (same values as the reference tables, ntt.cpp:124-128).
      std::vector<uint2> t2f((size_t)np * n), t2i((size_t)np * n);
#pragma omp parallel for schedule(static)
      for (int g = 0; g < (int)np; ++g) {
        const uint2* F = fwd.data() + (size_t)g * n;
        const uint2* I = inv.data() + (size_t)g * n;
        for (uint32_t r = 0; r < 256; ++r) {
          uint2* A = t2f.data() + ((size_t)g * 256 + r) * 256;
          uint2* B = t2i.data() + ((size_t)g * 256 + r) * 256;
          A[15] = B[255] = make_uint2(0, 0);
          for (uint32_t s = 0; s < 4; ++s)  // forward phase A: stage 8+s, blk < 2^s
            for (uint32_t blk = 0; blk < (1u << s); ++blk)
              A[(1u << s) - 1 + blk] = F[(256u << s) + (r << s) + blk];
          for (uint32_t s = 4; s < 8; ++s)  // forward phase B: stage 8+s, blk < 2^(s-4), thread tau
            for (uint32_t blk = 0; blk < (1u << (s - 4)); ++blk)
              for (uint32_t tau = 0; tau < 16; ++tau)
                A[16 + ((1u << (s - 4)) - 1 + blk) * 16 + tau] = F[(256u << s) + (r << s) + (tau << (s - 4)) + blk];
          for (uint32_t v = 0; v < 4; ++v) {  // inverse phase A: stage v, blk < 2^(3-v), thread tau
            const uint32_t off = 16 - (16 >> v);
            for (uint32_t blk = 0; blk < (8u >> v); ++blk)
              for (uint32_t tau = 0; tau < 16; ++tau)
                B[(off + blk) * 16 + tau] = I[(32768u >> v) + (r << (7 - v)) + (tau << (3 - v)) + blk];
          }
          for (uint32_t v = 4; v < 8; ++v) {  // inverse phase B: stage v, blk < 2^(7-v)
            const uint32_t off = 16 - (16 >> (v - 4));
            for (uint32_t blk = 0; blk < (128u >> v); ++blk)
              B[240 + off + blk] = I[(32768u >> v) + (r << (7 - v)) + blk];
          }
        }
      }
      CK_CUDA(cudaMalloc(&c->d_tw2f, t2f.size() * sizeof(uint2)));
      CK_CUDA(cudaMemcpy(c->d_tw2f, t2f.data(), t2f.size() * sizeof(uint2), cudaMemcpyHostToDevice));
      CK_CUDA(cudaMalloc(&c->d_tw2i, t2i.size() * sizeof(uint2)));
      CK_CUDA(cudaMemcpy(c->d_tw2i, t2i.data(), t2i.size() * sizeof(uint2), cudaMemcpyHostToDevice));
    } else if (n == 131072) {
      build_rowx_tables(fwd, inv, n, 9, np, &c->d_tw2f, &c->d_tw2i);
    }

    std::vector<uint32_t> pm(p.l);  // p_mont (ckks.cpp:171-175)
    for (uint32_t i = 0; i < p.l; ++i) {
      const uint32_t q = c->primes[i];
      uint32_t prod = 1 % q;
      for (uint32_t j = 0; j < p.alpha; ++j) prod = mulm(prod, c->primes[p.l + j] % q, q);
      pm[i] = to_mont(prod, q);
    }
    CK_CUDA(cudaMalloc(&c->d_pmont, p.l * sizeof(uint32_t)));
    CK_CUDA(cudaMemcpy(c->d_pmont, pm.data(), p.l * sizeof(uint32_t), cudaMemcpyHostToDevice));
    *out = reinterpret_cast<ck_context*>(c.release());
  });
}

ck_status ck_generate_basis(uint32_t n, uint32_t l, uint32_t alpha, uint32_t delta_bits, uint32_t* primes_out) {
  return guard([&] {
    if (!primes_out) throw InvalidArgument("null argument");
    const auto p = generate_basis(n, l, alpha, delta_bits);
    std::copy(p.begin(), p.end(), primes_out);
  });
}

ck_status ck_context_destroy(ck_context* ctx) {
  return guard([&] { delete C(ctx); });
}

ck_status ck_context_params(const ck_context* ctx, ck_params* out) {
  return guard([&] {
    if (!ctx || !out) throw InvalidArgument("null argument");
    *out = reinterpret_cast<const Context*>(ctx)->p;
  });
}

ck_status ck_context_primes(const ck_context* ctx, uint32_t* out) {
  return guard([&] {
    const Context* c = reinterpret_cast<const Context*>(ctx);
    if (!c || !out) throw InvalidArgument("null argument");
    std::copy(c->primes.begin(), c->primes.end(), out);
  });
}

ck_status ck_context_counters(const ck_context* ctx, uint64_t out[7]) {
  return guard([&] {
    const Context* c = reinterpret_cast<const Context*>(ctx);
    if (!c || !out) throw InvalidArgument("null argument");
    std::copy(c->counters, c->counters + 7, out);
  });
}
ck_status ck_context_reset_counters(ck_context* ctx) {
  return guard([&] { std::fill(C(ctx)->counters, C(ctx)->counters + 7, 0); });
}
ck_status ck_profile(ck_context* ctx, int enable) {
  return guard([&] {
    Context* c = C(ctx);
    CK_CUDA(cudaDeviceSynchronize());
    for (auto& r : c->prof_recs) {
      c->ev_pool.push_back(r.a);
      c->ev_pool.push_back(r.b);
    }
    c->prof_recs.clear();
    c->prof = enable != 0;
  });
}

ck_status ck_profile_read(ck_context* ctx, ck_prof_stat* out, uint32_t max_classes, uint32_t* count) {
  return guard([&] {
    Context* c = C(ctx);
    static const char* names[] = {"ntt_fwd", "ntt_inv", "bconv", "key_mult", "tensor", "combine", "hrot_tail",
                                  "conv_mid", "ntt_row+keymult", "ntt_fwd+combine", "ntt_fwd+rottail"};
    const uint32_t ncls = 11;
    if (!out || !count) throw InvalidArgument("null argument");
    CK_CUDA(cudaDeviceSynchronize());
    std::vector<ck_prof_stat> st(ncls);
    for (uint32_t i = 0; i < ncls; ++i) {
      std::memset(&st[i], 0, sizeof(ck_prof_stat));
      std::snprintf(st[i].name, sizeof(st[i].name), "%s", names[i]);
    }
    for (auto& r : c->prof_recs) {
      float ms = 0;
      CK_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
      st[r.cls].groups += 1;
      st[r.cls].launches += r.launches;
      st[r.cls].ms += ms;
      st[r.cls].bytes += r.bytes;
    }
    *count = std::min(ncls, max_classes);
    std::copy(st.begin(), st.begin() + *count, out);
  });
}

uint64_t ck_launch_count(const ck_context* ctx) {
  return ctx ? reinterpret_cast<const Context*>(ctx)->launches.load() : 0;
}

ck_status ck_malloc(ck_context* ctx, size_t bytes, void** dptr) {
  return guard([&] {
    CK_CUDA(cudaSetDevice(C(ctx)->device));
    CK_CUDA(cudaMalloc(dptr, std::max<size_t>(bytes, 16)));
  });
}
ck_status ck_free(ck_context* ctx, void* dptr) {
  return guard([&] {
    CK_CUDA(cudaSetDevice(C(ctx)->device));
    CK_CUDA(cudaFree(dptr));
  });
}
ck_status ck_memcpy_h2d(ck_context* ctx, void* dst, const void* src, size_t bytes, ck_stream stream) {
  return guard([&] { CK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, S(stream))); (void)ctx; });
}
ck_status ck_memcpy_d2h(ck_context* ctx, void* dst, const void* src, size_t bytes, ck_stream stream) {
  return guard([&] { CK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, S(stream))); (void)ctx; });
}
ck_status ck_memcpy_d2d(ck_context* ctx, void* dst, const void* src, size_t bytes, ck_stream stream) {
  return guard([&] { CK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, S(stream))); (void)ctx; });
}
// ---- the reference's randomness (host side, as in the reference) ----
// std::mt19937_64 consumed draw for draw like ckks.cpp: sample_gaussian
// (:33-40, Box-Muller on two 53-bit draws, llround), ternary_coeffs (:51-60,
// Fisher-Yates positions + sign bit), uniform_eval (:383-395, rng() % q row
// by row).  Compiled by the same g++/glibc as the reference, with the same
// expressions, so a seed reproduces the reference's keys and ciphertexts.
struct ck_rng {
  std::mt19937_64 g;
};
ck_status ck_rng_create(uint64_t seed, ck_rng** out) {
  return guard([&] {
    if (!out) throw InvalidArgument("null argument");
    *out = new ck_rng{std::mt19937_64(seed)};
  });
}
ck_status ck_rng_destroy(ck_rng* r) {
  return guard([&] { delete r; });
}
ck_status ck_rng_draws(ck_rng* r, uint64_t count, uint64_t* out) {
  return guard([&] {
    if (!r || (count && !out)) throw InvalidArgument("null argument");
    for (uint64_t i = 0; i < count; ++i) out[i] = r->g();
  });
}
ck_status ck_sample_gaussian(ck_rng* r, uint32_t n, double sigma, int64_t* out) {
  return guard([&] {
    if (!r || (n && !out)) throw InvalidArgument("null argument");
    constexpr double kPi = 3.141592653589793238462643383279502884;  // std::numbers::pi
    for (uint32_t i = 0; i < n; ++i) {
      const double u1 = (static_cast<double>(r->g() >> 11) + 0.5) * 0x1p-53;
      const double u2 = static_cast<double>(r->g() >> 11) * 0x1p-53;
      const double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * kPi * u2);
      out[i] = std::llround(z * sigma);
    }
  });
}
ck_status ck_sample_ternary(ck_rng* r, uint32_t n, uint32_t h, int64_t* out) {
  return guard([&] {
    if (!r || !out) throw InvalidArgument("null argument");
    if (h > n) throw InvalidArgument("hamming weight exceeds n");
    std::vector<uint32_t> idx(n);
    for (uint32_t i = 0; i < n; ++i) idx[i] = i;
    for (uint32_t i = 0; i < n; ++i) out[i] = 0;
    for (uint32_t i = 0; i < h; ++i) {
      const uint32_t j = i + static_cast<uint32_t>(r->g() % (n - i));
      std::swap(idx[i], idx[j]);
      out[idx[i]] = (r->g() & 1) ? 1 : -1;
    }
  });
}
ck_status ck_sample_uniform(ck_rng* r, const uint32_t* q, uint32_t rows, uint32_t n, uint32_t* out) {
  return guard([&] {
    if (!r || (rows && (!q || !out))) throw InvalidArgument("null argument");
    for (uint32_t i = 0; i < rows; ++i) {
      if (q[i] == 0) throw InvalidArgument("zero modulus");
      for (uint32_t k = 0; k < n; ++k) out[(size_t)i * n + k] = static_cast<uint32_t>(r->g() % q[i]);
    }
  });
}

ck_status ck_stream_create(ck_context* ctx, ck_stream* out) {
  return guard([&] {
    if (!ctx || !out) throw InvalidArgument("null argument");
    CK_CUDA(cudaSetDevice(C(ctx)->device));
    cudaStream_t st;
    CK_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    *out = st;
  });
}

ck_status ck_stream_destroy(ck_context* ctx, ck_stream stream) {
  return guard([&] {
    if (!ctx) throw InvalidArgument("null argument");
    if (stream) {
      CK_CUDA(cudaStreamSynchronize(S(stream)));
      Context* c = C(ctx);
      auto it = c->scratch.find(S(stream));  // the stream's scratch arena goes with it
      if (it != c->scratch.end()) {
        if (it->second.ptr) CK_CUDA(cudaFree(it->second.ptr));
        c->scratch.erase(it);
      }
      CK_CUDA(cudaStreamDestroy(S(stream)));
    }
  });
}

ck_status ck_stream_sync(ck_context* ctx, ck_stream stream) {
  return guard([&] { CK_CUDA(cudaStreamSynchronize(S(stream))); (void)ctx; });
}

ck_status ck_ntt_forward(ck_context* ctx, uint32_t* rows_dev, uint32_t rows, const uint32_t* gidx, ck_stream stream) {
  return guard([&] {
    CK_RANGE("ck_ntt_forward");
    Context* c = C(ctx);
    check_ptr(rows_dev);
    if (!gidx && rows) throw InvalidArgument("null prime index list");
    std::string key(1, 'F');
    key.append(reinterpret_cast<const char*>(gidx), sizeof(uint32_t) * rows);
    auto& pl = c->adhoc_ntt[key];
    if (!pl) {
      std::vector<RowJob> jobs;
      for (uint32_t i = 0; i < rows; ++i) {
        if (gidx[i] >= c->primes.size()) throw InvalidArgument("prime index out of range");
        jobs.push_back({i, i, (uint16_t)gidx[i], 0});
      }
      auto np = std::make_unique<NttPlan>();
      np->jobs_off = np->blob.add(jobs);
      np->njobs = (int)jobs.size();
      np->blob.upload();
      pl = std::move(np);
    }
    c->run_ntt(*pl, false, 1, rows_dev, 0, rows_dev, 0, 1, S(stream));
    check_launch();
    c->counters[2] += rows;
  });
}

static ck_status ntt_raw_impl(ck_context* ctx, int32_t* rows_dev, uint32_t rows, const uint32_t* gidx,
                              const uint32_t* epilogue_mont, int inverse, ck_stream stream) {
  return guard([&] {
    CK_RANGE("ck_ntt_raw");
    Context* c = C(ctx);
    check_ptr(rows_dev);
    if (!gidx && rows) throw InvalidArgument("null prime index list");
    if (!rows) return;
    std::vector<uint16_t> g16(rows);
    std::vector<uint32_t> epi(epilogue_mont ? rows : 0);
    for (uint32_t i = 0; i < rows; ++i) {
      if (gidx[i] >= c->primes.size()) throw InvalidArgument("prime index out of range");
      g16[i] = (uint16_t)gidx[i];
      if (epilogue_mont) epi[i] = epilogue_mont[i];
    }
    const RawNttConst* rc = c->raw_const();
    cudaStream_t st = S(stream);
    char* tmp = nullptr;  // stream-ordered: the per-call prime / epilogue lists
    const size_t bytes = rows * 2 + 16 + epi.size() * 4;
    CK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&tmp), bytes, st));
    CK_CUDA(cudaMemcpyAsync(tmp, g16.data(), rows * 2, cudaMemcpyHostToDevice, st));
    uint32_t* depi = nullptr;
    if (!epi.empty()) {
      depi = reinterpret_cast<uint32_t*>(tmp + ((rows * 2 + 15) & ~size_t(15)));
      CK_CUDA(cudaMemcpyAsync(depi, epi.data(), epi.size() * 4, cudaMemcpyHostToDevice, st));
    }
    ntt_raw((int)c->n, (int)c->logn, (int)rows, inverse, rows_dev, reinterpret_cast<const uint16_t*>(tmp), c->d_primes,
            rc, inverse ? c->d_inv : c->d_fwd, depi, st);
    CK_CUDA(cudaStreamSynchronize(st));  // the host lists are staged from pageable memory
    CK_CUDA(cudaFreeAsync(tmp, st));
    c->launches += c->logn;
    c->counters[inverse ? 3 : 2] += rows;
    check_launch();
  });
}

ck_status ck_ntt_forward_raw(ck_context* ctx, int32_t* rows_dev, uint32_t rows, const uint32_t* gidx,
                             ck_stream stream) {
  return ntt_raw_impl(ctx, rows_dev, rows, gidx, nullptr, 0, stream);
}
ck_status ck_intt_inverse_raw(ck_context* ctx, int32_t* rows_dev, uint32_t rows, const uint32_t* gidx,
                              const uint32_t* epilogue_mont, ck_stream stream) {
  return ntt_raw_impl(ctx, rows_dev, rows, gidx, epilogue_mont, 1, stream);
}

ck_status ck_intt_inverse(ck_context* ctx, uint32_t* rows_dev, uint32_t rows, const uint32_t* gidx,
                          const uint32_t* epilogue_mont, ck_stream stream) {
  return guard([&] {
    CK_RANGE("ck_intt_inverse");
    Context* c = C(ctx);
    check_ptr(rows_dev);
    if (!gidx && rows) throw InvalidArgument("null prime index list");
    // plan cache key: the raw prime-index and epilogue words (no per-call
    // modular arithmetic on a hit: the exit constants are built once)
    std::string key(1, 'I');
    key.append(reinterpret_cast<const char*>(gidx), sizeof(uint32_t) * rows);
    if (epilogue_mont) key.append(reinterpret_cast<const char*>(epilogue_mont), sizeof(uint32_t) * rows);
    auto& pl = c->adhoc_ntt[key];
    if (!pl) {
      std::vector<RowJob> jobs;
      std::vector<ExitConst> exits;
      for (uint32_t i = 0; i < rows; ++i) {
        if (gidx[i] >= c->primes.size()) throw InvalidArgument("prime index out of range");
        const uint32_t q = c->q(gidx[i]);
        // epilogue given in Montgomery form (ntt.hpp:72-73): plain factor = e * R^-1
        const uint32_t e = epilogue_mont ? mulm(epilogue_mont[i] % q, invm(r_mod(q), q), q) : 1u;
        jobs.push_back({i, i, (uint16_t)gidx[i], (uint16_t)i});
        exits.push_back(c->exit_const(gidx[i], e));
      }
      auto np = std::make_unique<NttPlan>();
      np->jobs_off = np->blob.add(jobs);
      np->exits_off = np->blob.add(exits);
      np->njobs = (int)jobs.size();
      np->blob.upload();
      pl = std::move(np);
    }
    c->run_ntt(*pl, true, 1, rows_dev, 0, rows_dev, 0, 0, S(stream));
    check_launch();
    c->counters[3] += rows;
  });
}

ck_status ck_bconv(ck_context* ctx, const uint32_t* src_dev, uint32_t src_count, const uint32_t* src_gidx,
                   uint32_t* dst_dev, uint32_t dst_count, const uint32_t* dst_gidx, ck_stream stream) {
  return guard([&] {
    CK_RANGE("ck_bconv");
    Context* c = C(ctx);
    check_ptr(src_dev);
    check_ptr(dst_dev);
    if (src_count == 0 || !src_gidx || !dst_gidx) throw InvalidArgument("empty conversion");
    std::vector<uint32_t> sg(src_gidx, src_gidx + src_count), dg(dst_gidx, dst_gidx + dst_count);
    for (uint32_t g : sg)
      if (g >= c->primes.size()) throw InvalidArgument("prime index out of range");
    for (uint32_t g : dg)
      if (g >= c->primes.size()) throw InvalidArgument("prime index out of range");
    c->check_bconv_width(sg);
    std::string key;
    for (uint32_t g : sg) key += std::to_string(g) + ",";
    key += "|";
    for (uint32_t g : dg) key += std::to_string(g) + ",";
    auto& pl = c->adhoc_bc[key];
    if (!pl) {
      pl = std::make_unique<BconvPlan>();
      std::vector<uint32_t> cmat, part1, drow(dst_count);
      std::vector<uint16_t> dprime(dst_count);
      c->bconv_consts(sg, dg, cmat, part1);
      for (uint32_t i = 0; i < dst_count; ++i) {
        drow[i] = i;
        dprime[i] = (uint16_t)dg[i];
      }
      std::vector<BconvGroup> groups = {{0, src_count, dst_count, 0, 0}};
      pl->groups_off = pl->blob.add(groups);
      pl->cmat_off = pl->blob.add(cmat);
      pl->row_off = pl->blob.add(drow);
      pl->prime_off = pl->blob.add(dprime);
      pl->ngroups = 1;
      pl->max_sc = (int)src_count;
      pl->src_rows = src_count;
      pl->dst_rows = dst_count;
      add_bconv_tc(*pl, groups, cmat, dprime, [&](uint32_t g) { return c->q(g); }, c->n);
      pl->blob.upload();
    }
    c->run_bconv(*pl, 1, src_dev, 0, dst_dev, 0, S(stream));
    check_launch();
    c->counters[5] += 1;
  });
}

ck_status ck_mod_switch(ck_context* ctx, const uint32_t* src_dev, uint32_t src_count, const uint32_t* src_gidx,
                        uint32_t* dst_dev, uint32_t dst_q, uint32_t dst_p, ck_stream stream) {
  // bconv.cpp:176-213: INTT with the part-1 epilogue, BConv part 2, forward NTT
  std::vector<uint32_t> sg, dg, part1_mont;
  Context* c = nullptr;
  uint32_t* work = nullptr;
  ck_status st0 = guard([&] {
    c = C(ctx);
    check_ptr(src_dev);
    check_ptr(dst_dev);
    if (src_count == 0 || !src_gidx) throw InvalidArgument("input rows do not match table source");
    if (dst_q > c->L || dst_p > c->alpha || dst_q + dst_p == 0)
      throw InvalidArgument("output rows do not match table destination");
    sg.assign(src_gidx, src_gidx + src_count);
    for (uint32_t g : sg)
      if (g >= c->primes.size()) throw InvalidArgument("source prime mismatch");
    for (uint32_t i = 0; i < dst_q; ++i) dg.push_back(i);
    for (uint32_t j = 0; j < dst_p; ++j) dg.push_back(c->L + j);
    std::vector<uint32_t> cmat, part1;
    c->bconv_consts(sg, dg, cmat, part1);
    for (size_t j = 0; j < sg.size(); ++j) part1_mont.push_back(to_mont(part1[j], c->q(sg[j])));
    work = static_cast<uint32_t*>(c->scratch_get((size_t)src_count * c->n * 4, S(stream)));
    CK_CUDA(cudaMemcpyAsync(work, src_dev, (size_t)src_count * c->n * 4, cudaMemcpyDeviceToDevice, S(stream)));
  });
  if (st0 != CK_OK) return st0;
  ck_status s1 = ck_intt_inverse(ctx, work, src_count, sg.data(), part1_mont.data(), stream);
  if (s1 != CK_OK) return s1;
  s1 = ck_bconv(ctx, work, src_count, sg.data(), dst_dev, (uint32_t)dg.size(), dg.data(), stream);
  if (s1 != CK_OK) return s1;
  return ck_ntt_forward(ctx, dst_dev, (uint32_t)dg.size(), dg.data(), stream);
}

ck_status ck_automorphism(ck_context* ctx, const uint32_t* in_dev, uint32_t* out_dev, uint32_t rows, int64_t r,
                          ck_stream stream) {
  return guard([&] {
    CK_RANGE("ck_automorphism");
    Context* c = C(ctx);
    check_ptr(in_dev);
    check_ptr(out_dev);
    if (in_dev == out_dev) throw InvalidArgument("automorphism is out-of-place");
    permute((int)c->n, (int)rows, 1, in_dev, 0, out_dev, 0, c->rotation_map(r), S(stream));
    ++c->launches;
    check_launch();
  });
}

ck_status ck_automorphism_galois(ck_context* ctx, const uint32_t* in_dev, uint32_t* out_dev, uint32_t q_rows,
                                 uint32_t p_rows, uint64_t galois, int coeff_domain, ck_stream stream) {
  return guard([&] {
    CK_RANGE("ck_automorphism_galois");
    Context* c = C(ctx);
    check_ptr(in_dev);
    check_ptr(out_dev);
    if (in_dev == out_dev) throw InvalidArgument("automorphism is out-of-place");
    const uint64_t two_n = 2ull * c->n;
    const uint64_t g = galois % two_n;
    if ((g & 1) == 0) throw InvalidArgument("Galois element must be odd");
    uint64_t gi = 1;  // g^-1 = g^(n-1) mod 2n: the unit group mod 2n has order n
    for (uint64_t e = c->n - 1, b = g; e; e >>= 1, b = b * b % two_n)
      if (e & 1) gi = gi * b % two_n;
    if (gi * g % two_n != 1) throw InvalidArgument("Galois element not invertible");
    automorphism_galois((int)c->n, (int)c->logn, (int)(q_rows + p_rows), (uint32_t)g, (uint32_t)gi, coeff_domain ? 1 : 0,
                        in_dev, out_dev, c->poly_row_primes(q_rows, p_rows), c->d_primes, S(stream));
    ++c->launches;
    check_launch();
  });
}

ck_status ck_ew_binary(ck_context* ctx, int op, const uint32_t* a, const uint32_t* b, uint32_t* out, uint32_t q_rows,
                       uint32_t p_rows, ck_stream stream) {
  return guard([&] {
    CK_RANGE("ck_ew_binary");
    Context* c = C(ctx);
    check_ptr(a);
    check_ptr(b);
    check_ptr(out);
    if (op < 0 || op > 6 || op == 3)
      throw InvalidArgument("element-wise op must be 0 (add), 1 (sub), 2 (mul) or 4 / 5 / 6 (raw add / sub / mul)");
    elementwise((int)c->n, (int)(q_rows + p_rows), 1, op, a, 0, b, 0, out, 0, c->poly_row_primes(q_rows, p_rows),
                c->d_primes, S(stream));
    ++c->launches;
    check_launch();
  });
}

static ck_status ew_mul_const_impl(ck_context* ctx, const uint32_t* a, const uint32_t* consts_mont, uint32_t* out,
                                   uint32_t q_rows, uint32_t p_rows, ck_stream stream, bool raw);
ck_status ck_ew_mul_const(ck_context* ctx, const uint32_t* a, const uint32_t* consts_mont, uint32_t* out,
                          uint32_t q_rows, uint32_t p_rows, ck_stream stream) {
  return ew_mul_const_impl(ctx, a, consts_mont, out, q_rows, p_rows, stream, false);
}
ck_status ck_ew_mul_const_raw(ck_context* ctx, const uint32_t* a, const uint32_t* consts_mont, uint32_t* out,
                              uint32_t q_rows, uint32_t p_rows, ck_stream stream) {
  return ew_mul_const_impl(ctx, a, consts_mont, out, q_rows, p_rows, stream, true);
}
static ck_status ew_mul_const_impl(ck_context* ctx, const uint32_t* a, const uint32_t* consts_mont, uint32_t* out,
                                   uint32_t q_rows, uint32_t p_rows, ck_stream stream, bool raw) {
  return guard([&] {
    CK_RANGE("ck_ew_mul_const");
    Context* c = C(ctx);
    check_ptr(a);
    check_ptr(out);
    check_ptr(consts_mont);
    const uint16_t* rp = c->poly_row_primes(q_rows, p_rows);
    const uint32_t rows = q_rows + p_rows;
    std::vector<uint32_t> k(rows);
    for (uint32_t i = 0; i < rows; ++i) {
      const uint32_t q = c->q(i < q_rows ? i : c->L + (i - q_rows));
      k[i] = raw ? consts_mont[i] : consts_mont[i] % q;  // canonical, poly.hpp:121-122 (raw: as the reference reads it)
    }
    uint32_t* d = nullptr;  // stream-ordered: safe for concurrent calls on other streams
    CK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), rows * 4, S(stream)));
    CK_CUDA(cudaMemcpyAsync(d, k.data(), rows * 4, cudaMemcpyHostToDevice, S(stream)));
    elementwise((int)c->n, (int)rows, 1, raw ? 7 : 3, a, 0, a, 0, out, 0, rp, c->d_primes, S(stream), 0, d);
    CK_CUDA(cudaFreeAsync(d, S(stream)));  // (a pageable-source copy has staged k before returning)
    ++c->launches;
    check_launch();
  });
}

ck_status ck_bconv_table(ck_context* ctx, const uint32_t* src_dev, uint32_t src_count, const uint32_t* src_gidx,
                         uint32_t* dst_dev, uint32_t dst_count, const uint32_t* dst_gidx, const int32_t* c_centered,
                         ck_stream stream) {
  return guard([&] {
    CK_RANGE("ck_bconv_table");
    Context* c = C(ctx);
    check_ptr(src_dev);
    check_ptr(dst_dev);
    check_ptr(c_centered);
    if (src_count == 0 || !src_gidx || !dst_gidx) throw InvalidArgument("empty conversion");
    std::vector<uint32_t> sg(src_gidx, src_gidx + src_count), dg(dst_gidx, dst_gidx + dst_count);
    for (uint32_t g : sg)
      if (g >= c->primes.size()) throw InvalidArgument("prime index out of range");
    for (uint32_t g : dg)
      if (g >= c->primes.size()) throw InvalidArgument("prime index out of range");
    c->check_bconv_width(sg);
    // the caller's table (BConvTable::c, centred Montgomery constants,
    // bconv.hpp:20-22) lifted to canonical [0, q_i): the same residue class,
    // so the canonical outputs equal the reference's
    std::vector<uint32_t> cmat((size_t)dst_count * src_count);
    for (uint32_t i = 0; i < dst_count; ++i) {
      const int64_t qi = c->q(dg[i]);
      for (uint32_t j = 0; j < src_count; ++j) {
        int64_t v = c_centered[(size_t)i * src_count + j] % qi;
        if (v < 0) v += qi;
        cmat[(size_t)i * src_count + j] = (uint32_t)v;
      }
    }
    std::string key("T");
    key.append(reinterpret_cast<const char*>(sg.data()), sg.size() * 4);
    key.append(reinterpret_cast<const char*>(dg.data()), dg.size() * 4);
    key.append(reinterpret_cast<const char*>(cmat.data()), cmat.size() * 4);
    auto& pl = c->adhoc_bc[key];
    if (!pl) {
      pl = std::make_unique<BconvPlan>();
      std::vector<uint32_t> drow(dst_count);
      std::vector<uint16_t> dprime(dst_count);
      for (uint32_t i = 0; i < dst_count; ++i) {
        drow[i] = i;
        dprime[i] = (uint16_t)dg[i];
      }
      std::vector<BconvGroup> groups = {{0, src_count, dst_count, 0, 0}};
      pl->groups_off = pl->blob.add(groups);
      pl->cmat_off = pl->blob.add(cmat);
      pl->row_off = pl->blob.add(drow);
      pl->prime_off = pl->blob.add(dprime);
      pl->ngroups = 1;
      pl->max_sc = (int)src_count;
      pl->src_rows = src_count;
      pl->dst_rows = dst_count;
      add_bconv_tc(*pl, groups, cmat, dprime, [&](uint32_t g) { return c->q(g); }, c->n);
      pl->blob.upload();
    }
    c->run_bconv(*pl, 1, src_dev, 0, dst_dev, 0, S(stream));
    check_launch();
    c->counters[5] += 1;
  });
}

static ck_status ew(ck_context* ctx, int op, const uint32_t* a, const uint32_t* b, uint32_t* out, uint32_t rows,
                    ck_stream stream) {
  return guard([&] {
    Context* c = C(ctx);
    check_ptr(a);
    check_ptr(b);
    check_ptr(out);
    if (rows > c->L) throw InvalidArgument("rows exceed the Q basis");
    elementwise((int)c->n, (int)rows, 1, op, a, 0, b, 0, out, 0, nullptr, c->d_primes, S(stream));
    ++c->launches;
    check_launch();
  });
}
ck_status ck_ew_add(ck_context* ctx, const uint32_t* a, const uint32_t* b, uint32_t* out, uint32_t rows,
                    ck_stream stream) {
  return ew(ctx, 0, a, b, out, rows, stream);
}
ck_status ck_ew_sub(ck_context* ctx, const uint32_t* a, const uint32_t* b, uint32_t* out, uint32_t rows,
                    ck_stream stream) {
  return ew(ctx, 1, a, b, out, rows, stream);
}
ck_status ck_ew_mul(ck_context* ctx, const uint32_t* a, const uint32_t* b, uint32_t* out, uint32_t rows,
                    ck_stream stream) {
  return ew(ctx, 2, a, b, out, rows, stream);
}

ck_status ck_mod_up(ck_context* ctx, uint32_t level, const uint32_t* d, uint32_t* hoist, ck_stream stream) {
  return guard([&] {
    CK_RANGE("ck_mod_up");
    Context* c = C(ctx);
    check_level(c, level);
    check_ptr(d);
    check_ptr(hoist);
    const uint64_t N = c->n;
    const uint32_t D = c->digits(level), rows = level + c->alpha;
    uint32_t* is = static_cast<uint32_t*>(c->scratch_get(level * N * 4, S(stream)));
    c->mod_up(level, 1, d, 0, is, hoist, S(stream));
    // the public HoistState carries the digit rows too (ckks.cpp:708-709)
    for (uint32_t k = 0; k < D; ++k) {
      const uint32_t b = k * c->alpha, e = std::min((k + 1) * c->alpha, level);
      CK_CUDA(cudaMemcpyAsync(hoist + ((size_t)k * rows + b) * N, d + (size_t)b * N, (size_t)(e - b) * N * 4,
                              cudaMemcpyDeviceToDevice, S(stream)));
    }
    check_launch();
  });
}

ck_status ck_key_mult(ck_context* ctx, uint32_t level, const uint32_t* hoist, const uint32_t* evk, uint32_t* v,
                      ck_stream stream) {
  return guard([&] {
    CK_RANGE("ck_key_mult");
    Context* c = C(ctx);
    check_level(c, level);
    check_ptr(hoist);
    check_ptr(evk);
    check_ptr(v);
    // key_mult_v reads each digit's own (pass-through) rows from a compact
    // level-row buffer; gather them out of the full HoistState first.
    const uint32_t rows = level + c->alpha;
    const uint64_t N = c->n;
    uint32_t* dd = static_cast<uint32_t*>(c->scratch_get(level * N * 4, S(stream)));
    const uint32_t D = c->digits(level);
    for (uint32_t k = 0; k < D; ++k) {
      const uint32_t b = k * c->alpha, e = std::min((k + 1) * c->alpha, level);
      CK_CUDA(cudaMemcpyAsync(dd + (size_t)b * N, hoist + ((size_t)k * rows + b) * N, (size_t)(e - b) * N * 4,
                              cudaMemcpyDeviceToDevice, S(stream)));
    }
    c->key_mult_v(level, 1, hoist, dd, 0, evk, nullptr, 0, v, S(stream));
    check_launch();
  });
}

ck_status ck_mod_down(ck_context* ctx, uint32_t level, const uint32_t* v, uint32_t* out, ck_stream stream) {
  return guard([&] {
    CK_RANGE("ck_mod_down");
    Context* c = C(ctx);
    check_level(c, level);
    check_ptr(v);
    check_ptr(out);
    if (c->alpha == 0) throw InvalidArgument("key switching needs P primes (alpha = 0)");
    const SwitchPlan& pl = c->switch_plan(0, level, 1);
    uint32_t* ts = static_cast<uint32_t*>(c->scratch_get((size_t)pl.sc * c->n * 4, S(stream)));
    c->drop_divide(pl, 1, v, 0, ts, out, true, S(stream));
    c->counters[1] += 1;
    check_launch();
  });
}

ck_status ck_key_switch(ck_context* ctx, uint32_t level, const uint32_t* d, const uint32_t* evk, uint32_t* out,
                        ck_stream stream) {
  return guard([&] {
    CK_RANGE("ck_key_switch");
    Context* c = C(ctx);
    check_level(c, level);
    check_ptr(d);
    check_ptr(evk);
    check_ptr(out);
    const uint64_t N = c->n;
    const uint32_t D = c->digits(level), rows = level + c->alpha;
    const SwitchPlan& pl = c->switch_plan(0, level, 2);
    const size_t is_w = level * N, ext_w = (size_t)D * rows * N, v_w = 2ull * rows * N, ts_w = 2ull * pl.sc * N;
    uint32_t* base = static_cast<uint32_t*>(c->scratch_get((is_w + ext_w + v_w + ts_w) * 4, S(stream)));
    uint32_t *is = base, *ext = is + is_w, *v = ext + ext_w, *ts = v + v_w;
    c->mod_up_key_mult(level, 1, d, 0, is, ext, evk, nullptr, 0, v, S(stream));
    c->drop_divide(pl, 1, v, 0, ts, out, true, S(stream));
    c->counters[1] += 1;
    check_launch();
  });
}

ck_status ck_rescale(ck_context* ctx, uint32_t level, uint32_t batch, const uint32_t* ct, uint32_t* out,
                     ck_stream stream) {
  return guard([&] {
    CK_RANGE("ck_rescale");
    Context* c = C(ctx);
    check_level(c, level, 4);
    check_ptr(ct);
    check_ptr(out);
    const SwitchPlan& pl = c->switch_plan(1, level, 2);
    uint32_t* ts = static_cast<uint32_t*>(c->scratch_get((size_t)batch * 2 * pl.sc * c->n * 4, S(stream)));
    c->drop_divide(pl, (int)batch, ct, 2ull * level * c->n, ts, out, true, S(stream));
    c->counters[6] += batch;
    check_launch();
  });
}

ck_status ck_hmult(ck_context* ctx, uint32_t level, uint32_t batch, const uint32_t* x, const uint32_t* y,
                   const uint32_t* relin_evk, uint32_t* out, ck_stream stream) {
  return guard([&] {
    CK_RANGE("ck_hmult");
    Context* c = C(ctx);
    check_level(c, level, 4);  // ckks.cpp:815
    check_ptr(x);
    check_ptr(y);
    check_ptr(relin_evk);
    check_ptr(out);
    if (batch == 0) return;
    const uint64_t N = c->n;
    const int B = (int)batch;
    const uint32_t D = c->digits(level), rows = level + c->alpha;
    const bool lazy = c->p.lazy_rescale != 0;
    const SwitchPlan& pl = lazy ? c->switch_plan(0, level, 2) : c->switch_plan(2, level, 2);
    const size_t t01_w = 2ull * level * N, d2_w = level * N, is_w = level * N, ext_w = (size_t)D * rows * N,
                 v_w = 2ull * rows * N, ts_w = 2ull * pl.sc * N, c_w = lazy ? 2ull * level * N : 0;
    const size_t per = t01_w + d2_w + is_w + ext_w + v_w + ts_w + c_w;
    uint32_t* base = static_cast<uint32_t*>(c->scratch_get(per * B * 4, S(stream)));
    uint32_t* t01 = base;
    uint32_t* d2 = t01 + t01_w * B;
    uint32_t* is = d2 + d2_w * B;
    uint32_t* ext = is + is_w * B;
    uint32_t* v = ext + ext_w * B;
    uint32_t* ts = v + v_w * B;
    uint32_t* cc = ts + ts_w * B;
    cudaStream_t st = S(stream);
    {
      Context::ProfScope ps(c, 4, 4.0 * N * level * 7 * B, 1, st);  // 4 rows in, 3 out
      tensor((int)N, (int)level, B, x, y, 2ull * level * N, t01, t01_w, d2, d2_w, c->d_primes, st);
    }
    ++c->launches;
    if (!lazy) {  // fold P*d0/1 fused; the merged switch's INTT pass A fused into the KeyMult epilogue
      const bool pre = c->mod_up_key_mult(level, B, d2, d2_w, is, ext, relin_evk, t01, t01_w, v, st, &pl, ts, ts_w);
      c->drop_divide(pl, B, v, v_w, ts, out, true, st, pre);
    } else {
      const bool pre = c->mod_up_key_mult(level, B, d2, d2_w, is, ext, relin_evk, nullptr, 0, v, st, &pl, ts, ts_w);
      c->drop_divide(pl, B, v, v_w, ts, cc, true, st, pre);
      // out.b = d0 + c0, out.a = d1 + c1 (ckks.cpp:857-858)
      elementwise((int)N, (int)(2 * level), B, 0, t01, t01_w, cc, c_w, out, 2ull * level * N, nullptr,
                  c->d_primes, st, (int)level);
      ++c->launches;
    }
    c->counters[1] += B;
    check_launch();
  });
}

ck_status ck_hrot(ck_context* ctx, uint32_t level, uint32_t batch, const uint32_t* ct, int64_t r,
                  const uint32_t* rot_evk, uint32_t* out, ck_stream stream) {
  return guard([&] {
    CK_RANGE("ck_hrot");
    Context* c = C(ctx);
    check_level(c, level);
    check_ptr(ct);
    check_ptr(rot_evk);
    check_ptr(out);
    if (batch == 0) return;
    if (ct == out) throw InvalidArgument("hrot is out-of-place");
    const uint64_t N = c->n;
    const int B = (int)batch;
    const uint32_t D = c->digits(level), rows = level + c->alpha;
    const SwitchPlan& pl = c->switch_plan(0, level, 2);
    const size_t is_w = level * N, ext_w = (size_t)D * rows * N, v_w = 2ull * rows * N, ts_w = 2ull * pl.sc * N,
                 o_w = 2ull * level * N;
    const size_t per = is_w + ext_w + v_w + ts_w + o_w;
    uint32_t* base = static_cast<uint32_t*>(c->scratch_get(per * B * 4, S(stream)));
    uint32_t* is = base;
    uint32_t* ext = is + is_w * B;
    uint32_t* v = ext + ext_w * B;
    uint32_t* ts = v + v_w * B;
    uint32_t* o = ts + ts_w * B;
    cudaStream_t st = S(stream);
    const uint64_t ct_bs = 2ull * level * N;
    const uint32_t* a = ct + level * N;
    const bool pre = c->mod_up_key_mult(level, B, a, ct_bs, is, ext, rot_evk, nullptr, 0, v, st, &pl, ts, ts_w);
    if (!c->drop_divide_hrot(pl, B, v, v_w, ts, o, ct, ct_bs, r, out, st, pre)) {
      c->drop_divide(pl, B, v, v_w, ts, o, false, st, pre);
      Context::ProfScope ps(c, 6, 4.0 * N * level * 7 * B, 1, st);  // v0 v1 o0 o1 b in, 2 out
      hrot_tail((int)N, (int)level, B, v, v_w, rows * N, o, o_w, level * N, ct, ct_bs, pl.consts.at<uint32_t>(0),
                c->rotation_map(r), out, ct_bs, c->d_primes, st, c->tail_gather ? nullptr : c->rotation_dest(r));
      ++c->launches;
    }
    c->counters[1] += B;
    check_launch();
  });
}

static ck_status ct_ew(ck_context* ctx, int op, uint32_t level, uint32_t batch, const uint32_t* x, const uint32_t* y,
                       bool y_is_pt, bool pt_only_b, uint32_t* out, ck_stream stream) {
  return guard([&] {
    Context* c = C(ctx);
    check_level(c, level);
    check_ptr(x);
    check_ptr(y);
    check_ptr(out);
    const uint64_t N = c->n, ct_bs = 2ull * level * N;
    cudaStream_t st = S(stream);
    if (!y_is_pt) {
      elementwise((int)N, (int)(2 * level), (int)batch, op, x, ct_bs, y, ct_bs, out, ct_bs, nullptr, c->d_primes, st,
                  (int)level);
      ++c->launches;
    } else {
      elementwise((int)N, (int)level, (int)batch, op, x, ct_bs, y, 0, out, ct_bs, nullptr, c->d_primes, st);
      ++c->launches;
      if (pt_only_b) {  // padd: a copied (ckks.cpp:578)
        CK_CUDA(cudaMemcpy2DAsync(out + level * N, ct_bs * 4, x + level * N, ct_bs * 4, level * N * 4, batch,
                                  cudaMemcpyDeviceToDevice, st));
      } else {
        elementwise((int)N, (int)level, (int)batch, op, x + level * N, ct_bs, y, 0, out + level * N, ct_bs, nullptr,
                    c->d_primes, st);
        ++c->launches;
      }
    }
    check_launch();
  });
}
ck_status ck_hadd(ck_context* ctx, uint32_t level, uint32_t batch, const uint32_t* x, const uint32_t* y,
                  uint32_t* out, ck_stream stream) {
  return ct_ew(ctx, 0, level, batch, x, y, false, false, out, stream);
}
ck_status ck_padd(ck_context* ctx, uint32_t level, uint32_t batch, const uint32_t* ct, const uint32_t* pt,
                  uint32_t* out, ck_stream stream) {
  return ct_ew(ctx, 0, level, batch, ct, pt, true, true, out, stream);
}
ck_status ck_pmult(ck_context* ctx, uint32_t level, uint32_t batch, const uint32_t* ct, const uint32_t* pt,
                   uint32_t* out, ck_stream stream) {
  return ct_ew(ctx, 2, level, batch, ct, pt, true, false, out, stream);
}

ck_status ck_encode(ck_context* ctx, const double* slots_dev, uint32_t count, double scale_log2, uint32_t level,
                    int p_extend, uint32_t* out_dev, ck_stream stream) {
  CK_RANGE("ck_encode");
  ck_status st0 = guard([&] {
    Context* c = C(ctx);
    check_level(c, level);
    check_ptr(out_dev);
    if (count > c->n / 2) throw InvalidArgument("too many slots");  // ckks.cpp:281-285
    if (count && !slots_dev) throw InvalidArgument("null slot pointer");
    if (!(scale_log2 <= 60.0)) throw InvalidArgument("scale out of the representable range");
    c->enc_tables();
    cudaStream_t st = S(stream);
    const uint32_t rows = level + (p_extend ? c->alpha : 0);
    const size_t N = c->n;
    char* base = static_cast<char*>(c->scratch_get(2 * N * sizeof(double2) + 4 * rows + 16, st));
    double2* a = reinterpret_cast<double2*>(base);
    uint32_t* rq = reinterpret_cast<uint32_t*>(base + 2 * N * sizeof(double2));
    std::vector<uint32_t> hq(rows);
    for (uint32_t i = 0; i < rows; ++i) hq[i] = c->q(c->gidx(level, i));
    CK_CUDA(cudaMemcpyAsync(rq, hq.data(), 4 * rows, cudaMemcpyHostToDevice, st));
    enc_scatter((int)N, reinterpret_cast<const double2*>(slots_dev), (int)count, c->d_jidx, a, st);
    fft_pow2_dev((int)c->logn, a, a + N, c->d_fft_inv, st);  // IDFT (1/n folded into enc_round)
    // the reference's scale: powl(2.0L, (long double)log2_rational(scale)) (ckks.cpp:297-299),
    // same glibc / x87 on the host; its 64-bit significand and exponent go to the kernel
    const long double scale_v = std::pow(2.0L, static_cast<long double>(scale_log2));
    int sexp = 0;
    const long double sfrac = std::frexp(scale_v, &sexp);  // [0.5, 1)
    const unsigned long long smant = static_cast<unsigned long long>(std::ldexp(sfrac, 64));
    enc_round((int)N, a + N, c->d_twist_enc, smant, sexp - 64, (int)rows, rq, out_dev, st);
    CK_CUDA(cudaStreamSynchronize(st));  // hq is pageable host memory
    c->launches += 4 + (c->logn > 12 ? c->logn - 12 : 0);
  });
  if (st0 != CK_OK) return st0;
  // coefficient (plain) -> evaluation (Montgomery), as ntt_forward does (ckks.cpp:316)
  Context* c = C(ctx);
  std::vector<uint32_t> g(level + (p_extend ? c->alpha : 0));
  for (uint32_t i = 0; i < g.size(); ++i) g[i] = c->gidx(level, i);
  return ck_ntt_forward(ctx, out_dev, (uint32_t)g.size(), g.data(), stream);
}

static ck_status decode_impl(ck_context* ctx, const uint32_t* pt_dev, uint32_t level, double scale_log2,
                             const RatScale& rs, double* slots_dev, ck_stream stream);

ck_status ck_decode(ck_context* ctx, const uint32_t* pt_dev, uint32_t level, double scale_log2, double* slots_dev,
                    ck_stream stream) {
  return decode_impl(ctx, pt_dev, level, scale_log2, RatScale{}, slots_dev, stream);
}

ck_status ck_decode_rational(ck_context* ctx, const uint32_t* pt_dev, uint32_t level, double scale_log2,
                             const uint32_t* scale_num, uint32_t num_words, const uint32_t* scale_den,
                             uint32_t den_words, double* slots_dev, ck_stream stream) {
  RatScale rs;
  const ck_status st = guard([&] {
    check_ptr(scale_num);
    check_ptr(scale_den);
    if (num_words == 0 || den_words == 0 || num_words > (uint32_t)kMaxRat || den_words > (uint32_t)kMaxRat)
      throw InvalidArgument("decode: scale numerator / denominator must have 1..8 32-bit words");
    bool nz = false, dz = false;
    for (uint32_t i = 0; i < num_words; ++i) nz |= (rs.num[i] = scale_num[i]) != 0;
    for (uint32_t i = 0; i < den_words; ++i) dz |= (rs.den[i] = scale_den[i]) != 0;
    if (!nz || !dz) throw InvalidArgument("decode: scale must be a positive rational");
    rs.nnum = (int)num_words;
    rs.nden = (int)den_words;
  });
  if (st != CK_OK) return st;
  return decode_impl(ctx, pt_dev, level, scale_log2, rs, slots_dev, stream);
}

static ck_status decode_impl(ck_context* ctx, const uint32_t* pt_dev, uint32_t level, double scale_log2,
                             const RatScale& rs, double* slots_dev, ck_stream stream) {
  return guard([&] {
    CK_RANGE("ck_decode");
    Context* c = C(ctx);
    check_level(c, level);
    check_ptr(pt_dev);
    check_ptr(slots_dev);
    // minimal Q prefix whose product dominates the scale with 40 bits of headroom (ckks.cpp:325-332)
    const double need_bits = scale_log2 + 40.0;
    uint32_t cnt = 1;
    double bits = std::log2(static_cast<double>(c->q(0)));
    while (cnt < level && bits < need_bits) {
      bits += std::log2(static_cast<double>(c->q(cnt)));
      ++cnt;
    }
    c->enc_tables();
    cudaStream_t st = S(stream);
    const size_t N = c->n;
    char* base = static_cast<char*>(c->scratch_get(2 * N * sizeof(double2) + 4 * N * cnt, st));
    double2* a = reinterpret_cast<double2*>(base);
    uint32_t* rows = reinterpret_cast<uint32_t*>(base + 2 * N * sizeof(double2));
    CK_CUDA(cudaMemcpyAsync(rows, pt_dev, 4 * N * cnt, cudaMemcpyDeviceToDevice, st));
    std::vector<uint32_t> g(cnt);
    for (uint32_t i = 0; i < cnt; ++i) g[i] = i;
    const ck_status si = ck_intt_inverse(ctx, rows, cnt, g.data(), nullptr, stream);
    if (si != CK_OK) throw std::runtime_error(ck_last_error());
    dec_crt((int)N, rows, c->crt_const(cnt), c->d_twist_dec, std::exp2(-scale_log2), a, st, rs);
    fft_pow2_dev((int)c->logn, a, a + N, c->d_fft_fwd, st);
    dec_gather((int)N, a + N, c->d_jidx, reinterpret_cast<double2*>(slots_dev), st);
    c->launches += 3 + (c->logn > 12 ? c->logn - 12 : 0);
  });
}

ck_status ck_decrypt(ck_context* ctx, uint32_t level, uint32_t batch, const uint32_t* ct, const uint32_t* s,
                     uint32_t* out, ck_stream stream) {
  return guard([&] {
    CK_RANGE("ck_decrypt");  // ckks.cpp:541-553
    Context* c = C(ctx);
    check_level(c, level);
    check_ptr(ct);
    check_ptr(s);
    check_ptr(out);
    crypt((int)c->n, (int)level, (int)batch, 0, ct, 2ull * level * c->n, s, nullptr, nullptr, nullptr, out,
          (uint64_t)level * c->n, c->d_primes, S(stream));
    ++c->launches;
    check_launch();
  });
}
ck_status ck_encrypt_sk(ck_context* ctx, uint32_t level, const uint32_t* pt, const uint32_t* a, const uint32_t* e,
                        const uint32_t* s, uint32_t* out, ck_stream stream) {
  return guard([&] {
    CK_RANGE("ck_encrypt_sk");  // ckks.cpp:497-516, randomness (a uniform, e Gaussian in eval form) supplied
    Context* c = C(ctx);
    check_level(c, level);
    for (const void* p : {(const void*)pt, (const void*)a, (const void*)e, (const void*)s, (const void*)out})
      check_ptr(p);
    crypt((int)c->n, (int)level, 1, 1, pt, 0, a, e, s, nullptr, out, 0, c->d_primes, S(stream));
    ++c->launches;
    check_launch();
  });
}
ck_status ck_encrypt_pk(ck_context* ctx, uint32_t level, const uint32_t* pt, const uint32_t* v, const uint32_t* e0,
                        const uint32_t* e1, const uint32_t* pk, uint32_t* out, ck_stream stream) {
  return guard([&] {
    CK_RANGE("ck_encrypt_pk");  // ckks.cpp:518-539, randomness (v ternary, e0 e1 Gaussian in eval form) supplied
    Context* c = C(ctx);
    check_level(c, level);
    for (const void* p : {(const void*)pt, (const void*)v, (const void*)e0, (const void*)e1, (const void*)pk,
                          (const void*)out})
      check_ptr(p);
    crypt((int)c->n, (int)level, 1, 2, pt, 0, v, e0, e1, pk, out, 0, c->d_primes, S(stream));
    ++c->launches;
    check_launch();
  });
}
ck_status ck_evk_digit(ck_context* ctx, const uint32_t* s_src, const uint32_t* s_dst, const uint32_t* a,
                       const uint32_t* e, const uint32_t* g_mont, int square_src, uint32_t* out_b, ck_stream stream) {
  return guard([&] {  // evk_gen digit (ckks.cpp:459-474) over the full L + alpha rows
    Context* c = C(ctx);
    for (const void* p : {(const void*)s_src, (const void*)s_dst, (const void*)a, (const void*)e, (const void*)out_b})
      check_ptr(p);
    if (!g_mont) throw InvalidArgument("null gadget constants");
    const uint32_t rows = c->L + c->alpha;
    char* base = static_cast<char*>(c->scratch_get(6 * rows + 16, S(stream)));
    uint32_t* d_g = reinterpret_cast<uint32_t*>(base);
    uint16_t* d_rp = reinterpret_cast<uint16_t*>(base + 4 * rows);
    std::vector<uint16_t> rp(rows);
    for (uint32_t i = 0; i < rows; ++i) rp[i] = (uint16_t)i;
    CK_CUDA(cudaMemcpyAsync(d_g, g_mont, 4 * rows, cudaMemcpyHostToDevice, S(stream)));
    CK_CUDA(cudaMemcpyAsync(d_rp, rp.data(), 2 * rows, cudaMemcpyHostToDevice, S(stream)));
    evk_digit((int)c->n, (int)rows, s_src, s_dst, a, e, d_g, d_rp, square_src, c->d_primes, out_b, S(stream));
    CK_CUDA(cudaStreamSynchronize(S(stream)));  // host arrays are pageable
    ++c->launches;
    check_launch();
  });
}

ck_status ck_coeffs_to_eval(ck_context* ctx, const int64_t* coeffs, uint32_t level, uint32_t p_rows, uint32_t* out,
                            ck_stream stream) {
  ck_status st0 = guard([&] {  // ckks.cpp:366-380: reduce mod every prime, then ntt_forward
    Context* c = C(ctx);
    check_level(c, level);
    check_ptr(coeffs);
    check_ptr(out);
    if (p_rows > c->alpha) throw InvalidArgument("too many P rows");
    const uint32_t rows = level + p_rows;
    std::vector<uint16_t> rp(rows);
    for (uint32_t i = 0; i < rows; ++i) rp[i] = (uint16_t)c->gidx(level, i);
    uint16_t* d_rp = static_cast<uint16_t*>(c->scratch_get(2 * rows + 16, S(stream)));
    CK_CUDA(cudaMemcpyAsync(d_rp, rp.data(), 2 * rows, cudaMemcpyHostToDevice, S(stream)));
    reduce_coeffs((int)c->n, (int)rows, reinterpret_cast<const long long*>(coeffs), d_rp, c->d_primes, out, S(stream));
    CK_CUDA(cudaStreamSynchronize(S(stream)));  // rp is pageable host memory
    ++c->launches;
    check_launch();
  });
  if (st0 != CK_OK) return st0;
  Context* c = C(ctx);
  std::vector<uint32_t> g(level + p_rows);
  for (uint32_t i = 0; i < g.size(); ++i) g[i] = c->gidx(level, i);
  return ck_ntt_forward(ctx, out, (uint32_t)g.size(), g.data(), stream);
}

ck_status ck_hoisted_rotations(ck_context* ctx, uint32_t level, const uint32_t* ct, uint32_t count,
                               const int64_t* rots, const uint32_t* const* evks, uint32_t* out, ck_stream stream) {
  return guard([&] {
    CK_RANGE("ck_hoisted_rotations");
    Context* c = C(ctx);
    check_level(c, level);
    check_ptr(ct);
    check_ptr(out);
    if (count && (!rots || !evks)) throw InvalidArgument("rotation/key count mismatch");
    const uint64_t N = c->n, ct_w = 2ull * level * N;
    const uint32_t D = c->digits(level), rows = level + c->alpha;
    const SwitchPlan& pl = c->switch_plan(0, level, 2);
    const size_t is_w = level * N, ext_w = (size_t)D * rows * N, v_w = 2ull * rows * N, ts_w = 2ull * pl.sc * N,
                 o_w = 2ull * level * N;
    uint32_t* base = static_cast<uint32_t*>(c->scratch_get((is_w + ext_w + v_w + ts_w + o_w) * 4, S(stream)));
    uint32_t *is = base, *ext = is + is_w, *v = ext + ext_w, *ts = v + v_w, *o = ts + ts_w;
    cudaStream_t st = S(stream);
    const uint32_t* a = ct + level * N;
    c->mod_up(level, 1, a, 0, is, ext, st);  // shared across all rotations
    for (uint32_t i = 0; i < count; ++i) {
      uint32_t* dst = out + i * ct_w;
      if (rots[i] == 0) {
        CK_CUDA(cudaMemcpyAsync(dst, ct, ct_w * 4, cudaMemcpyDeviceToDevice, st));
        continue;
      }
      if (!evks[i]) throw InvalidArgument("missing rotation key");
      c->key_mult_v(level, 1, ext, a, 0, evks[i], nullptr, 0, v, st);
      c->drop_divide(pl, 1, v, 0, ts, o, false, st);
      hrot_tail((int)N, (int)level, 1, v, 0, rows * N, o, 0, level * N, ct, 0, pl.consts.at<uint32_t>(0),
                c->rotation_map(rots[i]), dst, 0, c->d_primes, st,
                c->tail_gather ? nullptr : c->rotation_dest(rots[i]));
      ++c->launches;
      c->counters[1] += 1;
    }
    check_launch();
  });
}

ck_status ck_hoisted_rotate_accumulate(ck_context* ctx, uint32_t level, const uint32_t* ct, uint32_t count,
                                       const int64_t* rots, const uint32_t* const* pts,
                                       const uint32_t* const* evks, uint32_t* out, ck_stream stream) {
  return guard([&] {
    CK_RANGE("ck_hoisted_rotate_accumulate");
    Context* c = C(ctx);
    check_level(c, level);
    check_ptr(ct);
    check_ptr(out);
    if (count == 0 || !rots || !pts || !evks) throw InvalidArgument("rotation/plaintext/key count mismatch");
    const uint64_t N = c->n;
    const uint32_t D = c->digits(level), rows = level + c->alpha;
    const SwitchPlan& pl = c->switch_plan(0, level, 2);
    const size_t is_w = level * N, ext_w = (size_t)D * rows * N, v_w = 2ull * rows * N, ts_w = 2ull * pl.sc * N,
                 acc_w = 2ull * rows * N, o_w = 2ull * level * N;
    uint32_t* base = static_cast<uint32_t*>(c->scratch_get((is_w + ext_w + v_w + ts_w + acc_w + o_w) * 4, S(stream)));
    uint32_t *is = base, *ext = is + is_w, *v = ext + ext_w, *ts = v + v_w, *acc = ts + ts_w, *o = acc + acc_w;
    cudaStream_t st = S(stream);
    const uint32_t* b = ct;
    const uint32_t* a = ct + level * N;
    std::vector<uint16_t> rp(rows);
    for (uint32_t i = 0; i < rows; ++i) rp[i] = (uint16_t)c->gidx(level, i);
    // row->prime map for the (level + alpha)-row accumulators
    auto& blob = c->row_primes[level];
    if (!blob) {
      blob = std::make_unique<Blob>();
      blob->add(rp);
      blob->upload();
    }
    const uint16_t* d_rp = blob->at<uint16_t>(0);
    CK_CUDA(cudaMemsetAsync(acc, 0, acc_w * 4, st));
    CK_CUDA(cudaMemsetAsync(out, 0, o_w * 4, st));
    c->mod_up(level, 1, a, 0, is, ext, st);
    bool used_pq = false;
    for (uint32_t i = 0; i < count; ++i) {
      check_ptr(pts[i]);
      if (rots[i] == 0) {  // ckks.cpp:977-982
        addmul((int)N, (int)level, 1, out, 0, b, 0, pts[i], 0, nullptr, c->d_primes, st);
        addmul((int)N, (int)level, 1, out + level * N, 0, a, 0, pts[i], 0, nullptr, c->d_primes, st);
        c->launches += 2;
        continue;
      }
      if (!evks[i]) throw InvalidArgument("rotation key mismatch");
      const uint32_t* map = c->rotation_map(rots[i]);
      c->key_mult_v(level, 1, ext, a, 0, evks[i], nullptr, 0, v, st);
      addmul_permuted((int)N, (int)rows, 1, acc, 0, v, 0, pts[i], 0, map, d_rp, c->d_primes, st);
      addmul_permuted((int)N, (int)rows, 1, acc + rows * N, 0, v + rows * N, 0, pts[i], 0, map, d_rp, c->d_primes,
                      st);
      addmul_permuted((int)N, (int)level, 1, out, 0, b, 0, pts[i], 0, map, nullptr, c->d_primes, st);
      c->launches += 3;
      used_pq = true;
    }
    if (used_pq) {
      c->drop_divide(pl, 1, acc, 0, ts, o, true, st);
      elementwise((int)N, (int)(2 * level), 1, 0, out, 0, o, 0, out, 0, nullptr, c->d_primes, st, (int)level);
      ++c->launches;
      c->counters[1] += 1;
    }
    check_launch();
  });
}

/* ---- limb sharding ------------------------------------------------------ */
static Shard* SH(ck_shard* s) {
  if (!s) throw InvalidArgument("null shard");
  return reinterpret_cast<Shard*>(s);
}
static void check_kind(int kind) {
  if (kind < 0 || kind > 2) throw InvalidArgument("switch kind must be 0 (mod_down), 1 (rescale) or 2 (merged)");
}

ck_status ck_shard_create(ck_context* ctx, uint32_t world, uint32_t rank, ck_shard** out) {
  return guard([&] {
    Context* c = C(ctx);
    if (!out) throw InvalidArgument("null argument");
    if (world == 0 || rank >= world) throw InvalidArgument("rank out of range");
    if (world > c->L) throw InvalidArgument("more shards than Q primes");
    auto s = std::make_unique<Shard>();
    s->c = c;
    s->G = world;
    s->s = rank;
    s->qlo = s->q_lo(rank);
    s->qhi = s->q_hi(rank);
    s->plo = s->p_lo(rank);
    s->phi = s->p_hi(rank);
    for (uint32_t t = 0; t < world; ++t) {
      s->qmax = std::max(s->qmax, s->q_hi(t) - s->q_lo(t));
      s->pmax = std::max(s->pmax, s->p_hi(t) - s->p_lo(t));
    }
    *out = reinterpret_cast<ck_shard*>(s.release());
  });
}
ck_status ck_shard_destroy(ck_shard* sh) {
  return guard([&] { delete SH(sh); });
}
ck_status ck_shard_exchange_buffer(ck_shard* sh, void** base, uint64_t* bytes) {
  return guard([&] {
    if (!base) throw InvalidArgument("null argument");
    *base = SH(sh)->exchange_buffer(bytes);
  });
}
ck_status ck_shard_set_peers(ck_shard* sh, const uint64_t* bases, uint32_t world) {
  return guard([&] {
    check_ptr(bases);
    SH(sh)->set_peers(bases, world);
  });
}
ck_status ck_shard_set_timeout(ck_shard* sh, uint64_t timeout_ns) {
  return guard([&] { SH(sh)->timeout_ns = timeout_ns; });
}
ck_status ck_shard_peer_error(ck_shard* sh, uint32_t* err) {
  return guard([&] {
    if (!err) throw InvalidArgument("null argument");
    *err = SH(sh)->peer_error();
  });
}
ck_status ck_ipc_get_handle(const void* base, unsigned char handle[64]) {
  return guard([&] {
    if (!base || !handle) throw InvalidArgument("null argument");
    cudaIpcMemHandle_t h;
    CK_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(base)));
    static_assert(sizeof(h) == 64, "IPC handle size");
    std::memcpy(handle, &h, 64);
  });
}
ck_status ck_ipc_open_handle(const unsigned char handle[64], void** base) {
  return guard([&] {
    if (!base || !handle) throw InvalidArgument("null argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    CK_CUDA(cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess));
  });
}
ck_status ck_ipc_close(void* base) {
  return guard([&] {
    if (!base) throw InvalidArgument("null argument");
    CK_CUDA(cudaIpcCloseMemHandle(base));
  });
}
ck_status ck_shard_layout(const ck_shard* sh, uint32_t level, uint32_t out[8]) {
  return guard([&] {
    const Shard* s = reinterpret_cast<const Shard*>(sh);
    if (!s || !out) throw InvalidArgument("null argument");
    check_level(s->c, level);
    out[0] = s->qlo;
    out[1] = s->qhi;
    out[2] = s->plo;
    out[3] = s->phi;
    out[4] = s->lq(level);
    out[5] = s->qmax;
    out[6] = s->pmax;
    out[7] = s->G;
  });
}
ck_status ck_shard_modup_begin(ck_shard* sh, uint32_t level, const uint32_t* d, uint32_t* send, ck_stream stream) {
  return guard([&] {
    CK_RANGE("ck_shard_modup_begin");
    Shard* s = SH(sh);
    check_level(s->c, level);
    if (s->lq(level)) {
      check_ptr(d);
      if (!s->peer_mode()) check_ptr(send);
    }
    s->modup_begin(level, d, send, S(stream));
    check_launch();
  });
}
ck_status ck_shard_modup_keymult(ck_shard* sh, uint32_t level, const uint32_t* recv, const uint32_t* d,
                                 const uint32_t* evk, const uint32_t* fold, uint32_t* v, ck_stream stream) {
  return guard([&] {
    CK_RANGE("ck_shard_modup_keymult");
    Shard* s = SH(sh);
    check_level(s->c, level);
    if (!s->peer_mode()) check_ptr(recv);
    check_ptr(evk);
    if (s->up_plan(level).rows == 0) {  // nothing owned at this level (a peer rank still waits: buffer reuse)
      if (!recv) s->peer_wait(0, s->up_tab.at<uint64_t>(0), (int)s->c->L, S(stream));
      return;
    }
    check_ptr(v);
    if (s->lq(level)) check_ptr(d);
    s->modup_keymult(level, recv, d, evk, fold, v, S(stream));
    check_launch();
  });
}
ck_status ck_shard_switch_begin(ck_shard* sh, int kind, uint32_t level, const uint32_t* v, uint32_t* send,
                                ck_stream stream) {
  return guard([&] {
    CK_RANGE("ck_shard_switch_begin");
    Shard* s = SH(sh);
    check_kind(kind);
    check_level(s->c, level, kind == 0 ? 1 : 4);
    if (!s->peer_mode()) check_ptr(send);
    if (s->down_plan(kind, level).own_sc) check_ptr(v);
    s->switch_begin(kind, level, v, send, S(stream));
    check_launch();
  });
}
ck_status ck_shard_switch_end(ck_shard* sh, int kind, uint32_t level, const uint32_t* recv, const uint32_t* v,
                              const uint32_t* addend, uint32_t add_mask, int32_t rotate, int64_t r, uint32_t* out,
                              ck_stream stream) {
  return guard([&] {
    CK_RANGE("ck_shard_switch_end");
    Shard* s = SH(sh);
    check_kind(kind);
    check_level(s->c, level, kind == 0 ? 1 : 4);
    if (!s->peer_mode()) check_ptr(recv);
    const uint32_t lqo = s->down_plan(kind, level).lqo;
    if (lqo) {
      check_ptr(v);
      check_ptr(out);
    }
    const uint32_t* map = rotate && lqo ? s->c->rotation_map(r) : nullptr;
    s->switch_end(kind, level, recv, v, addend, add_mask, map, out, S(stream));
    check_launch();
  });
}
ck_status ck_shard_tensor(ck_shard* sh, uint32_t level, const uint32_t* x, const uint32_t* y, uint32_t* d01,
                          uint32_t* d2, ck_stream stream) {
  return guard([&] {
    CK_RANGE("ck_shard_tensor");
    Shard* s = SH(sh);
    check_level(s->c, level, 4);
    const uint32_t lq = s->lq(level);
    if (!lq) return;
    check_ptr(x);
    check_ptr(y);
    check_ptr(d01);
    check_ptr(d2);
    const uint64_t N = s->c->n;
    cudaStream_t st = S(stream);
    {
      Context::ProfScope ps(s->c, 4, 4.0 * N * lq * 7, 1, st);
      tensor((int)N, (int)lq, 1, x, y, 2ull * lq * N, d01, 2ull * lq * N, d2, lq * N, s->c->d_primes + s->qlo, st);
    }
    ++s->c->launches;
    check_launch();
  });
}

}  // extern "C"
