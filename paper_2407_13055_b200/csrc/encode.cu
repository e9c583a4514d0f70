// CKKS encode / decode on the GPU, restating
// ckks.cpp:278-362 of the reference:
//
//   encode: slots -> a[jidx[t]] = z_t, a[n-1-jidx[t]] = conj(z_t)       (scatter)
//           a = IDFT(a) by fft_pow2(invert) (ckks.cpp:63-87)             (FFT)
//           m_k = llround(Re(a_k * psi^-k) * scale)  mod every q_i       (round + reduce)
//           -> forward NTT (entry merge) in the caller                   (plaintext rows)
//   decode: INTT of the first c rows (caller) -> CRT lift of c <= 16 primes
//           (multi-precision limbs), centre, / scale -> a_k = coeff * (cos, sin)(pi k / n)
//           -> fft_pow2(forward) -> out[t] = a[jidx[t]]
//
// The FFT reproduces the reference's radix-2 iterative transform operation by
// operation: the same bit-reversed order, the same per-stage twiddle values
// (the host builds them with the reference's recurrence w *= wl in double),
// and complex products / sums rounded exactly as libstdc++ evaluates them
// (x86-64, no FMA): every product and sum below uses the _rn intrinsics so the
// compiler cannot contract them into FMAs; the final scaling and rounding
// replays the reference's 80-bit long double arithmetic on integers
// (llroundl_x87), so the encoded residues are bit-identical to the
// reference's for every scale.
#include <algorithm>

#include "ck_common.cuh"
#include "ck_kernels.h"

namespace ck {
namespace {

constexpr int kFftBlock = 4096;  // elements per shared-memory FFT block (64 KB)
constexpr int kFftThreads = 512;

__device__ __forceinline__ double2 cmul(double2 a, double2 w) {  // (a.x w.x - a.y w.y, a.x w.y + a.y w.x)
  return make_double2(__dsub_rn(__dmul_rn(a.x, w.x), __dmul_rn(a.y, w.y)),
                      __dadd_rn(__dmul_rn(a.x, w.y), __dmul_rn(a.y, w.x)));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y)); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y)); }

__device__ __forceinline__ uint32_t brev(uint32_t x, int bits) { return __brev(x) >> (32 - bits); }

// stages len = 2 .. B of one B-element block, input gathered in bit-reversed order
__global__ void __launch_bounds__(kFftThreads) k_fft_first(const double2* __restrict__ src, double2* __restrict__ dst,
                                                           const double2* __restrict__ tw, int logn, int B) {
  extern __shared__ double2 sa[];
  const int base = blockIdx.x * B;
  for (int i = threadIdx.x; i < B; i += blockDim.x) sa[i] = src[brev((uint32_t)(base + i), logn)];
  __syncthreads();
  for (int len = 2; len <= B; len <<= 1) {
    const int half = len >> 1;
    const double2* w = tw + (half - 1);
    for (int b = threadIdx.x; b < B / 2; b += blockDim.x) {
      const int i = (b / half) * len, j = b % half;
      const double2 u = sa[i + j];
      const double2 v = cmul(sa[i + j + half], w[j]);
      sa[i + j] = cadd(u, v);
      sa[i + j + half] = csub(u, v);
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < B; i += blockDim.x) dst[base + i] = sa[i];
}

// one radix-2 stage of length len, in place
__global__ void k_fft_stage(double2* __restrict__ a, const double2* __restrict__ tw, int n, int len) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n / 2) return;
  const int half = len >> 1;
  const int i = (b / half) * len, j = b % half;
  const double2 u = a[i + j];
  const double2 v = cmul(a[i + j + half], tw[(half - 1) + j]);
  a[i + j] = cadd(u, v);
  a[i + j + half] = csub(u, v);
}

__global__ void k_enc_scatter(int n, const double2* __restrict__ slots, int count, const uint32_t* __restrict__ jidx,
                              double2* __restrict__ a) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  const double2 z = slots[t];
  const uint32_t j = jidx[t];
  a[j] = z;
  a[n - 1 - j] = make_double2(z.x, -z.y);
}

// llroundl(c * S) exactly as the reference evaluates it on x86-64: c a double,
// S = ms * 2^es the 64-bit-significand long double scale (powl(2.0L, log2),
// ckks.cpp:297-305), the product rounded once to a 64-bit significand
// (x87 extended, round to nearest even), then to an integer (half away from
// zero).  Done on integers: c = mc * 2^ec (53-bit mc), P = mc * ms (<= 117
// bits, exact), round P to 64 significant bits, shift by ec + es.
__device__ __forceinline__ long long llroundl_x87(double c, unsigned long long ms, int es) {
  if (c == 0.0) return 0;
  int e;
  const double f = frexp(fabs(c), &e);                                  // |c| = f 2^e, f in [0.5, 1)
  const unsigned long long mc = (unsigned long long)ldexp(f, 53);        // exact 53-bit integer
  unsigned __int128 P = (unsigned __int128)mc * ms;
  int E = e - 53 + es;
  const int L = 128 - (int)((P >> 64) ? __clzll((unsigned long long)(P >> 64)) : 64 + __clzll((unsigned long long)P));
  if (L > 64) {  // round to 64 significant bits, nearest even
    const int d = L - 64;
    const unsigned __int128 half = (unsigned __int128)1 << (d - 1), mask = ((unsigned __int128)1 << d) - 1;
    const unsigned __int128 rem = P & mask;
    P >>= d;
    if (rem > half || (rem == half && (P & 1))) P += 1;
    E += d;
  }
  unsigned long long mag;
  if (E >= 0) {
    mag = (unsigned long long)(P << E);  // |c S| < 2^63 for the reference's scale bound
  } else {
    const int sft = -E;
    if (sft >= 127) mag = 0;
    else mag = (unsigned long long)((P + ((unsigned __int128)1 << (sft - 1))) >> sft);  // half away from zero
  }
  return c < 0 ? -(long long)mag : (long long)mag;
}

// m_k = llroundl((Re(a_k tw_k) / n) * S), then canonical m mod q for every row
__global__ void k_enc_round(int n, const double2* __restrict__ a, const double2* __restrict__ twist, double inv_n,
                            unsigned long long ms, int es, int rows, const uint32_t* __restrict__ row_q,
                            uint32_t* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double2 x = a[k], t = twist[k];
  const double re = __dsub_rn(__dmul_rn(x.x, t.x), __dmul_rn(x.y, t.y));
  const long long m = llroundl_x87(__dmul_rn(re, inv_n), ms, es);
  for (int i = 0; i < rows; ++i) {
    const long long q = row_q[i];
    long long r = m % q;  // correct() of modarith.hpp:46-50
    if (r < 0) r += q;
    out[(size_t)i * n + k] = (uint32_t)r;
  }
}

// correctly rounded conversion of a little-endian multi-limb magnitude to double
__device__ __forceinline__ double limbs_to_double(const uint32_t* v, int nl) {
  int top = nl - 1;
  while (top >= 0 && v[top] == 0) --top;
  if (top < 0) return 0.0;
  if (top <= 1) return __ull2double_rn(((uint64_t)(top == 1 ? v[1] : 0) << 32) | v[0]);
  // top 64 bits starting at the highest set bit, plus a sticky bit for everything below
  const int lz = __clz(v[top]);
  const int hb = 32 * top + 31 - lz;  // index of the highest set bit
  const int lo = hb - 63;             // bit index of the 64-bit window's lsb (>= 1 here)
  uint64_t w = 0;
  for (int i = 63; i >= 0; --i) {
    const int b = lo + i;
    w = (w << 1) | ((v[b >> 5] >> (b & 31)) & 1u);
  }
  bool sticky = false;
  for (int b = 0; b < lo && !sticky; ++b) sticky = (v[b >> 5] >> (b & 31)) & 1u;
  if (sticky) w |= 1;  // below the 53-bit rounding point: only breaks ties
  return ldexp(__ull2double_rn(w), lo);
}

// ---- correctly rounded |v| * den / num (the reference's
// static_cast<double>(Rational(v) / scale), ckks.cpp:353, with the round-to-
// nearest-even conversion of the oracle's Boost shim)
constexpr int kMaxA = kMaxCrt + 1 + kMaxRat + 1;

__device__ __forceinline__ int bitlen_w(const uint32_t* x, int n) {
  for (int i = n - 1; i >= 0; --i)
    if (x[i]) return 32 * i + 32 - __clz(x[i]);
  return 0;
}

// q = floor(u / v), returns whether the remainder is nonzero; u has nu words
// (destroyed), v has nv >= 1 words with v[nv-1] != 0, the quotient fits in 64
// bits (Knuth, TAOCP 4.3.1 algorithm D, 32-bit digits)
__device__ uint64_t divmod_small_q(uint32_t* u, int nu, const uint32_t* v, int nv, bool& rem_nz) {
  uint64_t q = 0;
  if (nv == 1) {
    uint64_t r = 0;
    for (int j = nu - 1; j >= 0; --j) {
      const uint64_t t = (r << 32) | u[j];
      const uint64_t d = t / v[0];
      r = t - d * v[0];
      if (j < 2) q |= d << (32 * j);
    }
    rem_nz = r != 0;
    return q;
  }
  const int sh = __clz(v[nv - 1]);
  uint32_t vn[kMaxRat], un[kMaxA + 1];
  for (int i = nv - 1; i > 0; --i) vn[i] = (v[i] << sh) | (sh ? (uint32_t)((uint64_t)v[i - 1] >> (32 - sh)) : 0u);
  vn[0] = v[0] << sh;
  un[nu] = sh ? (uint32_t)((uint64_t)u[nu - 1] >> (32 - sh)) : 0u;
  for (int i = nu - 1; i > 0; --i) un[i] = (u[i] << sh) | (sh ? (uint32_t)((uint64_t)u[i - 1] >> (32 - sh)) : 0u);
  un[0] = u[0] << sh;
  for (int j = nu - nv; j >= 0; --j) {
    const uint64_t top = ((uint64_t)un[j + nv] << 32) | un[j + nv - 1];
    uint64_t qhat = top / vn[nv - 1], rhat = top - qhat * vn[nv - 1];
    while (qhat >> 32 || qhat * vn[nv - 2] > ((rhat << 32) | un[j + nv - 2])) {
      --qhat;
      rhat += vn[nv - 1];
      if (rhat >> 32) break;
    }
    int64_t borrow = 0;
    uint64_t carry = 0;
    for (int i = 0; i < nv; ++i) {
      const uint64_t p = qhat * vn[i] + carry;
      carry = p >> 32;
      const int64_t t = (int64_t)un[i + j] - (int64_t)(uint32_t)p - borrow;
      un[i + j] = (uint32_t)t;
      borrow = t < 0;
    }
    const int64_t t = (int64_t)un[j + nv] - (int64_t)carry - borrow;
    un[j + nv] = (uint32_t)t;
    if (t < 0) {  // qhat one too large: add back
      --qhat;
      uint64_t c = 0;
      for (int i = 0; i < nv; ++i) {
        const uint64_t s2 = (uint64_t)un[i + j] + vn[i] + c;
        un[i + j] = (uint32_t)s2;
        c = s2 >> 32;
      }
      un[j + nv] += (uint32_t)c;
    }
    if (j < 2) q |= qhat << (32 * j);
  }
  rem_nz = false;
  for (int i = 0; i < nv; ++i) rem_nz |= un[i] != 0;
  return q;
}

__device__ double rat_to_double(const uint32_t* acc, int nl, const RatScale& rs) {
  uint32_t A[kMaxA];
  const int na = nl + rs.nden;
  for (int i = 0; i < na; ++i) A[i] = 0;
  for (int i = 0; i < nl; ++i) {  // A = |v| * den
    uint64_t carry = 0;
    for (int j = 0; j < rs.nden; ++j) {
      const uint64_t t = (uint64_t)acc[i] * rs.den[j] + A[i + j] + carry;
      A[i + j] = (uint32_t)t;
      carry = t >> 32;
    }
    A[i + rs.nden] = (uint32_t)carry;
  }
  const int nb = bitlen_w(A, na);
  if (nb == 0) return 0.0;
  const int db = bitlen_w(rs.num, rs.nnum);
  const int shift = 55 - (nb - db);  // the quotient gets 55 or 56 significant bits
  uint32_t U[kMaxA + 2];
  bool sticky = false;
  int nu;
  if (shift >= 0) {  // U = A << shift
    const int ws = shift >> 5, bs = shift & 31;
    nu = (nb + shift + 31) >> 5;
    for (int i = 0; i < nu; ++i) {
      const int src = i - ws;
      const uint32_t hi = (src >= 0 && src < na) ? A[src] : 0u;
      const uint32_t lo = (src - 1 >= 0 && src - 1 < na) ? A[src - 1] : 0u;
      U[i] = bs ? (hi << bs) | (lo >> (32 - bs)) : hi;
    }
  } else {  // U = A >> k, sticky = the bits shifted out (floor(floor(A / 2^k) / num) = floor(A / (num 2^k)))
    const int k = -shift, ws = k >> 5, bs = k & 31;
    for (int i = 0; i < ws && i < na; ++i) sticky |= A[i] != 0;
    if (bs && ws < na) sticky |= (A[ws] & ((1u << bs) - 1)) != 0;
    nu = (nb - k + 31) >> 5;
    for (int i = 0; i < nu; ++i) {
      const int src = i + ws;
      const uint32_t lo = src < na ? A[src] : 0u;
      const uint32_t hi = src + 1 < na ? A[src + 1] : 0u;
      U[i] = bs ? (lo >> bs) | (hi << (32 - bs)) : lo;
    }
  }
  int nv = rs.nnum;
  while (nv > 1 && rs.num[nv - 1] == 0) --nv;
  // U has db + 55 bits, so nu >= nv always (the quotient has 55 or 56 bits)
  bool rnz = false;
  const uint64_t qv = divmod_small_q(U, nu, rs.num, nv, rnz);
  sticky |= rnz;
  const int extra = (64 - __clzll(qv)) - 53;  // 2 or 3
  uint64_t mant = qv >> extra;
  const uint64_t rem = qv & ((1ull << extra) - 1), half = 1ull << (extra - 1);
  if (rem > half || (rem == half && (sticky || (mant & 1)))) ++mant;
  return ldexp((double)mant, extra - shift);
}

// CRT lift (multi-precision), centred, / scale, twisted: a_k = coeff (cos, sin)(pi k / n)
__global__ void k_dec_crt(int n, const uint32_t* __restrict__ rows, const CrtConst* __restrict__ ccp,
                          const double2* __restrict__ twist, double inv_scale, double2* __restrict__ a,
                          const __grid_constant__ RatScale rs) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const CrtConst& cc = *ccp;
  const int c = cc.c, nl = c + 1;
  uint32_t acc[kMaxCrt + 1];
  for (int j = 0; j < nl; ++j) acc[j] = 0;
  for (int i = 0; i < c; ++i) {  // acc += ((r_i y_i) mod q_i) * (M / q_i)
    const uint32_t r = rows[(size_t)i * n + k];
    const uint32_t t = (uint32_t)((uint64_t)r * cc.y[i] % cc.q[i]);
    uint64_t carry = 0;
    for (int j = 0; j < c; ++j) {
      const uint64_t s = (uint64_t)t * cc.mi[i][j] + acc[j] + carry;
      acc[j] = (uint32_t)s;
      carry = s >> 32;
    }
    for (int j = c; j < nl && carry; ++j) {
      const uint64_t s = (uint64_t)acc[j] + carry;
      acc[j] = (uint32_t)s;
      carry = s >> 32;
    }
  }
  auto geq_m = [&]() {  // acc >= M ?
    for (int j = nl - 1; j >= 0; --j) {
      const uint32_t mj = j < c ? cc.m[j] : 0u;
      if (acc[j] != mj) return acc[j] > mj;
    }
    return true;
  };
  while (geq_m()) {  // sum < c M: at most c subtractions
    int64_t borrow = 0;
    for (int j = 0; j < nl; ++j) {
      const int64_t s = (int64_t)acc[j] - (j < c ? cc.m[j] : 0u) - borrow;
      acc[j] = (uint32_t)s;
      borrow = s < 0;
    }
  }
  // centred lift (ckks.cpp:344): v > M / 2  <=>  2 v > M
  bool neg = false;
  {
    uint32_t carry = 0;
    int cmp = 0;  // compare 2 acc with M, from the top
    uint32_t twice[kMaxCrt + 1];
    for (int j = 0; j < nl; ++j) {
      twice[j] = (acc[j] << 1) | carry;
      carry = acc[j] >> 31;
    }
    for (int j = nl - 1; j >= 0 && cmp == 0; --j) {
      const uint32_t mj = j < c ? cc.m[j] : 0u;
      if (twice[j] != mj) cmp = twice[j] > mj ? 1 : -1;
    }
    neg = cmp > 0;
  }
  if (neg) {  // acc = M - acc
    int64_t borrow = 0;
    for (int j = 0; j < nl; ++j) {
      const int64_t s = (int64_t)(j < c ? cc.m[j] : 0u) - acc[j] - borrow;
      acc[j] = (uint32_t)s;
      borrow = s < 0;
    }
  }
  double coeff;
  if (rs.nnum > 0) {  // one correctly rounded division by the exact rational scale
    coeff = rat_to_double(acc, nl, rs);
    if (neg) coeff = -coeff;
  } else {  // |v| rounded once, times 2^-log2(scale): exact for power-of-two scales
    coeff = limbs_to_double(acc, nl);
    if (neg) coeff = -coeff;
    coeff = __dmul_rn(coeff, inv_scale);
  }
  const double2 tw = twist[k];
  a[k] = make_double2(__dmul_rn(coeff, tw.x), __dmul_rn(coeff, tw.y));
}

__global__ void k_dec_gather(int n, const double2* __restrict__ a, const uint32_t* __restrict__ jidx,
                             double2* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n / 2) out[t] = a[jidx[t]];
}

inline int cdiv(int a, int b) { return (a + b - 1) / b; }

}  // namespace

void fft_pow2_dev(int logn, const double2* src, double2* dst, const double2* tw, cudaStream_t st) {
  const int n = 1 << logn;
  const int B = std::min(n, kFftBlock);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_fft_first, cudaFuncAttributeMaxDynamicSharedMemorySize, kFftBlock * (int)sizeof(double2));
    attr = true;
  }
  k_fft_first<<<n / B, std::min(kFftThreads, std::max(32, B / 2)), B * sizeof(double2), st>>>(src, dst, tw, logn, B);
  for (int len = 2 * B; len <= n; len <<= 1) k_fft_stage<<<cdiv(n / 2, 256), 256, 0, st>>>(dst, tw, n, len);
}

void enc_scatter(int n, const double2* slots, int count, const uint32_t* jidx, double2* a, cudaStream_t st) {
  cudaMemsetAsync(a, 0, sizeof(double2) * n, st);
  if (count) k_enc_scatter<<<cdiv(count, 256), 256, 0, st>>>(n, slots, count, jidx, a);
}

void enc_round(int n, const double2* a, const double2* twist, unsigned long long scale_mant, int scale_exp, int rows,
               const uint32_t* row_q, uint32_t* out, cudaStream_t st) {
  k_enc_round<<<cdiv(n, 256), 256, 0, st>>>(n, a, twist, 1.0 / n, scale_mant, scale_exp, rows, row_q, out);
}

void dec_crt(int n, const uint32_t* rows, const CrtConst* cc_dev, const double2* twist, double inv_scale, double2* a,
             cudaStream_t st, const RatScale& rs) {
  k_dec_crt<<<cdiv(n, 128), 128, 0, st>>>(n, rows, cc_dev, twist, inv_scale, a, rs);
}

void dec_gather(int n, const double2* a, const uint32_t* jidx, double2* out, cudaStream_t st) {
  k_dec_gather<<<cdiv(n / 2, 256), 256, 0, st>>>(n, a, jidx, out);
}

}  // namespace ck
