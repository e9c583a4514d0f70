// Element-wise, base-conversion and key-switching kernels for sm_100a.
//
// All of these are HBM-bound integer kernels: every thread owns 4 adjacent
// coefficients (one 128-bit load/store per row), grids cover (columns, rows,
// batch), and per-row constants come from small device tables.  References:
//   bconv_part2        bconv.cpp:96-174   (int64 delayed accumulation, one reduction)
//   tensor             ckks.cpp:818-821
//   key_mult (+fold)   ckks.cpp:733-770, ckks.cpp:831-842
//   combine            ckks.cpp:643-651
//   hrot tail          ckks.cpp:875-882 + apply_automorphism automorphism.cpp:76-100
//   ew_*               poly.cpp:146-205;  addmul_rows ckks.cpp:930-941
#include "ck_common.cuh"
#include "ck_kernels.h"

namespace ck {
namespace {

constexpr int kT = 256;

__device__ __forceinline__ uint4 ld4(const uint32_t* p) { return *reinterpret_cast<const uint4*>(p); }
__device__ __forceinline__ void st4(uint32_t* p, uint4 v) { *reinterpret_cast<uint4*>(p) = v; }
__device__ __forceinline__ uint32_t getc(const uint4& v, int k) {
  return k == 0 ? v.x : (k == 1 ? v.y : (k == 2 ? v.z : v.w));
}

// ------------------------------------------------------------------ bconv --
// One thread = 4 adjacent coefficients x all destination rows of the group.
// Per-destination constants (matrix row, q, -q^-1, output row offset) are
// staged in shared memory so the MAC loop never waits on a global load; the
// destination loop is unrolled by two for independent accumulator chains.
template <int SC>
__global__ void __launch_bounds__(kT) k_bconv(BconvLaunch a, int n) {
  __shared__ uint32_t cm[kMaxRows * SC];
  __shared__ uint4 rc[kMaxRows];  // {q, qinv, dst row, 0}
  const BconvGroup G = a.groups[blockIdx.y];
  for (int e = threadIdx.x; e < G.dc * SC; e += kT) {
    const int i = e / SC, j = e % SC;
    cm[e] = j < (int)G.sc ? a.cmat[G.cmat_off + i * G.sc + j] : 0u;
  }
  for (int i = threadIdx.x; i < (int)G.dc; i += kT) {
    const PrimeDev P = a.primes[a.dst_prime[G.map_off + i]];
    rc[i] = make_uint4(P.q, P.qinv, a.dst_row[G.map_off + i], 0);
  }
  __syncthreads();
  const int x = (blockIdx.x * kT + threadIdx.x) * 4;
  if (x >= n) return;
  const uint32_t* src = a.src + blockIdx.z * a.src_bs + (size_t)G.src_off * n + x;
  uint4 s[SC];
  if (a.src_rows) {  // rows by absolute address (possibly peer memory); plain loads
#pragma unroll
    for (int j = 0; j < SC; ++j)
      s[j] = j < (int)G.sc ? ld4(reinterpret_cast<const uint32_t*>(a.src_rows[G.src_off + j]) + x)
                           : make_uint4(0, 0, 0, 0);
  } else {
#pragma unroll
    for (int j = 0; j < SC; ++j) s[j] = j < (int)G.sc ? ld4(src + (size_t)j * n) : make_uint4(0, 0, 0, 0);
  }
  uint32_t* dst = a.dst + blockIdx.z * a.dst_bs + x;
  auto one = [&](int i) {
    uint64_t acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
#pragma unroll
    for (int j = 0; j < SC; ++j) {
      const uint32_t c = cm[i * SC + j];
      acc0 = mac_wide(acc0, s[j].x, c);
      acc1 = mac_wide(acc1, s[j].y, c);
      acc2 = mac_wide(acc2, s[j].z, c);
      acc3 = mac_wide(acc3, s[j].w, c);
    }
    const uint4 R = rc[i];
    uint4 r;
    r.x = sub_if(mont_reduce64(acc0, R.x, R.y), R.x);
    r.y = sub_if(mont_reduce64(acc1, R.x, R.y), R.x);
    r.z = sub_if(mont_reduce64(acc2, R.x, R.y), R.x);
    r.w = sub_if(mont_reduce64(acc3, R.x, R.y), R.x);
    st4(dst + (size_t)R.z * n, r);
  };
  int i = 0;
  for (; i + 1 < (int)G.dc; i += 2) {
    one(i);
    one(i + 1);
  }
  if (i < (int)G.dc) one(i);
}

// ------------------------------------------------------- bconv, FP64 pipe --
// The CUDA-core BConv above is bound by the integer multiply pipe (IMAD.WIDE
// occupies fmaheavy for two issue slots; ncu: fmaheavy 79%, math-pipe
// throttle the top stall).  B200 has a full-rate FP64 pipe next to it, and
// the dot products sum_j s_j c_ij can be computed EXACTLY there:
//   c = c_lo + 2^15 c_hi (c_lo < 2^15, c_hi < 2^14 as c < q < 2^29),
//   s < 2^32, SC <= 16  =>  sum_j s_j c_lo < 2^51, sum_j s_j c_hi < 2^50;
// each partial sum is accumulated by DFMA on top of 2^52, where the spacing of
// doubles is exactly 1, so every product (< 2^49) and every partial sum is an
// exactly representable integer and no rounding ever happens.  The integer is
// then read straight from the bit pattern (bits(2^52 + S) = 0x4330... + S) and
// t = S_lo + 2^15 S_hi is the same 64-bit sum the IMAD.WIDE path forms, so
// the Montgomery reduction and the canonical output are bit-identical.
// MODE selects which destination rows go to the FP64 pipe: 1 = all, 2 = every
// other row (the rest on IMAD.WIDE), 3 = two of every three.  Two adjacent
// coefficients per thread (uint2) keep the double copies of the sources in
// registers.
constexpr int kTD = 256;
template <int SC, int MODE>
__global__ void __launch_bounds__(kTD) k_bconv_df(BconvLaunch a, int n) {
  __shared__ uint32_t cm[kMaxRows * SC];
  __shared__ double2 cd[kMaxRows * SC];
  __shared__ uint4 rc[kMaxRows];  // {q, qinv, dst row, 0}
  const BconvGroup G = a.groups[blockIdx.y];
  for (int e = threadIdx.x; e < G.dc * SC; e += kTD) {
    const int i = e / SC, j = e % SC;
    const uint32_t c = j < (int)G.sc ? a.cmat[G.cmat_off + i * G.sc + j] : 0u;
    cm[e] = c;
    cd[e] = make_double2((double)(c & 0x7fffu), (double)(c >> 15));
  }
  for (int i = threadIdx.x; i < (int)G.dc; i += kTD) {
    const PrimeDev P = a.primes[a.dst_prime[G.map_off + i]];
    rc[i] = make_uint4(P.q, P.qinv, a.dst_row[G.map_off + i], 0);
  }
  __syncthreads();
  const int x = (blockIdx.x * kTD + threadIdx.x) * 2;
  if (x >= n) return;
  const uint32_t* src = a.src + blockIdx.z * a.src_bs + (size_t)G.src_off * n + x;
  uint2 s[SC];
  double2 sd[SC];
#pragma unroll
  for (int j = 0; j < SC; ++j) {
    s[j] = j < (int)G.sc ? *reinterpret_cast<const uint2*>(src + (size_t)j * n) : make_uint2(0, 0);
    sd[j] = make_double2((double)s[j].x, (double)s[j].y);
  }
  uint32_t* dst = a.dst + blockIdx.z * a.dst_bs + x;
  auto store = [&](int i, uint64_t t0, uint64_t t1) {
    const uint4 R = rc[i];
    *reinterpret_cast<uint2*>(dst + (size_t)R.z * n) =
        make_uint2(sub_if(mont_reduce64(t0, R.x, R.y), R.x), sub_if(mont_reduce64(t1, R.x, R.y), R.x));
  };
  auto row_fp = [&](int i) {
    constexpr double kM = 4503599627370496.0;  // 2^52
    double l0 = kM, h0 = kM, l1 = kM, h1 = kM;
#pragma unroll
    for (int j = 0; j < SC; ++j) {
      const double2 c = cd[i * SC + j];
      l0 = __fma_rn(sd[j].x, c.x, l0);
      h0 = __fma_rn(sd[j].x, c.y, h0);
      l1 = __fma_rn(sd[j].y, c.x, l1);
      h1 = __fma_rn(sd[j].y, c.y, h1);
    }
    // (bits(l) - K) + ((bits(h) - K) << 15), K = bits(2^52), folded
    constexpr uint64_t kK = 0x4330000000000000ull, kKK = kK + (kK << 15);
    const uint64_t t0 = (uint64_t)__double_as_longlong(l0) + ((uint64_t)__double_as_longlong(h0) << 15) - kKK;
    const uint64_t t1 = (uint64_t)__double_as_longlong(l1) + ((uint64_t)__double_as_longlong(h1) << 15) - kKK;
    store(i, t0, t1);
  };
  auto row_int = [&](int i) {
    uint64_t a0 = 0, a1 = 0;
#pragma unroll
    for (int j = 0; j < SC; ++j) {
      const uint32_t c = cm[i * SC + j];
      a0 = mac_wide(a0, s[j].x, c);
      a1 = mac_wide(a1, s[j].y, c);
    }
    store(i, a0, a1);
  };
  int i = 0;
  if (MODE == 1) {
    for (; i + 1 < (int)G.dc; i += 2) {
      row_fp(i);
      row_fp(i + 1);
    }
  } else if (MODE == 2) {
    for (; i + 1 < (int)G.dc; i += 2) {
      row_fp(i);
      row_int(i + 1);
    }
  } else {
    for (; i + 2 < (int)G.dc; i += 3) {
      row_fp(i);
      row_int(i + 2);
      row_fp(i + 1);
    }
  }
  for (; i < (int)G.dc; ++i) row_fp(i);
}

// Generic-width pieces for the FP64 / warp-specialised variants: CPT adjacent
// coefficients per thread, rows [r0, r1) of group G.
template <int SC, int CPT>
struct BconvRows {
  const uint32_t* cm;
  const double2* cd;
  const uint4* rc;
  uint32_t* dst;
  int n;
  __device__ __forceinline__ void store(int i, const uint64_t (&t)[CPT]) const {
    const uint4 R = rc[i];
    uint32_t o[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k) o[k] = sub_if(mont_reduce64(t[k], R.x, R.y), R.x);
    uint32_t* p = dst + (size_t)R.z * n;
    if (CPT == 4) *reinterpret_cast<uint4*>(p) = make_uint4(o[0], o[1], o[2], o[3 % CPT]);
    else *reinterpret_cast<uint2*>(p) = make_uint2(o[0], o[1 % CPT]);
  }
  __device__ __forceinline__ void fp(int i, const double (&sd)[SC][CPT]) const {
    constexpr double kM = 4503599627370496.0;  // 2^52
    constexpr uint64_t kK = 0x4330000000000000ull, kKK = kK + (kK << 15);
    double l[CPT], h[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k) l[k] = h[k] = kM;
#pragma unroll
    for (int j = 0; j < SC; ++j) {
      const double2 c = cd[i * SC + j];
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        l[k] = __fma_rn(sd[j][k], c.x, l[k]);
        h[k] = __fma_rn(sd[j][k], c.y, h[k]);
      }
    }
    uint64_t t[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k)
      t[k] = (uint64_t)__double_as_longlong(l[k]) + ((uint64_t)__double_as_longlong(h[k]) << 15) - kKK;
    store(i, t);
  }
  __device__ __forceinline__ void in(int i, const uint32_t (&s)[SC][CPT]) const {
    uint64_t t[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k) t[k] = 0;
#pragma unroll
    for (int j = 0; j < SC; ++j) {
      const uint32_t c = cm[i * SC + j];
#pragma unroll
      for (int k = 0; k < CPT; ++k) t[k] = mac_wide(t[k], s[j][k], c);
    }
    store(i, t);
  }
};

template <int SC, int CPT>
__device__ __forceinline__ void bconv_load(const uint32_t* src, int n, int sc, uint32_t (&s)[SC][CPT]) {
#pragma unroll
  for (int j = 0; j < SC; ++j) {
    if (CPT == 4) {
      const uint4 v = j < sc ? *reinterpret_cast<const uint4*>(src + (size_t)j * n) : make_uint4(0, 0, 0, 0);
      s[j][0] = v.x, s[j][1 % CPT] = v.y, s[j][2 % CPT] = v.z, s[j][3 % CPT] = v.w;
    } else {
      const uint2 v = j < sc ? *reinterpret_cast<const uint2*>(src + (size_t)j * n) : make_uint2(0, 0);
      s[j][0] = v.x, s[j][1 % CPT] = v.y;
    }
  }
}

// Warp-specialised BConv: the first half of the CTA's warps runs the
// IMAD.WIDE dot products for destination rows [0, h), the second half the
// exact FP64 dot products for rows [h, dc), on the SAME coefficients, so the
// SM's fmaheavy and FP64 pipes work side by side.  h = dc - dc * FP / 6.
constexpr int kTW = 256;
template <int SC, int FP>
__global__ void __launch_bounds__(kTW) k_bconv_ws(BconvLaunch a, int n) {
  constexpr int CPT = 4;
  __shared__ uint32_t cm[kMaxRows * SC];
  __shared__ double2 cd[kMaxRows * SC];
  __shared__ uint4 rc[kMaxRows];
  const BconvGroup G = a.groups[blockIdx.y];
  for (int e = threadIdx.x; e < G.dc * SC; e += kTW) {
    const int i = e / SC, j = e % SC;
    const uint32_t c = j < (int)G.sc ? a.cmat[G.cmat_off + i * G.sc + j] : 0u;
    cm[e] = c;
    cd[e] = make_double2((double)(c & 0x7fffu), (double)(c >> 15));
  }
  for (int i = threadIdx.x; i < (int)G.dc; i += kTW) {
    const PrimeDev P = a.primes[a.dst_prime[G.map_off + i]];
    rc[i] = make_uint4(P.q, P.qinv, a.dst_row[G.map_off + i], 0);
  }
  __syncthreads();
  const bool fpw = threadIdx.x >= kTW / 2;
  const int t = threadIdx.x % (kTW / 2);
  const int x = (blockIdx.x * (kTW / 2) + t) * CPT;
  if (x >= n) return;
  const uint32_t* src = a.src + blockIdx.z * a.src_bs + (size_t)G.src_off * n + x;
  const BconvRows<SC, CPT> R{cm, cd, rc, a.dst + blockIdx.z * a.dst_bs + x, n};
  const int dc = (int)G.dc, h = dc - dc * FP / 6;
  uint32_t s[SC][CPT];
  bconv_load<SC, CPT>(src, n, (int)G.sc, s);
  if (!fpw) {
    int i = 0;
    for (; i + 1 < h; i += 2) {
      R.in(i, s);
      R.in(i + 1, s);
    }
    if (i < h) R.in(i, s);
  } else {
    double sd[SC][CPT];
#pragma unroll
    for (int j = 0; j < SC; ++j)
#pragma unroll
      for (int k = 0; k < CPT; ++k) sd[j][k] = (double)s[j][k];
    for (int i = h; i < dc; ++i) R.fp(i, sd);
  }
}

// ----------------------------------------------------------------- tensor --
__global__ void __launch_bounds__(kT) k_tensor(int n, int level, const uint32_t* __restrict__ x,
                                               const uint32_t* __restrict__ y, uint64_t ct_bs,
                                               uint32_t* __restrict__ d01, uint64_t d01_bs,
                                               uint32_t* __restrict__ d2, uint64_t d2_bs,
                                               const PrimeDev* __restrict__ primes) {
  const int xo = (blockIdx.x * kT + threadIdx.x) * 4;
  if (xo >= n) return;
  const int i = blockIdx.y, b = blockIdx.z;
  const PrimeDev P = primes[i];
  const size_t ro = (size_t)i * n + xo, ao = (size_t)(level + i) * n + xo;
  const uint4 xb = ld4(x + b * ct_bs + ro), xa = ld4(x + b * ct_bs + ao);
  const uint4 yb = ld4(y + b * ct_bs + ro), ya = ld4(y + b * ct_bs + ao);
  uint4 o0, o1, o2;
#define CK_T(c)                                                                              \
  {                                                                                          \
    const uint32_t bb = xb.c, ba = xa.c, cb = yb.c, ca = ya.c;                               \
    o0.c = sub_if(mont_mul(bb, cb, P.q, P.qinv), P.q);                                   \
    o1.c = sub_if(mont_reduce64(mac_wide(mac_wide(0ull, bb, ca), ba, cb), P.q, P.qinv), P.q); \
    o2.c = sub_if(mont_mul(ba, ca, P.q, P.qinv), P.q);                                   \
  }
  CK_T(x) CK_T(y) CK_T(z) CK_T(w)
#undef CK_T
  st4(d01 + b * d01_bs + ro, o0);
  st4(d01 + b * d01_bs + ao, o1);
  st4(d2 + b * d2_bs + ro, o2);
}

// --------------------------------------------------------------- key_mult --
__global__ void __launch_bounds__(kT) k_key_mult(KeyMultLaunch a, int n) {
  const int xo = (blockIdx.x * kT + threadIdx.x) * 4;
  if (xo >= n) return;
  const int i = blockIdx.y, b = blockIdx.z;
  const int rows = a.level + a.alpha;
  const int g = i < a.level ? i : a.L + (i - a.level);  // global prime index (poly.hpp:103-106)
  const PrimeDev P = a.primes[g];
  const uint32_t LA = (uint32_t)(a.L + a.alpha);
  uint64_t s0[4] = {0, 0, 0, 0}, s1[4] = {0, 0, 0, 0};
  int terms = 0;
  auto renorm = [&]() {  // keep the int64 sums below q*2^32 (acc value unchanged mod q, scaled back by R)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      s0[c] = shoup_mul(mont_reduce64(s0[c], P.q, P.qinv), P.r, P.r_sh, P.q);
      s1[c] = shoup_mul(mont_reduce64(s1[c], P.q, P.qinv), P.r, P.r_sh, P.q);
    }
  };
  for (int k = 0; k < a.D; ++k) {
    const int lo = k * a.alpha, hi = min((k + 1) * a.alpha, a.level);
    const uint32_t* op = (i >= lo && i < hi) ? a.d + b * a.d_bs + (size_t)i * n + xo
                                             : a.ext + b * a.ext_bs + ((size_t)k * rows + i) * n + xo;
    const uint4 dv = ld4(op);
    const uint4 eb = ld4(a.evk + (((size_t)k * 2 + 0) * LA + g) * n + xo);
    const uint4 ea = ld4(a.evk + (((size_t)k * 2 + 1) * LA + g) * n + xo);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      s0[c] = mac_wide(s0[c], getc(dv, c), getc(eb, c));
      s1[c] = mac_wide(s1[c], getc(dv, c), getc(ea, c));
    }
    if (++terms == 7) {
      renorm();
      terms = 1;
    }
  }
  if (a.fold && i < a.level) {
    const uint32_t pm = a.p_mont[i];
    const uint4 f0 = ld4(a.fold + b * a.fold_bs + (size_t)i * n + xo);
    const uint4 f1 = ld4(a.fold + b * a.fold_bs + (size_t)(a.level + i) * n + xo);
    if (terms == 7) renorm();
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      s0[c] = mac_wide(s0[c], getc(f0, c), pm);
      s1[c] = mac_wide(s1[c], getc(f1, c), pm);
    }
  }
  uint4 r0, r1;
  r0.x = sub_if(mont_reduce64(s0[0], P.q, P.qinv), P.q);
  r0.y = sub_if(mont_reduce64(s0[1], P.q, P.qinv), P.q);
  r0.z = sub_if(mont_reduce64(s0[2], P.q, P.qinv), P.q);
  r0.w = sub_if(mont_reduce64(s0[3], P.q, P.qinv), P.q);
  r1.x = sub_if(mont_reduce64(s1[0], P.q, P.qinv), P.q);
  r1.y = sub_if(mont_reduce64(s1[1], P.q, P.qinv), P.q);
  r1.z = sub_if(mont_reduce64(s1[2], P.q, P.qinv), P.q);
  r1.w = sub_if(mont_reduce64(s1[3], P.q, P.qinv), P.q);
  st4(a.v + b * a.v_bs + (size_t)i * n + xo, r0);
  st4(a.v + b * a.v_bs + (size_t)(rows + i) * n + xo, r1);
}

// ---------------------------------------------------------------- combine --
__global__ void __launch_bounds__(kT) k_combine(int n, const uint32_t* __restrict__ v, uint64_t v_ps, uint64_t v_bs,
                                                uint32_t* __restrict__ o, uint64_t o_ps, uint64_t o_bs,
                                                const uint32_t* __restrict__ dinv, const PrimeDev* __restrict__ primes,
                                                int npoly) {
  const int xo = (blockIdx.x * kT + threadIdx.x) * 4;
  if (xo >= n) return;
  const int i = blockIdx.y;
  const int b = blockIdx.z / npoly, p = blockIdx.z % npoly;
  const PrimeDev P = primes[i];
  const uint32_t di = dinv[i];
  const uint32_t* vp = v + b * v_bs + p * v_ps + (size_t)i * n + xo;
  uint32_t* op = o + b * o_bs + p * o_ps + (size_t)i * n + xo;
  const uint4 vv = ld4(vp), ov = ld4(op);
  uint4 r;
  r.x = sub_if(mont_mul(vv.x - ov.x + P.q, di, P.q, P.qinv), P.q);
  r.y = sub_if(mont_mul(vv.y - ov.y + P.q, di, P.q, P.qinv), P.q);
  r.z = sub_if(mont_mul(vv.z - ov.z + P.q, di, P.q, P.qinv), P.q);
  r.w = sub_if(mont_mul(vv.w - ov.w + P.q, di, P.q, P.qinv), P.q);
  st4(op, r);
}

// -------------------------------------------------------------- hrot tail --
__global__ void __launch_bounds__(kT) k_hrot_tail(int n, int level, const uint32_t* __restrict__ v, uint64_t v_bs,
                                                  uint64_t v_ps, const uint32_t* __restrict__ o, uint64_t o_bs,
                                                  uint64_t o_ps, const uint32_t* __restrict__ bb, uint64_t b_bs,
                                                  const uint32_t* __restrict__ dinv, const uint32_t* __restrict__ src,
                                                  uint32_t* __restrict__ out, uint64_t out_bs,
                                                  const PrimeDev* __restrict__ primes) {
  const int j = blockIdx.x * kT + threadIdx.x;
  if (j >= n) return;
  const int i = blockIdx.y, b = blockIdx.z;
  const PrimeDev P = primes[i];
  const uint32_t di = dinv[i];
  const uint32_t s = __ldg(&src[j]);
  const size_t r = (size_t)i * n + s;
  const uint32_t* vb = v + b * v_bs;
  const uint32_t* ob = o + b * o_bs;
  uint32_t c0 = sub_if(mont_mul(vb[r] - ob[r] + P.q, di, P.q, P.qinv), P.q);
  c0 = sub_if(c0 + bb[b * b_bs + r], P.q);
  const uint32_t c1 = sub_if(mont_mul(vb[v_ps + r] - ob[o_ps + r] + P.q, di, P.q, P.qinv), P.q);
  out[b * out_bs + (size_t)i * n + j] = c0;
  out[b * out_bs + (size_t)(level + i) * n + j] = c1;
}

// HRot tail, scatter form: thread = 4 consecutive SOURCE coefficients x..x+3
// (every operand read with one 16-B load: v0, o0, b, v1, o1) written to
// out[dest[x + m]] (the automorphism maps each aligned 32-block onto one
// aligned 32-block, so a warp's scattered 4-B stores fill whole lines in L2).
// 6 vector loads + 8 scalar stores per 4 coefficients instead of 24 scalar
// loads (the gather form above: one coefficient per thread).
__global__ void __launch_bounds__(kT) k_hrot_tail4(int n, int level, const uint32_t* __restrict__ v, uint64_t v_bs,
                                                   uint64_t v_ps, const uint32_t* __restrict__ o, uint64_t o_bs,
                                                   uint64_t o_ps, const uint32_t* __restrict__ bb, uint64_t b_bs,
                                                   const uint32_t* __restrict__ dinv,
                                                   const uint32_t* __restrict__ dest, uint32_t* __restrict__ out,
                                                   uint64_t out_bs, const PrimeDev* __restrict__ primes) {
  const int x = (blockIdx.x * kT + threadIdx.x) * 4;
  if (x >= n) return;
  const int i = blockIdx.y, b = blockIdx.z;
  const PrimeDev P = primes[i];
  const uint32_t di = dinv[i];
  const size_t r = (size_t)i * n + x;
  const uint32_t* vb = v + b * v_bs + r;
  const uint32_t* ob = o + b * o_bs + r;
  const uint4 d4 = __ldg(reinterpret_cast<const uint4*>(dest + x));
  const uint4 v0 = ld4(vb), o0 = ld4(ob), b0 = ld4(bb + b * b_bs + r), v1 = ld4(vb + v_ps), o1 = ld4(ob + o_ps);
  uint32_t* out0 = out + b * out_bs + (size_t)i * n;
  uint32_t* out1 = out + b * out_bs + (size_t)(level + i) * n;
#define CK_T(c)                                                                                   \
  {                                                                                               \
    const uint32_t c0 = sub_if(mont_mul(v0.c - o0.c + P.q, di, P.q, P.qinv), P.q);                \
    out0[d4.c] = sub_if(c0 + b0.c, P.q);                                                          \
    out1[d4.c] = sub_if(mont_mul(v1.c - o1.c + P.q, di, P.q, P.qinv), P.q);                       \
  }
  CK_T(x) CK_T(y) CK_T(z) CK_T(w)
#undef CK_T
}

// ------------------------------------------------------------ elementwise --
// op 0 add, 1 sub, 2 Montgomery mul (poly.cpp:146-164), 3 multiply row i by
// the canonical Montgomery constant rc[i] (ew_mul_const, poly.cpp:166-180);
// ops 4 / 5 / 6 / 7: the same four in the reference's raw representation
// (signed lazy int32 in (-q, q): narrow() and signed Montgomery, bit for bit).
// o may alias a or b (ew_add_inplace / ew_sub_inplace, poly.cpp:182-205):
// every thread reads its 4 words of each operand before writing them.
__global__ void __launch_bounds__(kT) k_elementwise(int n, int op, const uint32_t* a, uint64_t a_bs,
                                                    const uint32_t* bp, uint64_t b_bs, uint32_t* o, uint64_t o_bs,
                                                    const uint16_t* __restrict__ row_prime,
                                                    const PrimeDev* __restrict__ primes, int prime_mod,
                                                    const uint32_t* __restrict__ rc) {
  const int xo = (blockIdx.x * kT + threadIdx.x) * 4;
  if (xo >= n) return;
  const int i = blockIdx.y, b = blockIdx.z;
  const PrimeDev P = primes[row_prime ? row_prime[i] : i % prime_mod];
  const size_t r = (size_t)i * n + xo;
  const uint4 x = *reinterpret_cast<const uint4*>(a + b * a_bs + r);
  uint4 z;
  if (op >= 4) {  // raw: the reference's signed lazy int32 formulas (poly.cpp:121-180, modarith.hpp:20-36)
    const int32_t q = (int32_t)P.q;
    auto narrow = [&](int64_t v) -> uint32_t {
      if (v >= q) v -= q;
      else if (v <= -q) v += q;
      return (uint32_t)(int32_t)v;
    };
    auto mred = [&](int64_t v) -> uint32_t {  // signed Montgomery, (-q, q)
      const int32_t hi = (int32_t)(v >> 32), t = (int32_t)((uint32_t)v * P.qinv);
      return (uint32_t)(hi - (int32_t)(((int64_t)t * q) >> 32));
    };
    const int32_t* xs = reinterpret_cast<const int32_t*>(&x);
    uint32_t* zs = reinterpret_cast<uint32_t*>(&z);
    if (op == 7) {
      const int32_t c = (int32_t)rc[i];
#pragma unroll
      for (int e = 0; e < 4; ++e) zs[e] = mred((int64_t)xs[e] * c);
    } else {
      const uint4 y = *reinterpret_cast<const uint4*>(bp + b * b_bs + r);
      const int32_t* ys = reinterpret_cast<const int32_t*>(&y);
#pragma unroll
      for (int e = 0; e < 4; ++e)
        zs[e] = op == 4 ? narrow((int64_t)xs[e] + ys[e]) : op == 5 ? narrow((int64_t)xs[e] - ys[e])
                                                                   : mred((int64_t)xs[e] * ys[e]);
    }
    *reinterpret_cast<uint4*>(o + b * o_bs + r) = z;
    return;
  }
  if (op == 3) {
    const uint32_t c = rc[i];
    z = make_uint4(sub_if(mont_mul(x.x, c, P.q, P.qinv), P.q), sub_if(mont_mul(x.y, c, P.q, P.qinv), P.q),
                   sub_if(mont_mul(x.z, c, P.q, P.qinv), P.q), sub_if(mont_mul(x.w, c, P.q, P.qinv), P.q));
    *reinterpret_cast<uint4*>(o + b * o_bs + r) = z;
    return;
  }
  const uint4 y = *reinterpret_cast<const uint4*>(bp + b * b_bs + r);
  if (op == 0) {
    z = make_uint4(sub_if(x.x + y.x, P.q), sub_if(x.y + y.y, P.q), sub_if(x.z + y.z, P.q), sub_if(x.w + y.w, P.q));
  } else if (op == 1) {
    z = make_uint4(sub_if(x.x - y.x + P.q, P.q), sub_if(x.y - y.y + P.q, P.q), sub_if(x.z - y.z + P.q, P.q),
                   sub_if(x.w - y.w + P.q, P.q));
  } else {
    z = make_uint4(sub_if(mont_mul(x.x, y.x, P.q, P.qinv), P.q), sub_if(mont_mul(x.y, y.y, P.q, P.qinv), P.q),
                   sub_if(mont_mul(x.z, y.z, P.q, P.qinv), P.q), sub_if(mont_mul(x.w, y.w, P.q, P.qinv), P.q));
  }
  *reinterpret_cast<uint4*>(o + b * o_bs + r) = z;
}

// ------------------------------------------------------------ automorphism --
// apply_automorphism (automorphism.cpp:76-100) for any Galois element g (odd,
// mod 2n) with inverse gi, indices computed on the fly (no map table), as a
// gather so every warp writes 32 contiguous words:
//  * evaluation domain (bit-reversed columns): out[j] = in[src(j)] with
//    src(j) = brev(phi_gi(brev(j))), phi_g(i) = ((2i+1) g mod 2n - 1) / 2
//    (the inverse of dest(i) = brev(phi_g(brev(i))), automorphism.cpp:40-46);
//  * coefficient domain: the reference scatters coefficient k to
//    k * gi mod 2n with a sign flip past n (automorphism.cpp:50-61, :90-97);
//    gathered, out[m] = +in[k] if k = m g mod 2n < n, else -in[k - n],
//    negation canonical (q - v, 0 stays 0).
__global__ void __launch_bounds__(kT) k_automorphism_galois(int n, int logn, uint32_t g, uint32_t gi, int coeff,
                                                            const uint32_t* __restrict__ in,
                                                            uint32_t* __restrict__ out,
                                                            const uint16_t* __restrict__ row_prime,
                                                            const PrimeDev* __restrict__ primes) {
  const uint32_t j = blockIdx.x * kT + threadIdx.x;
  if (j >= (uint32_t)n) return;
  const size_t r = (size_t)blockIdx.y * n;
  const uint32_t mask2n = 2u * n - 1u;
  if (!coeff) {
    const uint32_t bj = __brev(j) >> (32 - logn);
    const uint32_t ph = (((2u * bj + 1u) * gi) & mask2n) >> 1;  // ((2i+1) gi mod 2n - 1) / 2
    out[r + j] = __ldg(&in[r + (__brev(ph) >> (32 - logn))]);
    return;
  }
  const uint32_t k = (j * g) & mask2n;
  if (k < (uint32_t)n) {
    out[r + j] = __ldg(&in[r + k]);
  } else {
    const uint32_t q = primes[row_prime[blockIdx.y]].q;
    const uint32_t v = __ldg(&in[r + k - n]);
    out[r + j] = v ? q - v : 0u;
  }
}

// ------------------------------------------------- encrypt / decrypt parts --
// Element-wise parts of decrypt / encrypt (ckks.cpp:497-553) on one batch of
// ciphertexts [B][2][level][n]; every operand is evaluation domain, Montgomery
// form, canonical.  op 0 decrypt: m = b + a s.  op 1 secret-key encrypt:
// b = m + e - a s, a = a.  op 2 public-key encrypt: b = v pk.b + e0 + m,
// a = v pk.a + e1.  (x, y, z, w) are the op's operands in that order.
__global__ void __launch_bounds__(kT) k_crypt(int n, int level, int op, const uint32_t* __restrict__ x,
                                              uint64_t x_bs, const uint32_t* __restrict__ y,
                                              const uint32_t* __restrict__ z, const uint32_t* __restrict__ w,
                                              const uint32_t* __restrict__ u, uint32_t* __restrict__ out,
                                              uint64_t out_bs, const PrimeDev* __restrict__ primes) {
  const int k = blockIdx.x * kT + threadIdx.x;
  if (k >= n) return;
  const int i = blockIdx.y, b = blockIdx.z;
  const PrimeDev P = primes[i];
  const uint32_t q = P.q;
  const size_t r = (size_t)i * n + k;
  if (op == 0) {  // x = ct [2][level], y = s
    const uint32_t cb = x[b * x_bs + r], ca = x[b * x_bs + (size_t)level * n + r];
    out[b * out_bs + r] = sub_if(cb + sub_if(mont_mul(ca, y[r], q, P.qinv), q), q);
  } else if (op == 1) {  // x = m, y = a, z = e, w = s
    const uint32_t as = sub_if(mont_mul(y[r], w[r], q, P.qinv), q);
    out[r] = sub_if(sub_if(x[r] + z[r], q) + q - as, q);
    out[(size_t)level * n + r] = y[r];
  } else {  // x = m, y = v, z = e0, w = e1, u = pk [2][level] (b then a)
    const uint32_t vb = sub_if(mont_mul(y[r], u[r], q, P.qinv), q);
    const uint32_t va = sub_if(mont_mul(y[r], u[(size_t)level * n + r], q, P.qinv), q);
    out[r] = sub_if(sub_if(vb + z[r], q) + x[r], q);
    out[(size_t)level * n + r] = sub_if(va + w[r], q);
  }
}

// One evaluation-key digit over the full PQ basis (evk_gen, ckks.cpp:459-474):
// b = e + s_src * g - a * s_dst, with s_src squared first for relinearisation.
__global__ void __launch_bounds__(kT) k_evk_digit(int n, const uint32_t* __restrict__ s_src,
                                                  const uint32_t* __restrict__ s_dst, const uint32_t* __restrict__ a,
                                                  const uint32_t* __restrict__ e, const uint32_t* __restrict__ gm,
                                                  const uint16_t* __restrict__ row_prime, int square,
                                                  const PrimeDev* __restrict__ primes, uint32_t* __restrict__ out) {
  const int k = blockIdx.x * kT + threadIdx.x;
  if (k >= n) return;
  const int i = blockIdx.y;
  const PrimeDev P = primes[row_prime[i]];
  const uint32_t q = P.q;
  const size_t r = (size_t)i * n + k;
  uint32_t src = s_src[r];
  if (square) src = sub_if(mont_mul(src, src, q, P.qinv), q);
  const uint32_t sg = sub_if(mont_mul(src, gm[i], q, P.qinv), q);
  const uint32_t as = sub_if(mont_mul(a[r], s_dst[r], q, P.qinv), q);
  out[r] = sub_if(sub_if(e[r] + sg, q) + q - as, q);
}

// int64 coefficients -> canonical residues of every row (coeffs_to_eval's
// reduction, ckks.cpp:366-380, correct() of modarith.hpp:46-50)
__global__ void __launch_bounds__(kT) k_reduce_coeffs(int n, const long long* __restrict__ c,
                                                      const uint16_t* __restrict__ row_prime,
                                                      const PrimeDev* __restrict__ primes, uint32_t* __restrict__ out) {
  const int k = blockIdx.x * kT + threadIdx.x;
  if (k >= n) return;
  const long long q = primes[row_prime[blockIdx.y]].q;
  long long v = c[k] % q;
  if (v < 0) v += q;
  out[(size_t)blockIdx.y * n + k] = (uint32_t)v;
}

__global__ void __launch_bounds__(kT) k_permute(int n, const uint32_t* __restrict__ in, uint64_t in_bs,
                                                uint32_t* __restrict__ out, uint64_t out_bs,
                                                const uint32_t* __restrict__ src) {
  const int j = blockIdx.x * kT + threadIdx.x;
  if (j >= n) return;
  const size_t r = (size_t)blockIdx.y * n;
  out[blockIdx.z * out_bs + r + j] = in[blockIdx.z * in_bs + r + __ldg(&src[j])];
}

__global__ void __launch_bounds__(kT) k_addmul(int n, uint32_t* __restrict__ acc, uint64_t acc_bs,
                                               const uint32_t* __restrict__ x, uint64_t x_bs,
                                               const uint32_t* __restrict__ y, uint64_t y_bs,
                                               const uint32_t* __restrict__ src, const uint16_t* __restrict__ row_prime,
                                               const PrimeDev* __restrict__ primes) {
  const int j = blockIdx.x * kT + threadIdx.x;
  if (j >= n) return;
  const int i = blockIdx.y, b = blockIdx.z;
  const PrimeDev P = primes[row_prime ? row_prime[i] : i];
  const size_t r = (size_t)i * n;
  const uint32_t xs = x[b * x_bs + r + (src ? __ldg(&src[j]) : (uint32_t)j)];
  const uint32_t ys = y[b * y_bs + r + j];
  uint32_t* a = acc + b * acc_bs + r + j;
  *a = sub_if(sub_if(*a + mont_mul(xs, ys, P.q, P.qinv), P.q2), P.q);
}

inline unsigned cdiv(unsigned a, unsigned b) { return (a + b - 1) / b; }

}  // namespace

void bconv(int n, const BconvLaunch& a, cudaStream_t st, int fp64_mode) {
  const int sc = a.max_sc;
  const BconvLaunch b = a;
  if (a.src_rows) fp64_mode = 0;  // the pointer-table form is implemented by k_bconv only
  if (fp64_mode >= 4 && fp64_mode <= 8 && sc <= 16) {  // warp-specialised, FP64 share (mode - 3) / 6 of the rows
    dim3 grid(cdiv(n / 4, kTW / 2), a.ngroups, a.batch);
    switch (sc * 16 + fp64_mode) {
#define CK_WS(S)                                                           \
  case S * 16 + 4: k_bconv_ws<S, 1><<<grid, kTW, 0, st>>>(b, n); break; \
  case S * 16 + 5: k_bconv_ws<S, 2><<<grid, kTW, 0, st>>>(b, n); break; \
  case S * 16 + 6: k_bconv_ws<S, 3><<<grid, kTW, 0, st>>>(b, n); break; \
  case S * 16 + 7: k_bconv_ws<S, 4><<<grid, kTW, 0, st>>>(b, n); break; \
  case S * 16 + 8: k_bconv_ws<S, 6><<<grid, kTW, 0, st>>>(b, n); break;
      CK_WS(1) CK_WS(2) CK_WS(3) CK_WS(4) CK_WS(5) CK_WS(6) CK_WS(7) CK_WS(8) CK_WS(9) CK_WS(10) CK_WS(11)
      CK_WS(12) CK_WS(13) CK_WS(14) CK_WS(15) CK_WS(16)
#undef CK_WS
      default: break;
    }
    return;
  }
  if (fp64_mode >= 1 && fp64_mode <= 3 && sc <= 16) {
    dim3 grid(cdiv(n / 2, kTD), a.ngroups, a.batch);
    switch (sc * 4 + fp64_mode) {
#define CK_DF(S)                                                       \
  case S * 4 + 1: k_bconv_df<S, 1><<<grid, kTD, 0, st>>>(b, n); break; \
  case S * 4 + 2: k_bconv_df<S, 2><<<grid, kTD, 0, st>>>(b, n); break; \
  case S * 4 + 3: k_bconv_df<S, 3><<<grid, kTD, 0, st>>>(b, n); break;
      CK_DF(1) CK_DF(2) CK_DF(3) CK_DF(4) CK_DF(5) CK_DF(6) CK_DF(7) CK_DF(8) CK_DF(9) CK_DF(10) CK_DF(11)
      CK_DF(12) CK_DF(13) CK_DF(14) CK_DF(15) CK_DF(16)
#undef CK_DF
      default: break;
    }
    return;
  }
  dim3 grid(cdiv(n / 4, kT), a.ngroups, a.batch);
  switch (sc) {
#define CK_SC(S) case S: k_bconv<S><<<grid, kT, 0, st>>>(b, n); break;
    CK_SC(1) CK_SC(2) CK_SC(3) CK_SC(4) CK_SC(5) CK_SC(6) CK_SC(7) CK_SC(8) CK_SC(9) CK_SC(10) CK_SC(11)
    CK_SC(12) CK_SC(13) CK_SC(14) CK_SC(15) CK_SC(16)
#undef CK_SC
    default: break;
  }
}

void tensor(int n, int level, int batch, const uint32_t* x, const uint32_t* y, uint64_t ct_bs, uint32_t* d01,
            uint64_t d01_bs, uint32_t* d2, uint64_t d2_bs, const PrimeDev* primes, cudaStream_t st) {
  dim3 grid(cdiv(n / 4, kT), level, batch);
  k_tensor<<<grid, kT, 0, st>>>(n, level, x, y, ct_bs, d01, d01_bs, d2, d2_bs, primes);
}

void key_mult(int n, const KeyMultLaunch& a, cudaStream_t st) {
  dim3 grid(cdiv(n / 4, kT), a.level + a.alpha, a.batch);
  k_key_mult<<<grid, kT, 0, st>>>(a, n);
}

void combine(int n, int rows, int npoly, int batch, const uint32_t* v, uint64_t v_ps, uint64_t v_bs, uint32_t* o,
             uint64_t o_ps, uint64_t o_bs, const uint32_t* div_inv_mont, const PrimeDev* primes, cudaStream_t st) {
  dim3 grid(cdiv(n / 4, kT), rows, batch * npoly);
  k_combine<<<grid, kT, 0, st>>>(n, v, v_ps, v_bs, o, o_ps, o_bs, div_inv_mont, primes, npoly);
}

void hrot_tail(int n, int level, int batch, const uint32_t* v, uint64_t v_bs, uint64_t v_ps, const uint32_t* o,
               uint64_t o_bs, uint64_t o_ps, const uint32_t* b, uint64_t b_bs, const uint32_t* div_inv_mont,
               const uint32_t* src_map, uint32_t* out, uint64_t out_bs, const PrimeDev* primes, cudaStream_t st,
               const uint32_t* dest_map) {
  if (dest_map && n % 4 == 0) {
    dim3 grid4(cdiv(n / 4, kT), level, batch);
    k_hrot_tail4<<<grid4, kT, 0, st>>>(n, level, v, v_bs, v_ps, o, o_bs, o_ps, b, b_bs, div_inv_mont, dest_map, out,
                                       out_bs, primes);
    return;
  }
  dim3 grid(cdiv(n, kT), level, batch);
  k_hrot_tail<<<grid, kT, 0, st>>>(n, level, v, v_bs, v_ps, o, o_bs, o_ps, b, b_bs, div_inv_mont, src_map, out,
                                   out_bs, primes);
}

void elementwise(int n, int rows, int batch, int op, const uint32_t* a, uint64_t a_bs, const uint32_t* b,
                 uint64_t b_bs, uint32_t* o, uint64_t o_bs, const uint16_t* row_prime, const PrimeDev* primes,
                 cudaStream_t st, int prime_mod, const uint32_t* row_consts) {
  dim3 grid(cdiv(n / 4, kT), rows, batch);
  k_elementwise<<<grid, kT, 0, st>>>(n, op, a, a_bs, b, b_bs, o, o_bs, row_prime, primes,
                                     prime_mod > 0 ? prime_mod : rows, row_consts);
}

void automorphism_galois(int n, int logn, int rows, uint32_t g, uint32_t gi, int coeff, const uint32_t* in,
                         uint32_t* out, const uint16_t* row_prime, const PrimeDev* primes, cudaStream_t st) {
  dim3 grid(cdiv(n, kT), rows);
  k_automorphism_galois<<<grid, kT, 0, st>>>(n, logn, g, gi, coeff, in, out, row_prime, primes);
}

void crypt(int n, int level, int batch, int op, const uint32_t* x, uint64_t x_bs, const uint32_t* y, const uint32_t* z,
           const uint32_t* w, const uint32_t* u, uint32_t* out, uint64_t out_bs, const PrimeDev* primes,
           cudaStream_t st) {
  dim3 grid(cdiv(n, kT), level, batch);
  k_crypt<<<grid, kT, 0, st>>>(n, level, op, x, x_bs, y, z, w, u, out, out_bs, primes);
}

void evk_digit(int n, int rows, const uint32_t* s_src, const uint32_t* s_dst, const uint32_t* a, const uint32_t* e,
               const uint32_t* gm, const uint16_t* row_prime, int square, const PrimeDev* primes, uint32_t* out,
               cudaStream_t st) {
  dim3 grid(cdiv(n, kT), rows);
  k_evk_digit<<<grid, kT, 0, st>>>(n, s_src, s_dst, a, e, gm, row_prime, square, primes, out);
}

void reduce_coeffs(int n, int rows, const long long* c, const uint16_t* row_prime, const PrimeDev* primes,
                   uint32_t* out, cudaStream_t st) {
  dim3 grid(cdiv(n, kT), rows);
  k_reduce_coeffs<<<grid, kT, 0, st>>>(n, c, row_prime, primes, out);
}

void permute(int n, int rows, int batch, const uint32_t* in, uint64_t in_bs, uint32_t* out, uint64_t out_bs,
             const uint32_t* src_map, cudaStream_t st) {
  dim3 grid(cdiv(n, kT), rows, batch);
  k_permute<<<grid, kT, 0, st>>>(n, in, in_bs, out, out_bs, src_map);
}

void addmul(int n, int rows, int batch, uint32_t* acc, uint64_t acc_bs, const uint32_t* x, uint64_t x_bs,
            const uint32_t* y, uint64_t y_bs, const uint16_t* row_prime, const PrimeDev* primes, cudaStream_t st) {
  dim3 grid(cdiv(n, kT), rows, batch);
  k_addmul<<<grid, kT, 0, st>>>(n, acc, acc_bs, x, x_bs, y, y_bs, nullptr, row_prime, primes);
}

void addmul_permuted(int n, int rows, int batch, uint32_t* acc, uint64_t acc_bs, const uint32_t* x, uint64_t x_bs,
                     const uint32_t* y, uint64_t y_bs, const uint32_t* src_map, const uint16_t* row_prime,
                     const PrimeDev* primes, cudaStream_t st) {
  dim3 grid(cdiv(n, kT), rows, batch);
  k_addmul<<<grid, kT, 0, st>>>(n, acc, acc_bs, x, x_bs, y, y_bs, src_map, row_prime, primes);
}

}  // namespace ck
