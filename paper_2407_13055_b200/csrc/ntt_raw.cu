// The reference's NTT in its RAW representation (ntt.cpp:15-96): signed
// lazy int32 values, signed Montgomery reduction (modarith.hpp:20-36), the
// (-2q, 2q) narrowing after every stage, the entry merge (x R, y psi^{N/2} R)
// and the tightened last stage of the forward transform, the exit constants
// (+ optional part-1 epilogue) of the inverse -- butterfly for butterfly, so
// the int32 rows equal the reference's forward_row_serial / inverse_row_serial
// (and therefore every NttPlan of the reference, which are bit-identical to
// them by construction: test_ntt.cpp:203-227).
//
// Compatibility mode for callers that compare raw rows; the product path
// works on canonical residues (ntt256.cu, ntt.cu).  Every butterfly's result
// depends only on its two inputs and the formula, so one launch per stage
// (one thread per butterfly, global memory) reproduces the serial order
// exactly; nothing here is tuned.
#include "ck_common.cuh"
#include "ck_kernels.h"

namespace ck {
namespace {

__device__ __forceinline__ int32_t mred_s(int64_t a, int32_t q, uint32_t m) {  // modarith.hpp:20-29
  const int32_t hi = (int32_t)(a >> 32);
  const int32_t t = (int32_t)((uint32_t)a * m);
  return hi - (int32_t)(((int64_t)t * q) >> 32);
}
__device__ __forceinline__ int64_t narrow_s(int64_t v, int64_t b) {
  if (v >= b) v -= b;
  else if (v <= -b) v += b;
  return v;
}

// the reference table's Montgomery-form twiddle psi^brev(i) R mod q (canonical)
// from the library's plain table entry {w, w'}
__device__ __forceinline__ int32_t tw_mont(uint2 w, const PrimeDev& P) {
  return (int32_t)sub_if(shoup_mul(w.x, P.r, P.r_sh, P.q), P.q);
}

__global__ void k_ntt_raw_stage(int32_t* __restrict__ d, int n, int logn, int s, int inv,
                                const uint16_t* __restrict__ gidx, const PrimeDev* __restrict__ primes,
                                const RawNttConst* __restrict__ rc, const uint2* __restrict__ tw,
                                const uint32_t* __restrict__ epi) {
  const int bfly = blockIdx.x * blockDim.x + threadIdx.x;
  if (bfly >= n / 2) return;
  const int row = blockIdx.y;
  const int g_ = gidx[row];
  const PrimeDev P = primes[g_];
  const RawNttConst C = rc[g_];
  const int32_t q = (int32_t)P.q;
  const int64_t q2 = 2 * (int64_t)q;
  int32_t* r = d + (size_t)row * n;
  if (!inv) {  // fwd_stages, stage s (m = 2^s, t = n >> (s + 1)), entry merge at s = 0, tightened last stage
    const int t = n >> (s + 1), g = bfly / t, j = bfly - g * t, m = 1 << s;
    int32_t* px = r + 2 * g * t + j;
    int32_t* py = px + t;
    int32_t x = *px;
    const int32_t w = s == 0 ? C.fwd1_r2 : tw_mont(tw[(size_t)g_ * n + m + g], P);
    const int32_t y = mred_s((int64_t)*py * w, q, P.qinv);
    if (s == 0) x = mred_s((int64_t)x * C.r2, q, P.qinv);
    int64_t u = narrow_s((int64_t)x + y, q2), v = narrow_s((int64_t)x - y, q2);
    if (s == logn - 1) {
      u = narrow_s(u, q);
      v = narrow_s(v, q);
    }
    *px = (int32_t)u;
    *py = (int32_t)v;
  } else {  // inv_stages, stage s (m = n >> (1 + s), t = 2^s), exit constants at m = 1
    const int m = n >> (1 + s), t = 1 << s, g = bfly / t, j = bfly - g * t;
    int32_t* px = r + 2 * g * t + j;
    int32_t* py = px + t;
    const int32_t x = *px, y = *py;
    const int64_t u = (int64_t)x + y, v2 = (int64_t)x - y;
    if (m == 1) {
      int32_t a0 = mred_s(u * C.exit_x, q, P.qinv), a1 = mred_s(v2 * C.exit_y, q, P.qinv);
      if (epi && epi[row]) {  // correct_lazy(mont_mul(a, epilogue)) -> [0, q)
        const int32_t e = (int32_t)epi[row];
        a0 = mred_s((int64_t)a0 * e, q, P.qinv);
        a1 = mred_s((int64_t)a1 * e, q, P.qinv);
        a0 = a0 < 0 ? a0 + q : a0;
        a1 = a1 < 0 ? a1 + q : a1;
      }
      *px = a0;
      *py = a1;
    } else {
      const int32_t w = tw_mont(tw[(size_t)g_ * n + m + g], P);
      *px = (int32_t)narrow_s(u, q2);
      *py = mred_s(v2 * w, q, P.qinv);
    }
  }
}

}  // namespace

void ntt_raw(int n, int logn, int rows, int inverse, int32_t* d, const uint16_t* gidx, const PrimeDev* primes,
             const RawNttConst* rc, const uint2* tw, const uint32_t* epi, cudaStream_t st) {
  dim3 grid((n / 2 + 255) / 256, rows);
  for (int s = 0; s < logn; ++s)
    k_ntt_raw_stage<<<grid, 256, 0, st>>>(d, n, logn, s, inverse, gidx, primes, rc, tw, epi);
}

}  // namespace ck
