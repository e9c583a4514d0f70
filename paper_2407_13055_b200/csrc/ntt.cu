// Batched negacyclic NTT / INTT for sm_100a.
//
// Restates the reference transforms (NttPlan::forward_row / inverse_row,
// ntt.cpp:176-272, serial form ntt.cpp:274-286) B200-first:
//   * an N = N1 x N2 two-pass decomposition (pass 1: N1-point column lines,
//     pass 2: N2-point row lines), one CTA per 4096-word tile, the tile held
//     in shared memory and processed in register phases of <= 4 radix-2
//     stages (radix-16 butterfly blocks per thread);
//   * Harvey-lazy Shoup butterflies (twiddle pair {w, floor(w*2^32/q)} per
//     table entry), values in [0, 4q) between stages; the reference's
//     entry merge (x*R, y*psi^{N/2}*R at stage 0, ntt.cpp:27-35) and the exit
//     merge (N^-1, psi^{-N/2} N^-1 plus the fused BConv part-1 constant,
//     ntt.cpp:76-84) are folded into Shoup constants;
//   * batched over a job list (row -> prime, exit slot) and a batch grid
//     dimension so one launch covers every row of a mechanism step.
// Twiddle index convention is the reference's (ntt.cpp:109-133): forward
// stage S group g uses psi^{brev(2^S + g)}, inverse stage v group g uses
// psi^{-brev(N/2^{v+1} + g)}.
#include <cstdio>

#include "ck_common.cuh"
#include "ck_kernels.h"

namespace ck {
namespace {

constexpr int kTile = 4096;
constexpr int kThreads = 256;

constexpr int cmin(int a, int b) { return a < b ? a : b; }
constexpr int cmax(int a, int b) { return a > b ? a : b; }
constexpr int nphases(int k) { return (k + 3) / 4; }
// start bit of phase p when k bits are split into near-equal phases of <= 4
constexpr int phase_start(int k, int p) {
  return p * (k / nphases(k)) + cmin(p, k % nphases(k));
}

template <int K1, int K2>
struct Shape {
  static constexpr int N1 = 1 << K1, N2 = 1 << K2;
  static constexpr int N = N1 * N2;
  static constexpr int TC = cmax(1, cmin(N2, kTile / N1));  // columns per pass-1 tile
  static constexpr int TCP = TC + (TC >= 16 ? 1 : 0);        // padded smem row stride
  static constexpr int TR = cmax(1, cmin(N1, kTile / N2));  // rows per pass-2 tile
  static constexpr int N2P = N2 + (N2 >= 32 ? 16 : 0);       // padded smem row stride
};

__device__ __forceinline__ int swz(int c, int n2) { return c ^ ((c >> 4) & 15 & (n2 - 1)); }

// ---- forward (DIF Cooley-Tukey, twiddle on y) on a register block ------------
// Local stages [S0, S1) of a line transform whose global stage offset is GOFF.
// Twiddle index for local stage s, block blk: 2^(GOFF+s) + prefix*2^s + hi*2^(s-S0) + blk.
template <int S0, int S1, int GOFF>
__device__ __forceinline__ void fwd_block(uint32_t (&v)[1 << (S1 - S0)], const uint2* __restrict__ tw,
                                          uint32_t prefix, uint32_t hi, uint32_t q, uint32_t q2,
                                          bool entry, const PrimeDev& P) {
  constexpr int E = 1 << (S1 - S0);
#pragma unroll
  for (int s = S0; s < S1; ++s) {
    const int b = S1 - 1 - s;  // pair distance 2^b inside the block
    const uint32_t tbase = (1u << (GOFF + s)) + (prefix << s) + (hi << (s - S0));
#pragma unroll
    for (int blk = 0; blk < (1 << (s - S0)); ++blk) {
      uint32_t w, wp;
      const bool ent = (GOFF + s == 0) && entry;
      if (ent) {
        w = P.w1r;
        wp = P.w1r_sh;
      } else {
        const uint2 t = __ldg(&tw[tbase + blk]);
        w = t.x;
        wp = t.y;
      }
#pragma unroll
      for (int jj = 0; jj < (1 << b); ++jj) {
        const int j = blk * (2 << b) + jj;
        uint32_t x = v[j];
        const uint32_t y = v[j + (1 << b)];
        if (ent)
          x = shoup_mul(x, P.r, P.r_sh, q);  // x*R, [0, 2q)
        else
          x = sub_if(x, q2);  // [0, 4q) -> [0, 2q)
        const uint32_t t = shoup_mul(y, w, wp, q);
        v[j] = x + t;                    // [0, 4q)
        v[j + (1 << b)] = x - t + q2;    // (0, 4q)
      }
    }
  }
  (void)E;
}

// ---- inverse (DIT Gentleman-Sande) on a register block ------------------------
// Local bit stages [V0, V1) of a line of 2^KL points, global stage offset VOFF.
// Twiddle index: 2^(LOGN-1-v) + prefix*2^(KL-1-vl) + hi*2^(V1-vl-1) + blk.
template <int V0, int V1, int KL, int VOFF, int LOGN>
__device__ __forceinline__ void inv_block(uint32_t (&v)[1 << (V1 - V0)], const uint2* __restrict__ tw,
                                          uint32_t prefix, uint32_t hi, uint32_t q, uint32_t q2,
                                          const ExitConst& ex) {
#pragma unroll
  for (int vl = V0; vl < V1; ++vl) {
    const int b = vl - V0;
    const int gv = VOFF + vl;
    const bool exit_stage = gv == LOGN - 1;
    const uint32_t tbase = (1u << (LOGN - 1 - gv)) + (prefix << (KL - 1 - vl)) + (hi << (V1 - vl - 1));
#pragma unroll
    for (int blk = 0; blk < (1 << (V1 - vl - 1)); ++blk) {
      uint2 t = make_uint2(0, 0);
      if (!exit_stage) t = __ldg(&tw[tbase + blk]);
#pragma unroll
      for (int jj = 0; jj < (1 << b); ++jj) {
        const int j = blk * (2 << b) + jj;
        const uint32_t x = v[j], y = v[j + (1 << b)];
        if (exit_stage) {
          const uint32_t u = x + y;         // [0, 4q)
          const uint32_t d = x - y + q2;    // (0, 4q)
          v[j] = sub_if(shoup_mul(u, ex.x, ex.y, q), q);             // canonical
          v[j + (1 << b)] = sub_if(shoup_mul(d, ex.z, ex.w, q), q);  // canonical
        } else {
          v[j] = sub_if(x + y, q2);                       // [0, 2q)
          v[j + (1 << b)] = shoup_mul(x - y + q2, t.x, t.y, q);  // [0, 2q)
        }
      }
    }
  }
}

// ---- pass 1 / pass B: column lines (line index = row r in [0, N1)) ---------------
template <int K1, int K2, int P>
__device__ __forceinline__ void col_phase_fwd(uint32_t* sm, const uint2* tw, uint32_t q, uint32_t q2,
                                              bool entry, const PrimeDev& PD) {
  using S = Shape<K1, K2>;
  constexpr int S0 = phase_start(K1, P), S1 = phase_start(K1, P + 1);
  constexpr int E = 1 << (S1 - S0), LOW = K1 - S1;
  constexpr int UNITS = S::TC * (S::N1 / E);
  for (int u = threadIdx.x; u < UNITS; u += kThreads) {
    const int c = u % S::TC, tau = u / S::TC;
    const int lo = tau & ((1 << LOW) - 1), hi = tau >> LOW;
    const int base = (hi << (K1 - S0)) + lo;
    uint32_t v[E];
#pragma unroll
    for (int j = 0; j < E; ++j) v[j] = sm[(base + (j << LOW)) * S::TCP + c];
    fwd_block<S0, S1, 0>(v, tw, 0u, (uint32_t)hi, q, q2, entry, PD);
#pragma unroll
    for (int j = 0; j < E; ++j) sm[(base + (j << LOW)) * S::TCP + c] = v[j];
  }
}

template <int K1, int K2, int P>
__device__ __forceinline__ void col_phase_inv(uint32_t* sm, const uint2* tw, uint32_t q, uint32_t q2,
                                              const ExitConst& ex) {
  using S = Shape<K1, K2>;
  constexpr int V0 = phase_start(K1, P), V1 = phase_start(K1, P + 1);
  constexpr int E = 1 << (V1 - V0);
  constexpr int UNITS = S::TC * (S::N1 / E);
  for (int u = threadIdx.x; u < UNITS; u += kThreads) {
    const int c = u % S::TC, tau = u / S::TC;
    const int lo = tau & ((1 << V0) - 1), hi = tau >> V0;
    const int base = (hi << V1) + lo;
    uint32_t v[E];
#pragma unroll
    for (int j = 0; j < E; ++j) v[j] = sm[(base + (j << V0)) * S::TCP + c];
    inv_block<V0, V1, K1, K2, K1 + K2>(v, tw, 0u, (uint32_t)hi, q, q2, ex);
#pragma unroll
    for (int j = 0; j < E; ++j) sm[(base + (j << V0)) * S::TCP + c] = v[j];
  }
}

// ---- pass 2 / pass A: row lines (line index = column c in [0, N2)) ----------------
template <int K1, int K2, int P>
__device__ __forceinline__ void row_phase_fwd(uint32_t* sm, const uint2* tw, uint32_t row0, uint32_t q,
                                              uint32_t q2, const PrimeDev& PD) {
  using S = Shape<K1, K2>;
  constexpr int S0 = phase_start(K2, P), S1 = phase_start(K2, P + 1);
  constexpr int E = 1 << (S1 - S0), LOW = K2 - S1;
  constexpr int PER_LINE = S::N2 / E;
  constexpr int UNITS = S::TR * PER_LINE;
  for (int u = threadIdx.x; u < UNITS; u += kThreads) {
    const int rho = u / PER_LINE, tau = u % PER_LINE;
    const int lo = tau & ((1 << LOW) - 1), hi = tau >> LOW;
    const int base = (hi << (K2 - S0)) + lo;
    uint32_t* line = sm + rho * S::N2P;
    uint32_t v[E];
#pragma unroll
    for (int j = 0; j < E; ++j) v[j] = line[swz(base + (j << LOW), S::N2)];
    fwd_block<S0, S1, K1>(v, tw, row0 + rho, (uint32_t)hi, q, q2, false, PD);
#pragma unroll
    for (int j = 0; j < E; ++j) line[swz(base + (j << LOW), S::N2)] = v[j];
  }
}

template <int K1, int K2, int P>
__device__ __forceinline__ void row_phase_inv(uint32_t* sm, const uint2* tw, uint32_t row0, uint32_t q,
                                              uint32_t q2) {
  using S = Shape<K1, K2>;
  constexpr int V0 = phase_start(K2, P), V1 = phase_start(K2, P + 1);
  constexpr int E = 1 << (V1 - V0);
  constexpr int PER_LINE = S::N2 / E;
  constexpr int UNITS = S::TR * PER_LINE;
  const ExitConst none = make_uint4(0, 0, 0, 0);
  for (int u = threadIdx.x; u < UNITS; u += kThreads) {
    const int rho = u / PER_LINE, tau = u % PER_LINE;
    const int lo = tau & ((1 << V0) - 1), hi = tau >> V0;
    const int base = (hi << V1) + lo;
    uint32_t* line = sm + rho * S::N2P;
    uint32_t v[E];
#pragma unroll
    for (int j = 0; j < E; ++j) v[j] = line[swz(base + (j << V0), S::N2)];
    inv_block<V0, V1, K2, 0, K1 + K2>(v, tw, row0 + rho, (uint32_t)hi, q, q2, none);
#pragma unroll
    for (int j = 0; j < E; ++j) line[swz(base + (j << V0), S::N2)] = v[j];
  }
}

template <int K, class F, int P = 0>
__device__ __forceinline__ void for_phases(F&& f) {
  if constexpr (P < nphases(K)) {
    f(std::integral_constant<int, P>{});
    __syncthreads();
    for_phases<K, F, P + 1>(static_cast<F&&>(f));
  }
}

// Column-tile copies between global (row stride N2) and smem (row stride TCP).
template <int K1, int K2>
__device__ __forceinline__ void col_load(uint32_t* sm, const uint32_t* __restrict__ g, int c0) {
  using S = Shape<K1, K2>;
  if constexpr (S::TC % 4 == 0) {
    for (int e = threadIdx.x; e < S::N1 * S::TC / 4; e += kThreads) {
      const int r = e / (S::TC / 4), c = (e % (S::TC / 4)) * 4;
      const uint4 x = *reinterpret_cast<const uint4*>(g + (size_t)r * S::N2 + c0 + c);
      uint32_t* d = sm + r * S::TCP + c;
      d[0] = x.x; d[1] = x.y; d[2] = x.z; d[3] = x.w;
    }
  } else {
    for (int e = threadIdx.x; e < S::N1 * S::TC; e += kThreads) {
      const int r = e / S::TC, c = e % S::TC;
      sm[r * S::TCP + c] = g[(size_t)r * S::N2 + c0 + c];
    }
  }
}
template <int K1, int K2>
__device__ __forceinline__ void col_store(const uint32_t* sm, uint32_t* __restrict__ g, int c0) {
  using S = Shape<K1, K2>;
  if constexpr (S::TC % 4 == 0) {
    for (int e = threadIdx.x; e < S::N1 * S::TC / 4; e += kThreads) {
      const int r = e / (S::TC / 4), c = (e % (S::TC / 4)) * 4;
      const uint32_t* s = sm + r * S::TCP + c;
      *reinterpret_cast<uint4*>(g + (size_t)r * S::N2 + c0 + c) = make_uint4(s[0], s[1], s[2], s[3]);
    }
  } else {
    for (int e = threadIdx.x; e < S::N1 * S::TC; e += kThreads) {
      const int r = e / S::TC, c = e % S::TC;
      g[(size_t)r * S::N2 + c0 + c] = sm[r * S::TCP + c];
    }
  }
}
template <int K1, int K2>
__device__ __forceinline__ void row_load(uint32_t* sm, const uint32_t* __restrict__ g) {
  using S = Shape<K1, K2>;
  if constexpr (S::N2 % 4 == 0) {
    for (int e = threadIdx.x; e < S::TR * S::N2 / 4; e += kThreads) {
      const int r = e / (S::N2 / 4), c = (e % (S::N2 / 4)) * 4;
      const uint4 x = *reinterpret_cast<const uint4*>(g + (size_t)r * S::N2 + c);
      uint32_t* line = sm + r * S::N2P;
      line[swz(c, S::N2)] = x.x;
      line[swz(c + 1, S::N2)] = x.y;
      line[swz(c + 2, S::N2)] = x.z;
      line[swz(c + 3, S::N2)] = x.w;
    }
  } else {
    for (int e = threadIdx.x; e < S::TR * S::N2; e += kThreads) {
      const int r = e / S::N2, c = e % S::N2;
      sm[r * S::N2P + swz(c, S::N2)] = g[(size_t)r * S::N2 + c];
    }
  }
}
// final store with an optional [0, 4q) -> [0, q) canonicalisation
template <int K1, int K2, bool CANON>
__device__ __forceinline__ void row_store(const uint32_t* sm, uint32_t* __restrict__ g, uint32_t q,
                                          uint32_t q2) {
  using S = Shape<K1, K2>;
  auto fix = [&](uint32_t x) { return CANON ? canon4(x, q, q2) : x; };
  if constexpr (S::N2 % 4 == 0) {
    for (int e = threadIdx.x; e < S::TR * S::N2 / 4; e += kThreads) {
      const int r = e / (S::N2 / 4), c = (e % (S::N2 / 4)) * 4;
      const uint32_t* line = sm + r * S::N2P;
      *reinterpret_cast<uint4*>(g + (size_t)r * S::N2 + c) =
          make_uint4(fix(line[swz(c, S::N2)]), fix(line[swz(c + 1, S::N2)]), fix(line[swz(c + 2, S::N2)]),
                     fix(line[swz(c + 3, S::N2)]));
    }
  } else {
    for (int e = threadIdx.x; e < S::TR * S::N2; e += kThreads) {
      const int r = e / S::N2, c = e % S::N2;
      g[(size_t)r * S::N2 + c] = fix(sm[r * S::N2P + swz(c, S::N2)]);
    }
  }
}

// ---------------------------------------------------------------- kernels ----
template <int K1, int K2>
__global__ void __launch_bounds__(kThreads) k_ntt_fwd_p1(const RowJob* __restrict__ jobs,
                                                         const uint32_t* __restrict__ src, uint64_t src_bs,
                                                         uint32_t* __restrict__ dst, uint64_t dst_bs,
                                                         const PrimeDev* __restrict__ primes,
                                                         const uint2* __restrict__ fwd_tw, int entry) {
  using S = Shape<K1, K2>;
  __shared__ uint32_t sm[S::N1 * S::TCP];
  const RowJob job = jobs[blockIdx.y];
  const uint32_t* g = src + blockIdx.z * src_bs + (size_t)job.src_off * S::N;
  uint32_t* o = dst + blockIdx.z * dst_bs + (size_t)job.dst_off * S::N;
  const int c0 = blockIdx.x * S::TC;
  const PrimeDev PD = primes[job.prime];
  const uint2* tw = fwd_tw + (size_t)job.prime * S::N;
  col_load<K1, K2>(sm, g, c0);
  __syncthreads();
  for_phases<K1>([&](auto p) { col_phase_fwd<K1, K2, decltype(p)::value>(sm, tw, PD.q, PD.q2, entry != 0, PD); });
  col_store<K1, K2>(sm, o, c0);
}

template <int K1, int K2>
__global__ void __launch_bounds__(kThreads) k_ntt_fwd_p2(const RowJob* __restrict__ jobs, uint32_t* __restrict__ dst,
                                                         uint64_t dst_bs, const PrimeDev* __restrict__ primes,
                                                         const uint2* __restrict__ fwd_tw) {
  using S = Shape<K1, K2>;
  __shared__ uint32_t sm[S::TR * S::N2P];
  const RowJob job = jobs[blockIdx.y];
  const int r0 = blockIdx.x * S::TR;
  uint32_t* o = dst + blockIdx.z * dst_bs + (size_t)job.dst_off * S::N + (size_t)r0 * S::N2;
  const PrimeDev PD = primes[job.prime];
  const uint2* tw = fwd_tw + (size_t)job.prime * S::N;
  row_load<K1, K2>(sm, o);
  __syncthreads();
  for_phases<K2>([&](auto p) { row_phase_fwd<K1, K2, decltype(p)::value>(sm, tw, (uint32_t)r0, PD.q, PD.q2, PD); });
  row_store<K1, K2, true>(sm, o, PD.q, PD.q2);
}

template <int K1, int K2>
__global__ void __launch_bounds__(kThreads) k_intt_pA(const RowJob* __restrict__ jobs,
                                                      const uint32_t* __restrict__ src, uint64_t src_bs,
                                                      uint32_t* __restrict__ dst, uint64_t dst_bs,
                                                      const PrimeDev* __restrict__ primes,
                                                      const uint2* __restrict__ inv_tw) {
  using S = Shape<K1, K2>;
  __shared__ uint32_t sm[S::TR * S::N2P];
  const RowJob job = jobs[blockIdx.y];
  const int r0 = blockIdx.x * S::TR;
  const uint32_t* g = src + blockIdx.z * src_bs + (size_t)job.src_off * S::N + (size_t)r0 * S::N2;
  uint32_t* o = dst + blockIdx.z * dst_bs + (size_t)job.dst_off * S::N + (size_t)r0 * S::N2;
  const PrimeDev PD = primes[job.prime];
  const uint2* tw = inv_tw + (size_t)job.prime * S::N;
  row_load<K1, K2>(sm, g);
  __syncthreads();
  for_phases<K2>([&](auto p) { row_phase_inv<K1, K2, decltype(p)::value>(sm, tw, (uint32_t)r0, PD.q, PD.q2); });
  row_store<K1, K2, false>(sm, o, PD.q, PD.q2);
}

template <int K1, int K2>
__global__ void __launch_bounds__(kThreads) k_intt_pB(const RowJob* __restrict__ jobs, uint32_t* __restrict__ dst,
                                                      uint64_t dst_bs, const PrimeDev* __restrict__ primes,
                                                      const uint2* __restrict__ inv_tw,
                                                      const ExitConst* __restrict__ exits) {
  using S = Shape<K1, K2>;
  __shared__ uint32_t sm[S::N1 * S::TCP];
  const RowJob job = jobs[blockIdx.y];
  uint32_t* o = dst + blockIdx.z * dst_bs + (size_t)job.dst_off * S::N;
  const int c0 = blockIdx.x * S::TC;
  const PrimeDev PD = primes[job.prime];
  const uint2* tw = inv_tw + (size_t)job.prime * S::N;
  const ExitConst ex = exits[job.epi];
  col_load<K1, K2>(sm, o, c0);
  __syncthreads();
  for_phases<K1>([&](auto p) { col_phase_inv<K1, K2, decltype(p)::value>(sm, tw, PD.q, PD.q2, ex); });
  col_store<K1, K2>(sm, o, c0);
}

template <int LOGN>
void launch_fwd(const NttLaunch& a, cudaStream_t st) {
  constexpr int K1 = LOGN / 2, K2 = LOGN - K1;
  using S = Shape<K1, K2>;
  dim3 g1(S::N2 / S::TC, a.njobs, a.batch), g2(S::N1 / S::TR, a.njobs, a.batch);
  k_ntt_fwd_p1<K1, K2><<<g1, kThreads, 0, st>>>(a.jobs, a.src, a.src_bs, a.dst, a.dst_bs, a.primes, a.tw, a.entry);
  k_ntt_fwd_p2<K1, K2><<<g2, kThreads, 0, st>>>(a.jobs, a.dst, a.dst_bs, a.primes, a.tw);
}
template <int LOGN>
void launch_inv(const NttLaunch& a, cudaStream_t st) {
  constexpr int K1 = LOGN / 2, K2 = LOGN - K1;
  using S = Shape<K1, K2>;
  dim3 g1(S::N1 / S::TR, a.njobs, a.batch), g2(S::N2 / S::TC, a.njobs, a.batch);
  k_intt_pA<K1, K2><<<g1, kThreads, 0, st>>>(a.jobs, a.src, a.src_bs, a.dst, a.dst_bs, a.primes, a.tw);
  k_intt_pB<K1, K2><<<g2, kThreads, 0, st>>>(a.jobs, a.dst, a.dst_bs, a.primes, a.tw, a.exits);
}

}  // namespace

void ntt_forward(int logn, const NttLaunch& a, cudaStream_t st) {
  switch (logn) {
#define CK_CASE(L) case L: launch_fwd<L>(a, st); break;
    CK_CASE(3) CK_CASE(4) CK_CASE(5) CK_CASE(6) CK_CASE(7) CK_CASE(8) CK_CASE(9) CK_CASE(10) CK_CASE(11)
    CK_CASE(12) CK_CASE(13) CK_CASE(14) CK_CASE(15) CK_CASE(16) CK_CASE(17)
#undef CK_CASE
    default: break;
  }
}
void ntt_inverse(int logn, const NttLaunch& a, cudaStream_t st) {
  switch (logn) {
#define CK_CASE(L) case L: launch_inv<L>(a, st); break;
    CK_CASE(3) CK_CASE(4) CK_CASE(5) CK_CASE(6) CK_CASE(7) CK_CASE(8) CK_CASE(9) CK_CASE(10) CK_CASE(11)
    CK_CASE(12) CK_CASE(13) CK_CASE(14) CK_CASE(15) CK_CASE(16) CK_CASE(17)
#undef CK_CASE
    default: break;
  }
}

}  // namespace ck
