// N = 2^16 NTT / INTT specialised for sm_100a (256 x 256 decomposition).
//
// Same transform as ntt.cpp:176-272 (and the generic kernels in ntt.cu), but
// every data movement is a full-width coalesced access and every twiddle is
// either a warp-broadcast or a coalesced load of a per-row table laid out in
// the order the threads consume it:
//
//  column pass (fwd stages 0-7, inverse stages 8-15 + exit):
//    a thread owns 4 adjacent columns (one uint4) x 16 rows.  Phase A reads
//    16 uint4 straight from HBM, runs 4 radix-2 stages on all 4 columns with
//    one twiddle per 4 butterflies, one smem transpose (uint4, conflict-free),
//    phase B runs the other 4 stages and writes 16 uint4 straight back.
//  row pass (fwd stages 8-15, inverse stages 0-7):
//    16 threads (half a warp) own one 256-point row, 16 elements each; the
//    exchange is a warp-local smem transpose (no CTA barrier).  The row's 30
//    twiddle pairs are held in registers and reused for every batch item of
//    the job (same prime), so twiddle traffic is amortised over the batch.
//
// Butterflies are Harvey-lazy Shoup (3 multiply-pipe ops each; IMAD.HI is
// quarter rate on sm_100a, see tools/microbench_int.cu): values in [0, 4q).
#include "ck_common.cuh"
#include "ck_kernels.h"

namespace ck {
namespace {

constexpr int kN = 65536;
constexpr int kR = 256;

__device__ __forceinline__ uint4 ldg4(const uint32_t* p) { return __ldg(reinterpret_cast<const uint4*>(p)); }
__device__ __forceinline__ void stg4(uint32_t* p, uint4 v) { *reinterpret_cast<uint4*>(p) = v; }

// forward CT butterfly on one lane, Harvey lazy: x,y in [0,4q) -> [0,4q)
__device__ __forceinline__ void ct(uint32_t& x, uint32_t& y, uint32_t w, uint32_t wp, uint32_t q, uint32_t q2) {
  const uint32_t xx = sub_if(x, q2);
  const uint32_t t = shoup_mul(y, w, wp, q);
  x = xx + t;
  y = xx - t + q2;
}
// inverse GS butterfly: x,y in [0,2q) -> [0,2q)
__device__ __forceinline__ void gs(uint32_t& x, uint32_t& y, uint32_t w, uint32_t wp, uint32_t q, uint32_t q2) {
  const uint32_t u = sub_if(x + y, q2);
  y = shoup_mul(x - y + q2, w, wp, q);
  x = u;
}
__device__ __forceinline__ void ct4(uint4& x, uint4& y, uint2 w, uint32_t q, uint32_t q2) {
  ct(x.x, y.x, w.x, w.y, q, q2);
  ct(x.y, y.y, w.x, w.y, q, q2);
  ct(x.z, y.z, w.x, w.y, q, q2);
  ct(x.w, y.w, w.x, w.y, q, q2);
}
__device__ __forceinline__ void gs4(uint4& x, uint4& y, uint2 w, uint32_t q, uint32_t q2) {
  gs(x.x, y.x, w.x, w.y, q, q2);
  gs(x.y, y.y, w.x, w.y, q, q2);
  gs(x.z, y.z, w.x, w.y, q, q2);
  gs(x.w, y.w, w.x, w.y, q, q2);
}

// Column tile: 256 rows x 64 columns; thread (tau = tid>>4, cq = tid&15).
constexpr int kColTileCols = 64;
constexpr int kColSmem = 256 * 16 * 16 + 256 * 8;  // uint4 tile + 256 twiddle pairs

// ------------------------------------------------------- forward, pass 1 --
__global__ void __launch_bounds__(256, 2) k_fwd_col(const RowJob* __restrict__ jobs, const uint32_t* __restrict__ src,
                                                    uint64_t src_bs, uint32_t* __restrict__ dst, uint64_t dst_bs,
                                                    int batch, const PrimeDev* __restrict__ primes,
                                                    const uint2* __restrict__ fwd_tw, int entry) {
  extern __shared__ uint4 smc[];
  uint4* tile = smc;                                   // [256][16]
  uint2* tw = reinterpret_cast<uint2*>(smc + 256 * 16);  // [256]
  const RowJob job = jobs[blockIdx.y];
  const PrimeDev P = primes[job.prime];
  const uint32_t q = P.q, q2 = P.q2;
  const int tid = threadIdx.x, cq = tid & 15, tau = tid >> 4;
  tw[tid] = __ldg(&fwd_tw[(size_t)job.prime * kN + tid]);
  const int c0 = blockIdx.x * kColTileCols + 4 * cq;
  __syncthreads();
  for (int b = 0; b < batch; ++b) {
    const uint32_t* g = src + b * src_bs + (size_t)job.src_off * kN + c0;
    uint32_t* o = dst + b * dst_bs + (size_t)job.dst_off * kN + c0;
    uint4 v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = ldg4(g + (tau + 16 * j) * kR);
    // phase A: stages 0..3, rows tau + 16j; twiddle 2^s + blk (shared by all threads)
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int d = 8 >> t;
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int blk = p / d, j = blk * 2 * d + p % d;
        const uint2 w = tw[(1 << t) + blk];
        {
          if (t == 0 && entry) {  // reference entry merge: x*R, y*psi^{N/2}*R (ntt.cpp:27-35)
            uint4& x = v[j];
            uint4& y = v[j + d];
#define CK_E(c)                                               \
  {                                                           \
    const uint32_t xx = shoup_mul(x.c, P.r, P.r_sh, q);       \
    const uint32_t tt = shoup_mul(y.c, P.w1r, P.w1r_sh, q);   \
    x.c = xx + tt;                                            \
    y.c = xx - tt + q2;                                       \
  }
            CK_E(x) CK_E(y) CK_E(z) CK_E(w)
#undef CK_E
          } else {
            ct4(v[j], v[j + d], w, q, q2);
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) tile[(tau + 16 * j) * 16 + cq] = v[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = tile[(16 * tau + j) * 16 + cq];
    // phase B: stages 4..7, rows 16 tau + j; twiddle 2^s + tau*2^(s-4) + blk
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int d = 8 >> t;
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int blk = p / d, j = blk * 2 * d + p % d;
        ct4(v[j], v[j + d], tw[(16 << t) + (tau << t) + blk], q, q2);
      }
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) stg4(o + (16 * tau + j) * kR, v[j]);
    __syncthreads();
  }
}

// ------------------------------------------------ inverse, pass B (columns) --
__global__ void __launch_bounds__(256) k_inv_col(const RowJob* __restrict__ jobs, uint32_t* __restrict__ dst,
                                                    uint64_t dst_bs, int batch, const PrimeDev* __restrict__ primes,
                                                    const uint2* __restrict__ inv_tw,
                                                    const ExitConst* __restrict__ exits) {
  extern __shared__ uint4 smc[];
  uint4* tile = smc;
  uint2* tw = reinterpret_cast<uint2*>(smc + 256 * 16);
  const RowJob job = jobs[blockIdx.y];
  const PrimeDev P = primes[job.prime];
  const ExitConst ex = exits[job.epi];
  const uint32_t q = P.q, q2 = P.q2;
  const int tid = threadIdx.x, cq = tid & 15, tau = tid >> 4;
  tw[tid] = __ldg(&inv_tw[(size_t)job.prime * kN + tid]);
  const int c0 = blockIdx.x * kColTileCols + 4 * cq;
  __syncthreads();
  for (int b = 0; b < batch; ++b) {
    uint32_t* o = dst + b * dst_bs + (size_t)job.dst_off * kN + c0;
    uint4 v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = ldg4(o + (16 * tau + j) * kR);
    // phase A: r bits 0..3 (global v = 8..11): twiddle 2^(7-t) + tau*2^(3-t) + blk
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int d = 1 << t;
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int blk = p / d, j = blk * 2 * d + p % d;
        gs4(v[j], v[j + d], tw[(128 >> t) + (tau << (3 - t)) + blk], q, q2);
      }
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) tile[(16 * tau + j) * 16 + cq] = v[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = tile[(tau + 16 * j) * 16 + cq];
    // phase B: r bits 4..7 (global v = 12..14), then the exit stage (v = 15)
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const int d = 1 << t;
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int blk = p / d, j = blk * 2 * d + p % d;
        gs4(v[j], v[j + d], tw[(8 >> t) + blk], q, q2);
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {  // exit merge (ntt.cpp:76-84): N^-1 R^-1 (x part1) constants
#define CK_X(c)                                                    \
  {                                                                \
    const uint32_t u = v[j].c + v[j + 8].c, dd = v[j].c - v[j + 8].c + q2; \
    v[j].c = sub_if(shoup_mul(u, ex.x, ex.y, q), q);               \
    v[j + 8].c = sub_if(shoup_mul(dd, ex.z, ex.w, q), q);          \
  }
      CK_X(x) CK_X(y) CK_X(z) CK_X(w)
#undef CK_X
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) stg4(o + (tau + 16 * j) * kR, v[j]);
    __syncthreads();
  }
}

// Row tile: 16 rows; the 16 threads of a row are one half-warp.
// smem position of element c in a row: c + 4*(c>>4) (conflict-free for both
// the stride-16 scalar and the contiguous uint4 access); row stride 336.
constexpr int kRowStride = 336;
__device__ __forceinline__ int rpos(int c) { return c + 4 * (c >> 4); }

// ------------------------------------------------------- forward, pass 2 --
__global__ void __launch_bounds__(256) k_fwd_row(const RowJob* __restrict__ jobs, uint32_t* __restrict__ dst,
                                                 uint64_t dst_bs, int batch, const PrimeDev* __restrict__ primes,
                                                 const uint2* __restrict__ tw2) {
  __shared__ __align__(16) uint32_t sm[16 * kRowStride];
  const RowJob job = jobs[blockIdx.y];
  const PrimeDev P = primes[job.prime];
  const uint32_t q = P.q, q2 = P.q2;
  const int tid = threadIdx.x, rho = tid >> 4, tau = tid & 15;
  const int r = blockIdx.x * 16 + rho;
  // per-row permuted twiddles: [0,15) phase A (shared by the row), 16 + k*16 + tau phase B
  const uint2* T = tw2 + ((size_t)job.prime * kR + r) * kR;
  uint2 wa[15], wb[15];
#pragma unroll
  for (int k = 0; k < 15; ++k) {
    wa[k] = __ldg(&T[k]);
    wb[k] = __ldg(&T[16 + k * 16 + tau]);
  }
  uint32_t* line = sm + rho * kRowStride;
  for (int b = 0; b < batch; ++b) {
    uint32_t* row = dst + b * dst_bs + (size_t)job.dst_off * kN + (size_t)r * kR;
    uint32_t v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = row[tau + 16 * j];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int d = 8 >> t;
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int blk = p / d, j = blk * 2 * d + p % d;
        const uint2 w = wa[(1 << t) - 1 + blk];
        ct(v[j], v[j + d], w.x, w.y, q, q2);
      }
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) line[rpos(tau + 16 * j)] = v[j];
    __syncwarp();
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const uint4 x = *reinterpret_cast<const uint4*>(line + rpos(16 * tau) + 4 * m);
      v[4 * m] = x.x;
      v[4 * m + 1] = x.y;
      v[4 * m + 2] = x.z;
      v[4 * m + 3] = x.w;
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int d = 8 >> t;
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int blk = p / d, j = blk * 2 * d + p % d;
        const uint2 w = wb[(1 << t) - 1 + blk];
        ct(v[j], v[j + d], w.x, w.y, q, q2);
      }
    }
#pragma unroll
    for (int m = 0; m < 4; ++m)
      stg4(row + 16 * tau + 4 * m, make_uint4(canon4(v[4 * m], q, q2), canon4(v[4 * m + 1], q, q2),
                                              canon4(v[4 * m + 2], q, q2), canon4(v[4 * m + 3], q, q2)));
  }
}

// ------------------------------------------------- inverse, pass A (rows) --
__global__ void __launch_bounds__(256) k_inv_row(const RowJob* __restrict__ jobs, const uint32_t* __restrict__ src,
                                                 uint64_t src_bs, uint32_t* __restrict__ dst, uint64_t dst_bs,
                                                 int batch, const PrimeDev* __restrict__ primes,
                                                 const uint2* __restrict__ tw2i) {
  __shared__ __align__(16) uint32_t sm[16 * kRowStride];
  const RowJob job = jobs[blockIdx.y];
  const PrimeDev P = primes[job.prime];
  const uint32_t q = P.q, q2 = P.q2;
  const int tid = threadIdx.x, rho = tid >> 4, tau = tid & 15;
  const int r = blockIdx.x * 16 + rho;
  // per-row permuted inverse twiddles: k*16 + tau (phase A, k < 15), 240 + k (phase B)
  const uint2* T = tw2i + ((size_t)job.prime * kR + r) * kR;
  uint2 wa[15], wb[15];
#pragma unroll
  for (int k = 0; k < 15; ++k) {
    wa[k] = __ldg(&T[k * 16 + tau]);
    wb[k] = __ldg(&T[240 + k]);
  }
  uint32_t* line = sm + rho * kRowStride;
  for (int b = 0; b < batch; ++b) {
    const uint32_t* in = src + b * src_bs + (size_t)job.src_off * kN + (size_t)r * kR;
    uint32_t* out = dst + b * dst_bs + (size_t)job.dst_off * kN + (size_t)r * kR;
    uint32_t v[16];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const uint4 x = ldg4(in + 16 * tau + 4 * m);
      v[4 * m] = x.x;
      v[4 * m + 1] = x.y;
      v[4 * m + 2] = x.z;
      v[4 * m + 3] = x.w;
    }
    // phase A: c bits 0..3; block offsets 0, 8, 12, 14
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int d = 1 << t;
      const int off = 16 - (16 >> t);
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int blk = p / d, j = blk * 2 * d + p % d;
        const uint2 w = wa[off + blk];
        gs(v[j], v[j + d], w.x, w.y, q, q2);
      }
    }
#pragma unroll
    for (int m = 0; m < 4; ++m)
      *reinterpret_cast<uint4*>(line + rpos(16 * tau) + 4 * m) =
          make_uint4(v[4 * m], v[4 * m + 1], v[4 * m + 2], v[4 * m + 3]);
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = line[rpos(tau + 16 * j)];
    __syncwarp();
    // phase B: c bits 4..7
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int d = 1 << t;
      const int off = 16 - (16 >> t);
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int blk = p / d, j = blk * 2 * d + p % d;
        const uint2 w = wb[off + blk];
        gs(v[j], v[j + d], w.x, w.y, q, q2);
      }
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) out[tau + 16 * j] = v[j];
  }
}

}  // namespace

bool ntt256_forward(const NttLaunch& a, const uint2* tw2, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_fwd_col, cudaFuncAttributeMaxDynamicSharedMemorySize, kColSmem);
    cudaFuncSetAttribute(k_inv_col, cudaFuncAttributeMaxDynamicSharedMemorySize, kColSmem);
    attr = true;
  }
  k_fwd_col<<<dim3(kR / kColTileCols, a.njobs), 256, kColSmem, st>>>(a.jobs, a.src, a.src_bs, a.dst, a.dst_bs,
                                                                      a.batch, a.primes, a.tw, a.entry);
  k_fwd_row<<<dim3(kR / 16, a.njobs), 256, 0, st>>>(a.jobs, a.dst, a.dst_bs, a.batch, a.primes, tw2);
  return true;
}

bool ntt256_inverse(const NttLaunch& a, const uint2* tw2i, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_fwd_col, cudaFuncAttributeMaxDynamicSharedMemorySize, kColSmem);
    cudaFuncSetAttribute(k_inv_col, cudaFuncAttributeMaxDynamicSharedMemorySize, kColSmem);
    attr = true;
  }
  k_inv_row<<<dim3(kR / 16, a.njobs), 256, 0, st>>>(a.jobs, a.src, a.src_bs, a.dst, a.dst_bs, a.batch, a.primes,
                                                     tw2i);
  k_inv_col<<<dim3(kR / kColTileCols, a.njobs), 256, kColSmem, st>>>(a.jobs, a.dst, a.dst_bs, a.batch, a.primes,
                                                                      a.tw, a.exits);
  return true;
}

}  // namespace ck
