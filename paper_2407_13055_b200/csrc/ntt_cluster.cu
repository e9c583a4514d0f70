// Single-pass N = 2^16 NTT / INTT on 8-CTA thread-block clusters (sm_100a).
//
// Same transform as ntt.cpp:176-272 (256 x 256 decomposition as ntt256.cu),
// but each limb crosses HBM exactly once in each direction: the pass-1 /
// pass-2 transpose goes through distributed shared memory instead of HBM.
//
//   cluster of 8 CTAs, CTA rank k:
//   forward  — pass 1 on columns [32k, 32k+32) of the limb (all 256 rows, in
//              its own smem), cluster barrier, pass 2 on rows [32k, 32k+32)
//              reading 7/8 of each row from the 7 peers' smem (DSMEM),
//              cluster barrier (the block may be refilled);
//   inverse  — pass A on rows [32k, 32k+32), cluster barrier, pass B (+exit,
//              +BConv part 1) on columns [32k, 32k+32) reading from peers,
//              cluster barrier.
// A CTA needs < 80 KB of shared memory and <= 128 registers per thread so two
// CTAs of different clusters share an SM: one cluster's loads and barriers
// overlap the other's butterflies.  Row-pass twiddles are read from the
// per-row permuted tables in L2 (warp-broadcast / coalesced).
#include <algorithm>

#include <cooperative_groups.h>

#include "ck_common.cuh"
#include "ck_kernels.h"

namespace cg = cooperative_groups;

namespace ck {
namespace {

constexpr int kN = 65536, kR = 256, kCl = 8, kB = 32, kT = 256;
constexpr int kRS = 336;  // padded row stride (words) for row-layout tiles: c -> c + 4*(c>>4)

__device__ __forceinline__ int rp(int c) { return c + 4 * (c >> 4); }
__device__ __forceinline__ void stg4(uint32_t* p, uint4 v) { *reinterpret_cast<uint4*>(p) = v; }
__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

__device__ __forceinline__ void ct(uint32_t& x, uint32_t& y, uint32_t w, uint32_t wp, uint32_t q, uint32_t q2) {
  const uint32_t xx = sub_if(x, q2);
  const uint32_t t = shoup_mul(y, w, wp, q);
  x = xx + t;
  y = xx - t + q2;
}
__device__ __forceinline__ void gs(uint32_t& x, uint32_t& y, uint32_t w, uint32_t wp, uint32_t q, uint32_t q2) {
  const uint32_t u = sub_if(x + y, q2);
  y = shoup_mul(x - y + q2, w, wp, q);
  x = u;
}
__device__ __forceinline__ void ct2(uint2& x, uint2& y, uint2 w, uint32_t q, uint32_t q2) {
  ct(x.x, y.x, w.x, w.y, q, q2);
  ct(x.y, y.y, w.x, w.y, q, q2);
}
__device__ __forceinline__ void gs2(uint2& x, uint2& y, uint2 w, uint32_t q, uint32_t q2) {
  gs(x.x, y.x, w.x, w.y, q, q2);
  gs(x.y, y.y, w.x, w.y, q, q2);
}

// ---------------------------------------------------------------- forward --
struct FwdSmem {
  uint32_t col[256 * kB];    // column block [row][32 cols] (32 KB)
  uint2 ctw[256];            // column-pass twiddles of the current prime
  uint32_t stage[16 * kRS];  // row exchange (16 rows at a time)
};

__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kT, 2)
    k_fwd_cluster(const RowJob* __restrict__ jobs, const uint32_t* __restrict__ src, uint64_t src_bs,
                  uint32_t* __restrict__ dst, uint64_t dst_bs, int batch, int njobs, const PrimeDev* __restrict__ primes,
                  const uint2* __restrict__ fwd_tw, const uint2* __restrict__ tw2, int entry) {
  extern __shared__ __align__(16) unsigned char smraw[];
  FwdSmem& S = *reinterpret_cast<FwdSmem*>(smraw);
  cg::cluster_group cluster = cg::this_cluster();
  const int k = (int)cluster.block_rank();
  const int cid = blockIdx.x / kCl, ncl = gridDim.x / kCl;
  const int tid = threadIdx.x;
  const int items = njobs * batch;
  const uint32_t* peer[kCl];
#pragma unroll
  for (int kk = 0; kk < kCl; ++kk) peer[kk] = cluster.map_shared_rank(S.col, kk);
  for (int it = cid; it < items; it += ncl) {
    const int job = it / batch, b = it % batch;
    const RowJob J = jobs[job];
    {  // load this CTA's column block and the prime's column twiddles
      const uint32_t* g = src + b * src_bs + (size_t)J.src_off * kN + kB * k;
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const int e = tid + m * kT, r = e >> 3, c4 = e & 7;
        cp16(&S.col[r * kB + 4 * c4], g + r * kR + 4 * c4);
      }
      if (tid < 128) cp16(&S.ctw[2 * tid], &fwd_tw[(size_t)J.prime * kN + 2 * tid]);
      cp_commit();
      cp_wait_all();
      __syncthreads();
    }
    const PrimeDev P = primes[J.prime];
    const uint32_t q = P.q, q2 = P.q2;
    // ---- pass 1: columns 2cp, 2cp+1 of the block, stages 0..7
    {
      const int tau = tid >> 4, cp = tid & 15;
      uint32_t* C = S.col + 2 * cp;
      uint2 v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = *reinterpret_cast<const uint2*>(C + (tau + 16 * j) * kB);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int d = 8 >> t;
#pragma unroll
        for (int p = 0; p < 8; ++p) {
          const int blk = p / d, j = blk * 2 * d + p % d;
          if (t == 0 && entry) {  // entry merge x*R, y*psi^{N/2}*R (ntt.cpp:27-35)
            const uint32_t x0 = shoup_mul(v[j].x, P.r, P.r_sh, q), t0 = shoup_mul(v[j + d].x, P.w1r, P.w1r_sh, q);
            const uint32_t x1 = shoup_mul(v[j].y, P.r, P.r_sh, q), t1 = shoup_mul(v[j + d].y, P.w1r, P.w1r_sh, q);
            v[j] = make_uint2(x0 + t0, x1 + t1);
            v[j + d] = make_uint2(x0 - t0 + q2, x1 - t1 + q2);
          } else {
            ct2(v[j], v[j + d], S.ctw[(1 << t) + blk], q, q2);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) *reinterpret_cast<uint2*>(C + (tau + 16 * j) * kB) = v[j];
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = *reinterpret_cast<const uint2*>(C + (16 * tau + j) * kB);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int d = 8 >> t;
#pragma unroll
        for (int p = 0; p < 8; ++p) {
          const int blk = p / d, j = blk * 2 * d + p % d;
          ct2(v[j], v[j + d], S.ctw[(16 << t) + (tau << t) + blk], q, q2);
        }
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) *reinterpret_cast<uint2*>(C + (16 * tau + j) * kB) = v[j];
    }
    cluster.sync();  // every CTA's pass-1 block is complete and visible
    // ---- pass 2: rows 32k .. 32k+31 (two rounds of 16), stages 8..15
    {
      const int rho = tid >> 4, tau = tid & 15;
      uint32_t* line = S.stage + rho * kRS;
#pragma unroll 1
      for (int round = 0; round < 2; ++round) {
        const int r = kB * k + 16 * round + rho;
        const uint2* W = tw2 + ((size_t)J.prime * kR + r) * kR;  // per-row permuted table (L2)
        uint32_t v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = peer[j >> 1][r * kB + tau + 16 * (j & 1)];  // c = tau + 16 j
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int d = 8 >> t;
#pragma unroll
          for (int p = 0; p < 8; ++p) {
            const int blk = p / d, j = blk * 2 * d + p % d;
            const uint2 w = __ldg(&W[(1 << t) - 1 + blk]);
            ct(v[j], v[j + d], w.x, w.y, q, q2);
          }
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) line[rp(tau + 16 * j)] = v[j];
        __syncwarp();
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const uint4 x = *reinterpret_cast<const uint4*>(line + rp(16 * tau) + 4 * m);
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
            const uint2 w = __ldg(&W[16 + ((1 << t) - 1 + blk) * 16 + tau]);
            ct(v[j], v[j + d], w.x, w.y, q, q2);
          }
        }
        uint32_t* orow = dst + b * dst_bs + (size_t)J.dst_off * kN + (size_t)r * kR + 16 * tau;
#pragma unroll
        for (int m = 0; m < 4; ++m)
          stg4(orow + 4 * m, make_uint4(canon4(v[4 * m], q, q2), canon4(v[4 * m + 1], q, q2),
                                        canon4(v[4 * m + 2], q, q2), canon4(v[4 * m + 3], q, q2)));
      }
    }
    cluster.sync();  // peers are done reading this block
  }
}

// ---------------------------------------------------------------- inverse --
struct InvSmem {
  uint32_t rows[kB * kRS];  // row block, padded row layout (43 KB)
  uint2 ctw[256];           // column-pass inverse twiddles
  uint32_t col[256 * kB];   // column-pass exchange (32 KB)
};

__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kT, 2)
    k_inv_cluster(const RowJob* __restrict__ jobs, const uint32_t* __restrict__ src, uint64_t src_bs,
                  uint32_t* __restrict__ dst, uint64_t dst_bs, int batch, int njobs, const PrimeDev* __restrict__ primes,
                  const uint2* __restrict__ inv_tw, const uint2* __restrict__ tw2i, const ExitConst* __restrict__ exits) {
  extern __shared__ __align__(16) unsigned char smraw[];
  InvSmem& S = *reinterpret_cast<InvSmem*>(smraw);
  cg::cluster_group cluster = cg::this_cluster();
  const int k = (int)cluster.block_rank();
  const int cid = blockIdx.x / kCl, ncl = gridDim.x / kCl;
  const int tid = threadIdx.x;
  const int items = njobs * batch;
  for (int it = cid; it < items; it += ncl) {
    const int job = it / batch, b = it % batch;
    const RowJob J = jobs[job];
    {
      const uint32_t* g = src + b * src_bs + (size_t)J.src_off * kN + (size_t)kB * k * kR;
#pragma unroll
      for (int m = 0; m < 8; ++m) {  // 32 rows x 64 chunks of 16 B
        const int e = tid + m * kT, r = e >> 6, c = (e & 63) * 4;
        cp16(&S.rows[r * kRS + rp(c)], g + r * kR + c);
      }
      if (tid < 128) cp16(&S.ctw[2 * tid], &inv_tw[(size_t)J.prime * kN + 2 * tid]);
      cp_commit();
      cp_wait_all();
      __syncthreads();
    }
    const PrimeDev P = primes[J.prime];
    const uint32_t q = P.q, q2 = P.q2;
    // ---- pass A: rows 32k .. 32k+31 (inverse stages 0..7), results stay in smem
    {
      const int rho = tid >> 4, tau = tid & 15;
#pragma unroll 1
      for (int round = 0; round < 2; ++round) {
        const int lr = 16 * round + rho;
        uint32_t* line = S.rows + lr * kRS;
        const uint2* W = tw2i + ((size_t)J.prime * kR + kB * k + lr) * kR;
        uint32_t v[16];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const uint4 x = *reinterpret_cast<const uint4*>(line + rp(16 * tau) + 4 * m);
          v[4 * m] = x.x;
          v[4 * m + 1] = x.y;
          v[4 * m + 2] = x.z;
          v[4 * m + 3] = x.w;
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int d = 1 << t, off = 16 - (16 >> t);
#pragma unroll
          for (int p = 0; p < 8; ++p) {
            const int blk = p / d, j = blk * 2 * d + p % d;
            const uint2 w = __ldg(&W[(off + blk) * 16 + tau]);
            gs(v[j], v[j + d], w.x, w.y, q, q2);
          }
        }
#pragma unroll
        for (int m = 0; m < 4; ++m)
          *reinterpret_cast<uint4*>(line + rp(16 * tau) + 4 * m) =
              make_uint4(v[4 * m], v[4 * m + 1], v[4 * m + 2], v[4 * m + 3]);
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = line[rp(tau + 16 * j)];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int d = 1 << t, off = 16 - (16 >> t);
#pragma unroll
          for (int p = 0; p < 8; ++p) {
            const int blk = p / d, j = blk * 2 * d + p % d;
            const uint2 w = __ldg(&W[240 + off + blk]);
            gs(v[j], v[j + d], w.x, w.y, q, q2);
          }
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) line[rp(tau + 16 * j)] = v[j];
        __syncwarp();
      }
    }
    cluster.sync();
    // ---- pass B: columns 32k + 2cp, +1 (inverse stages 8..15 + exit)
    {
      const int tau = tid >> 4, cp = tid & 15;
      const ExitConst ex = exits[J.epi];
      const int c = kB * k + 2 * cp;
      // rows 16 tau + j live in CTA tau >> 1 at local row 16 (tau & 1) + j
      const uint32_t* pr = cluster.map_shared_rank(S.rows, tau >> 1) + (16 * (tau & 1)) * kRS + rp(c);
      uint2 v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = *reinterpret_cast<const uint2*>(pr + j * kRS);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int d = 1 << t;
#pragma unroll
        for (int p = 0; p < 8; ++p) {
          const int blk = p / d, j = blk * 2 * d + p % d;
          gs2(v[j], v[j + d], S.ctw[(128 >> t) + (tau << (3 - t)) + blk], q, q2);
        }
      }
      uint32_t* C = S.col + 2 * cp;
#pragma unroll
      for (int j = 0; j < 16; ++j) *reinterpret_cast<uint2*>(C + (16 * tau + j) * kB) = v[j];
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = *reinterpret_cast<const uint2*>(C + (tau + 16 * j) * kB);
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        const int d = 1 << t;
#pragma unroll
        for (int p = 0; p < 8; ++p) {
          const int blk = p / d, j = blk * 2 * d + p % d;
          gs2(v[j], v[j + d], S.ctw[(8 >> t) + blk], q, q2);
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {  // exit merge (ntt.cpp:76-84)
        const uint32_t u0 = v[j].x + v[j + 8].x, d0 = v[j].x - v[j + 8].x + q2;
        const uint32_t u1 = v[j].y + v[j + 8].y, d1 = v[j].y - v[j + 8].y + q2;
        v[j] = make_uint2(sub_if(shoup_mul(u0, ex.x, ex.y, q), q), sub_if(shoup_mul(u1, ex.x, ex.y, q), q));
        v[j + 8] = make_uint2(sub_if(shoup_mul(d0, ex.z, ex.w, q), q), sub_if(shoup_mul(d1, ex.z, ex.w, q), q));
      }
      uint32_t* o = dst + b * dst_bs + (size_t)J.dst_off * kN + c;
#pragma unroll
      for (int j = 0; j < 16; ++j) *reinterpret_cast<uint2*>(o + (tau + 16 * j) * kR) = v[j];
    }
    cluster.sync();  // peers are done reading this row block; S.col free
  }
}

int g_fwd_clusters = 0, g_inv_clusters = 0;

int max_clusters(const void* fn, int smem) {
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kCl * 64, 1, 1);
  cfg.blockDim = dim3(kT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = kCl;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = 16;
  }
  return n;
}

}  // namespace

bool ntt_cluster_available() {
  static int ok = -1;
  if (ok < 0) {
    int dev = 0, cc = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&cc, cudaDevAttrClusterLaunch, dev);
    ok = cc ? 1 : 0;
    if (ok) {
      g_fwd_clusters = max_clusters((const void*)k_fwd_cluster, sizeof(FwdSmem));
      g_inv_clusters = max_clusters((const void*)k_inv_cluster, sizeof(InvSmem));
    }
  }
  return ok == 1;
}

void ntt_cluster_forward(const NttLaunch& a, const uint2* tw2, cudaStream_t st) {
  const int items = a.njobs * a.batch;
  const int ncl = std::max(1, std::min(g_fwd_clusters, items));
  k_fwd_cluster<<<ncl * kCl, kT, sizeof(FwdSmem), st>>>(a.jobs, a.src, a.src_bs, a.dst, a.dst_bs, a.batch, a.njobs,
                                                         a.primes, a.tw, tw2, a.entry);
}

void ntt_cluster_inverse(const NttLaunch& a, const uint2* tw2i, cudaStream_t st) {
  const int items = a.njobs * a.batch;
  const int ncl = std::max(1, std::min(g_inv_clusters, items));
  k_inv_cluster<<<ncl * kCl, kT, sizeof(InvSmem), st>>>(a.jobs, a.src, a.src_bs, a.dst, a.dst_bs, a.batch, a.njobs,
                                                         a.primes, a.tw, tw2i, a.exits);
}

int ntt_cluster_grid(bool inverse) { return inverse ? g_inv_clusters : g_fwd_clusters; }

}  // namespace ck
