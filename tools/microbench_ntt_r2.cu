// Round-2 NTT experiments, compute skeletons with no
// HBM traffic so the butterfly rate of each design is measured on its own
// (butterflies / clk / SM at the SM clock the run reports):
//
//   row_smem     the production row-pass shape (ntt256.cu k_row / k_row_keymult):
//                16 threads x 16 elements per 256-point row, 4 Shoup stages,
//                16 x 16 exchange through padded shared memory (warp-local),
//                4 stages; twiddles from a shared-memory table
//   row_shfl     the same with the exchange done by warp shuffles (butterfly
//                transpose: 4 rounds of __shfl_xor over 16 lanes)
//   row_ot       the same as row_smem with on-the-fly twiddles (ntt.cpp:208-229,
//                PAPER.md:397): w = lsb[u] * msb[v] (Montgomery) per distinct
//                twiddle, Montgomery butterflies (no Shoup companion exists
//                for a twiddle made on the fly)
//   col_1tile    the column-pass skeleton (k_col: v[16] uint4, smem transpose
//                with CTA barriers, 128 threads, 5 CTAs / SM)
//   col_2tile    two independent tiles interleaved per thread (v[2][16]):
//                twice the independent work between dependent multiplies,
//                twice the registers
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_ntt_r2 tools/microbench_ntt_r2.cu -lnvidia-ml
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t sub_if(uint32_t x, uint32_t m) { return min(x, x - m); }
// Shoup CT butterfly, Harvey lazy [0, 4q)
__device__ __forceinline__ void ct(uint32_t& x, uint32_t& y, uint32_t w, uint32_t wp, uint32_t q, uint32_t q2) {
  const uint32_t xx = sub_if(x, q2);
  const uint32_t t = y * w - __umulhi(y, wp) * q;
  x = xx + t;
  y = xx - t + q2;
}
// Montgomery product a b R^-1 mod q, result in [0, 2q) (q < 2^30, unsigned)
__device__ __forceinline__ uint32_t mont(uint32_t a, uint32_t b, uint32_t q, uint32_t qinv_neg) {
  const uint64_t t = (uint64_t)a * b;
  const uint32_t m = (uint32_t)t * qinv_neg;
  return (uint32_t)((t + (uint64_t)m * q) >> 32);
}
__device__ __forceinline__ void ct_mont(uint32_t& x, uint32_t& y, uint32_t w, uint32_t q, uint32_t q2,
                                        uint32_t qi) {
  const uint32_t xx = sub_if(x, q2);
  const uint32_t t = mont(y, w, q, qi);
  x = xx + t;
  y = xx - t + q2;
}

constexpr uint32_t kQ = 0x0f880001u;  // a 28-bit NTT prime (value irrelevant to timing)
constexpr int kStride = 336;
__device__ __forceinline__ int rpos(int c) { return c + 4 * (c >> 4); }

// ---- row pass: 8 rows per 128-thread CTA, 16 threads per row
template <int MODE>  // 0 smem exchange, 1 shuffle exchange, 2 OT twiddles + smem exchange
__global__ void __launch_bounds__(128, 8) k_rowskel(uint32_t* out, int iters) {
  __shared__ uint32_t line_all[8 * kStride];
  __shared__ uint2 tw[8 * 256];
  __shared__ uint32_t lsb[64], msb[64];
  const int tid = threadIdx.x, rho = tid >> 4, tau = tid & 15;
  const uint32_t q = kQ, q2 = 2 * q, qi = 0xf087ffffu;
  for (int e = tid; e < 8 * 256; e += 128) tw[e] = make_uint2(0x1234567u + e, 0x1f00000u + 3 * e);
  if (tid < 64) {
    lsb[tid] = 0x0345678u + 11 * tid;
    msb[tid] = 0x0456789u + 13 * tid;
  }
  uint32_t* line = line_all + rho * kStride;
  const uint2* W = tw + rho * 256;
  uint32_t v[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = (tid * 16 + j) % q;
  __syncthreads();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int d = 8 >> t;
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int blk = p / d, j = blk * 2 * d + p % d;
        if (MODE == 2) {  // twiddle made on the fly from the two half tables
          const uint32_t w = mont(lsb[(it + blk) & 63], msb[(t + blk) & 63], q, qi);
          ct_mont(v[j], v[j + d], w, q, q2, qi);
        } else {
          const uint2 w = W[(1 << t) - 1 + blk];
          ct(v[j], v[j + d], w.x, w.y, q, q2);
        }
      }
    }
    if (MODE == 1) {
      // 16 x 16 transpose across the 16 lanes of the row: after round s the
      // lane pair differing in bit s has swapped the element blocks differing in bit s
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const int m = 1 << s;
        const bool up = (tau >> s) & 1;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (((j >> s) & 1) == 0) {
            const uint32_t send = up ? v[j] : v[j + m];
            const uint32_t recv = __shfl_xor_sync(0xffffffffu, send, m, 16);
            if (up) v[j] = recv;
            else v[j + m] = recv;
          }
        }
      }
    } else {
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
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int d = 8 >> t;
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int blk = p / d, j = blk * 2 * d + p % d;
        if (MODE == 2) {
          const uint32_t w = mont(lsb[(tau + blk) & 63], msb[(it + t) & 63], q, qi);
          ct_mont(v[j], v[j + d], w, q, q2, qi);
        } else {
          const uint2 w = W[16 + ((1 << t) - 1 + blk) * 16 + tau];
          ct(v[j], v[j + d], w.x, w.y, q, q2);
        }
      }
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += v[j];
  if (s == 0x12345678u) out[blockIdx.x] = s;
}

// ---- column pass skeleton: T independent tiles per thread
template <int T>
__global__ void __launch_bounds__(128, (T == 1 ? 5 : 2)) k_colskel(uint32_t* out, int iters) {
  __shared__ uint4 tile[256 * 8];  // one transpose buffer, used by the T tiles in turn
  __shared__ uint2 tw[256];
  const int tid = threadIdx.x, cq = tid & 7, tau = tid >> 3;
  const uint32_t q = kQ, q2 = 2 * q;
  for (int e = tid; e < 256; e += 128) tw[e] = make_uint2(0x1234567u + e, 0x1f00000u + 3 * e);
  uint4 v[T][16];
#pragma unroll
  for (int u = 0; u < T; ++u)
#pragma unroll
    for (int j = 0; j < 16; ++j) v[u][j] = make_uint4(tid + j + u, tid * 3 + j, tid ^ j, tid + 7 * j);
  __syncthreads();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int d = 8 >> t;
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int blk = p / d, j = blk * 2 * d + p % d;
        const uint2 w = tw[(1 << t) + blk];
#pragma unroll
        for (int u = 0; u < T; ++u) {  // interleaved: T independent butterflies per twiddle
          ct(v[u][j].x, v[u][j + d].x, w.x, w.y, q, q2);
          ct(v[u][j].y, v[u][j + d].y, w.x, w.y, q, q2);
          ct(v[u][j].z, v[u][j + d].z, w.x, w.y, q, q2);
          ct(v[u][j].w, v[u][j + d].w, w.x, w.y, q, q2);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < T; ++u) {
#pragma unroll
      for (int j = 0; j < 16; ++j) tile[(tau + 16 * j) * 8 + cq] = v[u][j];
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 16; ++j) v[u][j] = tile[(16 * tau + j) * 8 + cq];
      __syncthreads();
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int d = 8 >> t;
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int blk = p / d, j = blk * 2 * d + p % d;
        const uint2 w = tw[(16 << t) + (tau << t) + blk];
#pragma unroll
        for (int u = 0; u < T; ++u) {
          ct(v[u][j].x, v[u][j + d].x, w.x, w.y, q, q2);
          ct(v[u][j].y, v[u][j + d].y, w.x, w.y, q, q2);
          ct(v[u][j].z, v[u][j + d].z, w.x, w.y, q, q2);
          ct(v[u][j].w, v[u][j + d].w, w.x, w.y, q, q2);
        }
      }
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int u = 0; u < T; ++u)
#pragma unroll
    for (int j = 0; j < 16; ++j) s += v[u][j].x + v[u][j].y + v[u][j].z + v[u][j].w;
  if (s == 0x12345678u) out[blockIdx.x] = s;
}

// ---- pipe probes for ncu (sm__inst_executed_pipe_fmaheavy vs sm__pipe_fmaheavy_cycles_active):
// 8 independent chains of one instruction kind, so the pipe, not latency, bounds them
template <int OP>  // 0 IMAD (mul.lo), 1 IMAD.HI (mul.hi.u32), 2 IMAD.WIDE (mad.wide.u32)
__global__ void __launch_bounds__(128, 8) k_probe(uint32_t* out, int iters) {
  uint32_t a[8];
  uint64_t w[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) a[c] = threadIdx.x * 7 + c, w[c] = c;
  const uint32_t m = 0x9e3779b9u + blockIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (OP == 0) a[c] = a[c] * m + c;
      else if (OP == 1) a[c] = __umulhi(a[c], m) ^ c;
      else w[c] = (uint64_t)(uint32_t)w[c] * m + (w[c] >> 32);  // mad.wide on a loop-carried value
    }
  }
  uint64_t s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += a[c] + w[c];
  if (s == 0x12345678u) out[blockIdx.x] = (uint32_t)s;
}

template <class K>
static void run(const char* name, K kern, int per_sm, double bfly_per_thread_iter, int iters) {
  int dev = 0, sms = 0, clk_khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 128, 0);
  const int grid = sms * (occ > 0 ? occ : per_sm);
  uint32_t* out;
  cudaMalloc(&out, grid * 4);
  kern<<<grid, 128>>>(out, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    kern<<<grid, 128>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double bfly = (double)grid * 128 * iters * bfly_per_thread_iter;
  const double per_clk_sm = bfly / (best * 1e-3) / (sms * clk_khz * 1e3);
  std::printf("%-10s %2d CTAs/SM  %.3f ms  %6.2f butterflies/clk/SM (at the %.0f MHz max clock)\n", name,
              occ, best, per_clk_sm, clk_khz / 1e3);
  cudaFree(out);
}

int main(int argc, char** argv) {
  const int iters = argc > 1 ? std::atoi(argv[1]) : 2000;
  // row skeleton: 16 elements x 8 stages / 2 per thread per iteration
  run("row_smem", k_rowskel<0>, 8, 64.0, iters);
  run("row_shfl", k_rowskel<1>, 8, 64.0, iters);
  run("row_ot", k_rowskel<2>, 8, 64.0, iters);
  // column skeleton: 64 elements x 8 stages / 2 per thread per tile
  run("col_1tile", k_colskel<1>, 5, 256.0, iters / 4);
  run("col_2tile", k_colskel<2>, 2, 512.0, iters / 4);
  // pipe probes (the "butterflies" column is meaningless for them; read them with ncu)
  run("probe_imad", k_probe<0>, 8, 8.0, iters);
  run("probe_hi", k_probe<1>, 8, 8.0, iters);
  run("probe_wide", k_probe<2>, 8, 8.0, iters);
  return 0;
}
