// Compute skeleton of the N = 2^16 column pass (ntt256.cu k_col<fwd>) with no
// global memory traffic: v[16] uint4 per thread, 4 CT stages with a
// warp-uniform twiddle from shared memory, smem transpose (+ CTA barrier),
// 4 stages with per-thread twiddles -- repeated.  Separates the compute /
// shared-memory ceiling of the pass from its HBM streaming.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_colpass tools/microbench_colpass.cu
#include <cstdint>
#include <cstdio>
__device__ __forceinline__ uint32_t sub_if(uint32_t x, uint32_t m) { return min(x, x - m); }
__device__ __forceinline__ void ct(uint32_t& x, uint32_t& y, uint2 w, uint32_t q, uint32_t q2) {
  const uint32_t xx = sub_if(x, q2);
  const uint32_t t = y * w.x - __umulhi(y, w.y) * q;
  x = xx + t;
  y = xx - t + q2;
}
__device__ __forceinline__ void ct4(uint4& x, uint4& y, uint2 w, uint32_t q, uint32_t q2) {
  ct(x.x, y.x, w, q, q2); ct(x.y, y.y, w, q, q2); ct(x.z, y.z, w, q, q2); ct(x.w, y.w, w, q, q2);
}
template <bool TRANSPOSE, bool BARRIER>
__global__ void __launch_bounds__(128, 5) kc(uint32_t* out, int iters) {
  __shared__ uint4 tile[256 * 8];
  __shared__ uint2 tw[256];
  const int tid = threadIdx.x, cq = tid & 7, tau = tid >> 3;
  const uint32_t q = 0x0f880001u, q2 = 2 * q;
  for (int e = tid; e < 256; e += 128) tw[e] = make_uint2(0x1234567u + e, 0x1f00000u + 3 * e);
  uint4 v[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = make_uint4(tid + j, tid * 3 + j, tid ^ j, tid + 7 * j);
  __syncthreads();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int d = 8 >> t;
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int blk = p / d, j = blk * 2 * d + p % d;
        ct4(v[j], v[j + d], tw[(1 << t) + blk], q, q2);
      }
    }
    if (TRANSPOSE) {
#pragma unroll
      for (int j = 0; j < 16; ++j) tile[(tau + 16 * j) * 8 + cq] = v[j];
      if (BARRIER) __syncthreads(); else __syncwarp();
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = tile[(16 * tau + j) * 8 + cq];
      if (BARRIER) __syncthreads(); else __syncwarp();
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int d = 8 >> t;
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int blk = p / d, j = blk * 2 * d + p % d;
        ct4(v[j], v[j + d], tw[(16 << t) + (tau << t) + blk], q, q2);
      }
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += v[j].x + v[j].y + v[j].z + v[j].w;
  out[blockIdx.x * 128 + tid] = s;
}
template <bool T, bool B>
void run(const char* name, int ctas_per_sm) {
  uint32_t* out;
  const int blocks = 148 * ctas_per_sm, iters = 256;
  cudaMalloc(&out, (size_t)blocks * 128 * 4);
  kc<T, B><<<blocks, 128>>>(out, 4);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kc<T, B><<<blocks, 128>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double bf = (double)blocks * 128 * iters * 256;
  printf("%-28s CTAs/SM=%d : %6.2f bf/clk/SM\n", name, ctas_per_sm, bf / (ms * 1e-3) / 148 / (clk * 1e3));
  cudaFree(out);
}
int main() {
  for (int c : {4, 5}) {
    run<false, false>("butterflies only", c);
    run<true, false>("+ smem transpose (syncwarp)", c);
    run<true, true>("+ smem transpose (barrier)", c);
  }
}
