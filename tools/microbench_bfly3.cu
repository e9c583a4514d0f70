// Shoup butterfly: quotient by IMAD.HI (__umulhi) vs by the high word of a
// 64-bit IMAD.WIDE (mul.wide.u32), data-dependent chains.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_bfly3 tools/microbench_bfly3.cu
#include <cstdint>
#include <cstdio>
constexpr int ITERS = 2048;
__device__ __forceinline__ uint32_t sub_if(uint32_t x, uint32_t m) { return min(x, x - m); }
__device__ __forceinline__ uint32_t hi_wide(uint32_t a, uint32_t b) {
  uint64_t d;
  asm("mul.wide.u32 %0, %1, %2;" : "=l"(d) : "r"(a), "r"(b));
  return (uint32_t)(d >> 32);
}
template <int MODE, int CH>
__global__ void kb(uint32_t* out, uint32_t seed, const uint2* tw) {
  uint32_t x[CH], y[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    x[c] = (seed * (threadIdx.x + c + 1)) & 0x0fffffff;
    y[c] = (seed ^ (c * 0x9e3779b9u)) & 0x0fffffff;
  }
  const uint32_t q = 0x0f880001u, q2 = 2 * q;
  for (int i = 0; i < ITERS; ++i) {
    const uint2 w = tw[i & 255];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const uint32_t xx = sub_if(x[c], q2);
      const uint32_t h = MODE == 0 ? __umulhi(y[c], w.y) : hi_wide(y[c], w.y);
      const uint32_t t = y[c] * w.x - h * q;
      x[c] = xx + t;
      y[c] = xx - t + q2;
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c] + y[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int MODE, int CH>
void run(int w, const uint2* tw) {
  uint32_t* out;
  const int threads = 128, blocks = 148 * w / 4;
  cudaMalloc(&out, (size_t)blocks * threads * 4);
  kb<MODE, CH><<<blocks, threads>>>(out, 7, tw);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kb<MODE, CH><<<blocks, threads>>>(out, 7, tw);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double bf = (double)blocks * threads * ITERS * CH;
  printf("%-12s chains=%2d warps/SM=%2d : %6.2f bf/clk/SM\n", MODE == 0 ? "IMAD.HI" : "IMAD.WIDE-hi", CH, w,
         bf / (ms * 1e-3) / 148 / (clk * 1e3));
  cudaFree(out);
}
int main() {
  uint2 h[256];
  const uint32_t q = 0x0f880001u;
  for (int i = 0; i < 256; ++i) {
    const uint32_t w = (0x0123457u * (i + 1)) % q;
    h[i] = make_uint2(w, (uint32_t)(((uint64_t)w << 32) / q));
  }
  uint2* tw;
  cudaMalloc(&tw, sizeof(h));
  cudaMemcpy(tw, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int w : {16, 32, 64}) {
    run<0, 8>(w, tw);
    run<1, 8>(w, tw);
    run<0, 16>(w, tw);
    run<1, 16>(w, tw);
  }
}
