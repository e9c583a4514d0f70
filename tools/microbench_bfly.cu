// Butterfly-throughput microbenchmark on sm_100a: Harvey-Shoup CT butterflies
// per SM-clock as a function of independent chains per thread (ILP) and
// resident warps per SM (TLP).  Separates latency limits from pipe limits for
// the NTT kernels.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_bfly tools/microbench_bfly.cu
#include <cstdint>
#include <cstdio>

constexpr int ITERS = 2048;

template <int CH>
__global__ void k(uint32_t* out, uint32_t seed) {
  uint32_t x[CH], y[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    x[c] = seed * (threadIdx.x + c + 1);
    y[c] = seed ^ (c * 0x9e3779b9u);
  }
  const uint32_t q = 0x0f880001u, wp = 0x8a3b1234u, w = 0x0123457u, q2 = 2 * q;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const uint32_t xx = min(x[c], x[c] - q2);
      const uint32_t t = y[c] * (w + i) - __umulhi(y[c], wp + i) * q;
      x[c] = xx + t;
      y[c] = xx - t + q2;
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c] + y[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// FP64-assisted Shoup: quotient k = round(y * w/q) from one DFMA with the
// 1.5*2^52 rounding constant; r = y*w - k*q in (-q, q) on the integer pipe.
template <int CH>
__global__ void k64(uint32_t* out, uint32_t seed) {
  uint32_t x[CH], y[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    x[c] = seed * (threadIdx.x + c + 1) & 0x0fffffff;
    y[c] = (seed ^ (c * 0x9e3779b9u)) & 0x3fffffff;
  }
  const uint32_t q = 0x0f880001u, q2 = 2 * q;
  for (int i = 0; i < ITERS; ++i) {
    const uint32_t w = 0x0123457u + i;
    const double wq = (double)w / (double)q;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const uint32_t xx = min(x[c], x[c] - q2);
      const double yd = __hiloint2double(0x43300000, (int)y[c]) - 4503599627370496.0;
      const double kd = fma(yd, wq, 6755399441055744.0);
      const uint32_t kk = (uint32_t)__double2loint(kd);
      const uint32_t r = y[c] * w - kk * q;  // (-q, q) as int32
      x[c] = xx + r + q;
      y[c] = xx - r + q;
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c] + y[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CH>
void run64(int warps_per_sm) {
  uint32_t* out;
  const int threads = 128, blocks = 148 * warps_per_sm / 4;
  cudaMalloc(&out, (size_t)blocks * threads * 4);
  k64<CH><<<blocks, threads>>>(out, 7);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k64<CH><<<blocks, threads>>>(out, 7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk_khz;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double bf = (double)blocks * threads * ITERS * CH;
  printf("FP64-quotient chains=%2d warps/SM=%2d : %6.2f bf/clk/SM\n", CH, warps_per_sm,
         bf / (ms * 1e-3) / 148 / (clk_khz * 1e3));
  cudaFree(out);
}

template <int CH>
void run(int warps_per_sm) {
  uint32_t* out;
  const int threads = 128, blocks = 148 * warps_per_sm / 4;
  cudaMalloc(&out, (size_t)blocks * threads * 4);
  k<CH><<<blocks, threads>>>(out, 7);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<CH><<<blocks, threads>>>(out, 7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk_khz;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double bf = (double)blocks * threads * ITERS * CH;
  printf("chains=%2d warps/SM=%2d : %6.2f bf/clk/SM (at %d MHz nominal), %.3f ms\n", CH, warps_per_sm,
         bf / (ms * 1e-3) / 148 / (clk_khz * 1e3), clk_khz / 1000, ms);
  cudaFree(out);
}

int main() {
  for (int w : {8, 16, 32, 64}) {
    run<4>(w);
    run<8>(w);
    run<16>(w);
    run<32>(w);
  }
  for (int w : {16, 32}) {
    run64<8>(w);
    run64<16>(w);
  }
  return 0;
}
