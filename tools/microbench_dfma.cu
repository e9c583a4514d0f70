#include <cstdio>
#include <cstdint>
template <int CH>
__global__ void kd(double* out, double seed) {
  double a[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) a[c] = seed + threadIdx.x + c;
  const double b = 1.0000001, d = 0.999999;
  for (int i = 0; i < 4096; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = fma(a[c], b, d);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CH>
__global__ void kmix(uint64_t* out, uint32_t seed) {  // IMAD.WIDE accumulate + DFMA side by side
  uint64_t acc[CH]; double da[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { acc[c] = seed + c; da[c] = seed * 0.5 + c; }
  uint32_t x = seed | 1, y = seed * 3;
  for (int i = 0; i < 4096; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      uint64_t d; asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(x + c), "r"(y), "l"(acc[c])); acc[c] = d;
      da[c] = fma(da[c], 1.0000001, 0.5);
    }
  }
  uint64_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c] + (uint64_t)da[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CH>
__global__ void kwide(uint64_t* out, uint32_t seed) {
  uint64_t acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = seed + c;
  uint32_t x = seed | 1, y = seed * 3;
  for (int i = 0; i < 4096; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) { uint64_t d; asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(x + c), "r"(y), "l"(acc[c])); acc[c] = d; }
  }
  uint64_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <class F>
float timeit(F f) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); return ms;
}
int main() {
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  void* out; cudaMalloc(&out, 1 << 26);
  for (int w : {16, 32, 64}) {
    const int threads = 128, blocks = 148 * w / 4;
    const double n = (double)blocks * threads * 4096 * 8;
    float ms = timeit([&] { kd<8><<<blocks, threads>>>((double*)out, 1.0); });
    printf("warps/SM %2d DFMA      %6.1f /clk/SM\n", w, n / (ms * 1e-3) / 148 / (clk * 1e3));
    ms = timeit([&] { kwide<8><<<blocks, threads>>>((uint64_t*)out, 7); });
    printf("warps/SM %2d IMAD.WIDE %6.1f /clk/SM\n", w, n / (ms * 1e-3) / 148 / (clk * 1e3));
    ms = timeit([&] { kmix<8><<<blocks, threads>>>((uint64_t*)out, 7); });
    printf("warps/SM %2d mixed: %6.1f IMAD.WIDE + %6.1f DFMA /clk/SM\n", w, n / (ms * 1e-3) / 148 / (clk * 1e3), n / (ms * 1e-3) / 148 / (clk * 1e3));
  }
}
