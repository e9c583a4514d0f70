// Butterfly throughput on sm_100a: integer Shoup (IMAD.HI + 2 IMAD) vs an
// FP64-quotient modmul (k = round(y * w/q) by one DFMA, r = y*w - k*q by two
// IMAD) vs a 1:1 mix that keeps both the integer and the FP64 pipe busy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_bfly2 tools/microbench_bfly2.cu
#include <cstdint>
#include <cstdio>
constexpr int ITERS = 2048;
__device__ __forceinline__ uint32_t sub_if(uint32_t x, uint32_t m) { return min(x, x - m); }

template <int MODE, int CH>  // MODE 0 int, 1 fp64 (magic conv), 2 fp64 (I2F), 3 mixed 0/1
__global__ void kb(uint32_t* out, uint32_t seed) {
  uint32_t x[CH], y[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    x[c] = (seed * (threadIdx.x + c + 1)) & 0x0fffffff;
    y[c] = (seed ^ (c * 0x9e3779b9u)) & 0x0fffffff;
  }
  const uint32_t q = 0x0f880001u, q2 = 2 * q;
  for (int i = 0; i < ITERS; ++i) {
    const uint32_t w = 0x0123457u + i;
    const uint32_t wp = (uint32_t)(((uint64_t)w << 32) / q);
    const double wq = (double)w / (double)q;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const bool fp = MODE == 1 || MODE == 2 || (MODE == 3 && (c & 1));
      if (!fp) {
        const uint32_t xx = sub_if(x[c], q2);
        const uint32_t t = y[c] * w - __umulhi(y[c], wp) * q;
        x[c] = xx + t;
        y[c] = xx - t + q2;
      } else {
        const uint32_t xx = sub_if(x[c], q2);
        double yd;
        if (MODE == 2) yd = (double)y[c];
        else yd = __hiloint2double(0x43300000, (int)y[c]) - 4503599627370496.0;
        const double kd = fma(yd, wq, 6755399441055744.0);
        const uint32_t k = (uint32_t)__double2loint(kd);
        const uint32_t r = y[c] * w - k * q;  // (-q/2, q/2) signed
        x[c] = xx + r + q;
        y[c] = xx - r + q;
      }
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c] + y[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE, int CH>
void run(int w) {
  uint32_t* out;
  const int threads = 128, blocks = 148 * w / 4;
  cudaMalloc(&out, (size_t)blocks * threads * 4);
  kb<MODE, CH><<<blocks, threads>>>(out, 7);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kb<MODE, CH><<<blocks, threads>>>(out, 7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double bf = (double)blocks * threads * ITERS * CH;
  const char* nm[] = {"int-shoup", "fp64-magic", "fp64-i2f", "mixed"};
  printf("%-10s chains=%2d warps/SM=%2d : %6.2f bf/clk/SM\n", nm[MODE], CH, w, bf / (ms * 1e-3) / 148 / (clk * 1e3));
  cudaFree(out);
}

int main() {
  for (int w : {16, 32}) {
    run<0, 16>(w);
    run<1, 16>(w);
    run<2, 16>(w);
    run<3, 16>(w);
    run<3, 32>(w);
  }
}
