// Integer-pipe microbenchmark on sm_100a: lane-ops per SM-clock for the
// instructions the NTT / BConv / KeyMult kernels are made of.  Used to pick
// the butterfly arithmetic (Shoup vs Montgomery) — see DESIGN.md.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench_int.cu && /tmp/mb
#include <cstdint>
#include <cstdio>

constexpr int ITERS = 4096;
constexpr int CH = 8;  // independent chains per thread

template <int OP>
__global__ void k(uint32_t* out, uint32_t seed, long long* cyc) {
  uint32_t a[CH], b[CH];
  uint64_t w[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    a[c] = seed * (threadIdx.x + c + 1);
    b[c] = seed ^ (c * 0x9e3779b9u);
    w[c] = a[c];
  }
  const uint32_t q = 0x0f880001u, wp = 0x8a3b1234u, q2 = 2 * q;
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (OP == 0) a[c] = __umulhi(a[c], b[c]) + 1;           // IMAD.HI (+ add folded?)
      if (OP == 1) a[c] = a[c] * b[c] + c;                     // IMAD
      if (OP == 2) w[c] += (uint64_t)a[c] * b[c], a[c] ^= (uint32_t)w[c];  // IMAD.WIDE
      if (OP == 3) a[c] = min(a[c] + b[c], a[c] - q2);         // IADD3 + IMNMX
      if (OP == 4) {                                           // Harvey-Shoup CT butterfly
        uint32_t x = min(a[c], a[c] - q2);
        uint32_t t = b[c] * wp - __umulhi(b[c], wp) * q;
        a[c] = x + t;
        b[c] = x - t + q2;
      }
    }
  }
  long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += a[c] + b[c] + (uint32_t)w[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int OP>
void run(const char* name, int ops_per_inner) {
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 8 * 1024 * 4);
  cudaMalloc(&cyc, 8);
  int blocks = 148 * 8, threads = 256;
  k<OP><<<blocks, threads>>>(out, 7, cyc);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<OP><<<blocks, threads>>>(out, 7, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  double lane_ops = (double)blocks * threads * ITERS * CH * ops_per_inner;
  int clk_khz;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  double tops = lane_ops / (ms * 1e-3) / 1e12;
  printf("%-28s %8.3f ms  %7.2f Tlane-op/s  (%6.1f lane-ops/clk/SM at %d MHz nominal)\n", name, ms, tops,
         lane_ops / (ms * 1e-3) / 148 / (clk_khz * 1e3), clk_khz / 1000);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<0>("umulhi (+1)", 1);
  run<1>("imad lo", 1);
  run<2>("imad.wide u64 accum", 1);
  run<3>("iadd+min", 2);
  run<4>("shoup CT butterfly (per bf)", 1);
  return 0;
}
