// Limb-sharded key switching (BASELINE config 4): the
// shard-local kernels that have no equivalent in the single-GPU path because
// a shard's rows are an arbitrary subset of the RNS basis.
//
// A shard owns a contiguous block of Q primes and a contiguous block of P
// primes; NTT/INTT and BConv reuse the generic row-job kernels, only KeyMult
// and the drop-and-divide tail need per-row prime/digit/key-row maps.
#include "ck_common.cuh"
#include "ck_kernels.h"

namespace ck {
namespace {

constexpr int kST = 256;
// Written instead of results when the peer exchange's error word is set: not a
// canonical residue of any prime (all q < 2^29), so it cannot pass for one.
constexpr uint32_t kPoison = 0xFFFFFFFFu;

__device__ __forceinline__ uint4 ld4(const uint32_t* p) { return __ldg(reinterpret_cast<const uint4*>(p)); }
__device__ __forceinline__ void st4(uint32_t* p, uint4 v) { *reinterpret_cast<uint4*>(p) = v; }
__device__ __forceinline__ uint32_t getc(const uint4& v, int c) { return c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w; }

// key_mult (ckks.cpp:733-770) over the shard's rows: v_c[r] = sum_k opnd_k[r] * evk_k.c[erow(r)]
// where opnd_k[r] is the ModUp input row itself when r belongs to digit k
// (pass-through, ckks.cpp:705-708) and the converted extension row otherwise;
// optional fold v_c[r] += P * fold_c[r] on Q rows (ckks.cpp:831-842).
__global__ void __launch_bounds__(kST) k_shard_key_mult(ShardKeyMultLaunch a, int n) {
  const int xo = (blockIdx.x * kST + threadIdx.x) * 4;
  if (xo >= n) return;
  const int r = blockIdx.y;
  const int g = a.prime[r], dig = a.digit[r], er = a.erow[r];
  const PrimeDev P = a.primes[g];
  uint64_t s0[4] = {0, 0, 0, 0}, s1[4] = {0, 0, 0, 0};
  int terms = 0;
  auto renorm = [&]() {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      s0[c] = shoup_mul(mont_reduce64(s0[c], P.q, P.qinv), P.r, P.r_sh, P.q);
      s1[c] = shoup_mul(mont_reduce64(s1[c], P.q, P.qinv), P.r, P.r_sh, P.q);
    }
  };
  for (int k = 0; k < a.D; ++k) {
    const uint32_t* op = dig == k ? a.d + (size_t)r * n + xo : a.ext + ((size_t)k * a.rows + r) * n + xo;
    const uint4 dv = ld4(op);
    const uint4 eb = ld4(a.evk + (((size_t)k * 2 + 0) * a.erows + er) * n + xo);
    const uint4 ea = ld4(a.evk + (((size_t)k * 2 + 1) * a.erows + er) * n + xo);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      s0[c] = mac_wide(s0[c], getc(dv, c), getc(eb, c));
      s1[c] = mac_wide(s1[c], getc(dv, c), getc(ea, c));
    }
    if (++terms == 7) {
      renorm();
      terms = 1;
    }
  }
  if (a.fold && r < a.lq) {
    const uint32_t pm = a.p_mont[g];
    const uint4 f0 = ld4(a.fold + (size_t)r * n + xo);
    const uint4 f1 = ld4(a.fold + (size_t)(a.lq + r) * n + xo);
    if (terms == 7) renorm();
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      s0[c] = mac_wide(s0[c], getc(f0, c), pm);
      s1[c] = mac_wide(s1[c], getc(f1, c), pm);
    }
  }
  uint4 r0, r1;
  r0.x = sub_if(mont_reduce64(s0[0], P.q, P.qinv), P.q);
  r0.y = sub_if(mont_reduce64(s0[1], P.q, P.qinv), P.q);
  r0.z = sub_if(mont_reduce64(s0[2], P.q, P.qinv), P.q);
  r0.w = sub_if(mont_reduce64(s0[3], P.q, P.qinv), P.q);
  r1.x = sub_if(mont_reduce64(s1[0], P.q, P.qinv), P.q);
  r1.y = sub_if(mont_reduce64(s1[1], P.q, P.qinv), P.q);
  r1.z = sub_if(mont_reduce64(s1[2], P.q, P.qinv), P.q);
  r1.w = sub_if(mont_reduce64(s1[3], P.q, P.qinv), P.q);
  if (a.err && *(volatile const uint32_t*)a.err) {  // a peer never arrived: poison, never silently wrong
    r0 = r1 = make_uint4(kPoison, kPoison, kPoison, kPoison);
  }
  st4(a.v + (size_t)r * n + xo, r0);
  st4(a.v + (size_t)(a.rows + r) * n + xo, r1);
}

// drop_and_divide tail (ckks.cpp:643-651) on the shard's output rows, with the
// HRot / lazy-HMult epilogue: out_c[r][j] = ((v_c - o_c) * div^-1 + add_c)[r][src(j)].
__global__ void __launch_bounds__(kST) k_shard_tail(ShardTailLaunch a, int n) {
  const int j = blockIdx.x * kST + threadIdx.x;
  if (j >= n) return;
  const int r = blockIdx.y, c = blockIdx.z;
  const PrimeDev P = a.primes[a.prime_base + r];
  const uint32_t s = a.src_map ? __ldg(&a.src_map[j]) : (uint32_t)j;
  const size_t e = (size_t)r * n + s;
  const uint32_t vv = a.v[(size_t)c * a.v_ps + e], oo = a.o[(size_t)c * a.o_ps + e];
  uint32_t x = sub_if(mont_mul(vv - oo + P.q, a.dinv[r], P.q, P.qinv), P.q);
  if (a.add && (a.add_mask >> c & 1)) x = sub_if(x + a.add[(size_t)c * a.add_ps + e], P.q);
  if (a.err && *(volatile const uint32_t*)a.err) x = kPoison;  // peer exchange timed out
  a.out[(size_t)c * a.out_ps + (size_t)r * n + j] = x;
}

// Peer exchange handshake.  Producer: after the phase-1 INTT (stream order)
// one thread per peer publishes the epoch into that peer's flag word for this
// rank with a system-scope release; the INTT's writes to the exchange buffer
// happen-before it.  Consumer: one thread per peer spins with system-scope
// acquire loads on its local flag word until the peer's epoch arrives; the
// BConv that reads the peers' buffers is the next kernel on the stream.  The
// spin is bounded (globaltimer) so a missing peer reports an error instead of
// hanging the GPU.
// The epoch lives in device memory (advanced by k_shard_advance at the head
// of phase 1), so no kernel of an exchange carries a host-chosen value and a
// captured step replays correctly.
__global__ void k_shard_advance(uint32_t* epoch, const RowJob* __restrict__ jobs2, RowJob* __restrict__ jobs_cur,
                                int njobs) {
  const uint32_t e = *epoch + 1;  // every thread reads the old value before thread 0 stores the new one
  for (int t = threadIdx.x; t < njobs; t += blockDim.x) jobs_cur[t] = jobs2[(e & 1) * njobs + t];
  __syncthreads();
  if (threadIdx.x == 0) *epoch = e;
}

__global__ void k_shard_signal(const uint64_t* __restrict__ sig, int G, const uint32_t* __restrict__ epoch) {
  const int t = threadIdx.x;
  if (t >= G) return;
  const uint32_t e = *epoch;
  uint32_t* p = reinterpret_cast<uint32_t*>(sig[t]);
  asm volatile("fence.sc.sys;\n" ::: "memory");
  asm volatile("st.release.sys.global.u32 [%0], %1;\n" ::"l"(p), "r"(e) : "memory");
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Phase 2 head: spin until every peer's flag reaches this rank's current
// epoch, then copy the epoch's parity of the BConv source-row table
// (rows2 [2][nrows]) into rows_cur, the table the BConv kernel reads.
__global__ void k_shard_wait(const uint32_t* __restrict__ flags, int G, const uint32_t* __restrict__ epoch,
                             uint32_t* err, uint64_t timeout_ns, const uint64_t* __restrict__ rows2,
                             uint64_t* __restrict__ rows_cur, int nrows) {
  const int t = threadIdx.x;
  const uint32_t e = *epoch;
  if (t < G) {
    const uint64_t t0 = globaltimer();
    while (true) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];\n" : "=r"(v) : "l"(flags + t) : "memory");
      if ((int32_t)(v - e) >= 0) break;
      if (globaltimer() - t0 > timeout_ns) {
        atomicExch(err, 1u);
        break;
      }
      __nanosleep(200);
    }
  }
  for (int r = t; r < nrows; r += blockDim.x) rows_cur[r] = rows2[(e & 1) * nrows + r];
}

}  // namespace

void shard_advance(uint32_t* epoch, const RowJob* jobs2, RowJob* jobs_cur, int njobs, cudaStream_t st) {
  k_shard_advance<<<1, 64, 0, st>>>(epoch, jobs2, jobs_cur, njobs);
}

void shard_signal(const uint64_t* sig, int G, const uint32_t* epoch, cudaStream_t st) {
  k_shard_signal<<<1, 32 * ((G + 31) / 32), 0, st>>>(sig, G, epoch);
}

void shard_wait(const uint32_t* flags, int G, const uint32_t* epoch, uint32_t* err, uint64_t timeout_ns,
                const uint64_t* rows2, uint64_t* rows_cur, int nrows, cudaStream_t st) {
  k_shard_wait<<<1, 64, 0, st>>>(flags, G, epoch, err, timeout_ns, rows2, rows_cur, nrows);
}

void shard_key_mult(int n, const ShardKeyMultLaunch& a, cudaStream_t st) {
  if (a.rows == 0) return;
  dim3 grid((n / 4 + kST - 1) / kST, a.rows);
  k_shard_key_mult<<<grid, kST, 0, st>>>(a, n);
}

void shard_tail(int n, int rows, const ShardTailLaunch& a, cudaStream_t st) {
  if (rows == 0) return;
  dim3 grid((n + kST - 1) / kST, rows, 2);
  k_shard_tail<<<grid, kST, 0, st>>>(a, n);
}

}  // namespace ck
