// Base conversion (bconv_part2, bconv.cpp:96-174) on the 5th-generation
// tensor cores: tcgen05.mma kind::i8 with the accumulator in TMEM.
//
//   dst[i][x] = mont_reduce( sum_j src[j][x] * C[i][j] )  mod q_i
//
// Split-word formulation (exact): write src[j][x] = sum_b 2^(8b) s_jb(x) with
// bytes s_jb, and precompute per destination prime
//   C'[i][j][b] = C[i][j] * 2^(8b) mod q_i = sum_a 2^(8a) c_ijab   (bytes c_ijab).
// Then   sum_j src[j][x] C[i][j]  ==  sum_a 2^(8a) acc_a(i, x)   (mod q_i),
//        acc_a(i, x) = sum_(j,b) c_ijab * s_jb(x)
// is ONE u8 x u8 -> s32 GEMM:  D[x][(i,a)] = A[x][(j,b)] . B[(i,a)][(j,b)]^T
// with M = 128 coefficients per tile, K = 4 sc bytes (32 or 64), N = 4 dc.
// Every acc_a < K * 255^2 < 2^22, so the int32 accumulator is exact, and
// v = sum_a 2^(8a) acc_a < 2^46 < q 2^32 is a valid Montgomery-reduction
// input congruent to the CUDA-core kernel's int64 sum: the canonical outputs
// are identical (canonical residues are the contract).
//
// Per CTA (128 threads = 4 warps, persistent over (group, batch, tile) items):
//   * raw source tiles [sc][128] u32 stream through a ring of NST smem stages
//     with cp.async (16 B, L1 bypass), NST-1 items ahead;
//   * each thread transposes its coefficient's sc words into the A tile in
//     the UMMA canonical K-major no-swizzle layout (8 x 16 B core matrices);
//   * thread 0 issues the MMA(s) and tcgen05.commit's to an mbarrier;
//   * the epilogue (warp w owns TMEM lanes 32w..32w+31 = coefficients) loads
//     32 columns (8 destination rows) at a time with tcgen05.ld, recombines
//     the 4 byte-planes into a 64-bit value, Montgomery-reduces and stores
//     coalesced rows.
// The B tables (canonical layout, bytes) are built by the host per plan.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "ck_common.cuh"
#include "ck_kernels.h"

namespace ck {
namespace {

constexpr int kTT = 128;   // threads = coefficients per tile (UMMA M)
constexpr int kNst = 4;    // raw-tile ring depth
#ifndef CK32_TC2_FAST3
#define CK32_TC2_FAST3 1
#endif
constexpr bool kTc2Fast3 = CK32_TC2_FAST3;  // k_bconv_tc2: straight-line epilogue for 24 consecutive-row destinations

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(K) : "memory");
}

// UMMA shared-memory descriptor, K-major, no swizzle (cute UMMA::SmemDescriptor):
// start >> 4 [0,14), LBO >> 4 [16,30) (K-direction core-matrix stride),
// SBO >> 4 [32,46) (M/N-direction 8-row-group stride), version 1 [46,48).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
// instruction descriptor: dense, D s32 (c_format 2), A/B u8, both K-major, N >> 3, M >> 4
__host__ __device__ constexpr uint32_t idesc_u8(int M, int N) {
  return (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_u8(uint32_t dtmem, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %5, %5, %5}, p;\n\t}\n" ::"r"(dtmem),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc), "r"(0u));
}
__device__ __forceinline__ void mma_commit(void* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(mbar))
               : "memory");
}
__device__ __forceinline__ void mbar_init(void* mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(void* mbar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(mbar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// 32 consecutive TMEM columns of this thread's lane
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
// wait for the outstanding tcgen05.ld's; the destination registers are tied
// to the wait so no use of them is scheduled above it
__device__ __forceinline__ void tmem_wait_ld(uint32_t (&r)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                 "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                 "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
               :
               : "memory");
}

// sum_a 2^(8a) acc_a  (< 2^46) Montgomery-reduced mod q, canonical
__device__ __forceinline__ uint32_t combine4(uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t q,
                                             uint32_t qinv_neg) {
  const uint32_t t1 = a0 + (a1 << 8), t2 = a2 + (a3 << 8);  // each < 2^31
  uint32_t lo, hi;
  asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, 0;\n" : "=r"(lo), "=r"(hi) : "r"(t1), "r"(t2 << 16), "r"(t2 >> 16));
  const uint32_t m = lo * qinv_neg;
  return sub_if(hi + __umulhi(m, q) + (lo != 0u), q);
}

struct __align__(16) TcDst {
  uint32_t q, qinv_neg, row, pad;
};

template <int KB, int NCOLS>
__global__ void __launch_bounds__(kTT) k_bconv_tc(BconvLaunch a, BconvTc t, int n) {
  // KB: A/B K extent in bytes (32 or 64); NCOLS: TMEM columns allocated (>= max N).
  // One accumulator buffer per CTA so that 4 CTAs fit the 512 TMEM columns of
  // an SM (a double-buffered variant at 2 CTAs/SM measured slower).
  extern __shared__ __align__(128) unsigned char smraw[];
  constexpr int kSbo = (KB / 16) * 128;  // bytes per 8-row group
  constexpr int kATile = kTT * KB;       // A tile bytes
  const int rawStage = a.max_sc * kTT;   // words per ring stage
  const int dcPad = (t.max_dc + 7) / 8 * 8;
  uint32_t* raw = reinterpret_cast<uint32_t*>(smraw);              // [kNst][max_sc][128] u32
  unsigned char* At = smraw + (size_t)kNst * rawStage * 4;         // A tile (128-B aligned)
  unsigned char* Bt = At + kATile;                                 // B table of the current group
  TcDst* dinfo = reinterpret_cast<TcDst*>(Bt + t.max_npad * KB);  // [dcPad] per destination row
  uint64_t* mbar = reinterpret_cast<uint64_t*>(dinfo + dcPad);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(mbar + 1);

  const int tid = threadIdx.x, warp = tid >> 5;
  const int tiles = n / kTT;
  const int items = a.ngroups * a.batch * tiles;  // (group, b, tile), tile fastest
  const int chunk = (items + gridDim.x - 1) / gridDim.x;
  const int i0 = blockIdx.x * chunk, i1 = min(items, i0 + chunk);
  if (i0 >= i1) return;

  if (warp == 0) {  // TMEM accumulator: 128 lanes x NCOLS columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tslot)),
                 "n"(NCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    mbar_init(mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);

  auto issue = [&](int it, int slot) {  // raw source tile of item `it` into ring slot `slot`
    if (it < i1) {
      const int tile = it % tiles, rest = it / tiles, b = rest % a.batch, g = rest / a.batch;
      const BconvGroup G = a.groups[g];
      const uint32_t* src = a.src + b * a.src_bs + (size_t)G.src_off * n + (size_t)tile * kTT;
      uint32_t* dst = raw + slot * rawStage;
      for (int e = tid; e < (int)G.sc * (kTT / 4); e += kTT) {
        const int j = e / (kTT / 4), c = e % (kTT / 4);
        cp16(dst + j * kTT + 4 * c, src + (size_t)j * n + 4 * c);
      }
    }
    cp_commit();
  };
#pragma unroll
  for (int s = 0; s < kNst - 1; ++s) issue(i0 + s, s);

  int cur_g = -1, sc = 0, dc = 0, npad = 16;
  uint32_t phase = 0;
  for (int it = i0, k = 0; it < i1; ++it, ++k) {
    cp_wait<kNst - 2>();
    __syncthreads();  // raw tile k landed for all threads; iteration k-1 fully done (A, B, TMEM free)
    issue(it + kNst - 1, (k + kNst - 1) % kNst);
    const int tile = it % tiles, rest = it / tiles, b = rest % a.batch, g = rest / a.batch;
    if (g != cur_g) {  // new group: its B table and destination constants
      cur_g = g;
      const BconvGroup G = a.groups[g];
      sc = (int)G.sc;
      dc = (int)G.dc;
      npad = (4 * dc + 15) / 16 * 16;
      const uint4* B = reinterpret_cast<const uint4*>(t.btab + t.boff[g]);
      uint4* Bs = reinterpret_cast<uint4*>(Bt);
      for (int e = tid; e < npad * KB / 16; e += kTT) Bs[e] = __ldg(B + e);
      for (int i = tid; i < dcPad; i += kTT) {
        TcDst d{1u, 0u, 0u, 0u};
        if (i < dc) {
          const PrimeDev P = a.primes[a.dst_prime[G.map_off + i]];
          d = TcDst{P.q, P.qinv_neg, a.dst_row[G.map_off + i] * (uint32_t)n, 0u};
        }
        dinfo[i] = d;
      }
    }
    {  // transpose: row x = tid, K chunk c holds the words src[4c .. 4c+3][x] (zero past sc)
      const uint32_t* R = raw + (k % kNst) * rawStage;
      uint32_t w[KB / 4];
#pragma unroll
      for (int j = 0; j < KB / 4; ++j) w[j] = j < sc ? R[j * kTT + tid] : 0u;
      unsigned char* row = At + (tid >> 3) * kSbo + (tid & 7) * 16;
#pragma unroll
      for (int c = 0; c < KB / 16; ++c)
        *reinterpret_cast<uint4*>(row + c * 128) = make_uint4(w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
    }
    fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor core (async proxy)
    __syncthreads();
    if (tid == 0) {
      fence_after();
      const uint32_t idesc = idesc_u8(kTT, npad);
      const uint32_t a0 = smem_u32(At), b0 = smem_u32(Bt);
#pragma unroll
      for (int kk = 0; kk < KB / 32; ++kk)  // K = 32 bytes per MMA: two 16-B core-matrix columns
        mma_u8(tmem, sdesc(a0 + kk * 256, 128, kSbo), sdesc(b0 + kk * 256, 128, kSbo), idesc, kk > 0);
      mma_commit(mbar);
    }
    mbar_wait(mbar, phase);
    phase ^= 1;
    fence_after();
    uint32_t* dbase = a.dst + b * a.dst_bs + (size_t)tile * kTT + tid;
    for (int ic = 0; ic < dc; ic += 8) {  // 8 destination rows (32 columns) per TMEM load
      uint32_t r[32];
      tmem_ld32(lane_addr + 4 * ic, r);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const TcDst d = dinfo[ic + u];
        const uint32_t v = combine4(r[4 * u], r[4 * u + 1], r[4 * u + 2], r[4 * u + 3], d.q, d.qinv_neg);
        if (ic + u < dc) dbase[d.row] = v;
      }
    }
    fence_before();  // TMEM reads ordered before the next iteration's barrier (next MMA overwrites)
  }
  cp_wait<0>();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(NCOLS));
}

// (group, batch item, tile) item cursor, tile fastest: advanced by one per
// item (a CTA owns a contiguous chunk), so the loop does no integer division
struct TcCursor {
  int tile, b, g;
  __device__ __forceinline__ void init(int it, int tiles, int batch) {
    tile = it % tiles;
    const int rest = it / tiles;
    b = rest % batch;
    g = rest / batch;
  }
  __device__ __forceinline__ void next(int tiles, int batch) {
    if (++tile == tiles) {
      tile = 0;
      if (++b == batch) {
        b = 0;
        ++g;
      }
    }
  }
};


// k_bconv_tc2 epilogue for 8 destination rows: r = the 32 TMEM columns (4 byte
// planes per row) of this thread's coefficient; dq = {q, q^-1}, doff = row * n
// ROWS > 0: the 8 destination rows are consecutive rows of ROWS words (the
// common case at N = 2^16): one address, then immediate offsets per store
template <bool FULL, int ROWS = 0>
__device__ __forceinline__ void tc2_store8(const uint32_t (&r)[32], const uint2* dq, const uint32_t* doff, int nv,
                                           uint32_t* dthr) {
  const uint4* dq4 = reinterpret_cast<const uint4*>(dq);
  uint32_t off[8];
  if (ROWS) {
    off[0] = doff[0];
  } else {
    const uint4 o0 = *reinterpret_cast<const uint4*>(doff), o1 = *reinterpret_cast<const uint4*>(doff + 4);
    off[0] = o0.x; off[1] = o0.y; off[2] = o0.z; off[3] = o0.w;
    off[4] = o1.x; off[5] = o1.y; off[6] = o1.z; off[7] = o1.w;
  }
  const uint64_t base = reinterpret_cast<uint64_t>(dthr);
  uint32_t* rbase = dthr + off[0];
#pragma unroll
  for (int u2 = 0; u2 < 4; ++u2) {
    const uint4 qq = dq4[u2];  // {q, q^-1} of rows 2 u2, 2 u2 + 1
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int u = 2 * u2 + e;
      const uint32_t q = e ? qq.z : qq.x, qi = e ? qq.w : qq.y;
      const uint32_t x = r[4 * u] + (r[4 * u + 1] << 8);      // < 2^31
      const uint32_t y = r[4 * u + 2] + (r[4 * u + 3] << 8);  // < 2^31
      uint32_t lo, hi;  // x + 2^16 y = sum_a 2^(8a) acc_a < 2^46
      asm("mad.lo.cc.u32 %0, %2, 65536, %3;\n\tmadc.hi.u32 %1, %2, 65536, 0;\n" : "=r"(lo), "=r"(hi) : "r"(y), "r"(x));
      const uint32_t v = sub_if(mont_reduce64s(lo, hi, q, qi), q);
      if (ROWS) {
        if (FULL || u < nv) rbase[u * ROWS] = v;
      } else {
        uint64_t addr;  // one IMAD.WIDE.U32 per store address
        asm("mad.wide.u32 %0, %1, 4, %2;" : "=l"(addr) : "r"(off[u]), "l"(base));
        if (FULL || u < nv) asm volatile("st.global.u32 [%0], %1;" ::"l"(addr), "r"(v) : "memory");
      }
    }
  }
}

// k_bconv_tc2: the same GEMM with a slimmer instruction stream (the kernel
// above is issue-bound at ~60% issue with ~800 warp instructions per item, a
// quarter of them integer divisions decoding the item twice):
//  * incremental item cursors (no division per item);
//  * epilogue per output: the 4 byte planes combined into (lo, hi) with two
//    shift-adds and one 64-bit shift-add, then the SUBTRACTIVE Montgomery
//    reduction hi - umulhi(lo q^-1, q) (no carry term) and one min for the
//    canonical residue -- identical canonical output;
//  * per-group destination constants staged as {q, q^-1} pairs and 32-bit
//    row offsets (vector loads, 8 rows at a time);
//  * the next 8-row block's tcgen05.ld is issued before the current block is
//    reduced (two 32-register buffers), so the TMEM load latency is hidden.
template <int KB, int NCOLS>
__global__ void __launch_bounds__(kTT) k_bconv_tc2(BconvLaunch a, BconvTc t, int n) {
  extern __shared__ __align__(128) unsigned char smraw[];
  constexpr int kSbo = (KB / 16) * 128;
  constexpr int kATile = kTT * KB;
  const int rawStage = a.max_sc * kTT;
  const int dcPad = (t.max_dc + 7) / 8 * 8;
  uint32_t* raw = reinterpret_cast<uint32_t*>(smraw);              // [kNst][max_sc][128] u32
  unsigned char* At = smraw + (size_t)kNst * rawStage * 4;         // A tile (128-B aligned)
  unsigned char* Bt = At + kATile;                                 // B table of the current group
  uint2* dq = reinterpret_cast<uint2*>(Bt + t.max_npad * KB);      // [dcPad] {q, q^-1}
  uint32_t* doff = reinterpret_cast<uint32_t*>(dq + dcPad);        // [dcPad] destination row * n
  uint32_t* dcont = doff + dcPad;                                   // [dcPad / 8] 8-row block = consecutive rows
  uint64_t* mbar = reinterpret_cast<uint64_t*>(doff + 2 * dcPad);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(mbar + 1);

  const int tid = threadIdx.x, warp = tid >> 5;
  const int tiles = n / kTT;
  const int items = a.ngroups * a.batch * tiles;
  const int chunk = (items + gridDim.x - 1) / gridDim.x;
  const int i0 = blockIdx.x * chunk, i1 = min(items, i0 + chunk);
  if (i0 >= i1) return;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tslot)),
                 "n"(NCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    mbar_init(mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);

  TcCursor ic;  // the next item to issue
  ic.init(i0, tiles, a.batch);
  int icount = i0, ig = -1;
  uint32_t isrc = 0, isc = 0;  // the issue group's source offset and row count (reloaded on group change)
  auto issue = [&](int slot) {  // raw source tile of item `ic` into ring slot `slot`, then advance
    if (icount < i1) {
      if (ic.g != ig) {
        ig = ic.g;
        isrc = a.groups[ig].src_off;
        isc = a.groups[ig].sc;
      }
      // source row j = warp + 4 m (m < 4: sc <= 16), 16-B chunk = lane (32 per 128-word row)
      const uint32_t* src = a.src + ic.b * a.src_bs + ((size_t)isrc + warp) * n + (size_t)ic.tile * kTT + 4 * (tid & 31);
      uint32_t* dst = raw + slot * rawStage + warp * kTT + 4 * (tid & 31);
#pragma unroll
      for (int m = 0; m < 4; ++m)
        if (warp + 4 * m < (int)isc) cp16(dst + 4 * m * kTT, src + (size_t)(4 * m) * n);
      ic.next(tiles, a.batch);
      ++icount;
    }
    cp_commit();
  };
#pragma unroll
  for (int s = 0; s < kNst - 1; ++s) issue(s);

  TcCursor pc;  // the item being processed
  pc.init(i0, tiles, a.batch);
  int cur_g = -1, sc = 0, dc = 0, npad = 16;
  uint32_t phase = 0;
  for (int it = i0, k = 0; it < i1; ++it, ++k) {
    cp_wait<kNst - 2>();
    __syncthreads();  // raw tile k landed for all threads; iteration k-1 fully done (A, B, TMEM free)
    issue((k + kNst - 1) % kNst);
    const int tile = pc.tile, b = pc.b, g = pc.g;
    pc.next(tiles, a.batch);
    if (g != cur_g) {  // new group: its B table and destination constants
      cur_g = g;
      const BconvGroup G = a.groups[g];
      sc = (int)G.sc;
      dc = (int)G.dc;
      npad = (4 * dc + 15) / 16 * 16;
      const uint4* B = reinterpret_cast<const uint4*>(t.btab + t.boff[g]);
      uint4* Bs = reinterpret_cast<uint4*>(Bt);
      for (int e = tid; e < npad * KB / 16; e += kTT) Bs[e] = __ldg(B + e);
      for (int i = tid; i < dcPad; i += kTT) {
        uint2 d = make_uint2(1u, 1u);
        uint32_t o = 0;
        if (i < dc) {
          const PrimeDev P = a.primes[a.dst_prime[G.map_off + i]];
          d = make_uint2(P.q, P.qinv);
          o = a.dst_row[G.map_off + i] * (uint32_t)n;
        }
        dq[i] = d;
        doff[i] = o;
      }
      for (int c = tid; c < dcPad / 8; c += kTT) {  // block c: rows 8c .. 8c+7 all valid and consecutive
        bool ok = 8 * c + 8 <= dc;
        for (int u = 1; ok && u < 8; ++u) ok = a.dst_row[G.map_off + 8 * c + u] == a.dst_row[G.map_off + 8 * c] + u;
        dcont[c] = ok;
      }
    }
    {  // transpose: row x = tid, K chunk c holds the words src[4c .. 4c+3][x] (zero past sc)
      const uint32_t* R = raw + (k % kNst) * rawStage;
      uint32_t w[KB / 4];
#pragma unroll
      for (int j = 0; j < KB / 4; ++j) w[j] = j < sc ? R[j * kTT + tid] : 0u;
      unsigned char* row = At + (tid >> 3) * kSbo + (tid & 7) * 16;
#pragma unroll
      for (int c = 0; c < KB / 16; ++c)
        *reinterpret_cast<uint4*>(row + c * 128) = make_uint4(w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
    }
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      fence_after();
      const uint32_t idesc = idesc_u8(kTT, npad);
      const uint32_t a0 = smem_u32(At), b0 = smem_u32(Bt);
#pragma unroll
      for (int kk = 0; kk < KB / 32; ++kk)
        mma_u8(tmem, sdesc(a0 + kk * 256, 128, kSbo), sdesc(b0 + kk * 256, 128, kSbo), idesc, kk > 0);
      mma_commit(mbar);
    }
    mbar_wait(mbar, phase);
    phase ^= 1;
    fence_after();
    uint32_t* dthr = a.dst + b * a.dst_bs + (size_t)tile * kTT + tid;
    uint32_t r[2][32];
    tmem_ld32_nowait(lane_addr, r[0]);
    tmem_wait_ld(r[0]);
    if (kTc2Fast3 && dc > 16 && dc <= 24 && n == 65536 && dcont[0] && dcont[1]) {
      // the common shapes (ModUp digits / ModDown at level 24: 24 destination rows,
      // the merged HMult drop-and-divide: 22) as three straight-line 8-row blocks,
      // the first two runs of consecutive rows: no per-block branches
      tmem_ld32_nowait(lane_addr + 32, r[1]);
      tc2_store8<true, 65536>(r[0], dq, doff, 8, dthr);
      tmem_wait_ld(r[1]);
      tmem_ld32_nowait(lane_addr + 64, r[0]);
      tc2_store8<true, 65536>(r[1], dq + 8, doff + 8, 8, dthr);
      tmem_wait_ld(r[0]);
      if (dc == 24 && dcont[2])
        tc2_store8<true, 65536>(r[0], dq + 16, doff + 16, 8, dthr);
      else
        tc2_store8<false>(r[0], dq + 16, doff + 16, dc - 16, dthr);
    } else
#pragma unroll 1
    for (int i8 = 0; i8 < dc; i8 += 16) {  // two 8-row blocks per trip: buffer 0, then buffer 1
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int ib = i8 + 8 * h;
        if (ib >= dc) break;
        if (ib + 8 < dc) tmem_ld32_nowait(lane_addr + 4 * (ib + 8), r[h ^ 1]);  // next block in flight
        if (ib + 8 <= dc) {
          if (n == 65536 && dcont[ib >> 3])
            tc2_store8<true, 65536>(r[h], dq + ib, doff + ib, 8, dthr);
          else
            tc2_store8<true>(r[h], dq + ib, doff + ib, 8, dthr);
        } else {
          tc2_store8<false>(r[h], dq + ib, doff + ib, dc - ib, dthr);
        }
        tmem_wait_ld(r[h ^ 1]);
      }
    }
    fence_before();
  }
  cp_wait<0>();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(NCOLS));
}

template <int KB, int NCOLS>
void launch_tc(const BconvLaunch& a, const BconvTc& t, int n, cudaStream_t st) {
  const int smem = kNst * a.max_sc * kTT * 4 + kTT * KB + t.max_npad * KB + ((t.max_dc + 7) / 8 * 8) * 16 + 16;
  static int grid = 0, smem_set = 0;
  if (smem > smem_set) {
    cudaFuncSetAttribute(k_bconv_tc<KB, NCOLS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_bconv_tc2<KB, NCOLS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    smem_set = smem;
    grid = 0;
  }
  if (!grid) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_bconv_tc<KB, NCOLS>, kTT, smem);
    if (std::getenv("CK32_DEBUG")) fprintf(stderr, "bconv_tc occupancy %d (%s) smem %d\n", per, cudaGetErrorString(e), smem);
    // the occupancy API reports 1 for kernels that allocate TMEM; the real
    // limits are smem / registers / threads and the 512 TMEM columns per SM
    per = std::max(per, std::min(227 * 1024 / (smem + 1024), 2048 / kTT));
    per = std::min(per, 512 / NCOLS);
    if (const char* e = std::getenv("CK32_BCONV_CTAS"))  // cap (A/B of the 2-stream overlap)
      if (std::atoi(e) > 0) per = std::min(per, std::atoi(e));
    grid = sms * std::max(1, per);
  }
  const int items = a.ngroups * a.batch * (n / kTT);
  if (t.variant == 1)
    k_bconv_tc<KB, NCOLS><<<std::min(grid, items), kTT, smem, st>>>(a, t, n);
  else
    k_bconv_tc2<KB, NCOLS><<<std::min(grid, items), kTT, smem, st>>>(a, t, n);
}

}  // namespace

bool bconv_tc_supported(int n, int max_sc, int max_dc) { return n % kTT == 0 && max_sc <= 16 && max_dc <= 64; }
// (max_dc <= 64: N = 4 dc <= 256 TMEM columns)

void bconv_tc(int n, const BconvLaunch& a, const BconvTc& t, cudaStream_t st) {
  const bool k64 = a.max_sc > 8;
  if (t.max_npad <= 128) {
    if (k64)
      launch_tc<64, 128>(a, t, n, st);
    else
      launch_tc<32, 128>(a, t, n, st);
  } else {
    if (k64)
      launch_tc<64, 256>(a, t, n, st);
    else
      launch_tc<32, 256>(a, t, n, st);
  }
}

}  // namespace ck
