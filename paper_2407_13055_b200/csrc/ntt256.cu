// N = 2^16 NTT / INTT specialised for sm_100a (256 x 256 decomposition).
//
// Same transform as ntt.cpp:176-272 (and the generic kernels in ntt.cu):
// forward = DIF Cooley-Tukey, natural -> bit-reversed, Montgomery entry merge;
// inverse = Gentleman-Sande, exit merge with the fused BConv part-1 factor.
//
// Structure (one kernel per pass, persistent CTAs):
//  * work items are tiles of one limb: 256 rows x 32 columns (column pass) or
//    16 rows x 256 (row pass); every CTA loops over its items and
//    double-buffers them in shared memory with cp.async (16-byte, L1
//    bypass), so HBM streaming of item k+1 overlaps the butterflies of item k;
//  * column pass: a thread owns 4 adjacent columns (uint4) x 16 rows, runs 4
//    radix-2 stages (one twiddle per 4 butterflies, warp-broadcast from the
//    tile's 256-entry table), writes back in place, then reads the transposed
//    16 rows and runs the other 4 stages, storing 16 uint4 straight to HBM;
//  * row pass: 16 threads (half a warp) own a 256-point row; the exchange is
//    warp-local (no CTA barrier); the row's 30 twiddle pairs live in
//    registers and are reused across consecutive batch items of the job.
// Butterflies: Harvey-lazy Shoup (IMAD.HI + 2 IMAD).  Inverse: values in
// [0, 2q).  Forward: values in [0, 8q) (q < 2^29), x reduced by 4q only at
// every other stage (`ctl`), the column pass hands [0, 8q) to the row pass
// through HBM and the row pass canonicalises once at the end.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <unordered_map>

#include "ck_common.cuh"
#include "ck_kernels.h"

namespace ck {
namespace {

constexpr int kN = 65536;
constexpr int kR = 256;

__device__ __forceinline__ void stg4(uint32_t* p, uint4 v) { *reinterpret_cast<uint4*>(p) = v; }
__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(K) : "memory");
}

// ---- TMA (cp.async.bulk.tensor) + mbarrier helpers for the column pass
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init1(uint64_t* mbar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_addr(mbar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(mbar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* mbar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "TMA_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TMA_WAIT_%=;\n\t}\n" ::"r"(smem_addr(mbar)),
      "r"(parity)
      : "memory");
}
// one [256 rows][32 columns] uint32 box of the 2D map (columns innermost)
__device__ __forceinline__ void tma_tile(void* dst, const CUtensorMap* map, int col, int row, uint64_t* mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
      ::"r"(smem_addr(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(col), "r"(row), "r"(smem_addr(mbar))
      : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(mbar))
               : "memory");
}

// ALU-pinned adds.  ptxas issues about half of the butterflies' two-input
// adds (x + t) as IMAD.IADD on the fmaheavy pipe -- the pipe that bounds the
// NTT (IMAD.HI = 4 cycles, IMAD = 2 per warp instruction) -- while the ALU
// pipe has slack.  min(a + b, bound) with a runtime bound the sum never
// reaches is the same value and compiles to ONE VIADDMNMX, which only the
// ALU pipe executes.  Measured neutral (r2s4: k_row<0, 3> -4%, the step
// unchanged: ptxas moves other work onto IMAD.MOV instead), so off by default.
#ifndef CK32_ALU_ADD
#define CK32_ALU_ADD 0
#endif
__device__ __forceinline__ uint32_t add_alu(uint32_t a, uint32_t b, uint32_t bound) {
  return CK32_ALU_ADD ? min(a + b, bound) : a + b;
}

// forward CT butterfly, Harvey lazy: x,y in [0,4q) -> [0,4q)
__device__ __forceinline__ void ct(uint32_t& x, uint32_t& y, uint32_t w, uint32_t wp, uint32_t q, uint32_t q2) {
  const uint32_t xx = sub_if(x, q2);
  const uint32_t t = shoup_mul(y, w, wp, q);
  x = xx + t;
  y = xx - t + q2;
}
// forward CT butterfly on the lazy [0, 8q) schedule (q < 2^29, so 8q < 2^32):
// RED reduces x from [0, 8q) to [0, 4q) (outputs [0, 6q)); without it the
// bound grows by 2q (outputs < B + 2q).  Reducing at every other stage keeps
// every value below 8q with half the sub_if work of `ct`.
template <bool RED>
__device__ __forceinline__ void ctl(uint32_t& x, uint32_t& y, uint32_t w, uint32_t wp, uint32_t q, uint32_t q2,
                                    uint32_t q4) {
  const uint32_t xx = RED ? sub_if(x, q4) : x;
  const uint32_t t = shoup_mul(y, w, wp, q);
  x = add_alu(xx, t, 2 * q4);  // < 8q
  y = xx - t + q2;
}
__device__ __forceinline__ uint32_t canon8(uint32_t x, uint32_t q, uint32_t q2, uint32_t q4) {
  return sub_if(sub_if(sub_if(x, q4), q2), q);  // [0, 8q) -> [0, q)
}
// inverse GS butterfly: x,y in [0,2q) -> [0,2q)
__device__ __forceinline__ void gs(uint32_t& x, uint32_t& y, uint32_t w, uint32_t wp, uint32_t q, uint32_t q2) {
  const uint32_t u = sub_if(add_alu(x, y, 2 * q2), q2);  // x + y < 4q
  y = shoup_mul(x - y + q2, w, wp, q);
  x = u;
}
__device__ __forceinline__ void ct4(uint4& x, uint4& y, uint2 w, uint32_t q, uint32_t q2) {
  ct(x.x, y.x, w.x, w.y, q, q2);
  ct(x.y, y.y, w.x, w.y, q, q2);
  ct(x.z, y.z, w.x, w.y, q, q2);
  ct(x.w, y.w, w.x, w.y, q, q2);
}
__device__ __forceinline__ void gs4(uint4& x, uint4& y, uint2 w, uint32_t q, uint32_t q2) {
  gs(x.x, y.x, w.x, w.y, q, q2);
  gs(x.y, y.y, w.x, w.y, q, q2);
  gs(x.z, y.z, w.x, w.y, q, q2);
  gs(x.w, y.w, w.x, w.y, q, q2);
}

// Four radix-2 CT stages over v[16] (uint4 lanes: 64 butterflies per stage),
// stage t pairing rows at distance 8 >> t with twiddle tw(t, blk).  The
// butterflies of a stage are issued in two groups of 16 with the three
// multiplies of every butterfly in separate passes (all IMAD.HI, then all
// q * hi, then all y * w - q * hi), so 16 independent multiplies sit between
// dependent ones instead of 4 (the `wait` stall of the per-butterfly order).
// RED: bit t set = stage t reduces x from [0, 8q) to [0, 4q) first (lazy
// schedule of `ctl`); clear = x is used as is.
#ifndef CK32_CT_PLAIN
#define CK32_CT_PLAIN 0
#endif
template <int T0, unsigned RED, class TWF>
__device__ __forceinline__ void ct_stages16(uint4 (&v)[16], TWF tw, uint32_t q, uint32_t q2, uint32_t q4) {
  if constexpr (CK32_CT_PLAIN != 0) {  // per-butterfly order (the round-1 skeleton's): measured 3% slower (r2s4)
#pragma unroll
    for (int t = T0; t < 4; ++t) {
      const int d = 8 >> t;
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int blk = p / d, j = blk * 2 * d + p % d;
        const uint2 w = tw(t, blk);
        uint32_t* x = &v[j].x;
        uint32_t* y = &v[j + d].x;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if ((RED >> t) & 1u) ctl<true>(x[c], y[c], w.x, w.y, q, q2, q4);
          else ctl<false>(x[c], y[c], w.x, w.y, q, q2, q4);
        }
      }
    }
  } else {
#pragma unroll
    for (int t = T0; t < 4; ++t) {
      const int d = 8 >> t;
      uint2 w[8];
#pragma unroll
      for (int blk = 0; blk < (1 << t); ++blk) w[blk] = tw(t, blk);
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        uint32_t h[16];
#pragma unroll
        for (int pp = 0; pp < 4; ++pp) {
          const int p = 4 * g + pp, blk = p / d, j = blk * 2 * d + p % d;
          h[4 * pp + 0] = __umulhi(v[j + d].x, w[blk].y);
          h[4 * pp + 1] = __umulhi(v[j + d].y, w[blk].y);
          h[4 * pp + 2] = __umulhi(v[j + d].z, w[blk].y);
          h[4 * pp + 3] = __umulhi(v[j + d].w, w[blk].y);
        }
#pragma unroll
        for (int e = 0; e < 16; ++e) h[e] *= q;
#pragma unroll
        for (int pp = 0; pp < 4; ++pp) {
          const int p = 4 * g + pp, blk = p / d, j = blk * 2 * d + p % d;
          const uint32_t ww = w[blk].x;
          uint32_t* y = &v[j + d].x;
          uint32_t* x = &v[j].x;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint32_t tt = y[c] * ww - h[4 * pp + c];  // shoup_mul: [0, 2q)
            const uint32_t xx = ((RED >> t) & 1u) ? sub_if(x[c], q4) : x[c];
            x[c] = add_alu(xx, tt, 2 * q4);  // < 8q
            y[c] = xx - tt + q2;
          }
        }
      }
    }
  }
}

// Inverse GS stages t = T0 .. T1-1 over v[16] (uint4 lanes), stage t pairing
// rows at distance 1 << t with twiddle tw(t, blk), blk = p >> t: the
// multiplies of each group of 16 butterflies issued as in ct_stages16 (all
// IMAD.HI, then all q * hi, then the rest).
template <int T0, int T1, class TWF>
__device__ __forceinline__ void gs_stages16(uint4 (&v)[16], TWF tw, uint32_t q, uint32_t q2) {
#pragma unroll
  for (int t = T0; t < T1; ++t) {
    const int d = 1 << t;
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      uint32_t dd[16], h[16];
      uint2 w[4];
#pragma unroll
      for (int pp = 0; pp < 4; ++pp) {
        const int p = 4 * g + pp, blk = p / d, j = blk * 2 * d + p % d;
        w[pp] = tw(t, blk);
        uint32_t* x = &v[j].x;
        uint32_t* y = &v[j + d].x;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          dd[4 * pp + c] = x[c] - y[c] + q2;
          x[c] = sub_if(add_alu(x[c], y[c], 2 * q2), q2);
        }
      }
#pragma unroll
      for (int e = 0; e < 16; ++e) h[e] = __umulhi(dd[e], w[e >> 2].y);
#pragma unroll
      for (int e = 0; e < 16; ++e) h[e] *= q;
#pragma unroll
      for (int pp = 0; pp < 4; ++pp) {
        const int p = 4 * g + pp, blk = p / d, j = blk * 2 * d + p % d;
        uint32_t* y = &v[j + d].x;
#pragma unroll
        for (int c = 0; c < 4; ++c) y[c] = dd[4 * pp + c] * w[pp].x - h[4 * pp + c];
      }
    }
  }
}

// One radix-2 stage over v[16] (8 butterflies, pairs at distance D, twiddle
// index blk = p / D) with the multiplies issued in groups as in
// ct_stages16: all IMAD.HI, then all q * hi, then the rest -- 8 independent
// multiplies between dependent ones instead of 1 (the row passes otherwise
// issue one Shoup multiply chain per butterfly and stall on its latency).
// Forward CT on the lazy schedule (RED: x reduced from [0, 8q) first).
template <int D, bool RED, class TWF>
__device__ __forceinline__ void ct_stage8(uint32_t (&v)[16], TWF tw, uint32_t q, uint32_t q2, uint32_t q4) {
  uint2 w[8];
  uint32_t h[8];
#pragma unroll
  for (int p = 0; p < 8; ++p) w[p] = tw(p / D);
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const int j = (p / D) * 2 * D + p % D;
    h[p] = __umulhi(v[j + D], w[p].y);
  }
#pragma unroll
  for (int p = 0; p < 8; ++p) h[p] *= q;
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const int j = (p / D) * 2 * D + p % D;
    const uint32_t tt = v[j + D] * w[p].x - h[p];
    const uint32_t xx = RED ? sub_if(v[j], q4) : v[j];
    v[j] = add_alu(xx, tt, 2 * q4);  // < 8q
    v[j + D] = xx - tt + q2;
  }
}
// Inverse GS stage over v[16] (pairs at distance D), grouped the same way.
template <int D, class TWF>
__device__ __forceinline__ void gs_stage8(uint32_t (&v)[16], TWF tw, uint32_t q, uint32_t q2) {
  uint2 w[8];
  uint32_t dd[8], h[8];
#pragma unroll
  for (int p = 0; p < 8; ++p) w[p] = tw(p / D);
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const int j = (p / D) * 2 * D + p % D;
    dd[p] = v[j] - v[j + D] + q2;
    v[j] = sub_if(add_alu(v[j], v[j + D], 2 * q2), q2);
  }
#pragma unroll
  for (int p = 0; p < 8; ++p) h[p] = __umulhi(dd[p], w[p].y);
#pragma unroll
  for (int p = 0; p < 8; ++p) h[p] *= q;
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const int j = (p / D) * 2 * D + p % D;
    v[j + D] = dd[p] * w[p].x - h[p];
  }
}

// ============================================================ column pass ==
#ifndef CK32_COL_GS_GROUPED
#define CK32_COL_GS_GROUPED 1
#endif
constexpr bool kColGsGrouped = CK32_COL_GS_GROUPED;  // inverse column pass: grouped GS multiplies (gs_stages16)
constexpr int kCT = 128;              // threads: tau = tid>>3 (16), cq = tid&7 (8)
constexpr int kCCols = 32;            // columns per tile
constexpr int kCTiles = kR / kCCols;  // 8 tiles per limb
struct ColBuf {
  uint4 tile[256 * (kCCols / 4)];  // [row][quad], 32 KB
  uint2 tw[256];                   // the prime's first 256 twiddle pairs
};

__device__ __forceinline__ void col_prefetch(ColBuf& B, const uint32_t* g, const uint2* tw) {
  // 256 rows x 128 B + 2 KB of twiddles, 16 B per cp.async
  for (int e = threadIdx.x; e < 256 * 8; e += kCT) {
    const int r = e >> 3, c4 = e & 7;
    cp16(&B.tile[r * 8 + c4], g + r * kR + 4 * c4);
  }
  cp16(&B.tw[2 * threadIdx.x], tw + 2 * threadIdx.x);
}

// Decode the i-th column-pass item: tile fastest, then batch, then job.
template <int TILES = kCTiles>
__device__ __forceinline__ void col_item(int it, int batch, int& job, int& b, int& tile) {
  tile = it % TILES;
  const int rest = it / TILES;
  b = rest % batch;
  job = rest / batch;
}

// TWR: the twiddle tables ride in their own 2-slot ring (slot = item parity)
// instead of inside the tile buffer, so phase B reads them from shared memory
// after the next item's prefetch has started (no 15 twiddle pairs in
// registers: 124 -> ~96 registers, MINB CTAs per SM).
// LOGR: log2 of the row length (8: N = 2^16 = 256 x 256; 9: N = 2^17 =
// 256 columns of a 256 x 512 matrix, the same 256-point column transform).
// TMA (LOGR = 8, TWR, single buffer): the tile arrives with ONE
// cp.async.bulk.tensor.2d per item (a [256][32] box of the limb matrix, one
// 2D tensor map over the whole source allocation: rows of 256 words) plus one
// 1D bulk copy of the 2 KB twiddle slice, completing on an mbarrier --
// instead of 16 cp.async (and their address arithmetic) per thread.
template <bool INV, bool DB, bool TWR = false, int MINB = 1, int LOGR = 8, bool TMA = false>
__global__ void __launch_bounds__(kCT, MINB) k_col(const RowJob* __restrict__ jobs, const uint32_t* __restrict__ src,
                                             uint64_t src_bs, uint32_t* __restrict__ dst, uint64_t dst_bs, int batch,
                                             int njobs, const PrimeDev* __restrict__ primes,
                                             const uint2* __restrict__ tw_full, const ExitConst* __restrict__ exits,
                                             int entry, const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(128) unsigned char smraw[];
  ColBuf* buf = reinterpret_cast<ColBuf*>(smraw);
  // [2][256] twiddle ring (TWR): right after the single tile buffer (ColBuf::tw unused)
  uint2* twring = reinterpret_cast<uint2*>(smraw + (DB ? 2 * sizeof(ColBuf) : (TWR ? sizeof(ColBuf::tile) : sizeof(ColBuf))));
  uint64_t* mbar = reinterpret_cast<uint64_t*>(twring + 512);  // TMA: one mbarrier after the ring
  const int tid = threadIdx.x, cq = tid & 7, tau = tid >> 3;
  constexpr int RS = 1 << LOGR, NT = 256 << LOGR, TILES = RS / kCCols;  // row stride, limb size, tiles per limb
  const int items = njobs * batch * TILES;
  if (TMA) {
    if (tid == 0) mbar_init1(mbar);
    __syncthreads();
  }
  // the item decoded (and its job loaded) when it is prefetched is reused
  // when it is processed
  int nb = 0, ntile = 0;
  RowJob nJ{};
  auto prefetch = [&](ColBuf& B, int it, int k) {
    int job;
    col_item<TILES>(it, batch, job, nb, ntile);
    nJ = jobs[job];
    if (TMA) {
      if (tid == 0) {
        // the CTA's generic-proxy accesses of the buffer (ordered by the
        // caller's barrier) happen before the async-proxy writes
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        const uint64_t word = INV ? nb * dst_bs + (uint64_t)nJ.dst_off * NT : nb * src_bs + (uint64_t)nJ.src_off * NT;
        mbar_expect_tx(mbar, (uint32_t)sizeof(ColBuf::tile) + 256 * 8);
        tma_tile(&B.tile[0], &tmap, ntile * kCCols, (int)(word / RS), mbar);
        bulk_copy(&twring[(k & 1) * 256], tw_full + (size_t)nJ.prime * NT, 256 * 8, mbar);
      }
      return;
    }
    const uint32_t* base = INV ? dst + nb * dst_bs + (size_t)nJ.dst_off * NT : src + nb * src_bs + (size_t)nJ.src_off * NT;
    if (TWR) {
      const uint32_t* g = base + ntile * kCCols;
      for (int e = threadIdx.x; e < 256 * 8; e += kCT) cp16(&B.tile[(e >> 3) * 8 + (e & 7)], g + (e >> 3) * RS + 4 * (e & 7));
      const uint2* tw = tw_full + (size_t)nJ.prime * NT;
      cp16(&twring[(k & 1) * 256 + 2 * threadIdx.x], tw + 2 * threadIdx.x);
    } else {
      col_prefetch(B, base + ntile * kCCols, tw_full + (size_t)nJ.prime * NT);  // LOGR = 8 only
    }
  };
  int it = blockIdx.x;
  if (it < items) prefetch(buf[0], it, 0);
  cp_commit();
  for (int k = 0; it < items; ++k, it += gridDim.x) {
    ColBuf& B = buf[DB ? (k & 1) : 0];
    const int nxt = it + gridDim.x;
    const int b = nb, tile = ntile;
    const RowJob J = nJ;
    if (TMA) {
      mbar_wait_parity(mbar, k & 1);  // item k's tile and twiddles have landed
    } else {
      if (DB) {
        if (nxt < items) prefetch(buf[(k + 1) & 1], nxt, k + 1);
        cp_commit();
        cp_wait<1>();
      } else {
        cp_wait<0>();
      }
      __syncthreads();
    }
    const PrimeDev P = primes[J.prime];
    const uint32_t q = P.q, q2 = P.q2, q4 = 2 * P.q2;
    const uint2* TW = TWR ? twring + (k & 1) * 256 : B.tw;
    uint32_t* out = dst + b * dst_bs + (size_t)J.dst_off * NT + tile * kCCols + 4 * cq;
    uint4 v[16];
    if (!INV) {
      // ---- forward, stages 0..7 (r bits 7..0). phase A rows tau + 16 j.
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = B.tile[(tau + 16 * j) * 8 + cq];
      if (entry) {  // stage 0 with the entry merge x*R, y*psi^{N/2}*R (ntt.cpp:27-35)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
#define CK_E(c)                                                    \
  {                                                                \
    const uint32_t xx = shoup_mul(v[j].c, P.r, P.r_sh, q);         \
    const uint32_t tt = shoup_mul(v[j + 8].c, P.w1r, P.w1r_sh, q); \
    v[j].c = xx + tt;                                              \
    v[j + 8].c = xx - tt + q2;                                     \
  }
          CK_E(x) CK_E(y) CK_E(z) CK_E(w)
#undef CK_E
        }
        ct_stages16<1, 0x4>(v, [&](int t, int blk) { return TW[(1 << t) + blk]; }, q, q2, q4);
      } else {
        ct_stages16<0, 0x4>(v, [&](int t, int blk) { return TW[(1 << t) + blk]; }, q, q2, q4);
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) B.tile[(tau + 16 * j) * 8 + cq] = v[j];
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = B.tile[(16 * tau + j) * 8 + cq];
      uint2 twb[TWR ? 1 : 15];  // phase-B twiddles to registers so the buffer can be refilled
      if (!TWR) {
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
          for (int blk = 0; blk < (1 << t); ++blk) twb[(1 << t) - 1 + blk] = B.tw[(16 << t) + (tau << t) + blk];
      }
      if (!DB) {
        if (TMA) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // my reads/writes before TMA's
        __syncthreads();
        if (nxt < items) prefetch(buf[0], nxt, k + 1);
        cp_commit();
      }
      // phase B rows 16 tau + j: twiddle 2^s + tau 2^(s-4) + blk
      ct_stages16<0, 0x5>(
          v, [&](int t, int blk) { return TWR ? TW[(16 << t) + (tau << t) + blk] : twb[(1 << t) - 1 + blk]; }, q, q2, q4);
#pragma unroll
      for (int j = 0; j < 16; ++j) stg4(out + (16 * tau + j) * RS, v[j]);
    } else {
      const ExitConst ex = exits[J.epi];
      // ---- inverse, stages 8..15 (r bits 0..7). phase A rows 16 tau + j.
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = B.tile[(16 * tau + j) * 8 + cq];
      if (kColGsGrouped) {
        gs_stages16<0, 4>(v, [&](int t, int blk) { return TW[(128 >> t) + (tau << (3 - t)) + blk]; }, q, q2);
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int d = 1 << t;
#pragma unroll
          for (int p = 0; p < 8; ++p) {
            const int blk = p / d, j = blk * 2 * d + p % d;
            gs4(v[j], v[j + d], TW[(128 >> t) + (tau << (3 - t)) + blk], q, q2);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) B.tile[(16 * tau + j) * 8 + cq] = v[j];
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = B.tile[(tau + 16 * j) * 8 + cq];
      uint2 twb[TWR ? 1 : 15];  // index (8>>t)-1+blk, t < 3
      if (!TWR) {
#pragma unroll
        for (int t = 0; t < 3; ++t)
#pragma unroll
          for (int blk = 0; blk < (8 >> t); ++blk) twb[(8 >> t) - 1 + blk] = B.tw[(8 >> t) + blk];
      }
      if (!DB) {
        if (TMA) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // my reads/writes before TMA's
        __syncthreads();
        if (nxt < items) prefetch(buf[0], nxt, k + 1);
        cp_commit();
      }
      if (kColGsGrouped && TWR) {
        gs_stages16<0, 3>(v, [&](int t, int blk) { return TW[(8 >> t) + blk]; }, q, q2);
      } else {
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          const int d = 1 << t;
#pragma unroll
          for (int p = 0; p < 8; ++p) {
            const int blk = p / d, j = blk * 2 * d + p % d;
            gs4(v[j], v[j + d], TWR ? TW[(8 >> t) + blk] : twb[(8 >> t) - 1 + blk], q, q2);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {  // exit merge (ntt.cpp:76-84)
#define CK_X(c)                                                            \
  {                                                                        \
    const uint32_t u = v[j].c + v[j + 8].c, dd = v[j].c - v[j + 8].c + q2; \
    v[j].c = sub_if(shoup_mul(u, ex.x, ex.y, q), q);                       \
    v[j + 8].c = sub_if(shoup_mul(dd, ex.z, ex.w, q), q);                  \
  }
        CK_X(x) CK_X(y) CK_X(z) CK_X(w)
#undef CK_X
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) stg4(out + (tau + 16 * j) * RS, v[j]);
    }
    if (DB) __syncthreads();  // buffer k&1 is refilled by the prefetch of iteration k+1
  }
  cp_wait<0>();
}

// k_col_tma: the TMA column pass (k_col<.., TMA>) with its per-item
// descriptors pipelined one item ahead.  In k_col the next item's RowJob is
// loaded right before thread 0 issues its TMA (so warp 0 stalls on that
// load in the middle of the item) and the item's PrimeDev / exit constants
// are loaded after the tile wait (a dependent global load at every item
// start: the R2UR / IMAD.HI long-scoreboard stalls of the source-level ncu
// profile).  Here the next RowJob is requested at the top of the current
// item, its PrimeDev / exit constants right after its TMA is issued, and
// both are in registers when the item starts.  Same arithmetic, same smem.
template <bool INV>
__global__ void __launch_bounds__(kCT, 5) k_col_tma(const RowJob* __restrict__ jobs, uint64_t src_bs,
                                                   uint32_t* __restrict__ dst, uint64_t dst_bs, int batch, int njobs,
                                                   const PrimeDev* __restrict__ primes,
                                                   const uint2* __restrict__ tw_full,
                                                   const ExitConst* __restrict__ exits, int entry,
                                                   const __grid_constant__ CUtensorMap tmap, int dbg) {
  extern __shared__ __align__(128) unsigned char smraw[];
  uint4* tileb = reinterpret_cast<uint4*>(smraw);                              // [256][8] uint4, 32 KB
  uint2* twring = reinterpret_cast<uint2*>(smraw + sizeof(ColBuf::tile));     // [2][256]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(twring + 512);
  const int tid = threadIdx.x, cq = tid & 7, tau = tid >> 3;
  constexpr int NT = kN;
  const int items = njobs * batch * kCTiles;
  int it = blockIdx.x;
  if (it >= items) return;
  if (tid == 0) mbar_init1(mbar);
  __syncthreads();
  auto issue = [&](int b, int tile, const RowJob& J, int k) {  // thread 0: item's tile + twiddles -> smem
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    const uint64_t word = INV ? b * dst_bs + (uint64_t)J.dst_off * NT : b * src_bs + (uint64_t)J.src_off * NT;
    mbar_expect_tx(mbar, (uint32_t)sizeof(ColBuf::tile) + 256 * 8);
    tma_tile(tileb, &tmap, tile * kCCols, (int)(word / kR), mbar);
    bulk_copy(&twring[(k & 1) * 256], tw_full + (size_t)J.prime * NT, 256 * 8, mbar);
  };
  int b, tile, job;
  col_item<kCTiles>(it, batch, job, b, tile);
  RowJob J = jobs[job];
  PrimeDev P = primes[J.prime];
  ExitConst ex{};
  if (INV) ex = exits[J.epi];
  if (tid == 0) issue(b, tile, J, 0);
  // dbg (timing experiments only, CK32_COL_DBG; outputs are garbage): bit 0 = no
  // global stores, bit 1 = no TMA after the first item (the tile is reused)
  for (int k = 0;; ++k) {
    const int nxt = it + gridDim.x;
    const bool more = nxt < items;
    int nb = 0, ntile = 0, njob = 0;
    RowJob nJ{};
    if (more) {  // next item's descriptor: requested now, used after phase A
      col_item<kCTiles>(nxt, batch, njob, nb, ntile);
      nJ = jobs[njob];
    }
    if (!(dbg & 2) || k == 0) mbar_wait_parity(mbar, k & 1);  // item k's tile and twiddles have landed
    const uint32_t q = P.q, q2 = P.q2, q4 = 2 * P.q2;
    const uint2* TW = twring + (k & 1) * 256;
    uint32_t* out = dst + b * dst_bs + (size_t)J.dst_off * NT + tile * kCCols + 4 * cq;
    uint4 v[16];
    PrimeDev nP{};
    ExitConst nex{};
    if (!INV) {
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = tileb[(tau + 16 * j) * 8 + cq];
      if (entry) {  // stage 0 with the entry merge x*R, y*psi^{N/2}*R (ntt.cpp:27-35)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
#define CK_E(c)                                                    \
  {                                                                \
    const uint32_t xx = shoup_mul(v[j].c, P.r, P.r_sh, q);         \
    const uint32_t tt = shoup_mul(v[j + 8].c, P.w1r, P.w1r_sh, q); \
    v[j].c = xx + tt;                                              \
    v[j + 8].c = xx - tt + q2;                                     \
  }
          CK_E(x) CK_E(y) CK_E(z) CK_E(w)
#undef CK_E
        }
        ct_stages16<1, 0x4>(v, [&](int t, int blk) { return TW[(1 << t) + blk]; }, q, q2, q4);
      } else {
        ct_stages16<0, 0x4>(v, [&](int t, int blk) { return TW[(1 << t) + blk]; }, q, q2, q4);
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) tileb[(tau + 16 * j) * 8 + cq] = v[j];
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = tileb[(16 * tau + j) * 8 + cq];
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncthreads();
      if (more) {
        if (tid == 0 && !(dbg & 2)) issue(nb, ntile, nJ, k + 1);
        nP = primes[nJ.prime];
      }
      ct_stages16<0, 0x5>(v, [&](int t, int blk) { return TW[(16 << t) + (tau << t) + blk]; }, q, q2, q4);
      if (!(dbg & 1)) {
#pragma unroll
        for (int j = 0; j < 16; ++j) stg4(out + (16 * tau + j) * kR, v[j]);
      } else {  // keep the result live without a store
        uint32_t acc = 0;
        for (int j = 0; j < 16; ++j) acc ^= v[j].x ^ v[j].y ^ v[j].z ^ v[j].w;
        if (acc == 0x12345678u) out[0] = acc;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = tileb[(16 * tau + j) * 8 + cq];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int d = 1 << t;
#pragma unroll
        for (int p = 0; p < 8; ++p) {
          const int blk = p / d, j = blk * 2 * d + p % d;
          gs4(v[j], v[j + d], TW[(128 >> t) + (tau << (3 - t)) + blk], q, q2);
        }
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) tileb[(16 * tau + j) * 8 + cq] = v[j];
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = tileb[(tau + 16 * j) * 8 + cq];
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncthreads();
      if (more) {
        if (tid == 0 && !(dbg & 2)) issue(nb, ntile, nJ, k + 1);
        nP = primes[nJ.prime];
        nex = exits[nJ.epi];
      }
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        const int d = 1 << t;
#pragma unroll
        for (int p = 0; p < 8; ++p) {
          const int blk = p / d, j = blk * 2 * d + p % d;
          gs4(v[j], v[j + d], TW[(8 >> t) + blk], q, q2);
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {  // exit merge (ntt.cpp:76-84)
#define CK_X(c)                                                            \
  {                                                                        \
    const uint32_t u = v[j].c + v[j + 8].c, dd = v[j].c - v[j + 8].c + q2; \
    v[j].c = sub_if(shoup_mul(u, ex.x, ex.y, q), q);                       \
    v[j + 8].c = sub_if(shoup_mul(dd, ex.z, ex.w, q), q);                  \
  }
        CK_X(x) CK_X(y) CK_X(z) CK_X(w)
#undef CK_X
      }
      if (!(dbg & 1)) {
#pragma unroll
        for (int j = 0; j < 16; ++j) stg4(out + (tau + 16 * j) * kR, v[j]);
      } else {
        uint32_t acc = 0;
        for (int j = 0; j < 16; ++j) acc ^= v[j].x ^ v[j].y ^ v[j].z ^ v[j].w;
        if (acc == 0x12345678u) out[0] = acc;
      }
    }
    if (!more) break;
    it = nxt;
    b = nb;
    tile = ntile;
    J = nJ;
    P = nP;
    ex = nex;
  }
}

// =============================================================== row pass ==
// 8 rows per tile, 16 threads (half a warp) per row.  The tile's per-row
// permuted twiddle tables (256 pairs per row) are staged in shared memory
// once per (job, row tile) and reused for every batch item; data tiles are
// double-buffered with cp.async.
constexpr int kRT = 128;
#ifndef CK32_ROW_GROUPED
#define CK32_ROW_GROUPED 0
#endif
constexpr bool kRowGrouped = CK32_ROW_GROUPED;  // k_row stages with grouped multiplies (ct_stage8 / gs_stage8): measured equal (r2ap), off
constexpr int kRRows = kRT / 16;
constexpr int kRowStride = 336;  // element c at c + 4*(c>>4): conflict-free for both access shapes
__device__ __forceinline__ int rpos(int c) { return c + 4 * (c >> 4); }
constexpr int kRowBufWords = kRRows * kRowStride;
constexpr int kRowSmem = 2 * kRowBufWords * 4 + kRRows * kR * 8;

// the two rows (2 warp, 2 warp + 1) of a kRRows x 256 tile that warp `warp` owns
__device__ __forceinline__ void row_prefetch_warp(uint32_t* buf, const uint32_t* g, int warp, int lane) {
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int e = lane + 32 * m, r = 2 * warp + (e >> 6), c = (e & 63) * 4;
    cp16(buf + r * kRowStride + rpos(c), g + r * kR + c);
  }
}

// (job, row tile, b) item cursor, b fastest; TILES row tiles per limb
template <int TILES>
struct RowCursorT {
  int b, tile, job;
  __device__ __forceinline__ void init(int it, int batch) {
    b = it % batch;
    const int key = it / batch;
    tile = key % TILES;
    job = key / TILES;
  }
  __device__ __forceinline__ void next(int batch) {
    if (++b == batch) {
      b = 0;
      if (++tile == TILES) {
        tile = 0;
        ++job;
      }
    }
  }
};

// (job, row tile, b) item cursor, b fastest
struct RowCursor {
  int b, tile, job;
  __device__ __forceinline__ void init(int it, int batch) {
    b = it % batch;
    const int key = it / batch;
    tile = key % (kR / kRRows);
    job = key / (kR / kRRows);
  }
  __device__ __forceinline__ void next(int batch) {
    if (++b == batch) {
      b = 0;
      if (++tile == kR / kRRows) {
        tile = 0;
        ++job;
      }
    }
  }
};

// COMB (forward only): drop-and-divide combine fused into the store,
// out = (v - NTT(.)) * divisor^-1 (ckks.cpp:643-651), so the NTT output never
// makes the extra HBM round trip through k_combine.
// COMB == 2: the combine's operand rows v are loaded at the start of the item
// (into registers, their latency hidden by the 8 butterfly stages) instead of
// right before the store (round 1: long-scoreboard 4.1 per issue there).
template <bool INV, int COMB = 0>
__global__ void __launch_bounds__(kRT) k_row(const RowJob* __restrict__ jobs, const uint32_t* __restrict__ src,
                                             uint64_t src_bs, uint32_t* __restrict__ dst, uint64_t dst_bs, int batch,
                                             int njobs, const PrimeDev* __restrict__ primes,
                                             const uint2* __restrict__ tw2, CombineArgs cb = CombineArgs{}) {
  extern __shared__ __align__(128) unsigned char smraw[];
  uint32_t* sbuf = reinterpret_cast<uint32_t*>(smraw);
  uint2* tws = reinterpret_cast<uint2*>(smraw + 2 * kRowBufWords * 4);  // [kRRows][256]
  const int tid = threadIdx.x, rho = tid >> 4, tau = tid & 15;
  constexpr int kTiles = kR / kRRows;
  // items: (job, row tile, b), b fastest; contiguous chunk per CTA
  const int items = njobs * kTiles * batch;
  const int chunk = (items + gridDim.x - 1) / gridDim.x;
  const int i0 = blockIdx.x * chunk, i1 = min(items, i0 + chunk);
  if (i0 >= i1) return;
  // item cursors (job, row tile, b), advanced incrementally: no divisions and
  // no dependent job/prime loads inside the loop except at (job, tile) changes
  RowCursor c;
  c.init(i0, batch);
  RowJob Jc = jobs[c.job];
  RowCursor nx = c;
  RowJob Jn = Jc;
  auto in_ptr = [&](const RowCursor& x, const RowJob& J) {
    // forward pass 2 works in place on dst; inverse pass A reads src
    return INV ? src + x.b * src_bs + (size_t)J.src_off * kN + x.tile * kRRows * kR
               : dst + x.b * dst_bs + (size_t)J.dst_off * kN + x.tile * kRRows * kR;
  };
  const int warp = tid >> 5, lane = tid & 31;
  row_prefetch_warp(sbuf, in_ptr(nx, Jn), warp, lane);
  cp_commit();
  // this thread's 15 per-thread twiddle pairs (forward phase B / inverse phase
  // A), kept in registers across the batch items of one (job, row tile)
  uint2 twr[15];
  uint32_t q = 0, q2 = 0, q4 = 0;
  uint32_t di_c = 0, qinv_c = 0;  // COMB: the job's divisor inverse and q^-1, loaded with the job (not at the store)
  for (int it = i0, k = 0; it < i1; ++it, ++k) {
    uint32_t* line_buf = sbuf + (k & 1) * kRowBufWords;
    const int b = c.b, tile = c.tile;
    const RowJob J = Jc;
    const bool reload = it == i0 || b == 0;
    if (reload) {  // stage this warp's two rows of the tile's twiddle tables (2 x 2 KB)
      __syncwarp();
      const uint2* T = tw2 + ((size_t)J.prime * kR + tile * kRRows + 2 * warp) * kR;
      for (int e = lane; e < kR; e += 32) cp16(&tws[2 * warp * kR + 2 * e], &T[2 * e]);
      cp_commit();
    }
    if (it + 1 < i1) {
      const int pj = nx.job;
      nx.next(batch);
      if (nx.job != pj) Jn = jobs[nx.job];
      row_prefetch_warp(sbuf + ((k + 1) & 1) * kRowBufWords, in_ptr(nx, Jn), warp, lane);
    }
    cp_commit();
    cp_wait<1>();
    __syncwarp();  // each warp owns its two rows of every buffer: no CTA barrier
    const int r = tile * kRRows + rho;
    const uint2* W = tws + rho * kR;
    if (reload) {
      const PrimeDev P = primes[J.prime];
      q = P.q;
      q2 = P.q2;
      q4 = 2 * P.q2;
      if (COMB) {
        qinv_c = P.qinv;
        di_c = cb.dinv[J.dst_off % cb.out_q];
      }
    }
    if (reload) {
#pragma unroll
      for (int i = 0; i < 15; ++i) twr[i] = INV ? W[i * 16 + tau] : W[16 + i * 16 + tau];
    }
    uint32_t* line = line_buf + rho * kRowStride;
    uint32_t* orow = dst + b * dst_bs + (size_t)J.dst_off * kN + (size_t)r * kR;
    uint32_t v[16];
    uint4 vvr[COMB == 2 ? 4 : 1];
    if (COMB >= 3 && lane < 16) {  // L2 prefetch of the warp's 2 v rows (16 lines of 128 B)
      const uint32_t pi = J.dst_off / cb.out_q, i = J.dst_off - pi * cb.out_q;
      const size_t lofs = (size_t)(tile * kRRows + 2 * warp) * kR + lane * 32;
      const uint32_t* vr = cb.v + b * cb.v_bs + ((size_t)pi * cb.prow + i) * kN + lofs;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(vr));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(vr + kR));
      if (COMB == 4 && pi == 0) {  // HRot tail: the b rows too
        const uint32_t* br = cb.add + b * cb.add_bs + (size_t)i * kN + lofs;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(br));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(br + kR));
      }
    }
    if (COMB == 2) {  // J.dst_off = p * out_q + i; v row p * prow + i
      const uint32_t pi = J.dst_off / cb.out_q, i = J.dst_off - pi * cb.out_q;
      const uint32_t* vr = cb.v + b * cb.v_bs + ((size_t)pi * cb.prow + i) * kN + (size_t)r * kR + 16 * tau;
#pragma unroll
      for (int m = 0; m < 4; ++m) vvr[m] = __ldg(reinterpret_cast<const uint4*>(vr + 4 * m));
    }
    if (!INV) {
      // phase A: c = tau + 16 j, stages 8..11 (row-shared twiddles W[0..14])
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = line[rpos(tau + 16 * j)];
      if (kRowGrouped) {
        ct_stage8<8, true>(v, [&](int blk) { return W[blk]; }, q, q2, q4);
        ct_stage8<4, false>(v, [&](int blk) { return W[1 + blk]; }, q, q2, q4);
        ct_stage8<2, true>(v, [&](int blk) { return W[3 + blk]; }, q, q2, q4);
        ct_stage8<1, false>(v, [&](int blk) { return W[7 + blk]; }, q, q2, q4);
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int d = 8 >> t;
#pragma unroll
          for (int p = 0; p < 8; ++p) {
            const int blk = p / d, j = blk * 2 * d + p % d;
            const uint2 w = W[(1 << t) - 1 + blk];
            if (t % 2 == 0) ctl<true>(v[j], v[j + d], w.x, w.y, q, q2, q4);
            else ctl<false>(v[j], v[j + d], w.x, w.y, q, q2, q4);
          }
        }
      }
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
      // phase B: c = 16 tau + j, stages 12..15 (W[16 + k*16 + tau])
      if (kRowGrouped) {
        ct_stage8<8, true>(v, [&](int blk) { return twr[blk]; }, q, q2, q4);
        ct_stage8<4, false>(v, [&](int blk) { return twr[1 + blk]; }, q, q2, q4);
        ct_stage8<2, true>(v, [&](int blk) { return twr[3 + blk]; }, q, q2, q4);
        ct_stage8<1, false>(v, [&](int blk) { return twr[7 + blk]; }, q, q2, q4);
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int d = 8 >> t;
#pragma unroll
          for (int p = 0; p < 8; ++p) {
            const int blk = p / d, j = blk * 2 * d + p % d;
            const uint2 w = twr[(1 << t) - 1 + blk];
            if (t % 2 == 0) ctl<true>(v[j], v[j + d], w.x, w.y, q, q2, q4);
            else ctl<false>(v[j], v[j + d], w.x, w.y, q, q2, q4);
          }
        }
      }
      if (COMB == 4) {
        // HRot tail (ckks.cpp:875-882) fused: c_p = (v_p - NTT) d^-1 (+ b for
        // p = 0) at position x = 256 r + 16 tau + m, stored at dest(x) of the
        // rotation: the automorphism maps every aligned 32-block to one
        // aligned 32-block (acceptance criterion 6), so the two threads of a
        // block fill one 128 B line with their scattered stores
        const uint32_t pi = J.dst_off / cb.out_q, i = J.dst_off - pi * cb.out_q;
        const size_t xo = (size_t)r * kR + 16 * tau;
        const uint32_t* vr = cb.v + b * cb.v_bs + ((size_t)pi * cb.prow + i) * kN + xo;
        const uint32_t* br = cb.add + b * cb.add_bs + (size_t)i * kN + xo;
        uint32_t* orow_t = cb.out + b * cb.out_bs + ((size_t)pi * cb.out_q + i) * kN;
        const uint32_t di = di_c, qinv = qinv_c;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const uint4 vv = *reinterpret_cast<const uint4*>(vr + 4 * m);
          const uint4 ds = __ldg(reinterpret_cast<const uint4*>(cb.dest + xo + 4 * m));
          uint32_t o0 = sub_if(mont_mul(vv.x - canon8(v[4 * m], q, q2, q4) + q, di, q, qinv), q);
          uint32_t o1 = sub_if(mont_mul(vv.y - canon8(v[4 * m + 1], q, q2, q4) + q, di, q, qinv), q);
          uint32_t o2 = sub_if(mont_mul(vv.z - canon8(v[4 * m + 2], q, q2, q4) + q, di, q, qinv), q);
          uint32_t o3 = sub_if(mont_mul(vv.w - canon8(v[4 * m + 3], q, q2, q4) + q, di, q, qinv), q);
          if (pi == 0) {
            const uint4 bb = *reinterpret_cast<const uint4*>(br + 4 * m);
            o0 = sub_if(o0 + bb.x, q);
            o1 = sub_if(o1 + bb.y, q);
            o2 = sub_if(o2 + bb.z, q);
            o3 = sub_if(o3 + bb.w, q);
          }
          // stage at (block, dest & 31) in this row's (now free) line buffer
          const int x = 16 * tau + 4 * m, blk = x & ~31;
          line[blk + (ds.x & 31)] = o0;
          line[blk + (ds.y & 31)] = o1;
          line[blk + (ds.z & 31)] = o2;
          line[blk + (ds.w & 31)] = o3;
        }
        __syncwarp();
        {  // whole 32-word destination blocks: lanes 2k, 2k+1 write block k's two halves
          const int blk = (tau >> 1) * 32, half = (tau & 1) * 16;
          const uint32_t dbase = __ldg(cb.dest + (size_t)r * kR + blk) & ~31u;
#pragma unroll
          for (int m = 0; m < 4; ++m)
            stg4(orow_t + dbase + half + 4 * m, *reinterpret_cast<const uint4*>(line + blk + half + 4 * m));
        }
        __syncwarp();  // the line buffer is refilled by the prefetch of item k + 2
      } else if (COMB) {  // J.dst_off = p * out_q + i; v row p * prow + i; prime i
        const uint32_t pi = J.dst_off / cb.out_q, i = J.dst_off - pi * cb.out_q;
        const uint32_t* vr = cb.v + b * cb.v_bs + ((size_t)pi * cb.prow + i) * kN + (size_t)r * kR + 16 * tau;
        const uint32_t di = di_c, qinv = qinv_c;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const uint4 vv = COMB == 2 ? vvr[m] : *reinterpret_cast<const uint4*>(vr + 4 * m);
          uint4 o;
          o.x = sub_if(mont_mul(vv.x - canon8(v[4 * m], q, q2, q4) + q, di, q, qinv), q);
          o.y = sub_if(mont_mul(vv.y - canon8(v[4 * m + 1], q, q2, q4) + q, di, q, qinv), q);
          o.z = sub_if(mont_mul(vv.z - canon8(v[4 * m + 2], q, q2, q4) + q, di, q, qinv), q);
          o.w = sub_if(mont_mul(vv.w - canon8(v[4 * m + 3], q, q2, q4) + q, di, q, qinv), q);
          stg4(orow + 16 * tau + 4 * m, o);
        }
      } else {
#pragma unroll
        for (int m = 0; m < 4; ++m)
          stg4(orow + 16 * tau + 4 * m, make_uint4(canon8(v[4 * m], q, q2, q4), canon8(v[4 * m + 1], q, q2, q4),
                                                   canon8(v[4 * m + 2], q, q2, q4), canon8(v[4 * m + 3], q, q2, q4)));
      }
    } else {
      // phase A: c = 16 tau + j, inverse stages 0..3 (W[k*16 + tau])
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const uint4 x = *reinterpret_cast<const uint4*>(line + rpos(16 * tau) + 4 * m);
        v[4 * m] = x.x;
        v[4 * m + 1] = x.y;
        v[4 * m + 2] = x.z;
        v[4 * m + 3] = x.w;
      }
      if (kRowGrouped) {
        gs_stage8<1>(v, [&](int blk) { return twr[blk]; }, q, q2);
        gs_stage8<2>(v, [&](int blk) { return twr[8 + blk]; }, q, q2);
        gs_stage8<4>(v, [&](int blk) { return twr[12 + blk]; }, q, q2);
        gs_stage8<8>(v, [&](int blk) { return twr[14 + blk]; }, q, q2);
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int d = 1 << t;
          const int off = 16 - (16 >> t);
#pragma unroll
          for (int p = 0; p < 8; ++p) {
            const int blk = p / d, j = blk * 2 * d + p % d;
            const uint2 w = twr[off + blk];
            gs(v[j], v[j + d], w.x, w.y, q, q2);
          }
        }
      }
#pragma unroll
      for (int m = 0; m < 4; ++m)
        *reinterpret_cast<uint4*>(line + rpos(16 * tau) + 4 * m) =
            make_uint4(v[4 * m], v[4 * m + 1], v[4 * m + 2], v[4 * m + 3]);
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = line[rpos(tau + 16 * j)];
      // phase B: c = tau + 16 j, inverse stages 4..7 (row-shared W[240 + k])
      if (kRowGrouped) {
        gs_stage8<1>(v, [&](int blk) { return W[240 + blk]; }, q, q2);
        gs_stage8<2>(v, [&](int blk) { return W[248 + blk]; }, q, q2);
        gs_stage8<4>(v, [&](int blk) { return W[252 + blk]; }, q, q2);
        gs_stage8<8>(v, [&](int blk) { return W[254 + blk]; }, q, q2);
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int d = 1 << t;
          const int off = 16 - (16 >> t);
#pragma unroll
          for (int p = 0; p < 8; ++p) {
            const int blk = p / d, j = blk * 2 * d + p % d;
            const uint2 w = W[240 + off + blk];
            gs(v[j], v[j + d], w.x, w.y, q, q2);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) orow[tau + 16 * j] = v[j];
    }
    c = nx;
    Jc = Jn;
    __syncwarp();  // this warp's rows of buffer k&1 are refilled by the prefetch of iteration k+1
  }
  cp_wait<0>();
}

int g_col_grid[2] = {0, 0}, g_row_grid = 0;
int env_cap(const char* name) {  // a positive integer from the environment, else "no cap"
  const char* e = std::getenv(name);
  const int v = e ? std::atoi(e) : 0;
  return v > 0 ? v : 1 << 20;
}
bool g_col_db = false;
int g_col_var = 3;  // CK32_COL: 0 = twiddles in registers, 1 = twiddle ring (4 CTAs/SM), 2 = ring, 5 CTAs/SM (cp.async), 3 = ring, 5 CTAs/SM, TMA tile loads (default)
constexpr int kColRingSmem = (int)sizeof(ColBuf::tile) + 2 * 256 * 8;  // 36 KB (6 CTAs/SM measured no faster than 5)
constexpr int kColTmaSmem = kColRingSmem + 16;                             // + the TMA mbarrier

void init_grids() {
  if (g_row_grid) return;
  const char* v = std::getenv("CK32_NTT_COL_DB");
  g_col_db = v && v[0] == '1';
  if (const char* cv = std::getenv("CK32_COL")) g_col_var = std::atoi(cv);
  cudaFuncSetAttribute(k_col<false, false, true, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, kColRingSmem);
  cudaFuncSetAttribute(k_col<true, false, true, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, kColRingSmem);
  cudaFuncSetAttribute(k_col<false, false, true, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, kColRingSmem);
  cudaFuncSetAttribute(k_col<true, false, true, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, kColRingSmem);

  const int col_smem_db = 2 * (int)sizeof(ColBuf), col_smem_sb = (int)sizeof(ColBuf);
  cudaFuncSetAttribute(k_col<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, col_smem_db);
  cudaFuncSetAttribute(k_col<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, col_smem_db);
  cudaFuncSetAttribute(k_col<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, col_smem_sb);
  cudaFuncSetAttribute(k_col<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, col_smem_sb);
  cudaFuncSetAttribute(k_row<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRowSmem);
  cudaFuncSetAttribute(k_row<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRowSmem);
  int dev = 0, sms = 148, c1 = 1, c2 = 1, r1 = 1, r2 = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute(k_col<false, false, true, 5, 8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kColTmaSmem);
  cudaFuncSetAttribute(k_col<true, false, true, 5, 8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kColTmaSmem);
  cudaFuncSetAttribute(k_col<false, false, true, 6, 8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kColTmaSmem);
  cudaFuncSetAttribute(k_col<true, false, true, 6, 8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kColTmaSmem);
  cudaFuncSetAttribute(k_col_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kColTmaSmem);
  cudaFuncSetAttribute(k_col_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kColTmaSmem);
  if (g_col_var == 4) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c1, k_col_tma<false>, kCT, kColTmaSmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c2, k_col_tma<true>, kCT, kColTmaSmem);
  } else if (g_col_var == 5) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c1, k_col<false, false, true, 6, 8, true>, kCT, kColTmaSmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c2, k_col<true, false, true, 6, 8, true>, kCT, kColTmaSmem);
  } else if (g_col_var == 3) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c1, k_col<false, false, true, 5, 8, true>, kCT, kColTmaSmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c2, k_col<true, false, true, 5, 8, true>, kCT, kColTmaSmem);
  } else if (g_col_var == 1 || g_col_var == 2) {
    if (g_col_var == 1) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c1, k_col<false, false, true, 4>, kCT, kColRingSmem);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c2, k_col<true, false, true, 4>, kCT, kColRingSmem);
    } else {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c1, k_col<false, false, true, 5>, kCT, kColRingSmem);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c2, k_col<true, false, true, 5>, kCT, kColRingSmem);
    }
  } else if (g_col_db) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c1, k_col<false, true>, kCT, col_smem_db);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c2, k_col<true, true>, kCT, col_smem_db);
  } else {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c1, k_col<false, false>, kCT, col_smem_sb);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c2, k_col<true, false>, kCT, col_smem_sb);
  }
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r1, k_row<false>, kRT, kRowSmem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r2, k_row<true>, kRT, kRowSmem);
  // CK32_COL_CTAS / CK32_ROW_CTAS: cap the persistent grids' CTAs per SM (A/B
  // of leaving SM room for the other stream's kernels)
  const int ccap = env_cap("CK32_COL_CTAS"), rcap = env_cap("CK32_ROW_CTAS");
  g_col_grid[0] = sms * max(1, min(c1, ccap));
  g_col_grid[1] = sms * max(1, min(c2, ccap));
  g_row_grid = sms * max(1, min(min(r1, r2), rcap));
}

// 2D tensor map over a limb matrix: rows of 256 uint32 starting at `base`,
// box = [256 rows][32 columns] (one column-pass tile).  The map spans 2^31
// rows: only boxes inside the caller's allocation are ever requested.
// Encoded on the host once per base address (cuTensorMapEncodeTiled through
// the runtime's driver entry point).
const CUtensorMap& col_tensor_map(const void* base) {
  static std::mutex mu;
  static std::unordered_map<const void*, CUtensorMap> cache;
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(base);
  if (it != cache.end()) return it->second;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  CUtensorMap m;
  const cuuint64_t dims[2] = {(cuuint64_t)kR, (cuuint64_t)1 << 31};
  const cuuint64_t strides[1] = {(cuuint64_t)kR * 4};
  const cuuint32_t box[2] = {(cuuint32_t)kCCols, 256u};
  const cuuint32_t estr[2] = {1u, 1u};
  const CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed");
  if (cache.size() > 4096) cache.clear();
  return cache.emplace(base, m).first->second;
}
template <bool INV>
void launch_col(const NttLaunch& a, const uint32_t* src, uint64_t src_bs, cudaStream_t st) {
  const int items = a.njobs * a.batch * kCTiles;
  const int grid = min(g_col_grid[INV], items);
  if (g_col_var == 4) {  // TMA staging, descriptors one item ahead (k_col_tma)
    const CUtensorMap& m = col_tensor_map(INV ? a.dst : src);
    static const int dbg = std::getenv("CK32_COL_DBG") ? std::atoi(std::getenv("CK32_COL_DBG")) : 0;
    k_col_tma<INV><<<grid, kCT, kColTmaSmem, st>>>(a.jobs, src_bs, a.dst, a.dst_bs, a.batch, a.njobs, a.primes, a.tw,
                                                   a.exits, a.entry, m, dbg);
    return;
  }
  if (g_col_var == 5) {  // TMA staging at 6 CTAs / SM (register-capped)
    const CUtensorMap& m = col_tensor_map(INV ? a.dst : src);
    k_col<INV, false, true, 6, 8, true><<<grid, kCT, kColTmaSmem, st>>>(a.jobs, src, src_bs, a.dst, a.dst_bs, a.batch,
                                                                       a.njobs, a.primes, a.tw, a.exits, a.entry, m);
    return;
  }
  if (g_col_var == 3) {  // TMA staging (the tile source is dst for the inverse pass, as in prefetch)
    const CUtensorMap& m = col_tensor_map(INV ? a.dst : src);
    k_col<INV, false, true, 5, 8, true><<<grid, kCT, kColTmaSmem, st>>>(a.jobs, src, src_bs, a.dst, a.dst_bs, a.batch,
                                                                       a.njobs, a.primes, a.tw, a.exits, a.entry, m);
    return;
  }
  if (g_col_var == 1)
    k_col<INV, false, true, 4><<<grid, kCT, kColRingSmem, st>>>(a.jobs, src, src_bs, a.dst, a.dst_bs, a.batch, a.njobs,
                                                                 a.primes, a.tw, a.exits, a.entry, CUtensorMap{});
  else if (g_col_var == 2)
    k_col<INV, false, true, 5><<<grid, kCT, kColRingSmem, st>>>(a.jobs, src, src_bs, a.dst, a.dst_bs, a.batch, a.njobs,
                                                                 a.primes, a.tw, a.exits, a.entry, CUtensorMap{});
  else if (g_col_db)
    k_col<INV, true><<<grid, kCT, 2 * sizeof(ColBuf), st>>>(a.jobs, src, src_bs, a.dst, a.dst_bs, a.batch, a.njobs,
                                                            a.primes, a.tw, a.exits, a.entry, CUtensorMap{});
  else
    k_col<INV, false><<<grid, kCT, sizeof(ColBuf), st>>>(a.jobs, src, src_bs, a.dst, a.dst_bs, a.batch, a.njobs,
                                                         a.primes, a.tw, a.exits, a.entry, CUtensorMap{});
}

// ===================================================== fused ModUp / ModDown ==
// k_conv_mid: INTT pass B (+ exit, + BConv part 1) of the sc source rows,
// BConv part 2 to the dc destination rows, and forward NTT pass 1 of every
// destination row, for one 256 x 8 column tile, in one kernel:
//   reference chain  inverse_row(part1) -> bconv_part2 -> forward_row
//   (ckks.cpp:698-724 for ModUp, ckks.cpp:621-640 for drop_and_divide).
// The converted rows never visit HBM between BConv and the first NTT pass;
// the source tiles are read once from HBM (INTT pass-A output).
// Layout: source tiles [s][256][2 quads] uint4 in smem with row swizzle
// r ^ ((r>>4)&3) (conflict-free for both the stride-16 and the contiguous
// row patterns), one 8 KB staging tile per warp for the destination
// transpose.  Warp w runs the INTT of sources w, w+8, .. then the
// destination rows w, w+8, ..; lane = (tau = lane>>1, cq = lane&1).
constexpr int kMTC = 8;  // columns per tile
constexpr int kMTiles = kR / kMTC;
__device__ __forceinline__ int msw(int r) { return r ^ ((r >> 4) & 3); }

template <int SC>
__global__ void __launch_bounds__(256, 1) k_conv_mid(ConvMidLaunch a) {
  extern __shared__ __align__(128) unsigned char smraw[];
  uint4* srct = reinterpret_cast<uint4*>(smraw);                 // [SC][256][2]
  uint4* stg = srct + SC * 512 + (threadIdx.x >> 5) * 512;       // per-warp [256][2]
  const ConvMidGroup G = a.groups[blockIdx.y];
  const int b = blockIdx.z, c0 = blockIdx.x * kMTC;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tau = lane >> 1, cq = lane & 1;
  // ---- load the source tiles (INTT pass-A output, [0, 2q))
  const uint32_t* sbase = a.src + b * a.src_bs + (size_t)G.src_off * kN + c0;
  for (int e = threadIdx.x; e < (int)G.sc * 512; e += 256) {
    const int s = e >> 9, r = (e >> 1) & 255, h = e & 1;
    cp16(&srct[s * 512 + msw(r) * 2 + h], sbase + (size_t)s * kN + r * kR + 4 * h);
  }
  cp_commit();
  cp_wait<0>();
  __syncthreads();
  // ---- phase I: inverse column pass of each source (exit folds N^-1 R^-1 part1)
  for (int s = warp; s < (int)G.sc; s += 8) {
    const int g = a.src_prime[G.src_map_off + s];
    const PrimeDev P = a.primes[g];
    const uint32_t q = P.q, q2 = P.q2;
    const ExitConst ex = a.src_exit[G.src_map_off + s];
    const uint2* tw = a.inv_tw + (size_t)g * kN;
    uint4* T = srct + s * 512;
    uint4 v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = T[msw(16 * tau + j) * 2 + cq];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int d = 1 << t;
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int blk = p / d, j = blk * 2 * d + p % d;
        gs4(v[j], v[j + d], __ldg(&tw[(128 >> t) + (tau << (3 - t)) + blk]), q, q2);
      }
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) T[msw(16 * tau + j) * 2 + cq] = v[j];
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = T[msw(tau + 16 * j) * 2 + cq];
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const int d = 1 << t;
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int blk = p / d, j = blk * 2 * d + p % d;
        gs4(v[j], v[j + d], __ldg(&tw[(8 >> t) + blk]), q, q2);
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#define CK_X(c)                                                            \
  {                                                                        \
    const uint32_t u = v[j].c + v[j + 8].c, dd = v[j].c - v[j + 8].c + q2; \
    v[j].c = sub_if(shoup_mul(u, ex.x, ex.y, q), q);                       \
    v[j + 8].c = sub_if(shoup_mul(dd, ex.z, ex.w, q), q);                  \
  }
      CK_X(x) CK_X(y) CK_X(z) CK_X(w)
#undef CK_X
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) T[msw(tau + 16 * j) * 2 + cq] = v[j];  // canonical coefficients
  }
  __syncthreads();
  // ---- phase II: BConv (x R folded into the matrix) + forward pass 1 per destination
  for (int i = warp; i < (int)G.dc; i += 8) {
    const int g = a.dst_prime[G.map_off + i];
    const PrimeDev P = a.primes[g];
    const uint32_t q = P.q, q2 = P.q2;
    const uint32_t* cm = a.cmat + G.cmat_off + i * G.sc;
    uint32_t c[SC];
#pragma unroll
    for (int s = 0; s < SC; ++s) c[s] = s < (int)G.sc ? __ldg(&cm[s]) : 0u;
    uint4 v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int rr = msw(tau + 16 * j) * 2 + cq;
      uint64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
      for (int s = 0; s < SC; ++s) {
        if (s < (int)G.sc) {
          const uint4 x = srct[s * 512 + rr];
          a0 = mac_wide(a0, x.x, c[s]);
          a1 = mac_wide(a1, x.y, c[s]);
          a2 = mac_wide(a2, x.z, c[s]);
          a3 = mac_wide(a3, x.w, c[s]);
        }
      }
      v[j] = make_uint4(mont_reduce64(a0, q, P.qinv), mont_reduce64(a1, q, P.qinv),
                        mont_reduce64(a2, q, P.qinv), mont_reduce64(a3, q, P.qinv));  // [0, 2q)
    }
    const uint2* tw = a.fwd_tw + (size_t)g * kN;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int d = 8 >> t;
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int blk = p / d, j = blk * 2 * d + p % d;
        ct4(v[j], v[j + d], __ldg(&tw[(1 << t) + blk]), q, q2);
      }
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) stg[msw(tau + 16 * j) * 2 + cq] = v[j];
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = stg[msw(16 * tau + j) * 2 + cq];
    __syncwarp();
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int d = 8 >> t;
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int blk = p / d, j = blk * 2 * d + p % d;
        ct4(v[j], v[j + d], __ldg(&tw[(16 << t) + (tau << t) + blk]), q, q2);
      }
    }
    uint32_t* o = a.dst + b * a.dst_bs + (size_t)a.dst_row[G.map_off + i] * kN + c0 + 4 * cq;
#pragma unroll
    for (int j = 0; j < 16; ++j) stg4(o + (16 * tau + j) * kR, v[j]);
  }
}

// ============================================ NTT pass 2 fused with KeyMult ==
// k_row_keymult: for output row i of v = [v0; v1] (level + alpha rows) and a
// tile of 8 coefficient rows, run the forward row pass on every digit's
// ModUp extension row (pass-1 output) — or take the digit's own row straight
// from d (evaluation domain) — and accumulate the KeyMult products with both
// key halves in int64, plus the merged-HMult fold P*d0 / P*d1:
//   reference  forward_row (mod_up, ckks.cpp:718-724) -> key_mult
//              (ckks.cpp:744-767) -> fold (ckks.cpp:831-842).
// The extension never returns to HBM after its row pass.
constexpr int kKT = 128;  // 8 rows x 16 threads
constexpr int kKBuf = kRRows * kRowStride;
constexpr int kKSmem = 2 * kKBuf * 4 + kRRows * kR * 8;

// EARLY: the key halves of digit k are loaded into registers before its row
// pass (their L2 latency hides behind the butterflies) at MINB CTAs per SM.
// ALLD (D <= 3): the extension tiles of all D digits of an item are requested
// together at the item start (one cp.async group per digit, one buffer per
// digit), so only the first digit's load latency is exposed; digit k waits
// for its own group.  Otherwise each digit's tile is loaded when needed.
// WL (with ALLD): every warp stages its own two rows of the tile and of the
// twiddle tables, so the CTA never synchronises: the four warps are
// independent pipelines (no __syncthreads in the loop).
// L2PF: at the item start every warp asks L2 for the lines of the rows it
// will read with plain loads later (the digit's own rows of d and the fold
// rows d0 / d1), so those loads hit L2 instead of going to HBM on the
// critical path (prefetch.global.L2: no registers, no shared memory).
template <bool EARLY = false, int MINB = 1, bool ALLD = false, bool WL = false, bool L2PF = false>
__global__ void __launch_bounds__(kKT, MINB) k_row_keymult(KeyMultLaunch a, const uint2* __restrict__ tw2) {
  extern __shared__ __align__(128) unsigned char smraw[];
  uint32_t* sbuf = reinterpret_cast<uint32_t*>(smraw);
  uint2* tws = reinterpret_cast<uint2*>(smraw + (ALLD ? 3 : 2) * kKBuf * 4);
  const int tid = threadIdx.x, rho = tid >> 4, tau = tid & 15;
  constexpr int kTiles = kR / kRRows;
  const int rows = a.level + a.alpha, B = a.batch;
  const uint32_t LA = (uint32_t)(a.L + a.alpha);
  const int items = rows * kTiles * B;  // (row i, tile, b), b fastest
  const int chunk = (items + gridDim.x - 1) / gridDim.x;
  const int i0 = blockIdx.x * chunk, i1 = min(items, i0 + chunk);
  int cur_key = -1;
  int kbuf = 0;
  for (int it = i0; it < i1; ++it) {
    const int b = it % B, key = it / B, tile = key % kTiles, i = key / kTiles;
    const int g = i < a.level ? i : a.L + (i - a.level);
    const PrimeDev P = a.primes[g];
    const uint32_t q = P.q, q2 = P.q2, q4 = 2 * P.q2;
    const int warp = tid >> 5, lane = tid & 31;
    if (ALLD) {  // every thread (warp) is done with the previous item's tile buffers
      if (WL) __syncwarp();
      else __syncthreads();
    }
    if (key != cur_key) {
      if (!ALLD) __syncthreads();
      const uint2* T = tw2 + ((size_t)g * kR + tile * kRRows) * kR;
      if (WL) {  // this warp's two rows of the tables
        for (int e = lane; e < 2 * kR / 2; e += 32) cp16(&tws[2 * warp * kR + 2 * e], &T[2 * warp * kR + 2 * e]);
      } else {
        for (int e = tid; e < kRRows * kR / 2; e += kKT) cp16(&tws[2 * e], &T[2 * e]);
      }
      cp_commit();
      cur_key = key;
    }
    if (ALLD) {
      for (int k = 0; k < a.D; ++k) {
        const int lo = k * a.alpha, hi = min((k + 1) * a.alpha, a.level);
        if (!(i >= lo && i < hi)) {
          const uint32_t* gsrc = a.ext + b * a.ext_bs + ((size_t)k * rows + i) * kN + (size_t)tile * kRRows * kR;
          uint32_t* buf = sbuf + k * kKBuf;
          if (WL) {  // this warp's two rows
#pragma unroll
            for (int m = 0; m < 4; ++m) {
              const int e = lane + 32 * m, rr = 2 * warp + (e >> 6), c = (e & 63) * 4;
              cp16(buf + rr * kRowStride + rpos(c), gsrc + rr * kR + c);
            }
          } else {
#pragma unroll
            for (int m = 0; m < kRRows * 64 / kKT; ++m) {
              const int e = tid + m * kKT, rr = e >> 6, c = (e & 63) * 4;
              cp16(buf + rr * kRowStride + rpos(c), gsrc + rr * kR + c);
            }
          }
        }
        cp_commit();
      }
    }
    const int r = tile * kRRows + rho;
    const uint2* W = tws + rho * kR;
    uint64_t s0[16], s1[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) s0[j] = s1[j] = 0;
    const size_t rofs = (size_t)r * kR + 16 * tau;  // this thread's 16 coefficients after the row pass
    if (L2PF && i < a.level) {  // the warp's 2 rows = 16 lines of 128 B per array; lane -> one line
      const size_t line_ofs = (size_t)(tile * kRRows + 2 * warp) * kR + (lane & 15) * 32;
      const uint32_t* own = a.d + b * a.d_bs + (size_t)i * kN + line_ofs;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(own + (lane >> 4) * kR));
      if (a.fold) {
        const uint32_t* f = a.fold + b * a.fold_bs + (size_t)(lane < 16 ? i : a.level + i) * kN + line_ofs;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(f));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(f + kR));
      }
    }
    for (int k = 0; k < a.D; ++k) {
      const int lo = k * a.alpha, hi = min((k + 1) * a.alpha, a.level);
      uint4 kb[4], ka[4];
      if (EARLY) {
        const uint32_t* eb = a.evk + (((size_t)k * 2 + 0) * LA + g) * kN + rofs;
        const uint32_t* ea = a.evk + (((size_t)k * 2 + 1) * LA + g) * kN + rofs;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          kb[m] = __ldg(reinterpret_cast<const uint4*>(eb + 4 * m));
          ka[m] = __ldg(reinterpret_cast<const uint4*>(ea + 4 * m));
        }
      }
      uint32_t v[16];
      if (i >= lo && i < hi) {  // the digit's own row: ModUp passes it through unchanged
        const uint32_t* dr = a.d + b * a.d_bs + (size_t)i * kN + rofs;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const uint4 x = *reinterpret_cast<const uint4*>(dr + 4 * m);
          v[4 * m] = x.x;
          v[4 * m + 1] = x.y;
          v[4 * m + 2] = x.z;
          v[4 * m + 3] = x.w;
        }
      } else {
        uint32_t* buf;
        if (ALLD) {
          buf = sbuf + k * kKBuf;
          const int pend = a.D - 1 - k;  // later digits' groups may still be in flight
          if (pend >= 2) cp_wait<2>();
          else if (pend == 1) cp_wait<1>();
          else cp_wait<0>();
          if (WL) __syncwarp();
          else __syncthreads();
        } else {
          buf = sbuf + kbuf * kKBuf;
          kbuf ^= 1;
          const uint32_t* gsrc = a.ext + b * a.ext_bs + ((size_t)k * rows + i) * kN + (size_t)tile * kRRows * kR;
#pragma unroll
          for (int m = 0; m < kRRows * 64 / kKT; ++m) {
            const int e = tid + m * kKT, rr = e >> 6, c = (e & 63) * 4;
            cp16(buf + rr * kRowStride + rpos(c), gsrc + rr * kR + c);
          }
          cp_commit();
          cp_wait<0>();
          __syncthreads();
        }
        uint32_t* line = buf + rho * kRowStride;
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = line[rpos(tau + 16 * j)];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int d = 8 >> t;
#pragma unroll
          for (int p = 0; p < 8; ++p) {
            const int blk = p / d, j = blk * 2 * d + p % d;
            const uint2 w = W[(1 << t) - 1 + blk];
            if (t % 2 == 0) ctl<true>(v[j], v[j + d], w.x, w.y, q, q2, q4);
            else ctl<false>(v[j], v[j + d], w.x, w.y, q, q2, q4);
          }
        }
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
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int d = 8 >> t;
#pragma unroll
          for (int p = 0; p < 8; ++p) {
            const int blk = p / d, j = blk * 2 * d + p % d;
            const uint2 w = W[16 + ((1 << t) - 1 + blk) * 16 + tau];
            if (t % 2 == 0) ctl<true>(v[j], v[j + d], w.x, w.y, q, q2, q4);
            else ctl<false>(v[j], v[j + d], w.x, w.y, q, q2, q4);
          }
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = canon8(v[j], q, q2, q4);
      }
      // KeyMult MACs with both key halves (rows indexed by the global prime, ckks.cpp:747)
      const uint32_t* eb = a.evk + (((size_t)k * 2 + 0) * LA + g) * kN + rofs;
      const uint32_t* ea = a.evk + (((size_t)k * 2 + 1) * LA + g) * kN + rofs;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const uint4 xb = EARLY ? kb[m] : __ldg(reinterpret_cast<const uint4*>(eb + 4 * m));
        const uint4 xa = EARLY ? ka[m] : __ldg(reinterpret_cast<const uint4*>(ea + 4 * m));
        s0[4 * m] = mac_wide(s0[4 * m], v[4 * m], xb.x);
        s0[4 * m + 1] = mac_wide(s0[4 * m + 1], v[4 * m + 1], xb.y);
        s0[4 * m + 2] = mac_wide(s0[4 * m + 2], v[4 * m + 2], xb.z);
        s0[4 * m + 3] = mac_wide(s0[4 * m + 3], v[4 * m + 3], xb.w);
        s1[4 * m] = mac_wide(s1[4 * m], v[4 * m], xa.x);
        s1[4 * m + 1] = mac_wide(s1[4 * m + 1], v[4 * m + 1], xa.y);
        s1[4 * m + 2] = mac_wide(s1[4 * m + 2], v[4 * m + 2], xa.z);
        s1[4 * m + 3] = mac_wide(s1[4 * m + 3], v[4 * m + 3], xa.w);
      }
      if ((k % 6) == 5) {  // keep the sums below q 2^32 (value unchanged mod q, rescaled by R)
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          s0[j] = shoup_mul(mont_reduce64(s0[j], q, P.qinv), P.r, P.r_sh, q);
          s1[j] = shoup_mul(mont_reduce64(s1[j], q, P.qinv), P.r, P.r_sh, q);
        }
      }
    }
    if (a.fold && i < a.level) {  // merged HMult: v += P * d0 / d1 (ckks.cpp:831-842)
      const uint32_t pm = a.p_mont[i];
      const uint32_t* f0 = a.fold + b * a.fold_bs + (size_t)i * kN + rofs;
      const uint32_t* f1 = a.fold + b * a.fold_bs + (size_t)(a.level + i) * kN + rofs;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const uint4 x0 = *reinterpret_cast<const uint4*>(f0 + 4 * m);
        const uint4 x1 = *reinterpret_cast<const uint4*>(f1 + 4 * m);
        s0[4 * m] = mac_wide(s0[4 * m], x0.x, pm);
        s0[4 * m + 1] = mac_wide(s0[4 * m + 1], x0.y, pm);
        s0[4 * m + 2] = mac_wide(s0[4 * m + 2], x0.z, pm);
        s0[4 * m + 3] = mac_wide(s0[4 * m + 3], x0.w, pm);
        s1[4 * m] = mac_wide(s1[4 * m], x1.x, pm);
        s1[4 * m + 1] = mac_wide(s1[4 * m + 1], x1.y, pm);
        s1[4 * m + 2] = mac_wide(s1[4 * m + 2], x1.z, pm);
        s1[4 * m + 3] = mac_wide(s1[4 * m + 3], x1.w, pm);
      }
    }
    uint32_t* o0 = a.v + b * a.v_bs + (size_t)i * kN + rofs;
    uint32_t* o1 = a.v + b * a.v_bs + (size_t)(rows + i) * kN + rofs;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      stg4(o0 + 4 * m, make_uint4(sub_if(mont_reduce64(s0[4 * m], q, P.qinv), q),
                                  sub_if(mont_reduce64(s0[4 * m + 1], q, P.qinv), q),
                                  sub_if(mont_reduce64(s0[4 * m + 2], q, P.qinv), q),
                                  sub_if(mont_reduce64(s0[4 * m + 3], q, P.qinv), q)));
      stg4(o1 + 4 * m, make_uint4(sub_if(mont_reduce64(s1[4 * m], q, P.qinv), q),
                                  sub_if(mont_reduce64(s1[4 * m + 1], q, P.qinv), q),
                                  sub_if(mont_reduce64(s1[4 * m + 2], q, P.qinv), q),
                                  sub_if(mont_reduce64(s1[4 * m + 3], q, P.qinv), q)));
    }
  }
  cp_wait<0>();
}

// k_row_keymult_pf: the warp-local (WL), all-digits-at-once (ALLD),
// key-ahead (EARLY) variant with NOTHING left on the critical path from HBM:
// besides the extension tiles, the digit's own rows (pass-through rows of d)
// go into that digit's (otherwise unused) tile buffer with the same cp.async
// group, and the fold rows d0 / d1 of the merged HMult go into tile buffers as
// soon as the row pass of an earlier digit has released them -- so every
// load of an item is in flight while the butterflies of the previous digit
// run (round 1 loaded own rows and fold rows with plain global loads right
// before use: long-scoreboard 1.87 per issue).  Shared memory is unchanged
// (3 tile buffers + the row tile's twiddles per CTA).
template <int MINB>
__global__ void __launch_bounds__(kKT, MINB) k_row_keymult_pf(KeyMultLaunch a, const uint2* __restrict__ tw2) {
  extern __shared__ __align__(128) unsigned char smraw[];
  uint32_t* sbuf = reinterpret_cast<uint32_t*>(smraw);
  uint2* tws = reinterpret_cast<uint2*>(smraw + 3 * kKBuf * 4);
  const int tid = threadIdx.x, rho = tid >> 4, tau = tid & 15;
  const int warp = tid >> 5, lane = tid & 31;
  constexpr int kTiles = kR / kRRows;
  const int rows = a.level + a.alpha, B = a.batch, D = a.D;
  const uint32_t LA = (uint32_t)(a.L + a.alpha);
  const int items = rows * kTiles * B;  // (row i, tile, b), b fastest
  const int chunk = (items + gridDim.x - 1) / gridDim.x;
  const int i0 = blockIdx.x * chunk, i1 = min(items, i0 + chunk);
  // this warp's two rows of a [8][256] row tile -> buffer (rpos layout), one cp.async each 16 B
  auto stage = [&](uint32_t* buf, const uint32_t* g) {
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int e = lane + 32 * m, rr = 2 * warp + (e >> 6), c = (e & 63) * 4;
      cp16(buf + rr * kRowStride + rpos(c), g + rr * kR + c);
    }
  };
  // cp.async.wait_group with a runtime count (<= 4 groups in flight)
  auto wait_groups = [](int pending) {
    if (pending >= 4) cp_wait<4>();
    else if (pending == 3) cp_wait<3>();
    else if (pending == 2) cp_wait<2>();
    else if (pending == 1) cp_wait<1>();
    else cp_wait<0>();
  };
  int cur_key = -1;
  for (int it = i0; it < i1; ++it) {
    const int b = it % B, key = it / B, tile = key % kTiles, i = key / kTiles;
    const int g = i < a.level ? i : a.L + (i - a.level);
    const PrimeDev P = a.primes[g];
    const uint32_t q = P.q, q2 = P.q2, q4 = 2 * P.q2;
    const bool fold = a.fold && i < a.level;
    __syncwarp();  // the warp is done with the previous item's buffers
    if (key != cur_key) {
      const uint2* T = tw2 + ((size_t)g * kR + tile * kRRows) * kR;
      for (int e = lane; e < kR; e += 32) cp16(&tws[2 * warp * kR + 2 * e], &T[2 * warp * kR + 2 * e]);
      cp_commit();
      cur_key = key;
    }
    const size_t tofs = (size_t)tile * kRRows * kR;
    int committed = 0;  // groups committed for this item: digit k = group k, then the fold groups
    for (int k = 0; k < D; ++k) {
      const int lo = k * a.alpha, hi = min((k + 1) * a.alpha, a.level);
      const uint32_t* gsrc = (i >= lo && i < hi) ? a.d + b * a.d_bs + (size_t)i * kN + tofs
                                                 : a.ext + b * a.ext_bs + ((size_t)k * rows + i) * kN + tofs;
      stage(sbuf + k * kKBuf, gsrc);
      cp_commit();
      ++committed;
    }
    // fold halves: into the buffers no digit uses (D < 3), else into the
    // buffer of digit 0 / 1 once its row pass has finished with it
    int fb0 = 0, fb1 = 0, nf = 0;  // buffers holding fold halves 0 / 1, halves issued
    const uint32_t* fsrc0 = a.fold + b * a.fold_bs + (size_t)i * kN + tofs;
    const uint32_t* fsrc1 = a.fold + b * a.fold_bs + (size_t)(a.level + i) * kN + tofs;
    auto issue_fold = [&](int buf) {
      if (nf == 0) fb0 = buf;
      else fb1 = buf;
      stage(sbuf + buf * kKBuf, nf == 0 ? fsrc0 : fsrc1);
      cp_commit();
      ++committed;
      ++nf;
    };
    if (fold)
      for (int f = D; f < 3 && nf < 2; ++f) issue_fold(f);
    const int r = tile * kRRows + rho;
    const uint2* W = tws + rho * kR;
    uint64_t s0[16], s1[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) s0[j] = s1[j] = 0;
    const size_t rofs = (size_t)r * kR + 16 * tau;  // this thread's 16 coefficients after the row pass
    for (int k = 0; k < D; ++k) {
      const int lo = k * a.alpha, hi = min((k + 1) * a.alpha, a.level);
      uint4 kb[4], ka[4];
      {
        const uint32_t* eb = a.evk + (((size_t)k * 2 + 0) * LA + g) * kN + rofs;
        const uint32_t* ea = a.evk + (((size_t)k * 2 + 1) * LA + g) * kN + rofs;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          kb[m] = __ldg(reinterpret_cast<const uint4*>(eb + 4 * m));
          ka[m] = __ldg(reinterpret_cast<const uint4*>(ea + 4 * m));
        }
      }
      wait_groups(committed - (k + 1));
      __syncwarp();
      uint32_t* line = sbuf + k * kKBuf + rho * kRowStride;
      uint32_t v[16];
      if (i >= lo && i < hi) {  // the digit's own row (ModUp pass-through), already in evaluation form
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const uint4 x = *reinterpret_cast<const uint4*>(line + rpos(16 * tau) + 4 * m);
          v[4 * m] = x.x;
          v[4 * m + 1] = x.y;
          v[4 * m + 2] = x.z;
          v[4 * m + 3] = x.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = line[rpos(tau + 16 * j)];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int d = 8 >> t;
#pragma unroll
          for (int p = 0; p < 8; ++p) {
            const int blk = p / d, j = blk * 2 * d + p % d;
            const uint2 w = W[(1 << t) - 1 + blk];
            if (t % 2 == 0) ctl<true>(v[j], v[j + d], w.x, w.y, q, q2, q4);
            else ctl<false>(v[j], v[j + d], w.x, w.y, q, q2, q4);
          }
        }
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
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int d = 8 >> t;
#pragma unroll
          for (int p = 0; p < 8; ++p) {
            const int blk = p / d, j = blk * 2 * d + p % d;
            const uint2 w = W[16 + ((1 << t) - 1 + blk) * 16 + tau];
            if (t % 2 == 0) ctl<true>(v[j], v[j + d], w.x, w.y, q, q2, q4);
            else ctl<false>(v[j], v[j + d], w.x, w.y, q, q2, q4);
          }
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = canon8(v[j], q, q2, q4);
      }
      if (fold && nf < 2 && k < 2) {  // buffer k is free now: the next fold half goes there
        __syncwarp();
        issue_fold(k);
      }
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        s0[4 * m] = mac_wide(s0[4 * m], v[4 * m], kb[m].x);
        s0[4 * m + 1] = mac_wide(s0[4 * m + 1], v[4 * m + 1], kb[m].y);
        s0[4 * m + 2] = mac_wide(s0[4 * m + 2], v[4 * m + 2], kb[m].z);
        s0[4 * m + 3] = mac_wide(s0[4 * m + 3], v[4 * m + 3], kb[m].w);
        s1[4 * m] = mac_wide(s1[4 * m], v[4 * m], ka[m].x);
        s1[4 * m + 1] = mac_wide(s1[4 * m + 1], v[4 * m + 1], ka[m].y);
        s1[4 * m + 2] = mac_wide(s1[4 * m + 2], v[4 * m + 2], ka[m].z);
        s1[4 * m + 3] = mac_wide(s1[4 * m + 3], v[4 * m + 3], ka[m].w);
      }
    }
    if (fold) {  // merged HMult: v += P * d0 / d1 (ckks.cpp:831-842)
      const uint32_t pm = a.p_mont[i];
      wait_groups(0);
      __syncwarp();
      const uint32_t* l0 = sbuf + fb0 * kKBuf + rho * kRowStride + rpos(16 * tau);
      const uint32_t* l1 = sbuf + fb1 * kKBuf + rho * kRowStride + rpos(16 * tau);
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const uint4 x0 = *reinterpret_cast<const uint4*>(l0 + 4 * m);
        const uint4 x1 = *reinterpret_cast<const uint4*>(l1 + 4 * m);
        s0[4 * m] = mac_wide(s0[4 * m], x0.x, pm);
        s0[4 * m + 1] = mac_wide(s0[4 * m + 1], x0.y, pm);
        s0[4 * m + 2] = mac_wide(s0[4 * m + 2], x0.z, pm);
        s0[4 * m + 3] = mac_wide(s0[4 * m + 3], x0.w, pm);
        s1[4 * m] = mac_wide(s1[4 * m], x1.x, pm);
        s1[4 * m + 1] = mac_wide(s1[4 * m + 1], x1.y, pm);
        s1[4 * m + 2] = mac_wide(s1[4 * m + 2], x1.z, pm);
        s1[4 * m + 3] = mac_wide(s1[4 * m + 3], x1.w, pm);
      }
    }
    uint32_t* o0 = a.v + b * a.v_bs + (size_t)i * kN + rofs;
    uint32_t* o1 = a.v + b * a.v_bs + (size_t)(rows + i) * kN + rofs;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      stg4(o0 + 4 * m, make_uint4(sub_if(mont_reduce64(s0[4 * m], q, P.qinv), q),
                                  sub_if(mont_reduce64(s0[4 * m + 1], q, P.qinv), q),
                                  sub_if(mont_reduce64(s0[4 * m + 2], q, P.qinv), q),
                                  sub_if(mont_reduce64(s0[4 * m + 3], q, P.qinv), q)));
      stg4(o1 + 4 * m, make_uint4(sub_if(mont_reduce64(s1[4 * m], q, P.qinv), q),
                                  sub_if(mont_reduce64(s1[4 * m + 1], q, P.qinv), q),
                                  sub_if(mont_reduce64(s1[4 * m + 2], q, P.qinv), q),
                                  sub_if(mont_reduce64(s1[4 * m + 3], q, P.qinv), q)));
    }
  }
  cp_wait<0>();
}

// k_row_keymult8: the fused row pass + KeyMult with 8 coefficients per
// thread (32 threads per 256-point row, one row per warp, 4-row tiles)
// instead of 16: 2 x 8 int64 accumulators instead of 2 x 16, so ~80
// registers and 6 CTAs (24 warps) per SM instead of 4 (16 warps) -- the
// kernel is latency-bound at 16 warps.  The row transform runs as 3 + 3 + 2
// radix-2 stages with two warp-local exchanges through padded shared memory
// (pad(c) = c + 4 (c >> 5): conflict-free for all three layouts); twiddles in
// natural per-row order T_r[2^s - 1 + B] = F[(256 << s) + (r << s) + B]
// (the reference's forward table, ntt.cpp:124-128), staged once per
// (prime, row tile) and reused for every batch item.
#ifndef CK32_KM_LAZY
#define CK32_KM_LAZY 1
#endif
constexpr bool kKmLazy = CK32_KM_LAZY;  // keymult8 (KPF 0): MAC inputs in [0, 8q), one canonicalisation of the output
constexpr int kK8Rows = 4;                       // rows per CTA (one per warp)
constexpr int kK8Stride = 288;                   // 256 + 32 padding words
__device__ __forceinline__ int pad8(int c) { return c + 4 * (c >> 5); }
constexpr int kK8SmemBase = (3 * kK8Rows * kK8Stride) * 4 + kK8Rows * 256 * 8;  // 3 digit tiles + fwd twiddles
constexpr int kK8Smem = kK8SmemBase + kK8Rows * 256 * 8;  // + inverse twiddles (fused INTT pass A)

// EARLY: the key halves of digit k are loaded before its row pass (16
// registers live across it); without, they are loaded after it (more CTAs).
// KPF (with !EARLY): 1 = the digit's key lines are requested into L1
// (prefetch.global.L1) before its row pass, 2 = the next digit's during this
// digit's row pass (the first digit's at the item start).
template <int MINB, bool EARLY = true, int KPF = 0, int DD = 0>
__global__ void __launch_bounds__(128, MINB) k_row_keymult8(KeyMultLaunch a, const uint2* __restrict__ fwd) {
  extern __shared__ __align__(128) unsigned char smraw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t* sbuf = reinterpret_cast<uint32_t*>(smraw);                          // [3][4][288]
  uint2* tws = reinterpret_cast<uint2*>(smraw + 3 * kK8Rows * kK8Stride * 4);   // [4][256] forward, [4][256] inverse
  uint2* T = tws + warp * 256;
  uint2* Ti = tws + (kK8Rows + warp) * 256;  // inverse row twiddles (fused INTT pass A), natural order per stage
  uint32_t* Ks = reinterpret_cast<uint32_t*>(smraw + kK8Smem) + warp * (3 * 2 * 256);  // KPF 3: key slice [D][2][256]
  uint32_t* Kd = reinterpret_cast<uint32_t*>(smraw + kK8SmemBase) + warp * (2 * 256);  // KPF 6: one digit's key [2][256]
  constexpr int kTiles = kR / kK8Rows;
  // KPF 7 (the MACs after all digits' row passes) is instantiated per digit count
  const int Dn = (KPF == 7 && DD > 0) ? DD : a.D;
  constexpr bool LAZY = KPF == 0 && kKmLazy;  // the default variant (D <= 3 by construction of keymult8's dispatch)
  const int rows = a.level + a.alpha, B = a.batch;
  const uint32_t LA = (uint32_t)(a.L + a.alpha);
  const int items = rows * kTiles * B;  // (row i, tile, b), b fastest
  const int chunk = (items + gridDim.x - 1) / gridDim.x;
  const int i0 = blockIdx.x * chunk, i1 = min(items, i0 + chunk);
  const int lhi = lane >> 2, llo = lane & 3;
  if (i0 >= i1) return;
  // item cursor (row i, tile, b), b fastest: advanced incrementally (no
  // divisions per item), per-(i, tile) values refreshed when b wraps
  int b = i0 % B, tile = (i0 / B) % kTiles, i = (i0 / B) / kTiles;
  int g = 0, r = 0;
  PrimeDev P{};
  uint32_t q = 0, q2 = 0, q4 = 0;
  for (int it = i0, left = i1 - i0; left > 0; ++it, --left) {  // a count: no i1 live across the loop
    __syncwarp();  // the warp is done with the previous item's buffers
    if (it == i0 || b == 0) {  // new (row, tile): prime, and this row's 255 forward twiddles (natural order)
      g = i < a.level ? i : a.L + (i - a.level);
      r = tile * kK8Rows + warp;  // this warp's row of the 256 x 256 limb matrix
      P = a.primes[g];
      q = P.q;
      q2 = P.q2;
      q4 = 2 * P.q2;
      const uint2* F = fwd + (size_t)g * kN;
      if (KPF == 6 || KPF == 0 || KPF == 7) {  // asynchronously (one group, older than the item's extension groups)
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = lane + 32 * u;
          if (e < 255) {
            const int s = 31 - __clz(e + 1), blk = e + 1 - (1 << s);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(&T[e]))),
                         "l"(&F[(256 << s) + (r << s) + blk])
                         : "memory");
          }
        }
        cp_commit();
      } else {
        for (int e = lane; e < 255; e += 32) {
          const int s = 31 - __clz(e + 1), blk = e + 1 - (1 << s);
          T[e] = __ldg(&F[(256 << s) + (r << s) + blk]);
        }
      }
      if (a.ts && i >= a.src_lo) {  // inverse stage v of row r: I[(N >> (v+1)) + (r << (7-v)) + blk] at 256 - (256 >> v) + blk
        const uint2* I = a.inv_full + (size_t)g * kN;
#pragma unroll
        for (int v = 0; v < 8; ++v)
          for (int blk = lane; blk < (128 >> v); blk += 32)
            Ti[256 - (256 >> v) + blk] = __ldg(&I[(kN >> (v + 1)) + (r << (7 - v)) + blk]);
      }
      if (KPF == 3) {  // this row's key slice (D digits x 2 halves x 256 words) into shared memory, reused for all b
        for (int k = 0; k < Dn; ++k)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t* kr = a.evk + (((size_t)k * 2 + h) * LA + g) * kN + (size_t)r * kR;
#pragma unroll
            for (int m = 0; m < 2; ++m) cp16(Ks + (k * 2 + h) * 256 + 4 * (lane + 32 * m), kr + 4 * (lane + 32 * m));
          }
        cp_commit();  // older than the extension groups below: complete at the first digit's wait
      }
    }
    // the next item of this CTA's chunk (b fastest): KPF 5 requests its
    // extension rows digit by digit as soon as this item's digit buffer is free
    int nb5 = b + 1, ntile5 = tile, ni5 = i;
    if (nb5 == B) {
      nb5 = 0;
      if (++ntile5 == kTiles) {
        ntile5 = 0;
        ++ni5;
      }
    }
    const bool next5 = KPF == 5 && left > 1;
    // all digits' extension rows at once (one cp.async group per digit); KPF 5: the first item only
    for (int k = 0; k < Dn && (KPF != 5 || it == i0); ++k) {
      const int lo = k * a.alpha, hi = min((k + 1) * a.alpha, a.level);
      if (!(i >= lo && i < hi)) {
        const uint32_t* gsrc = a.ext + b * a.ext_bs + ((size_t)k * rows + i) * kN + (size_t)r * kR;
        uint32_t* line = sbuf + (k * kK8Rows + warp) * kK8Stride;
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          const int c = 4 * (lane + 32 * m);
          cp16(line + pad8(c), gsrc + c);
        }
      } else if (KPF == 4) {  // the digit's own row (ModUp pass-through) into its otherwise unused buffer
        const uint32_t* gsrc = a.d + b * a.d_bs + (size_t)i * kN + (size_t)r * kR;
        uint32_t* line = sbuf + (k * kK8Rows + warp) * kK8Stride;
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          const int c = 4 * (lane + 32 * m);
          cp16(line + pad8(c), gsrc + c);
        }
      }
      cp_commit();
    }
    const size_t rofs = (size_t)r * kR + 8 * lane;  // this thread's 8 coefficients after the transform
    if (i < a.level && (lane & 3) == 0) {  // own-digit and fold rows into L2 now (plain loads later), 1 per line
      if (KPF != 4) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.d + b * a.d_bs + (size_t)i * kN + rofs));
      if (a.fold) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.fold + b * a.fold_bs + (size_t)i * kN + rofs));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.fold + b * a.fold_bs + (size_t)(a.level + i) * kN + rofs));
      }
    }
    uint64_t s0[8], s1[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) s0[j] = s1[j] = 0;
    auto key_l1 = [&](int kk) {  // one lane per 128 B line of this thread's key coefficients
      if ((lane & 3) == 0) {
        asm volatile("prefetch.global.L1 [%0];" ::"l"(a.evk + (((size_t)kk * 2 + 0) * LA + g) * kN + rofs));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(a.evk + (((size_t)kk * 2 + 1) * LA + g) * kN + rofs));
      }
    };
    if (KPF == 2) key_l1(0);
    uint32_t vd[KPF == 7 ? 3 : 1][8];  // KPF 7: every digit's row-pass output, multiplied after the loop
#pragma unroll(KPF == 7 ? 3 : 1)
    for (int k = 0; k < Dn; ++k) {
      const int lo = k * a.alpha, hi = min((k + 1) * a.alpha, a.level);
      uint4 kb[2], ka[2];  // key halves (EARLY: first, their L2 latency hides behind the butterflies)
      const uint32_t* eb = a.evk + (((size_t)k * 2 + 0) * LA + g) * kN + rofs;
      const uint32_t* ea = a.evk + (((size_t)k * 2 + 1) * LA + g) * kN + rofs;
      if (KPF == 1) key_l1(k);
      if (KPF == 2 && k + 1 < Dn) key_l1(k + 1);
      if (KPF == 6) {  // this digit's key slice (2 halves x 256 words) by cp.async: lands during the row pass
        __syncwarp();  // every lane has read the previous digit's slice
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t* kr = a.evk + (((size_t)k * 2 + h) * LA + g) * kN + (size_t)r * kR;
#pragma unroll
          for (int m = 0; m < 2; ++m) cp16(Kd + h * 256 + 4 * (lane + 32 * m), kr + 4 * (lane + 32 * m));
        }
        cp_commit();
      }
      if (EARLY) {
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          kb[m] = __ldg(reinterpret_cast<const uint4*>(eb + 4 * m));
          ka[m] = __ldg(reinterpret_cast<const uint4*>(ea + 4 * m));
        }
      }
      uint32_t v[8];
      if (KPF == 4 && i >= lo && i < hi) {  // own row, staged by cp.async at the item start
        if (Dn >= 3) cp_wait<2>();
        else if (Dn == 2) cp_wait<1>();
        else cp_wait<0>();
        __syncwarp();
        const uint32_t* line = sbuf + (k * kK8Rows + warp) * kK8Stride;
        const uint4 x0 = *reinterpret_cast<const uint4*>(line + pad8(8 * lane));
        const uint4 x1 = *reinterpret_cast<const uint4*>(line + pad8(8 * lane + 4));
        v[0] = x0.x; v[1] = x0.y; v[2] = x0.z; v[3] = x0.w;
        v[4] = x1.x; v[5] = x1.y; v[6] = x1.z; v[7] = x1.w;
      } else if (i >= lo && i < hi) {  // the digit's own row (ModUp pass-through), evaluation form already
        if (KPF == 3 && k == 0) {  // no extension wait precedes this digit: wait for the key group here
          if (Dn >= 3) cp_wait<2>();
          else if (Dn == 2) cp_wait<1>();
          else cp_wait<0>();
          __syncwarp();
        }
        const uint32_t* dr = a.d + b * a.d_bs + (size_t)i * kN + rofs;
        const uint4 x0 = *reinterpret_cast<const uint4*>(dr), x1 = *reinterpret_cast<const uint4*>(dr + 4);
        v[0] = x0.x; v[1] = x0.y; v[2] = x0.z; v[3] = x0.w;
        v[4] = x1.x; v[5] = x1.y; v[6] = x1.z; v[7] = x1.w;
      } else {
        // KPF 4: one post group per finished digit keeps D - 1 groups younger than this digit's;
        // KPF 5: this item's later digits + the next item's earlier ones, D - 1 as well
        // KPF 6: digit 0 waits behind the later digits' groups and its key group; the later
        // digits' extension groups completed at the previous digit's key wait (only its key is younger)
        const int pend = (KPF == 4 || KPF == 5) ? Dn - 1 : KPF == 6 ? (k == 0 ? Dn : 1) : Dn - 1 - k;
        if (pend >= 3) cp_wait<3>();
        else if (pend == 2) cp_wait<2>();
        else if (pend == 1) cp_wait<1>();
        else cp_wait<0>();
        __syncwarp();
        uint32_t* line = sbuf + (k * kK8Rows + warp) * kK8Stride;
        // phase A: c = lane + 32 j, stages 0..2 (bits 7..5), row-uniform twiddles
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = line[pad8(lane + 32 * j)];
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          const int d = 4 >> t;
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            const int blk = p / d, j = blk * 2 * d + p % d;
            const uint2 w = T[(1 << t) - 1 + blk];
            if (t % 2 == 0) ctl<true>(v[j], v[j + d], w.x, w.y, q, q2, q4);
            else ctl<false>(v[j], v[j + d], w.x, w.y, q, q2, q4);
          }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) line[pad8(lane + 32 * j)] = v[j];
        __syncwarp();
        // phase B: c = 32 lhi + 4 j + llo, stages 3..5 (bits 4..2)
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = line[pad8(32 * lhi + 4 * j + llo)];
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          const int d = 4 >> t, sg = 3 + t;
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            const int blk = p / d, j = blk * 2 * d + p % d;
            const uint2 w = T[(1 << sg) - 1 + (lhi << t) + blk];
            if (sg % 2 == 0) ctl<true>(v[j], v[j + d], w.x, w.y, q, q2, q4);
            else ctl<false>(v[j], v[j + d], w.x, w.y, q, q2, q4);
          }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) line[pad8(32 * lhi + 4 * j + llo)] = v[j];
        __syncwarp();
        // phase C: c = 8 lane + j, stages 6, 7 (bits 1, 0)
        {
          const uint4 x0 = *reinterpret_cast<const uint4*>(line + pad8(8 * lane));
          const uint4 x1 = *reinterpret_cast<const uint4*>(line + pad8(8 * lane + 4));
          v[0] = x0.x; v[1] = x0.y; v[2] = x0.z; v[3] = x0.w;
          v[4] = x1.x; v[5] = x1.y; v[6] = x1.z; v[7] = x1.w;
        }
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int d = 2 >> t, sg = 6 + t;
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            const int blk = p / d, j = blk * 2 * d + p % d;
            const uint2 w = T[(1 << sg) - 1 + (lane << (t + 1)) + blk];
            if (sg % 2 == 0) ctl<true>(v[j], v[j + d], w.x, w.y, q, q2, q4);
            else ctl<false>(v[j], v[j + d], w.x, w.y, q, q2, q4);
          }
        }
        // LAZY: v stays in [0, 8q) for the MACs (the D <= 3 products + fold sum
        // below 25 q^2, so the Montgomery reduction lands in (0, 4.2 q) and the
        // output is canonicalised once instead of every digit's input)
        if (!LAZY || a.ts) {
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] = canon8(v[j], q, q2, q4);
        }
      }
      if constexpr (KPF == 7) {
#pragma unroll
        for (int j = 0; j < 8; ++j) vd[k][j] = v[j];
        continue;
      }
      if (KPF == 5) {  // digit buffer k is free: the next item's digit-k extension row into it
        if (next5 && !(ni5 >= lo && ni5 < hi)) {
          __syncwarp();
          const uint32_t* gsrc =
              a.ext + nb5 * a.ext_bs + ((size_t)k * rows + ni5) * kN + (size_t)(ntile5 * kK8Rows + warp) * kR;
          uint32_t* line = sbuf + (k * kK8Rows + warp) * kK8Stride;
#pragma unroll
          for (int m = 0; m < 2; ++m) {
            const int c = 4 * (lane + 32 * m);
            cp16(line + pad8(c), gsrc + c);
          }
        }
        cp_commit();  // one group per (item, digit), empty for own rows / past the chunk
      }
      if (KPF == 6) {
        cp_wait<0>();
        __syncwarp();
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          kb[m] = *reinterpret_cast<const uint4*>(Kd + 8 * lane + 4 * m);
          ka[m] = *reinterpret_cast<const uint4*>(Kd + 256 + 8 * lane + 4 * m);
        }
      } else if (KPF == 3) {
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          kb[m] = *reinterpret_cast<const uint4*>(Ks + (k * 2 + 0) * 256 + 8 * lane + 4 * m);
          ka[m] = *reinterpret_cast<const uint4*>(Ks + (k * 2 + 1) * 256 + 8 * lane + 4 * m);
        }
      } else if (!EARLY) {
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          kb[m] = __ldg(reinterpret_cast<const uint4*>(eb + 4 * m));
          ka[m] = __ldg(reinterpret_cast<const uint4*>(ea + 4 * m));
        }
      }
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        s0[4 * m] = mac_wide(s0[4 * m], v[4 * m], kb[m].x);
        s0[4 * m + 1] = mac_wide(s0[4 * m + 1], v[4 * m + 1], kb[m].y);
        s0[4 * m + 2] = mac_wide(s0[4 * m + 2], v[4 * m + 2], kb[m].z);
        s0[4 * m + 3] = mac_wide(s0[4 * m + 3], v[4 * m + 3], kb[m].w);
        s1[4 * m] = mac_wide(s1[4 * m], v[4 * m], ka[m].x);
        s1[4 * m + 1] = mac_wide(s1[4 * m + 1], v[4 * m + 1], ka[m].y);
        s1[4 * m + 2] = mac_wide(s1[4 * m + 2], v[4 * m + 2], ka[m].z);
        s1[4 * m + 3] = mac_wide(s1[4 * m + 3], v[4 * m + 3], ka[m].w);
      }
      if (KPF == 4) {  // this digit's buffer is free: the fold row k (digits 0, 1 of a 3-digit key) into it
        if (a.fold && i < a.level && k < 2 && Dn == 3) {
          __syncwarp();
          const uint32_t* gsrc = a.fold + b * a.fold_bs + (size_t)(k * a.level + i) * kN + (size_t)r * kR;
          uint32_t* line = sbuf + (k * kK8Rows + warp) * kK8Stride;
#pragma unroll
          for (int m = 0; m < 2; ++m) {
            const int c = 4 * (lane + 32 * m);
            cp16(line + pad8(c), gsrc + c);
          }
        }
        cp_commit();
      }
      if ((k % 6) == 5) {  // keep the sums below q 2^32 (value unchanged mod q, rescaled by R)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          s0[j] = shoup_mul(mont_reduce64s((uint32_t)(s0[j]), (uint32_t)((s0[j]) >> 32), q, P.qinv), P.r, P.r_sh, q);
          s1[j] = shoup_mul(mont_reduce64s((uint32_t)(s1[j]), (uint32_t)((s1[j]) >> 32), q, P.qinv), P.r, P.r_sh, q);
        }
      }
    }
    if constexpr (KPF == 7) {
      // the key MACs of all digits at once: per output, DD products (+ the
      // fold) summed in one expression -- IMAD.WIDE per product and 3-input
      // adds with carry, instead of a split IMAD.WIDE + IADD3 + IADD3.X per
      // loop-carried MAC -- then reduced and stored; one exposed key-load
      // latency per item instead of one per digit
      const bool fold = a.fold && i < a.level;
      const uint32_t pm = fold ? a.p_mont[i] : 0u;
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // key half b (-> v0), then a (-> v1): 12 key registers live at a time
        uint32_t* o = a.v + b * a.v_bs + (size_t)(h * rows + i) * kN + rofs;
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          uint4 kh[3];
#pragma unroll
          for (int k = 0; k < DD; ++k)
            kh[k] = __ldg(reinterpret_cast<const uint4*>(a.evk + (((size_t)k * 2 + h) * LA + g) * kN + rofs + 4 * m));
          uint4 f = make_uint4(0, 0, 0, 0);
          if (fold) f = *reinterpret_cast<const uint4*>(a.fold + b * a.fold_bs + (size_t)(h * a.level + i) * kN + rofs + 4 * m);
          uint32_t rr[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint64_t t = (uint64_t)(&f.x)[c] * pm;
#pragma unroll
            for (int k = 0; k < DD; ++k) t += (uint64_t)vd[k][4 * m + c] * (&kh[k].x)[c];
            rr[c] = sub_if(mont_reduce64s((uint32_t)t, (uint32_t)(t >> 32), q, P.qinv), q);
          }
          stg4(o + 4 * m, make_uint4(rr[0], rr[1], rr[2], rr[3]));
        }
      }
    } else {
    if (a.fold && i < a.level) {  // merged HMult: v += P * d0 / d1 (ckks.cpp:831-842)
      const uint32_t pm = a.p_mont[i];
      const uint32_t* f0 = a.fold + b * a.fold_bs + (size_t)i * kN + rofs;
      const uint32_t* f1 = a.fold + b * a.fold_bs + (size_t)(a.level + i) * kN + rofs;
      const bool staged = KPF == 4 && Dn == 3;
      if (staged) {  // fold rows staged in digit buffers 0 / 1
        cp_wait<0>();
        __syncwarp();
        f0 = sbuf + warp * kK8Stride + pad8(8 * lane);
        f1 = sbuf + (kK8Rows + warp) * kK8Stride + pad8(8 * lane);
      }
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const uint4 x0 = *reinterpret_cast<const uint4*>(f0 + 4 * m);
        const uint4 x1 = *reinterpret_cast<const uint4*>(f1 + 4 * m);
        s0[4 * m] = mac_wide(s0[4 * m], x0.x, pm);
        s0[4 * m + 1] = mac_wide(s0[4 * m + 1], x0.y, pm);
        s0[4 * m + 2] = mac_wide(s0[4 * m + 2], x0.z, pm);
        s0[4 * m + 3] = mac_wide(s0[4 * m + 3], x0.w, pm);
        s1[4 * m] = mac_wide(s1[4 * m], x1.x, pm);
        s1[4 * m + 1] = mac_wide(s1[4 * m + 1], x1.y, pm);
        s1[4 * m + 2] = mac_wide(s1[4 * m + 2], x1.z, pm);
        s1[4 * m + 3] = mac_wide(s1[4 * m + 3], x1.w, pm);
      }
    }
    if (a.ts && i >= a.src_lo) {
      // this row is a source of the following drop-and-divide: run its INTT
      // pass A (the inverse row pass, GS stages v = 0..7) here and write the
      // result where that INTT's pass B reads it (ts), not into v
      const int tsrow = i < a.level ? i - a.src_lo : a.ts_q + (i - a.level);
#pragma unroll
      for (int pp = 0; pp < 2; ++pp) {
        uint32_t u[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) u[j] = sub_if(mont_reduce64s((uint32_t)(pp ? s1[j] : s0[j]), (uint32_t)((pp ? s1[j] : s0[j]) >> 32), q, P.qinv), q);
        uint32_t* line = sbuf + (pp * kK8Rows + warp) * kK8Stride;  // digit buffers 0 / 1 are free now
        // stages v = 0, 1 on c = 8 lane + k
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int d = 1 << v;
#pragma unroll
          for (int p4 = 0; p4 < 4; ++p4) {
            const int blk = p4 / d, k = blk * 2 * d + p4 % d;
            const uint2 w = Ti[256 - (256 >> v) + (lane << (2 - v)) + blk];
            gs(u[k], u[k + d], w.x, w.y, q, q2);
          }
        }
        *reinterpret_cast<uint4*>(line + pad8(8 * lane)) = make_uint4(u[0], u[1], u[2], u[3]);
        *reinterpret_cast<uint4*>(line + pad8(8 * lane + 4)) = make_uint4(u[4], u[5], u[6], u[7]);
        __syncwarp();
        // stages v = 2, 3, 4 on c = 32 lhi + 4 j + llo
#pragma unroll
        for (int j = 0; j < 8; ++j) u[j] = line[pad8(32 * lhi + 4 * j + llo)];
#pragma unroll
        for (int v = 2; v < 5; ++v) {
          const int d = 1 << (v - 2);
#pragma unroll
          for (int p4 = 0; p4 < 4; ++p4) {
            const int blk = p4 / d, j = blk * 2 * d + p4 % d;
            const uint2 w = Ti[256 - (256 >> v) + (lhi << (4 - v)) + blk];
            gs(u[j], u[j + d], w.x, w.y, q, q2);
          }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) line[pad8(32 * lhi + 4 * j + llo)] = u[j];
        __syncwarp();
        // stages v = 5, 6, 7 on c = lane + 32 j (row-uniform twiddles)
#pragma unroll
        for (int j = 0; j < 8; ++j) u[j] = line[pad8(lane + 32 * j)];
#pragma unroll
        for (int v = 5; v < 8; ++v) {
          const int d = 1 << (v - 5);
#pragma unroll
          for (int p4 = 0; p4 < 4; ++p4) {
            const int blk = p4 / d, j = blk * 2 * d + p4 % d;
            const uint2 w = Ti[256 - (256 >> v) + blk];
            gs(u[j], u[j + d], w.x, w.y, q, q2);
          }
        }
        uint32_t* trow = a.ts + b * a.ts_bs + ((size_t)pp * a.ts_sc + tsrow) * kN + (size_t)r * kR;
#pragma unroll
        for (int j = 0; j < 8; ++j) trow[lane + 32 * j] = u[j];
      }
    } else {
      uint32_t* o0 = a.v + b * a.v_bs + (size_t)i * kN + rofs;
      uint32_t* o1 = a.v + b * a.v_bs + (size_t)(rows + i) * kN + rofs;
      if (LAZY) {  // (0, 4.2 q) -> [0, q)
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          uint32_t r0[4], r1[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            r0[c] = canon8(mont_reduce64s((uint32_t)s0[4 * m + c], (uint32_t)(s0[4 * m + c] >> 32), q, P.qinv), q, q2, q4);
            r1[c] = canon8(mont_reduce64s((uint32_t)s1[4 * m + c], (uint32_t)(s1[4 * m + c] >> 32), q, P.qinv), q, q2, q4);
          }
          stg4(o0 + 4 * m, make_uint4(r0[0], r0[1], r0[2], r0[3]));
          stg4(o1 + 4 * m, make_uint4(r1[0], r1[1], r1[2], r1[3]));
        }
      } else
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        stg4(o0 + 4 * m, make_uint4(sub_if(mont_reduce64s((uint32_t)(s0[4 * m]), (uint32_t)((s0[4 * m]) >> 32), q, P.qinv), q),
                                    sub_if(mont_reduce64s((uint32_t)(s0[4 * m + 1]), (uint32_t)((s0[4 * m + 1]) >> 32), q, P.qinv), q),
                                    sub_if(mont_reduce64s((uint32_t)(s0[4 * m + 2]), (uint32_t)((s0[4 * m + 2]) >> 32), q, P.qinv), q),
                                    sub_if(mont_reduce64s((uint32_t)(s0[4 * m + 3]), (uint32_t)((s0[4 * m + 3]) >> 32), q, P.qinv), q)));
        stg4(o1 + 4 * m, make_uint4(sub_if(mont_reduce64s((uint32_t)(s1[4 * m]), (uint32_t)((s1[4 * m]) >> 32), q, P.qinv), q),
                                    sub_if(mont_reduce64s((uint32_t)(s1[4 * m + 1]), (uint32_t)((s1[4 * m + 1]) >> 32), q, P.qinv), q),
                                    sub_if(mont_reduce64s((uint32_t)(s1[4 * m + 2]), (uint32_t)((s1[4 * m + 2]) >> 32), q, P.qinv), q),
                                    sub_if(mont_reduce64s((uint32_t)(s1[4 * m + 3]), (uint32_t)((s1[4 * m + 3]) >> 32), q, P.qinv), q)));
      }
    }
    }  // KPF != 7
    if (++b == B) {
      b = 0;
      if (++tile == kTiles) {
        tile = 0;
        ++i;
      }
    }
  }
  cp_wait<0>();
}

// k_row_keymult8b: k_row_keymult8 with the CTA's 4 warps on the SAME row r
// of limb i for 4 consecutive batch items (warp w: b = 4 bg + w) instead of
// 4 rows of one item.  The row's 255 forward twiddles and its key slice
// (D digits x 2 halves x 256 words) are then shared by the warps: staged in
// shared memory once per (i, r) -- the key with cp.async together with the
// item's extension rows -- and read from shared memory after each digit's
// row pass.  k_row_keymult8 loads the key halves from L2 right before the
// MACs (64 registers leave no room to load them earlier), and that load is
// the kernel's top stall (13% of the samples, long scoreboard, on the first
// IMAD.WIDE of each digit); here the key crosses L2 once per 4 batch items.
// Items (i, r, bg), bg fastest.  D <= 3; no fused INTT pass A.
constexpr int kK8bSmem = (3 * kK8Rows * kK8Stride) * 4 + 258 * 8 + 3 * 2 * 256 * 4;
template <int MINB>
__global__ void __launch_bounds__(128, MINB) k_row_keymult8b(KeyMultLaunch a, const uint2* __restrict__ fwd) {
  extern __shared__ __align__(128) unsigned char smraw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t* sbuf = reinterpret_cast<uint32_t*>(smraw);                         // [3][4][288] per-warp ext rows
  // [255] row twiddles (shared), one entry past a 16-B boundary so that the
  // 16-B cp.async chunks (odd indices 2^s - 1 + 2c) are aligned
  uint2* T = reinterpret_cast<uint2*>(smraw + 3 * kK8Rows * kK8Stride * 4) + 1;
  uint32_t* Ks = reinterpret_cast<uint32_t*>(T + 257);                        // [3][2][256] key slice (shared)
  const int rows = a.level + a.alpha, B = a.batch, BG = (B + 3) >> 2;
  const uint32_t LA = (uint32_t)(a.L + a.alpha);
  const int items = rows * kR * BG;  // (row i, r, bg), bg fastest
  const int chunk = (items + gridDim.x - 1) / gridDim.x;
  const int i0 = blockIdx.x * chunk, i1 = min(items, i0 + chunk);
  const int lhi = lane >> 2, llo = lane & 3;
  if (i0 >= i1) return;
  int bg = i0 % BG, r = (i0 / BG) % kR, i = (i0 / BG) / kR;
  int g = 0;
  PrimeDev P{};
  uint32_t q = 0, q2 = 0, q4 = 0;
  for (int it = i0; it < i1; ++it) {
    const bool reload = it == i0 || bg == 0;
    const int b = 4 * bg + warp;
    const bool active = b < B;
    if (reload) {  // new (i, r): prime, the row's twiddles and key slice
      __syncthreads();  // every warp is done with the previous (i, r)'s T and Ks
      g = i < a.level ? i : a.L + (i - a.level);
      P = a.primes[g];
      q = P.q;
      q2 = P.q2;
      q4 = 2 * P.q2;
      // the row's twiddles T[2^s - 1 + blk] = F[(256 << s) + (r << s) + blk]:
      // stage s >= 1 is 2^(s-1) aligned 16-B chunks, stage 0 one 8-B pair
      const uint2* F = fwd + (size_t)g * kN;
      if (tid < 127) {
        const int sg = 32 - __clz(tid + 1), c = tid + 1 - (1 << (sg - 1));  // stage 1..7, chunk c
        cp16(&T[(1 << sg) - 1 + 2 * c], &F[(256 << sg) + (r << sg) + 2 * c]);
      } else {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(&T[0]))),
                     "l"(&F[256 + r])
                     : "memory");
      }
      for (int e = tid; e < a.D * 2 * 64; e += 128) {  // D x 2 rows of 64 x 16 B
        const int kh = e >> 6, c = 4 * (e & 63);
        cp16(Ks + kh * 256 + c, a.evk + ((size_t)kh * LA + g) * kN + (size_t)r * kR + c);
      }
    }
    cp_commit();  // the key group (empty unless reload): older than the extension groups
    for (int k = 0; k < a.D; ++k) {
      const int lo = k * a.alpha, hi = min((k + 1) * a.alpha, a.level);
      if (active && !(i >= lo && i < hi)) {
        const uint32_t* gsrc = a.ext + b * a.ext_bs + ((size_t)k * rows + i) * kN + (size_t)r * kR;
        uint32_t* line = sbuf + (k * kK8Rows + warp) * kK8Stride;
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          const int c = 4 * (lane + 32 * m);
          cp16(line + pad8(c), gsrc + c);
        }
      }
      cp_commit();
    }
    const size_t rofs = (size_t)r * kR + 8 * lane;
    if (active && i < a.level && (lane & 3) == 0) {
      asm volatile("prefetch.global.L2 [%0];" ::"l"(a.d + b * a.d_bs + (size_t)i * kN + rofs));
      if (a.fold) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.fold + b * a.fold_bs + (size_t)i * kN + rofs));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.fold + b * a.fold_bs + (size_t)(a.level + i) * kN + rofs));
      }
    }
    if (reload) {  // the key group (oldest) has landed for every thread; T stores visible
      if (a.D >= 3) cp_wait<3>();
      else if (a.D == 2) cp_wait<2>();
      else cp_wait<1>();
      __syncthreads();
    }
    if (active) {
      uint64_t s0[8], s1[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) s0[j] = s1[j] = 0;
      for (int k = 0; k < a.D; ++k) {
        const int lo = k * a.alpha, hi = min((k + 1) * a.alpha, a.level);
        uint32_t v[8];
        if (i >= lo && i < hi) {  // the digit's own row (ModUp pass-through), evaluation form already
          const uint32_t* dr = a.d + b * a.d_bs + (size_t)i * kN + rofs;
          const uint4 x0 = *reinterpret_cast<const uint4*>(dr), x1 = *reinterpret_cast<const uint4*>(dr + 4);
          v[0] = x0.x; v[1] = x0.y; v[2] = x0.z; v[3] = x0.w;
          v[4] = x1.x; v[5] = x1.y; v[6] = x1.z; v[7] = x1.w;
        } else {
          const int pend = a.D - 1 - k;
          if (pend >= 2) cp_wait<2>();
          else if (pend == 1) cp_wait<1>();
          else cp_wait<0>();
          __syncwarp();
          uint32_t* line = sbuf + (k * kK8Rows + warp) * kK8Stride;
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] = line[pad8(lane + 32 * j)];
#pragma unroll
          for (int t = 0; t < 3; ++t) {
            const int d = 4 >> t;
#pragma unroll
            for (int p = 0; p < 4; ++p) {
              const int blk = p / d, j = blk * 2 * d + p % d;
              const uint2 w = T[(1 << t) - 1 + blk];
              if (t % 2 == 0) ctl<true>(v[j], v[j + d], w.x, w.y, q, q2, q4);
              else ctl<false>(v[j], v[j + d], w.x, w.y, q, q2, q4);
            }
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) line[pad8(lane + 32 * j)] = v[j];
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] = line[pad8(32 * lhi + 4 * j + llo)];
#pragma unroll
          for (int t = 0; t < 3; ++t) {
            const int d = 4 >> t, sg = 3 + t;
#pragma unroll
            for (int p = 0; p < 4; ++p) {
              const int blk = p / d, j = blk * 2 * d + p % d;
              const uint2 w = T[(1 << sg) - 1 + (lhi << t) + blk];
              if (sg % 2 == 0) ctl<true>(v[j], v[j + d], w.x, w.y, q, q2, q4);
              else ctl<false>(v[j], v[j + d], w.x, w.y, q, q2, q4);
            }
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) line[pad8(32 * lhi + 4 * j + llo)] = v[j];
          __syncwarp();
          {
            const uint4 x0 = *reinterpret_cast<const uint4*>(line + pad8(8 * lane));
            const uint4 x1 = *reinterpret_cast<const uint4*>(line + pad8(8 * lane + 4));
            v[0] = x0.x; v[1] = x0.y; v[2] = x0.z; v[3] = x0.w;
            v[4] = x1.x; v[5] = x1.y; v[6] = x1.z; v[7] = x1.w;
          }
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const int d = 2 >> t, sg = 6 + t;
#pragma unroll
            for (int p = 0; p < 4; ++p) {
              const int blk = p / d, j = blk * 2 * d + p % d;
              const uint2 w = T[(1 << sg) - 1 + (lane << (t + 1)) + blk];
              if (sg % 2 == 0) ctl<true>(v[j], v[j + d], w.x, w.y, q, q2, q4);
              else ctl<false>(v[j], v[j + d], w.x, w.y, q, q2, q4);
            }
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] = canon8(v[j], q, q2, q4);
        }
        const uint4* kr = reinterpret_cast<const uint4*>(Ks + k * 512 + 8 * lane);
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          const uint4 kb = kr[m], ka = kr[64 + m];  // halves 0 / 1 of digit k
          s0[4 * m] = mac_wide(s0[4 * m], v[4 * m], kb.x);
          s0[4 * m + 1] = mac_wide(s0[4 * m + 1], v[4 * m + 1], kb.y);
          s0[4 * m + 2] = mac_wide(s0[4 * m + 2], v[4 * m + 2], kb.z);
          s0[4 * m + 3] = mac_wide(s0[4 * m + 3], v[4 * m + 3], kb.w);
          s1[4 * m] = mac_wide(s1[4 * m], v[4 * m], ka.x);
          s1[4 * m + 1] = mac_wide(s1[4 * m + 1], v[4 * m + 1], ka.y);
          s1[4 * m + 2] = mac_wide(s1[4 * m + 2], v[4 * m + 2], ka.z);
          s1[4 * m + 3] = mac_wide(s1[4 * m + 3], v[4 * m + 3], ka.w);
        }
      }
      if (a.fold && i < a.level) {  // merged HMult: v += P * d0 / d1 (ckks.cpp:831-842)
        const uint32_t pm = a.p_mont[i];
        const uint32_t* f0 = a.fold + b * a.fold_bs + (size_t)i * kN + rofs;
        const uint32_t* f1 = a.fold + b * a.fold_bs + (size_t)(a.level + i) * kN + rofs;
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          const uint4 x0 = *reinterpret_cast<const uint4*>(f0 + 4 * m);
          const uint4 x1 = *reinterpret_cast<const uint4*>(f1 + 4 * m);
          s0[4 * m] = mac_wide(s0[4 * m], x0.x, pm);
          s0[4 * m + 1] = mac_wide(s0[4 * m + 1], x0.y, pm);
          s0[4 * m + 2] = mac_wide(s0[4 * m + 2], x0.z, pm);
          s0[4 * m + 3] = mac_wide(s0[4 * m + 3], x0.w, pm);
          s1[4 * m] = mac_wide(s1[4 * m], x1.x, pm);
          s1[4 * m + 1] = mac_wide(s1[4 * m + 1], x1.y, pm);
          s1[4 * m + 2] = mac_wide(s1[4 * m + 2], x1.z, pm);
          s1[4 * m + 3] = mac_wide(s1[4 * m + 3], x1.w, pm);
        }
      }
      uint32_t* o0 = a.v + b * a.v_bs + (size_t)i * kN + rofs;
      uint32_t* o1 = a.v + b * a.v_bs + (size_t)(rows + i) * kN + rofs;
#pragma unroll
      for (int m = 0; m < 2; ++m) {
#define CK_R(s, j) sub_if(mont_reduce64s((uint32_t)(s[j]), (uint32_t)((s[j]) >> 32), q, P.qinv), q)
        stg4(o0 + 4 * m, make_uint4(CK_R(s0, 4 * m), CK_R(s0, 4 * m + 1), CK_R(s0, 4 * m + 2), CK_R(s0, 4 * m + 3)));
        stg4(o1 + 4 * m, make_uint4(CK_R(s1, 4 * m), CK_R(s1, 4 * m + 1), CK_R(s1, 4 * m + 2), CK_R(s1, 4 * m + 3)));
#undef CK_R
      }
    } else {
      cp_wait<0>();
    }
    __syncwarp();
    if (++bg == BG) {
      bg = 0;
      if (++r == kR) {
        r = 0;
        ++i;
      }
    }
  }
  cp_wait<0>();
}

// k_row8: the N = 2^16 row passes with 8 coefficients per thread (one
// 256-point row per warp, 4-row tiles, 3 + 3 + 2 stages through two padded
// warp-local exchanges -- the layout of k_row_keymult8) instead of 16: half
// the registers and shared memory per row, so ~2x the warps per SM.
// Forward (stages 8..15 of the NTT, lazy [0, 8q) schedule, canonical
// output; COMB 3: the drop-and-divide combine fused, v rows requested into
// L2 at the item start) in place on dst; inverse (stages 0..7, output
// [0, 2q) for the column pass) src -> dst.  Twiddles come from the full
// per-prime tables (a.tw) in natural order per row, staged once per
// (job, row tile) and reused for the batch.
template <bool INV, int COMB = 0>
__global__ void __launch_bounds__(128, 8) k_row8(NttLaunch a, CombineArgs cb) {
  extern __shared__ __align__(128) unsigned char smraw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t* lines = reinterpret_cast<uint32_t*>(smraw) + warp * 2 * kK8Stride;  // this warp's 2 input buffers
  uint2* T = reinterpret_cast<uint2*>(smraw + kK8Rows * 2 * kK8Stride * 4) + warp * 256;
  constexpr int kTiles = kR / kK8Rows;
  const int B = a.batch;
  const int items = a.njobs * kTiles * B;
  const int chunk = (items + gridDim.x - 1) / gridDim.x;
  const int i0 = blockIdx.x * chunk, i1 = min(items, i0 + chunk);
  if (i0 >= i1) return;
  const int lhi = lane >> 2, llo = lane & 3;
  // cursors (job, tile, b), b fastest
  int b = i0 % B, tile = (i0 / B) % kTiles, job = (i0 / B) / kTiles;
  int nb = b, ntile = tile, njob = job;
  auto advance = [&](int& bb, int& tt, int& jj) {
    if (++bb == B) {
      bb = 0;
      if (++tt == kTiles) {
        tt = 0;
        ++jj;
      }
    }
  };
  auto in_row = [&](int bb, int tt, const RowJob& J) {
    const int r = tt * kK8Rows + warp;
    return INV ? a.src + bb * a.src_bs + (size_t)J.src_off * kN + (size_t)r * kR
               : a.dst + bb * a.dst_bs + (size_t)J.dst_off * kN + (size_t)r * kR;
  };
  auto stage_row = [&](uint32_t* line, const uint32_t* g) {
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const int c = 4 * (lane + 32 * m);
      cp16(line + pad8(c), g + c);
    }
  };
  RowJob J = a.jobs[job], Jn = J;
  stage_row(lines, in_row(b, tile, J));
  cp_commit();
  uint32_t q = 0, q2 = 0, q4 = 0, qinv = 0, di = 0;
  for (int it = i0, k = 0; it < i1; ++it, ++k) {
    uint32_t* line = lines + (k & 1) * kK8Stride;
    const int r = tile * kK8Rows + warp;
    if (it == i0 || b == 0) {  // new (job, tile): prime and this row's 255 twiddles (natural order)
      __syncwarp();
      const PrimeDev P = a.primes[J.prime];
      q = P.q;
      q2 = P.q2;
      q4 = 2 * P.q2;
      qinv = P.qinv;
      const uint2* F = a.tw + (size_t)J.prime * kN;
      if (!INV) {
        for (int e = lane; e < 255; e += 32) {
          const int s = 31 - __clz(e + 1), blk = e + 1 - (1 << s);
          T[e] = __ldg(&F[(256 << s) + (r << s) + blk]);
        }
      } else {
#pragma unroll
        for (int v = 0; v < 8; ++v)
          for (int blk = lane; blk < (128 >> v); blk += 32)
            T[256 - (256 >> v) + blk] = __ldg(&F[(kN >> (v + 1)) + (r << (7 - v)) + blk]);
      }
      if (COMB) di = cb.dinv[J.dst_off - (J.dst_off / cb.out_q) * cb.out_q];
    }
    if (it + 1 < i1) {  // prefetch the next item's row into the other buffer
      advance(nb, ntile, njob);
      if (njob != job) Jn = a.jobs[njob];
      stage_row(lines + ((k + 1) & 1) * kK8Stride, in_row(nb, ntile, Jn));
    }
    cp_commit();
    if (COMB == 3) {  // the combine's v row into L2 now (plain loads at the end); one lane per 128 B line
      const uint32_t pi = J.dst_off / cb.out_q, i = J.dst_off - pi * cb.out_q;
      if ((lane & 3) == 0)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(cb.v + b * cb.v_bs + ((size_t)pi * cb.prow + i) * kN +
                                                       (size_t)r * kR + 8 * lane));
    }
    cp_wait<1>();
    __syncwarp();
    uint32_t u[8];
    if (!INV) {
#pragma unroll
      for (int j = 0; j < 8; ++j) u[j] = line[pad8(lane + 32 * j)];
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        const int d = 4 >> t;
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const int blk = p / d, j = blk * 2 * d + p % d;
          const uint2 w = T[(1 << t) - 1 + blk];
          if (t % 2 == 0) ctl<true>(u[j], u[j + d], w.x, w.y, q, q2, q4);
          else ctl<false>(u[j], u[j + d], w.x, w.y, q, q2, q4);
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) line[pad8(lane + 32 * j)] = u[j];
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 8; ++j) u[j] = line[pad8(32 * lhi + 4 * j + llo)];
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        const int d = 4 >> t, sg = 3 + t;
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const int blk = p / d, j = blk * 2 * d + p % d;
          const uint2 w = T[(1 << sg) - 1 + (lhi << t) + blk];
          if (sg % 2 == 0) ctl<true>(u[j], u[j + d], w.x, w.y, q, q2, q4);
          else ctl<false>(u[j], u[j + d], w.x, w.y, q, q2, q4);
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) line[pad8(32 * lhi + 4 * j + llo)] = u[j];
      __syncwarp();
      {
        const uint4 x0 = *reinterpret_cast<const uint4*>(line + pad8(8 * lane));
        const uint4 x1 = *reinterpret_cast<const uint4*>(line + pad8(8 * lane + 4));
        u[0] = x0.x; u[1] = x0.y; u[2] = x0.z; u[3] = x0.w;
        u[4] = x1.x; u[5] = x1.y; u[6] = x1.z; u[7] = x1.w;
      }
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int d = 2 >> t, sg = 6 + t;
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const int blk = p / d, j = blk * 2 * d + p % d;
          const uint2 w = T[(1 << sg) - 1 + (lane << (t + 1)) + blk];
          if (sg % 2 == 0) ctl<true>(u[j], u[j + d], w.x, w.y, q, q2, q4);
          else ctl<false>(u[j], u[j + d], w.x, w.y, q, q2, q4);
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) u[j] = canon8(u[j], q, q2, q4);
      if (COMB) {  // out = (v - NTT) d^-1 (ckks.cpp:643-651); J.dst_off = p * out_q + i
        const uint32_t pi = J.dst_off / cb.out_q, i = J.dst_off - pi * cb.out_q;
        const uint32_t* vr = cb.v + b * cb.v_bs + ((size_t)pi * cb.prow + i) * kN + (size_t)r * kR + 8 * lane;
        const uint4 v0 = *reinterpret_cast<const uint4*>(vr), v1 = *reinterpret_cast<const uint4*>(vr + 4);
        const uint32_t vv[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
        for (int j = 0; j < 8; ++j) u[j] = sub_if(mont_mul(vv[j] - u[j] + q, di, q, qinv), q);
      }
      uint32_t* orow = a.dst + b * a.dst_bs + (size_t)J.dst_off * kN + (size_t)r * kR + 8 * lane;
      stg4(orow, make_uint4(u[0], u[1], u[2], u[3]));
      stg4(orow + 4, make_uint4(u[4], u[5], u[6], u[7]));
    } else {
      {
        const uint4 x0 = *reinterpret_cast<const uint4*>(line + pad8(8 * lane));
        const uint4 x1 = *reinterpret_cast<const uint4*>(line + pad8(8 * lane + 4));
        u[0] = x0.x; u[1] = x0.y; u[2] = x0.z; u[3] = x0.w;
        u[4] = x1.x; u[5] = x1.y; u[6] = x1.z; u[7] = x1.w;
      }
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int d = 1 << v;
#pragma unroll
        for (int p4 = 0; p4 < 4; ++p4) {
          const int blk = p4 / d, kk = blk * 2 * d + p4 % d;
          const uint2 w = T[256 - (256 >> v) + (lane << (2 - v)) + blk];
          gs(u[kk], u[kk + d], w.x, w.y, q, q2);
        }
      }
      *reinterpret_cast<uint4*>(line + pad8(8 * lane)) = make_uint4(u[0], u[1], u[2], u[3]);
      *reinterpret_cast<uint4*>(line + pad8(8 * lane + 4)) = make_uint4(u[4], u[5], u[6], u[7]);
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 8; ++j) u[j] = line[pad8(32 * lhi + 4 * j + llo)];
#pragma unroll
      for (int v = 2; v < 5; ++v) {
        const int d = 1 << (v - 2);
#pragma unroll
        for (int p4 = 0; p4 < 4; ++p4) {
          const int blk = p4 / d, j = blk * 2 * d + p4 % d;
          const uint2 w = T[256 - (256 >> v) + (lhi << (4 - v)) + blk];
          gs(u[j], u[j + d], w.x, w.y, q, q2);
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) line[pad8(32 * lhi + 4 * j + llo)] = u[j];
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 8; ++j) u[j] = line[pad8(lane + 32 * j)];
#pragma unroll
      for (int v = 5; v < 8; ++v) {
        const int d = 1 << (v - 5);
#pragma unroll
        for (int p4 = 0; p4 < 4; ++p4) {
          const int blk = p4 / d, j = blk * 2 * d + p4 % d;
          const uint2 w = T[256 - (256 >> v) + blk];
          gs(u[j], u[j + d], w.x, w.y, q, q2);
        }
      }
      uint32_t* orow = a.dst + b * a.dst_bs + (size_t)J.dst_off * kN + (size_t)r * kR;
#pragma unroll
      for (int j = 0; j < 8; ++j) orow[lane + 32 * j] = u[j];
    }
    __syncwarp();  // this warp's buffer k&1 is refilled by the prefetch of iteration k+1
    b = nb;
    tile = ntile;
    job = njob;
    J = Jn;
  }
  cp_wait<0>();
}

}  // namespace

// CK32_KM selects the k_row_keymult variant for A/B runs: 7 = k_row_keymult8
// (default when D <= 3), 6 = 0 + L2 prefetch of own / fold rows, 5 =
// k_row_keymult_pf; 0 = key halves
// loaded before the row pass, all digit tiles of an item requested at once
// (default when D <= 3), 3 = the same with per-digit tile loads (4.83 TB/s),
// 1 = per-digit loads at 3 CTAs/SM (4.20), 2 = key halves loaded after the
// row pass (the first version, 4.77).
template <bool EARLY, int MINB, bool ALLD = false, bool WL = false, bool L2PF = false>
static void launch_km(const KeyMultLaunch& a, const uint2* tw2, int items, cudaStream_t st) {
  static int grid = 0;
  constexpr int smem = ALLD ? kKSmem + kKBuf * 4 : kKSmem;
  if (!grid) {
    cudaFuncSetAttribute(k_row_keymult<EARLY, MINB, ALLD, WL, L2PF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         smem);
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_row_keymult<EARLY, MINB, ALLD, WL, L2PF>, kKT, smem);
    grid = sms * std::max(1, per);
  }
  k_row_keymult<EARLY, MINB, ALLD, WL, L2PF><<<std::min(grid, items), kKT, smem, st>>>(a, tw2);
}

static int km_version() {
  static int ver = -1;
  if (ver < 0) {  // default: the 8-coefficient-per-thread kernel, keys after the row pass, 8 CTAs / SM (r2z:
                  // 268 vs 277 us for KM=7 and 288 us for round 1's kernel; +1.1% / +4% ops/s)
    const char* e = std::getenv("CK32_KM");
    ver = e ? std::atoi(e) : 8;
  }
  return ver;
}

// The switch's INTT pass A in the KeyMult epilogue (CK32_KM_INTT=1): bit-exact
// and it removes that pass's HBM round trip, but the extra butterflies land
// on the latency-bound KeyMult kernel -- measured neutral to slightly slower
// (r2aa: 16.90k vs 16.96k ops/s), so opt-in.
bool row_keymult_fuses_intt(const KeyMultLaunch& a) {
  static int on = -1;
  if (on < 0) on = std::getenv("CK32_KM_INTT") != nullptr;
  const int v = km_version();
  return on && v >= 7 && v <= 11 && a.D <= 3;
}

template <int MINB, bool EARLY, int KPF = 0, int DD = 0>
static void launch_km8(const KeyMultLaunch& a, const uint2* fwd, int items, cudaStream_t st) {
  static int grid[2] = {0, 0};
  const int fi = a.ts ? 1 : 0;  // the inverse twiddle region only when the INTT pass A is fused
  const int smem = KPF == 3 ? kK8Smem + kK8Rows * 3 * 2 * 256 * 4
                   : KPF == 6 ? kK8SmemBase + kK8Rows * 2 * 256 * 4
                   : fi       ? kK8Smem
                              : kK8SmemBase;
  if (!grid[fi]) {
    cudaFuncSetAttribute(k_row_keymult8<MINB, EARLY, KPF, DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_row_keymult8<MINB, EARLY, KPF, DD>, 128, smem);
    grid[fi] = sms * std::max(1, std::min(per, env_cap("CK32_KM_CTAS")));
  }
  k_row_keymult8<MINB, EARLY, KPF, DD><<<std::min(grid[fi], items), 128, smem, st>>>(a, fwd);
}

template <int MINB>
static void launch_km_pf(const KeyMultLaunch& a, const uint2* tw2, int items, cudaStream_t st) {
  static int grid = 0;
  constexpr int smem = kKSmem + kKBuf * 4;
  if (!grid) {
    cudaFuncSetAttribute(k_row_keymult_pf<MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_row_keymult_pf<MINB>, kKT, smem);
    grid = sms * std::max(1, per);
  }
  k_row_keymult_pf<MINB><<<std::min(grid, items), kKT, smem, st>>>(a, tw2);
}

void row_keymult(const KeyMultLaunch& a, const uint2* tw2, cudaStream_t st, const uint2* fwd_full) {
  const int ver = km_version();
  const int items = (a.level + a.alpha) * (kR / kRRows) * a.batch;
  if (ver == 5 && a.D <= 3) {
    launch_km_pf<4>(a, tw2, items, st);
    return;
  }
  if (ver == 6 && a.D <= 3) {
    launch_km<true, 4, true, true, true>(a, tw2, items, st);
    return;
  }
  if (ver == 12 && a.D <= 3 && fwd_full && !a.ts && a.batch >= 4) {  // batch-shared key / twiddles
    const int items8b = (a.level + a.alpha) * kR * ((a.batch + 3) / 4);
    static int grid = 0;
    if (!grid) {
      cudaFuncSetAttribute(k_row_keymult8b<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, kK8bSmem);
      int dev = 0, sms = 148, per = 1;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_row_keymult8b<8>, 128, kK8bSmem);
      grid = sms * std::max(1, per);
    }
    k_row_keymult8b<8><<<std::min(grid, items8b), 128, kK8bSmem, st>>>(a, fwd_full);
    return;
  }
  if (ver >= 7 && ver <= 16 && a.D <= 3 && fwd_full) {  // 8 coefficients per thread
    const int items8 = (a.level + a.alpha) * (kR / kK8Rows) * a.batch;
    if (ver == 13 && !a.ts)
      launch_km8<8, false, 4>(a, fwd_full, items8, st);  // own / fold rows through cp.async into freed digit buffers
    else if (ver == 14 && !a.ts)
      launch_km8<8, false, 5>(a, fwd_full, items8, st);  // next item's extension rows into each freed digit buffer
    else if (ver == 15 && !a.ts)
      launch_km8<7, false, 6>(a, fwd_full, items8, st);  // per-digit key slice + row twiddles by cp.async, 7 CTAs / SM
    else if (ver == 16 && !a.ts) {  // the MACs after all digits' row passes (per digit count)
      if (a.D == 3)
        launch_km8<8, false, 7, 3>(a, fwd_full, items8, st);
      else if (a.D == 2)
        launch_km8<8, false, 7, 2>(a, fwd_full, items8, st);
      else
        launch_km8<8, false, 7, 1>(a, fwd_full, items8, st);
    }
    else if (ver == 11)
      launch_km8<4, false, 3>(a, fwd_full, items8, st);  // key slice staged in shared memory per (row, tile), 4 CTAs / SM
    else if (ver == 9)
      launch_km8<8, false, 1>(a, fwd_full, items8, st);  // + the digit's key lines into L1 before its row pass
    else if (ver == 10)
      launch_km8<8, false, 2>(a, fwd_full, items8, st);  // + the next digit's key lines into L1 one digit ahead
    else if (ver == 7)
      launch_km8<6, true>(a, fwd_full, items8, st);  // keys ahead of the row pass, 6 CTAs / SM
    else
      launch_km8<8, false>(a, fwd_full, items8, st);  // keys after it, 64 registers, 8 CTAs / SM
    return;
  }
  if (ver == 1)
    launch_km<true, 3>(a, tw2, items, st);
  else if (ver == 2)
    launch_km<false, 4>(a, tw2, items, st);
  else if (ver == 3 || a.D > 3)
    launch_km<true, 4>(a, tw2, items, st);
  else if (ver == 4)
    launch_km<true, 4, true>(a, tw2, items, st);
  else
    launch_km<true, 4, true, true>(a, tw2, items, st);
}

void conv_mid(const ConvMidLaunch& a, cudaStream_t st) {
  const int smem = (a.max_sc * 512 + 8 * 512) * 16;
  dim3 grid(kMTiles, a.ngroups, a.batch);
  switch (a.max_sc) {
#define CK_SC(S)                                                                              \
  case S: {                                                                                   \
    static bool attr = false;                                                                 \
    if (!attr) {                                                                              \
      cudaFuncSetAttribute(k_conv_mid<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
      attr = true;                                                                            \
    }                                                                                         \
    k_conv_mid<S><<<grid, 256, smem, st>>>(a);                                                \
    break;                                                                                    \
  }
    CK_SC(1) CK_SC(2) CK_SC(3) CK_SC(4) CK_SC(5) CK_SC(6) CK_SC(7) CK_SC(8) CK_SC(9) CK_SC(10)
#undef CK_SC
    default: break;
  }
}


// CK32_ROW8=1: the plain row passes run as k_row8 (8 coefficients per thread)
constexpr int kRow8Smem = kK8Rows * 2 * kK8Stride * 4 + kK8Rows * 256 * 8;  // 2 input buffers + twiddles, 17 KB
static bool use_row8() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("CK32_ROW8");
    v = e && e[0] == '1';
  }
  return v == 1;
}
template <bool INV, int COMB>
static void launch_row8(const NttLaunch& a, const CombineArgs& cb, cudaStream_t st) {
  static int grid = 0;
  if (!grid) {
    cudaFuncSetAttribute(k_row8<INV, COMB>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRow8Smem);
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_row8<INV, COMB>, 128, kRow8Smem);
    grid = sms * std::max(1, per);
  }
  const int items = a.njobs * (kR / kK8Rows) * a.batch;
  k_row8<INV, COMB><<<std::min(grid, items), 128, kRow8Smem, st>>>(a, cb);
}

// Individual passes (used when the fused kernels replace the other pass).
void ntt256_pass(int which, const NttLaunch& a, const uint2* tw2, cudaStream_t st) {
  init_grids();
  const int row_items = a.njobs * (kR / kRRows) * a.batch;
  switch (which) {
    case 0:
      launch_col<false>(a, a.src, a.src_bs, st);
      break;
    case 1:  // forward row pass, in place on dst
      if (use_row8()) {
        launch_row8<false, 0>(a, CombineArgs{}, st);
        break;
      }
      k_row<false><<<min(g_row_grid, row_items), kRT, kRowSmem, st>>>(a.jobs, a.dst, a.dst_bs, a.dst, a.dst_bs,
                                                                      a.batch, a.njobs, a.primes, tw2);
      break;
    case 2:  // inverse row pass src -> dst
      if (use_row8()) {
        launch_row8<true, 0>(a, CombineArgs{}, st);
        break;
      }
      k_row<true><<<min(g_row_grid, row_items), kRT, kRowSmem, st>>>(a.jobs, a.src, a.src_bs, a.dst, a.dst_bs,
                                                                     a.batch, a.njobs, a.primes, tw2);
      break;
    default: {
      NttLaunch b = a;
      b.entry = 0;
      launch_col<true>(b, a.dst, a.dst_bs, st);
    }
  }
}

// ================================================ N = 2^17: 512-point rows ==
// N = 2^17 as 256 columns x 512-point rows (x = 512 r + c): the column pass is
// k_col<.., LOGR = 9> (stages 0-7), the row pass below runs the other 9
// stages on rows of 512.  16 threads per row, 32 elements per thread:
//   forward  phase A: c = tau + 16 j, stages 8-12 (row-shared twiddles W[0..30])
//            phase B: c = 32 tau + j, stages 13-16 (per-thread twiddles)
//   inverse  phase A: c = 32 tau + j, stages v = 0-3 (per-thread twiddles)
//            phase B: c = tau + 16 j, stages v = 4-8 (row-shared)
// Row layout in shared memory: c -> c + 4 (c >> 5) (the 32-word chunks of
// phase B start on distinct bank quads), rows 592 words apart (the two rows
// of a warp sit on opposite bank halves for the stride-16 accesses).  Each
// warp stages its own two rows of the data tile and of the per-row twiddle
// tables (512 pairs, host-permuted in consumption order): no CTA barrier.
constexpr int kR5 = 512;
__device__ __forceinline__ int rpos5(int c) { return c + 4 * (c >> 5); }
// Row-pass geometry for rows of R = 2^LOGR (LOGR = 8 or 9), 32 elements per
// thread: TPR threads per row, RPC rows per 128-thread CTA, padded stride.
template <int LOGR>
struct RowX {
  static constexpr int R = 1 << LOGR, N = 256 * R, TPR = R / 32, RPC = 128 / TPR, RPW = 32 / TPR;
  static constexpr int STRIDE = R + R / 8 + (TPR == 16 ? 16 : 8);  // rows of a warp on distinct bank groups
  static constexpr int BUF = RPC * STRIDE;
  static constexpr int SMEM = 2 * BUF * 4 + RPC * R * 8;
  static constexpr int PB = LOGR - 5;                  // phase-B forward stages / phase-A inverse stages + 1
  static constexpr int RS_BASE = TPR * (32 - (1 << (5 - PB)));  // inverse: per-thread entries before the row-shared ones
};

template <bool INV, int LOGR>
__global__ void __launch_bounds__(kRT) k_rowx(const RowJob* __restrict__ jobs, const uint32_t* __restrict__ src,
                                              uint64_t src_bs, uint32_t* __restrict__ dst, uint64_t dst_bs, int batch,
                                              int njobs, const PrimeDev* __restrict__ primes,
                                              const uint2* __restrict__ tw2) {
  using G = RowX<LOGR>;
  extern __shared__ __align__(128) unsigned char smraw[];
  uint32_t* sbuf = reinterpret_cast<uint32_t*>(smraw);
  uint2* tws = reinterpret_cast<uint2*>(smraw + 2 * G::BUF * 4);  // [RPC][R]
  const int tid = threadIdx.x, rho = tid / G::TPR, tau = tid % G::TPR, warp = tid >> 5, lane = tid & 31;
  constexpr int kTiles = 256 / G::RPC;
  const int items = njobs * kTiles * batch;
  const int chunk = (items + gridDim.x - 1) / gridDim.x;
  const int i0 = blockIdx.x * chunk, i1 = min(items, i0 + chunk);
  if (i0 >= i1) return;
  RowCursorT<kTiles> c;
  c.init(i0, batch);
  RowJob Jc = jobs[c.job];
  RowCursorT<kTiles> nx = c;
  RowJob Jn = Jc;
  auto in_ptr = [&](const RowCursorT<kTiles>& x, const RowJob& J) {
    return INV ? src + x.b * src_bs + (size_t)J.src_off * G::N + x.tile * G::RPC * G::R
               : dst + x.b * dst_bs + (size_t)J.dst_off * G::N + x.tile * G::RPC * G::R;
  };
  auto prefetch = [&](uint32_t* buf, const uint32_t* g) {  // this warp's RPW rows, 16 B per cp.async
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const int e = lane + 32 * m, r = G::RPW * warp + e / (G::R / 4), cc = (e % (G::R / 4)) * 4;
      cp16(buf + r * G::STRIDE + rpos5(cc), g + r * G::R + cc);
    }
  };
  prefetch(sbuf, in_ptr(nx, Jn));
  cp_commit();
  uint32_t q = 0, q2 = 0, q4 = 0;
  for (int it = i0, k = 0; it < i1; ++it, ++k) {
    uint32_t* line_buf = sbuf + (k & 1) * G::BUF;
    const int b = c.b, tile = c.tile;
    const RowJob J = Jc;
    const bool reload = it == i0 || b == 0;
    if (reload) {  // this warp's rows of the tile's twiddle tables (1024 pairs)
      __syncwarp();
      const uint2* T = tw2 + ((size_t)J.prime * 256 + tile * G::RPC + G::RPW * warp) * G::R;
      for (int e = lane; e < 512; e += 32) cp16(&tws[G::RPW * warp * G::R + 2 * e], &T[2 * e]);
      cp_commit();
    }
    if (it + 1 < i1) {
      const int pj = nx.job;
      nx.next(batch);
      if (nx.job != pj) Jn = jobs[nx.job];
      prefetch(sbuf + ((k + 1) & 1) * G::BUF, in_ptr(nx, Jn));
    }
    cp_commit();
    cp_wait<1>();
    __syncwarp();
    if (reload) {
      const PrimeDev P = primes[J.prime];
      q = P.q;
      q2 = P.q2;
      q4 = 2 * P.q2;
    }
    const int r = tile * G::RPC + rho;
    const uint2* W = tws + rho * G::R;
    uint32_t* line = line_buf + rho * G::STRIDE;
    uint32_t* orow = dst + b * dst_bs + (size_t)J.dst_off * G::N + (size_t)r * G::R;
    uint32_t v[32];
    if (!INV) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = line[rpos5(tau + G::TPR * j)];
#pragma unroll
      for (int t = 0; t < 5; ++t) {  // row stage t: pairs (j, j + (16 >> t)), twiddle W[2^t - 1 + (j >> (5 - t))]
        const int d = 16 >> t;
#pragma unroll
        for (int p = 0; p < 16; ++p) {
          const int blk = p / d, j = blk * 2 * d + p % d;
          const uint2 w = W[(1 << t) - 1 + blk];
          if (t % 2 == 0) ctl<true>(v[j], v[j + d], w.x, w.y, q, q2, q4);
          else ctl<false>(v[j], v[j + d], w.x, w.y, q, q2, q4);
        }
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) line[rpos5(tau + G::TPR * j)] = v[j];
      __syncwarp();
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const uint4 x = *reinterpret_cast<const uint4*>(line + rpos5(32 * tau) + 4 * m);
        v[4 * m] = x.x;
        v[4 * m + 1] = x.y;
        v[4 * m + 2] = x.z;
        v[4 * m + 3] = x.w;
      }
#pragma unroll
      for (int t = 5; t < LOGR; ++t) {  // row stage t: pairs (j, j + (R/2 >> t)), per-thread twiddles
        const int d = (G::R / 2) >> t, cnt0 = 1 << (5 - G::PB), off = (1 << (t - G::PB)) - cnt0;
#pragma unroll
        for (int p = 0; p < 16; ++p) {
          const int blk = p / d, j = blk * 2 * d + p % d;
          const uint2 w = W[32 + (off + blk) * G::TPR + tau];
          if (t % 2 == 0) ctl<true>(v[j], v[j + d], w.x, w.y, q, q2, q4);
          else ctl<false>(v[j], v[j + d], w.x, w.y, q, q2, q4);
        }
      }
#pragma unroll
      for (int m = 0; m < 8; ++m)
        stg4(orow + 32 * tau + 4 * m, make_uint4(canon8(v[4 * m], q, q2, q4), canon8(v[4 * m + 1], q, q2, q4),
                                                 canon8(v[4 * m + 2], q, q2, q4), canon8(v[4 * m + 3], q, q2, q4)));
    } else {
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const uint4 x = *reinterpret_cast<const uint4*>(line + rpos5(32 * tau) + 4 * m);
        v[4 * m] = x.x;
        v[4 * m + 1] = x.y;
        v[4 * m + 2] = x.z;
        v[4 * m + 3] = x.w;
      }
      constexpr int kOffI[4] = {0, 16, 24, 28};
#pragma unroll
      for (int t = 0; t < G::PB; ++t) {  // inverse stages t: pairs (j, j + 2^t), per-thread twiddles
        const int d = 1 << t;
#pragma unroll
        for (int p = 0; p < 16; ++p) {
          const int blk = p / d, j = blk * 2 * d + p % d;
          const uint2 w = W[(kOffI[t] + blk) * G::TPR + tau];
          gs(v[j], v[j + d], w.x, w.y, q, q2);
        }
      }
#pragma unroll
      for (int m = 0; m < 8; ++m)
        *reinterpret_cast<uint4*>(line + rpos5(32 * tau) + 4 * m) =
            make_uint4(v[4 * m], v[4 * m + 1], v[4 * m + 2], v[4 * m + 3]);
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = line[rpos5(tau + G::TPR * j)];
      constexpr int kOffR[5] = {0, 16, 24, 28, 30};
#pragma unroll
      for (int t = 0; t < 5; ++t) {  // inverse stages PB + t: pairs (j, j + 2^t), row-shared twiddles
        const int d = 1 << t;
#pragma unroll
        for (int p = 0; p < 16; ++p) {
          const int blk = p / d, j = blk * 2 * d + p % d;
          const uint2 w = W[G::RS_BASE + kOffR[t] + blk];
          gs(v[j], v[j + d], w.x, w.y, q, q2);
        }
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) orow[tau + G::TPR * j] = v[j];
    }
    c = nx;
    Jc = Jn;
    __syncwarp();
  }
  cp_wait<0>();
}

template <bool INV>
void launch_col9(const NttLaunch& a, const uint32_t* src, uint64_t src_bs, cudaStream_t st) {
  static int grid = 0;
  if (!grid) {
    cudaFuncSetAttribute(k_col<INV, false, true, 5, 9>, cudaFuncAttributeMaxDynamicSharedMemorySize, kColRingSmem);
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_col<INV, false, true, 5, 9>, kCT, kColRingSmem);
    grid = sms * std::max(1, per);
  }
  const int items = a.njobs * a.batch * (kR5 / kCCols);
  k_col<INV, false, true, 5, 9><<<min(grid, items), kCT, kColRingSmem, st>>>(
      a.jobs, src, src_bs, a.dst, a.dst_bs, a.batch, a.njobs, a.primes, a.tw, a.exits, a.entry, CUtensorMap{});
}

template <bool INV, int LOGR>
void launch_rowx(const NttLaunch& a, const uint32_t* src, uint64_t src_bs, const uint2* tw2, cudaStream_t st) {
  using G = RowX<LOGR>;
  static int grid = 0;
  if (!grid) {
    cudaFuncSetAttribute(k_rowx<INV, LOGR>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_rowx<INV, LOGR>, kRT, G::SMEM);
    grid = sms * std::max(1, per);
  }
  const int items = a.njobs * (256 / G::RPC) * a.batch;
  k_rowx<INV, LOGR><<<min(grid, items), kRT, G::SMEM, st>>>(a.jobs, src, src_bs, a.dst, a.dst_bs, a.batch, a.njobs,
                                                             a.primes, tw2);
}

bool ntt131k_forward(const NttLaunch& a, const uint2* tw2, cudaStream_t st) {
  launch_col9<false>(a, a.src, a.src_bs, st);
  launch_rowx<false, 9>(a, a.dst, a.dst_bs, tw2, st);  // in place on dst
  return true;
}

bool ntt131k_inverse(const NttLaunch& a, const uint2* tw2i, cudaStream_t st) {
  launch_rowx<true, 9>(a, a.src, a.src_bs, tw2i, st);
  NttLaunch b = a;
  b.entry = 0;
  launch_col9<true>(b, a.dst, a.dst_bs, st);
  return true;
}

bool ntt256_forward(const NttLaunch& a, const uint2* tw2, cudaStream_t st) {
  init_grids();
  const int row_items = a.njobs * (kR / kRRows) * a.batch;
  launch_col<false>(a, a.src, a.src_bs, st);
  if (use_row8()) {
    launch_row8<false, 0>(a, CombineArgs{}, st);
    return true;
  }
  k_row<false><<<min(g_row_grid, row_items), kRT, kRowSmem, st>>>(a.jobs, a.dst, a.dst_bs, a.dst, a.dst_bs, a.batch,
                                                                  a.njobs, a.primes, tw2);
  return true;
}

template <int COMB>
static void launch_row_comb(const NttLaunch& a, const uint2* tw2, const CombineArgs& cb, int items, cudaStream_t st) {
  static int grid = 0;
  if (!grid) {
    cudaFuncSetAttribute(k_row<false, COMB>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRowSmem);
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_row<false, COMB>, kRT, kRowSmem);
    grid = sms * std::max(1, per);
  }
  k_row<false, COMB><<<min(grid, items), kRT, kRowSmem, st>>>(a.jobs, a.dst, a.dst_bs, a.dst, a.dst_bs, a.batch,
                                                               a.njobs, a.primes, tw2, cb);
}

bool ntt256_forward_hrot_tail(const NttLaunch& a, const uint2* tw2, const CombineArgs& cb, cudaStream_t st) {
  init_grids();
  const int row_items = a.njobs * (kR / kRRows) * a.batch;
  launch_col<false>(a, a.src, a.src_bs, st);
  launch_row_comb<4>(a, tw2, cb, row_items, st);
  return true;
}

bool ntt256_forward_combine(const NttLaunch& a, const uint2* tw2, const CombineArgs& cb, cudaStream_t st) {
  init_grids();
  // CK32_COMB_EARLY: 2 = the combine operand rows are requested into L2 at
  // the item start (default: +7-10% on this class, r2i), 1 = loaded into
  // registers at the item start, 0 = loaded right before the store (round 1)
  static int early = -1;
  if (early < 0) {
    const char* e = std::getenv("CK32_COMB_EARLY");
    early = e ? std::atoi(e) : 2;
  }
  const int row_items = a.njobs * (kR / kRRows) * a.batch;
  launch_col<false>(a, a.src, a.src_bs, st);
  if (early == 2 && use_row8()) launch_row8<false, 3>(a, cb, st);
  else if (early == 2) launch_row_comb<3>(a, tw2, cb, row_items, st);
  else if (early) launch_row_comb<2>(a, tw2, cb, row_items, st);
  else launch_row_comb<1>(a, tw2, cb, row_items, st);
  return true;
}

bool ntt256_inverse(const NttLaunch& a, const uint2* tw2i, cudaStream_t st) {
  init_grids();
  const int row_items = a.njobs * (kR / kRRows) * a.batch;
  if (use_row8())
    launch_row8<true, 0>(a, CombineArgs{}, st);
  else
    k_row<true><<<min(g_row_grid, row_items), kRT, kRowSmem, st>>>(a.jobs, a.src, a.src_bs, a.dst, a.dst_bs, a.batch,
                                                                   a.njobs, a.primes, tw2i);
  NttLaunch b = a;
  b.entry = 0;
  launch_col<true>(b, a.dst, a.dst_bs, st);
  return true;
}

}  // namespace ck
