// Device-side building blocks shared by every ck32-b200 kernel.
//
// Arithmetic model (B200-first restatement of the reference's signed
// Montgomery core, modarith.hpp:11-60):
//   * residues are stored canonical [0, q) as uint32 in HBM; evaluation-domain
//     polynomials carry the reference's Montgomery factor R = 2^32 (the stored
//     value is X*R mod q, exactly the reference's canonical residue);
//   * constant x variable products (twiddles, BConv part 1, exit constants,
//     divisor inverses) use Shoup multiplication with a precomputed
//     w' = floor(w * 2^32 / q): 3 integer-pipe ops, output in [0, 2q);
//   * variable x variable products (tensor, KeyMult) and the int64 BConv /
//     KeyMult accumulators use unsigned Montgomery reduction, output [0, 2q);
//   * NTT butterflies are Harvey-lazy: values live in [0, 4q) between stages
//     (q < 2^29 is guaranteed by generate_basis' cap, rns.cpp:71-72).
// Canonical outputs are a pure function of canonical inputs,
// so the results are bit-identical to the reference after correct_lazy.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ck {

constexpr int kMaxRows = 96;  // max rows of one polynomial (L + alpha)

// Per-prime constants (device copy; built by the host in ck_context.cu).
struct PrimeDev {
  uint32_t q, q2;        // q, 2q
  uint32_t qinv_neg;     // -q^{-1} mod 2^32 (unsigned Montgomery)
  uint32_t r, r_sh;      // R mod q and its Shoup companion (entry x*R)
  uint32_t w1r, w1r_sh;  // psi^{N/2} * R mod q (entry-merged stage-0 twiddle)
  uint32_t qinv;         // q^{-1} mod 2^32 (subtractive Montgomery, mont_reduce64s)
};

// One row transform: source/destination row offsets (in units of N words,
// relative to the launch's base pointers), prime index, exit-constant slot.
struct RowJob {
  uint32_t src_off, dst_off;
  uint16_t prime, epi;
};

// Inverse-NTT exit constants (reference exit_x/exit_y with the fused BConv
// part-1 factor, ntt.cpp:76-84), Shoup pairs: {cx, cx', cy, cy'}.
using ExitConst = uint4;

__device__ __forceinline__ uint32_t shoup_mul(uint32_t a, uint32_t w, uint32_t wp, uint32_t q) {
  return a * w - __umulhi(a, wp) * q;  // [0, 2q) for any a < 2^32
}
__device__ __forceinline__ uint32_t sub_if(uint32_t x, uint32_t m) { return min(x, x - m); }
__device__ __forceinline__ uint32_t canon4(uint32_t x, uint32_t q, uint32_t q2) {
  return sub_if(sub_if(x, q2), q);  // [0, 4q) -> [0, q)
}
// unsigned Montgomery a*b*2^-32 for a*b < q*2^32 -> (0, 2q), subtractive
// form (qinv = q^-1 mod 2^32; see mont_reduce64s)
__device__ __forceinline__ uint32_t mont_mul(uint32_t a, uint32_t b, uint32_t q, uint32_t qinv) {
  const uint32_t lo = a * b;
  const uint32_t hi = __umulhi(a, b);
  return hi - __umulhi(lo * qinv, q) + q;
}
// acc + a*b with a, b < 2^32: one IMAD.WIDE.U32 (the compiler otherwise
// sometimes widens a register-promoted operand and emits a 64x32 multiply)
__device__ __forceinline__ uint64_t mac_wide(uint64_t acc, uint32_t a, uint32_t b) {
  uint64_t d;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(acc));
  return d;
}
// Subtractive Montgomery reduction of t < q*2^32 -> [0, 2q), congruent to
// t 2^-32: with m = lo q^-1, t - m q is divisible by 2^32 with no borrow out
// of the low word, so (t - m q) / 2^32 = hi - umulhi(m, q) in (-q, q) exactly
// (one instruction fewer than the additive form: no carry term)
__device__ __forceinline__ uint32_t mont_reduce64s(uint32_t lo, uint32_t hi, uint32_t q, uint32_t qinv) {
  return hi - __umulhi(lo * qinv, q) + q;
}
// Montgomery reduction of a 64-bit accumulator t < q*2^32 -> (0, 2q)
// (subtractive form, qinv = q^-1 mod 2^32)
__device__ __forceinline__ uint32_t mont_reduce64(uint64_t t, uint32_t q, uint32_t qinv) {
  return mont_reduce64s(static_cast<uint32_t>(t), static_cast<uint32_t>(t >> 32), q, qinv);
}

}  // namespace ck
