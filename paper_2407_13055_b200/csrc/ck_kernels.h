// Launch interface between the host runtime (ck_context.cu) and the kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "ck_common.cuh"

namespace ck {

struct NttLaunch {
  const RowJob* jobs = nullptr;  // device
  int njobs = 0;
  int batch = 1;
  const uint32_t* src = nullptr;
  uint64_t src_bs = 0;  // batch stride (words)
  uint32_t* dst = nullptr;
  uint64_t dst_bs = 0;
  const PrimeDev* primes = nullptr;
  const uint2* tw = nullptr;  // [prime][N] {w, w'}
  const ExitConst* exits = nullptr;
  int entry = 0;  // forward: multiply the input by R (reference entry merge)
};
void ntt_forward(int logn, const NttLaunch& a, cudaStream_t st);
void ntt_inverse(int logn, const NttLaunch& a, cudaStream_t st);
// N = 2^16 specialisation (ntt256.cu); tw2 / tw2i are the per-row permuted
// row-pass tables built by the host ([prime][256 rows][256] {w, w'}).
bool ntt256_forward(const NttLaunch& a, const uint2* tw2, cudaStream_t st);
bool ntt256_inverse(const NttLaunch& a, const uint2* tw2i, cudaStream_t st);
// N = 2^17 (256 columns x 512-point rows; row tables [prime][256][512])
bool ntt131k_forward(const NttLaunch& a, const uint2* tw2, cudaStream_t st);
bool ntt131k_inverse(const NttLaunch& a, const uint2* tw2i, cudaStream_t st);
// forward NTT whose row pass also applies the drop-and-divide combine
// (ckks.cpp:643-651): dst row (p, i) <- (v[p * prow + i] - NTT) * dinv[i]
struct CombineArgs {
  const uint32_t* v = nullptr;  // [B][npoly][prow][n]
  uint64_t v_bs = 0;
  uint32_t prow = 0, out_q = 1;
  const uint32_t* dinv = nullptr;  // [out_q] divisor^-1, Montgomery
  // HRot tail (ntt256_forward_hrot_tail): + add (the ciphertext's b rows,
  // [B][out_q][n], batch stride add_bs) on poly 0, results stored at
  // dest[x] of the rotation into out [B][2][out_q][n] (batch stride out_bs)
  const uint32_t* add = nullptr;
  uint64_t add_bs = 0;
  const uint32_t* dest = nullptr;
  uint32_t* out = nullptr;
  uint64_t out_bs = 0;
};
bool ntt256_forward_combine(const NttLaunch& a, const uint2* tw2, const CombineArgs& cb, cudaStream_t st);
// forward NTT of the ModDown conversion with the whole HRot tail fused into
// the row pass: combine, + b, automorphism (scattered stores within 32-blocks)
bool ntt256_forward_hrot_tail(const NttLaunch& a, const uint2* tw2, const CombineArgs& cb, cudaStream_t st);
// single-pass cluster/DSMEM variant (ntt_cluster.cu)
bool ntt_cluster_available();
void ntt_cluster_forward(const NttLaunch& a, const uint2* tw2, cudaStream_t st);
void ntt_cluster_inverse(const NttLaunch& a, const uint2* tw2i, cudaStream_t st);
// single pass: 0 fwd column, 1 fwd row (in place on dst), 2 inv row (src->dst), 3 inv column (in place on dst)
void ntt256_pass(int which, const NttLaunch& a, const uint2* tw2, cudaStream_t st);

// Fused INTT pass B (+part 1) -> BConv -> forward NTT pass 1 (ntt256.cu).
struct ConvMidGroup {
  uint32_t src_off;      // first source row (rows contiguous in src)
  uint32_t sc, dc;       // source / destination row counts
  uint32_t cmat_off;     // dc x sc constants ((P/P_j) mod q_i) R^2 mod q_i
  uint32_t map_off;      // into dst_row / dst_prime
  uint32_t src_map_off;  // into src_prime / src_exit
};
struct ConvMidLaunch {
  const ConvMidGroup* groups = nullptr;
  int ngroups = 0, batch = 1, max_sc = 1;
  const uint32_t* src = nullptr;  // INTT pass-A output
  uint64_t src_bs = 0;
  uint32_t* dst = nullptr;        // forward pass-1 output (row pass pending)
  uint64_t dst_bs = 0;
  const uint32_t* cmat = nullptr;
  const uint32_t* dst_row = nullptr;
  const uint16_t* dst_prime = nullptr;
  const uint16_t* src_prime = nullptr;
  const ExitConst* src_exit = nullptr;
  const PrimeDev* primes = nullptr;
  const uint2* fwd_tw = nullptr;
  const uint2* inv_tw = nullptr;
};
void conv_mid(const ConvMidLaunch& a, cudaStream_t st);

// One base-conversion group: src rows [src_off, src_off+sc) of the source
// buffer, dc destination rows dst_row[map_off + i] (row offsets in the
// destination buffer) with primes dst_prime[map_off + i], constants
// cmat[cmat_off + i*sc + j] = ((P/P_j) mod q_i) * R mod q_i.
struct BconvGroup {
  uint32_t src_off, sc, dc, cmat_off, map_off;
};
struct BconvLaunch {
  const BconvGroup* groups = nullptr;  // device
  int ngroups = 0;
  int batch = 1;
  int max_sc = 1;  // max source rows over groups (template dispatch)
  const uint32_t* src = nullptr;
  uint64_t src_bs = 0;
  uint32_t* dst = nullptr;
  uint64_t dst_bs = 0;
  const uint32_t* cmat = nullptr;
  const uint32_t* dst_row = nullptr;
  const uint16_t* dst_prime = nullptr;
  const PrimeDev* primes = nullptr;
  // optional (batch 1): source row r of the launch is the absolute address
  // src_rows[r] instead of src + r * n -- rows may live in PEER GPUs' memory
  // (limb-sharded exchange through peer-mapped loads, shard.cu)
  const uint64_t* src_rows = nullptr;
};
// fp64_mode 0: IMAD.WIDE dot products (k_bconv); 1-3: exact dot products on
// the FP64 pipe for all / every other / two of three destination rows
void bconv(int n, const BconvLaunch& a, cudaStream_t st, int fp64_mode = 0);
// tensor-core BConv (bconv_tc.cu): tcgen05 u8 split-word GEMM, TMEM accumulator
struct BconvTc {
  const unsigned char* btab = nullptr;  // per-group B tables (canonical UMMA layout)
  const uint32_t* boff = nullptr;       // byte offset of each group's table
  int max_npad = 0, max_dc = 0;
  int variant = 2;  // 1: k_bconv_tc, 2: k_bconv_tc2 (CK32_TC, read at context creation)
};
bool bconv_tc_supported(int n, int max_sc, int max_dc);
void bconv_tc(int n, const BconvLaunch& a, const BconvTc& t, cudaStream_t st);

// CKKS encode / decode (encode.cu, ckks.cpp:278-362)
constexpr int kMaxCrt = 16;  // decode: CRT lift over up to 16 primes (~460 bits)
struct CrtConst {  // CRT over the first c primes, multi-precision (32-bit limbs, little endian)
  int c = 0;
  uint32_t q[kMaxCrt] = {};
  uint32_t y[kMaxCrt] = {};                // (M / q_i)^-1 mod q_i
  uint32_t mi[kMaxCrt][kMaxCrt] = {};      // M / q_i (c limbs)
  uint32_t m[kMaxCrt + 1] = {};            // M (c limbs)
};
// reference fft_pow2 (ckks.cpp:63-87) on n = 2^logn points: src gathered in
// bit-reversed order, result in dst; tw = per-stage twiddles (stage len at
// offset len/2 - 1), built by the host with the reference's recurrence
void fft_pow2_dev(int logn, const double2* src, double2* dst, const double2* tw, cudaStream_t st);
void enc_scatter(int n, const double2* slots, int count, const uint32_t* jidx, double2* a, cudaStream_t st);
// scale = scale_mant * 2^scale_exp: the reference's long double scale (64-bit significand)
void enc_round(int n, const double2* a, const double2* twist, unsigned long long scale_mant, int scale_exp, int rows,
               const uint32_t* row_q, uint32_t* out, cudaStream_t st);
// the reference's NTT in its raw representation (ntt_raw.cu): per-prime
// constants of its NttPrimeTable (ntt.cpp:124-131) as signed int32
struct RawNttConst {
  int32_t r2 = 0, fwd1_r2 = 0, exit_x = 0, exit_y = 0;
};
void ntt_raw(int n, int logn, int rows, int inverse, int32_t* d, const uint16_t* gidx, const PrimeDev* primes,
             const RawNttConst* rc, const uint2* tw, const uint32_t* epi, cudaStream_t st);

// decode's scale as an exact rational num / den (32-bit limbs, little endian):
// the coefficient is then the correctly rounded double of v * den / num, as
// the reference's static_cast<double>(Rational(v) / scale) (ckks.cpp:353)
constexpr int kMaxRat = 8;
struct RatScale {
  uint32_t num[kMaxRat] = {}, den[kMaxRat] = {};
  int nnum = 0, nden = 0;  // 0 words: use inv_scale (power-of-two scales are exact either way)
};
void dec_crt(int n, const uint32_t* rows, const CrtConst* cc_dev, const double2* twist, double inv_scale, double2* a,
             cudaStream_t st, const RatScale& rs = RatScale{});
void dec_gather(int n, const double2* a, const uint32_t* jidx, double2* out, cudaStream_t st);

// tensor product of two ciphertexts (ckks.cpp:818-821): d0 = b b', d1 = b a' + a b', d2 = a a'
void tensor(int n, int level, int batch, const uint32_t* x, const uint32_t* y, uint64_t ct_bs, uint32_t* d01,
            uint64_t d01_bs, uint32_t* d2, uint64_t d2_bs, const PrimeDev* primes, cudaStream_t st);

// KeyMult (ckks.cpp:733-770) with the ModUp pass-through rows read from `d`
// and an optional fold v += P*d0/1 (ckks.cpp:831-842).
struct KeyMultLaunch {
  int level = 0, alpha = 0, L = 0, D = 0, batch = 1;
  const uint32_t* ext = nullptr;  // [B][D][level+alpha][n]
  uint64_t ext_bs = 0;
  const uint32_t* d = nullptr;    // [B][level][n] ModUp input (pass-through rows)
  uint64_t d_bs = 0;
  const uint32_t* evk = nullptr;  // [D][2][L+alpha][n]
  const uint32_t* fold = nullptr; // [B][2][level][n] (d0 then d1) or null
  uint64_t fold_bs = 0;
  const uint32_t* p_mont = nullptr;  // [level] P mod q_i in Montgomery form
  uint32_t* v = nullptr;          // [B][2][level+alpha][n]
  uint64_t v_bs = 0;
  const PrimeDev* primes = nullptr;
  // Optional (k_row_keymult8): the following drop-and-divide's INTT pass A
  // done in the epilogue.  Rows i >= src_lo are that switch's sources: they
  // are written row-transformed (inverse row pass, [0, 2q)) into ts
  // [B][2][ts_sc][n] (row ts_q + (i - level) for P rows, i - src_lo for the
  // ts_q tail Q rows) instead of into v.  inv_full: [prime][N] inverse tables.
  uint32_t* ts = nullptr;
  uint64_t ts_bs = 0;
  int src_lo = 1 << 30, ts_q = 0, ts_sc = 0;
  const uint2* inv_full = nullptr;
};
void key_mult(int n, const KeyMultLaunch& a, cudaStream_t st);
// N = 2^16: forward NTT row pass of every digit's extension row fused with
// KeyMult (ntt256.cu); `ext` holds the column-pass output.
// fwd_full: the per-prime forward tables [prime][N] {w, w'} (the
// 8-coefficient-per-thread variant reads its row twiddles from them)
void row_keymult(const KeyMultLaunch& a, const uint2* tw2, cudaStream_t st, const uint2* fwd_full = nullptr);
// whether row_keymult runs a kernel that honours KeyMultLaunch::ts (the fused INTT pass A)
bool row_keymult_fuses_intt(const KeyMultLaunch& a);

// drop-and-divide combine (ckks.cpp:643-651): o = (v - o) * div_inv (Montgomery)
void combine(int n, int rows, int npoly, int batch, const uint32_t* v, uint64_t v_ps, uint64_t v_bs, uint32_t* o,
             uint64_t o_ps, uint64_t o_bs, const uint32_t* div_inv_mont, const PrimeDev* primes, cudaStream_t st);

// HRot tail (ckks.cpp:875-882): combine both halves, c0 += b, permute.
void hrot_tail(int n, int level, int batch, const uint32_t* v, uint64_t v_bs, uint64_t v_ps, const uint32_t* o,
               uint64_t o_bs, uint64_t o_ps, const uint32_t* b, uint64_t b_bs, const uint32_t* div_inv_mont,
               const uint32_t* src_map, uint32_t* out, uint64_t out_bs, const PrimeDev* primes, cudaStream_t st,
               const uint32_t* dest_map = nullptr);  // dest_map: the scatter kernel (4 coefficients per thread)

// element-wise (poly.cpp:146-205): op 0 add, 1 sub, 2 mul (Montgomery).
// Row i uses prime row_prime[i] if given, else i % prime_mod (prime_mod = rows
// of one polynomial when several polynomials are stacked; <= 0 means `rows`).
void elementwise(int n, int rows, int batch, int op, const uint32_t* a, uint64_t a_bs, const uint32_t* b,
                 uint64_t b_bs, uint32_t* o, uint64_t o_bs, const uint16_t* row_prime, const PrimeDev* primes,
                 cudaStream_t st, int prime_mod = 0, const uint32_t* row_consts = nullptr);
// apply_automorphism for Galois element g (inverse gi), evaluation or
// coefficient domain (automorphism.cpp:76-100), out-of-place gather
void automorphism_galois(int n, int logn, int rows, uint32_t g, uint32_t gi, int coeff, const uint32_t* in,
                         uint32_t* out, const uint16_t* row_prime, const PrimeDev* primes, cudaStream_t st);
// decrypt / encrypt element-wise parts (ckks.cpp:497-553), see kernels.cu
void crypt(int n, int level, int batch, int op, const uint32_t* x, uint64_t x_bs, const uint32_t* y, const uint32_t* z,
           const uint32_t* w, const uint32_t* u, uint32_t* out, uint64_t out_bs, const PrimeDev* primes,
           cudaStream_t st);
void evk_digit(int n, int rows, const uint32_t* s_src, const uint32_t* s_dst, const uint32_t* a, const uint32_t* e,
               const uint32_t* gm, const uint16_t* row_prime, int square, const PrimeDev* primes, uint32_t* out,
               cudaStream_t st);
void reduce_coeffs(int n, int rows, const long long* c, const uint16_t* row_prime, const PrimeDev* primes,
                   uint32_t* out, cudaStream_t st);
// out[i][j] = in[i][src[j]] (automorphism.cpp:82-87)
void permute(int n, int rows, int batch, const uint32_t* in, uint64_t in_bs, uint32_t* out, uint64_t out_bs,
             const uint32_t* src_map, cudaStream_t st);
// acc = acc + x*y (Montgomery), addmul_rows (ckks.cpp:930-941)
void addmul(int n, int rows, int batch, uint32_t* acc, uint64_t acc_bs, const uint32_t* x, uint64_t x_bs,
            const uint32_t* y, uint64_t y_bs, const uint16_t* row_prime, const PrimeDev* primes, cudaStream_t st);
// permuted accumulate: acc[i][j] += x[i][src[j]] * y[i][j]
void addmul_permuted(int n, int rows, int batch, uint32_t* acc, uint64_t acc_bs, const uint32_t* x, uint64_t x_bs,
                     const uint32_t* y, uint64_t y_bs, const uint32_t* src_map, const uint16_t* row_prime,
                     const PrimeDev* primes, cudaStream_t st);

// Limb-sharded key switching (shard.cu): KeyMult over a shard's rows (any
// subset of Q_l + P) with per-row maps, and the drop-and-divide tail.
struct ShardKeyMultLaunch {
  int rows = 0, lq = 0, D = 0, erows = 0;
  const uint32_t* ext = nullptr;   // [D][rows][n]
  const uint32_t* d = nullptr;     // [lq][n] ModUp input (pass-through rows)
  const uint32_t* evk = nullptr;   // [D][2][erows][n] shard-local key rows
  const uint32_t* fold = nullptr;  // [2][lq][n] or null
  const int16_t* digit = nullptr;  // [rows] digit of the row (-1 for P rows)
  const uint16_t* prime = nullptr; // [rows] global prime index
  const uint16_t* erow = nullptr;  // [rows] row in the shard-local key
  const uint32_t* p_mont = nullptr;
  uint32_t* v = nullptr;           // [2][rows][n]
  const PrimeDev* primes = nullptr;
  const uint32_t* err = nullptr;   // peer exchange error word: when set, v is poisoned (0xFFFFFFFF)
};
void shard_key_mult(int n, const ShardKeyMultLaunch& a, cudaStream_t st);
struct ShardTailLaunch {
  const uint32_t* v = nullptr;  // poly stride v_ps, rows [0, rows) are the output rows
  uint64_t v_ps = 0;
  const uint32_t* o = nullptr;  // converted rows, poly stride o_ps
  uint64_t o_ps = 0;
  const uint32_t* dinv = nullptr;  // [rows] divisor^-1 (Montgomery)
  int prime_base = 0;              // global prime of row 0
  const uint32_t* add = nullptr;   // optional addend, poly stride add_ps
  uint64_t add_ps = 0;
  uint32_t add_mask = 0;           // bit c: add to poly c
  const uint32_t* src_map = nullptr;  // optional automorphism gather
  uint32_t* out = nullptr;
  uint64_t out_ps = 0;
  const PrimeDev* primes = nullptr;
  const uint32_t* err = nullptr;   // peer exchange error word: when set, out is poisoned (0xFFFFFFFF)
};
void shard_tail(int n, int rows, const ShardTailLaunch& a, cudaStream_t st);
// peer exchange handshake (shard.cu): signal stores the epoch (release,
// system scope) to the G flag words sig[0..G); wait spins (acquire, system
// scope) until flags[t] >= epoch for every t < G, or sets *err and gives up
// after `timeout_ns`.
// Epochs live in device memory (*epoch): advance increments it and selects
// the parity of the phase-1 INTT job table (jobs2 [2][njobs] -> jobs_cur);
// wait also selects the parity of the BConv row table (rows2 [2][nrows] ->
// rows_cur).  Nothing host-chosen per exchange: graph-capturable.
void shard_advance(uint32_t* epoch, const RowJob* jobs2, RowJob* jobs_cur, int njobs, cudaStream_t st);
void shard_signal(const uint64_t* sig, int G, const uint32_t* epoch, cudaStream_t st);
void shard_wait(const uint32_t* flags, int G, const uint32_t* epoch, uint32_t* err, uint64_t timeout_ns,
                const uint64_t* rows2, uint64_t* rows_cur, int nrows, cudaStream_t st);

}  // namespace ck
