/*
 * ck32_b200.h — the drop-in C ABI of the B200-native 32-bit RNS-CKKS hot path.
 *
 * Replaces the compute bodies behind the reference's C++ evaluator API
 * (/root/reference/proj/include/ckks32/ckks.hpp, ntt.hpp, bconv.hpp,
 * automorphism.hpp, poly.hpp).  Plain pointers and sizes only; no torch or
 * C++ types.  Every entry point cites the reference interface it replaces.
 *
 * Data model (mirrors Polynomial, poly.hpp:74-119):
 *   * a polynomial is `rows x n` uint32 residues, row-major, device memory;
 *     rows [0, level) are the Q-prefix, then (when present) the alpha P rows;
 *   * every value is CANONICAL in [0, q) — the reference's correct_lazy()
 *     view of its signed lazy residues (modarith.hpp:39-43);
 *   * evaluation-domain polynomials carry the Montgomery factor R = 2^32
 *     exactly as the reference's (mont flag = true);
 *   * a ciphertext at level l is `2 x l x n` (b rows then a rows,
 *     ckks.hpp:61-66); batches of B ciphertexts are contiguous;
 *   * an evaluation key is `D x 2 x (L+alpha) x n` (digit k: b_k rows then
 *     a_k rows over the full PQ basis, global row order, ckks.hpp:79-84),
 *     D = ceil(L / alpha).
 * All compute calls are asynchronous on the given CUDA stream (NULL = legacy
 * default stream).  A context is single-threaded like the reference's
 * CkksContext (its caches are unsynchronised, ckks.hpp:141-144); use one
 * context per host thread / device.
 *
 * Errors: every function returns a ck_status; ck_last_error() returns a
 * thread-local message.  CK_INVALID_ARGUMENT maps to the reference's
 * std::invalid_argument, CK_RUNTIME_ERROR to std::runtime_error.
 */
#ifndef CK32_B200_H
#define CK32_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CK_OK = 0,
  CK_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
  CK_RUNTIME_ERROR = 2,    /* std::runtime_error / BasisExhausted */
  CK_CUDA_ERROR = 3,
} ck_status;

typedef struct ck_context ck_context;
typedef void* ck_stream; /* cudaStream_t */

/* CkksParams subset that fixes the residue arithmetic (ckks.hpp:46-54). */
typedef struct {
  uint32_t n;          /* ring degree, power of two, 8 <= n <= 2^17 */
  uint32_t l;          /* number of Q primes (even) */
  uint32_t alpha;      /* number of P primes (= digit size) */
  uint32_t delta_bits; /* scale bits used by generate_basis */
  int32_t lazy_rescale;/* hmult: 0 merged ModDown+rescale, 1 lazy (ckks.cpp:822-863) */
} ck_params;

const char* ck_last_error(void);
const char* ck_version(void);

/* CkksContext::CkksContext (ckks.cpp:160-176): generate_basis (rns.cpp:63-117)
 * + build_twiddles (ntt.cpp:100-135) + P mod q (ckks.cpp:171-175), uploaded to
 * `device`.  primes == NULL generates the basis; otherwise l+alpha primes (Q then
 * P, e.g. from deserialize_basis, rns.cpp:189-216) are used verbatim. */
ck_status ck_context_create(const ck_params* params, const uint32_t* primes, int device, ck_context** out);
ck_status ck_context_destroy(ck_context* ctx);
/* generate_basis (rns.cpp:63-117) on the host only: l Q primes then alpha P
 * primes, identical to the reference's deterministic choice. */
ck_status ck_generate_basis(uint32_t n, uint32_t l, uint32_t alpha, uint32_t delta_bits, uint32_t* primes_out);
/* the parameters the context was created with (CkksParams subset) */
ck_status ck_context_params(const ck_context* ctx, ck_params* out);
/* RnsBasis q_primes then p_primes (rns.hpp:23-40) */
ck_status ck_context_primes(const ck_context* ctx, uint32_t* primes_out);
/* OpCounters (ckks.hpp:34-44): modup, moddown, ntt, intt, keymult, bconv, rescale */
ck_status ck_context_counters(const ck_context* ctx, uint64_t counters_out[7]);
ck_status ck_context_reset_counters(ck_context* ctx);

/* Device memory helpers for callers without their own allocator. */
ck_status ck_malloc(ck_context* ctx, size_t bytes, void** dptr);
ck_status ck_free(ck_context* ctx, void* dptr);
ck_status ck_memcpy_h2d(ck_context* ctx, void* dst, const void* src, size_t bytes, ck_stream stream);
ck_status ck_memcpy_d2h(ck_context* ctx, void* dst, const void* src, size_t bytes, ck_stream stream);
ck_status ck_memcpy_d2d(ck_context* ctx, void* dst, const void* src, size_t bytes, ck_stream stream);
ck_status ck_stream_sync(ck_context* ctx, ck_stream stream);
/* a non-blocking CUDA stream on the context's device, for callers without
 * the CUDA runtime headers (the C++ mirror's CkksContext::set_stream) */
ck_status ck_stream_create(ck_context* ctx, ck_stream* out);
ck_status ck_stream_destroy(ck_context* ctx, ck_stream stream);

/* ---- kernel-level entry points ------------------------------------------ */
/* ntt_forward (ntt.cpp:288-299) over `rows` rows in place; gidx[i] = global
 * prime index of row i (poly.hpp:103-106), host array.  Input coefficient
 * domain (plain), output evaluation domain (Montgomery). */
ck_status ck_ntt_forward(ck_context* ctx, uint32_t* rows_dev, uint32_t rows, const uint32_t* gidx,
                         ck_stream stream);
/* intt_inverse (ntt.cpp:301-312) / NttPlan::inverse_row with the fused part-1
 * epilogue (ntt.hpp:72-73): epilogue_mont[i] (host, canonical Montgomery form)
 * or NULL. */
ck_status ck_intt_inverse(ck_context* ctx, uint32_t* rows_dev, uint32_t rows, const uint32_t* gidx,
                          const uint32_t* epilogue_mont, ck_stream stream);
/* The reference's NTT / INTT in its RAW representation (ntt.cpp:15-96):
 * int32 rows as its Polynomial holds them (signed lazy values), its signed
 * Montgomery butterflies, (-2q, 2q) narrowing, forward entry merge and
 * tightened last stage, inverse exit constants (+ epilogue, canonical) --
 * butterfly for butterfly, so the rows equal the reference's
 * forward_row_serial / inverse_row_serial (and every NttPlan of it).  A
 * compatibility mode for callers that compare raw rows: one launch per
 * stage, untuned; the entry points above are the fast path. */
ck_status ck_ntt_forward_raw(ck_context* ctx, int32_t* rows_dev, uint32_t rows, const uint32_t* gidx,
                             ck_stream stream);
ck_status ck_intt_inverse_raw(ck_context* ctx, int32_t* rows_dev, uint32_t rows, const uint32_t* gidx,
                              const uint32_t* epilogue_mont, ck_stream stream);
/* make_bconv_table + bconv_part2 (bconv.cpp:13-46, 96-174): src is src_count
 * contiguous canonical rows (coefficient domain), dst dst_count rows. */
ck_status ck_bconv(ck_context* ctx, const uint32_t* src_dev, uint32_t src_count, const uint32_t* src_gidx,
                   uint32_t* dst_dev, uint32_t dst_count, const uint32_t* dst_gidx, ck_stream stream);
/* apply_automorphism, evaluation domain (automorphism.cpp:76-100), rotation r */
/* mod_switch (bconv.cpp:176-213): src rows (evaluation, Montgomery) over the
 * primes src_gidx -> dst rows over Q_[0, dst_q) then P_[0, dst_p)
 * (evaluation, Montgomery): INTT with the part-1 epilogue, BConv part 2,
 * forward NTT.  dst_dev holds dst_q + dst_p rows. */
ck_status ck_mod_switch(ck_context* ctx, const uint32_t* src_dev, uint32_t src_count, const uint32_t* src_gidx,
                        uint32_t* dst_dev, uint32_t dst_q, uint32_t dst_p, ck_stream stream);
ck_status ck_automorphism(ck_context* ctx, const uint32_t* in_dev, uint32_t* out_dev, uint32_t rows, int64_t r,
                          ck_stream stream);
/* apply_automorphism (automorphism.cpp:76-100) for any Galois element
 * (AutomorphismMap::rotation: 5^-r mod 2n; ::conjugation: 2n-1), evaluation
 * domain (bit-reversed column gather) or coefficient domain (coeff_domain = 1:
 * a(X) -> a(X^(g^-1)) with the negacyclic sign flips, canonical negation),
 * over a polynomial of q_rows Q-prefix rows then p_rows P rows. */
ck_status ck_automorphism_galois(ck_context* ctx, const uint32_t* in_dev, uint32_t* out_dev, uint32_t q_rows,
                                 uint32_t p_rows, uint64_t galois, int coeff_domain, ck_stream stream);
/* ew_add / ew_sub / ew_mul (op 0 / 1 / 2, poly.cpp:121-164) over a polynomial
 * of q_rows Q-prefix rows then p_rows P rows (P-extended operands as the
 * reference accepts them); out may alias a or b (ew_add_inplace /
 * ew_sub_inplace, poly.cpp:182-205).  Ops 4 / 5 / 6: the same in the
 * reference's raw representation -- int32 values in (-q, q) as its
 * Polynomial rows hold them, its narrow() and signed Montgomery reduction,
 * bit for bit (for callers that compare raw rows; every other entry point
 * takes and returns canonical residues). */
ck_status ck_ew_binary(ck_context* ctx, int op, const uint32_t* a, const uint32_t* b, uint32_t* out, uint32_t q_rows,
                       uint32_t p_rows, ck_stream stream);
/* ew_mul_const (poly.hpp:127-128): row i times consts_mont[i] (host array of
 * q_rows + p_rows canonical Montgomery constants); out may alias a. */
ck_status ck_ew_mul_const(ck_context* ctx, const uint32_t* a, const uint32_t* consts_mont, uint32_t* out,
                          uint32_t q_rows, uint32_t p_rows, ck_stream stream);
/* ew_mul_const in the reference's raw representation (as ops 4-6 above;
 * the constants are taken as the reference reads them, unreduced). */
ck_status ck_ew_mul_const_raw(ck_context* ctx, const uint32_t* a, const uint32_t* consts_mont, uint32_t* out,
                              uint32_t q_rows, uint32_t p_rows, ck_stream stream);
/* bconv_part2 (bconv.cpp:96-174) with the caller's BConvTable::c (centred
 * Montgomery constants, [dst_count][src_count], bconv.hpp:20-22) instead of
 * the library's own table: src canonical (coefficient domain) rows. */
ck_status ck_bconv_table(ck_context* ctx, const uint32_t* src_dev, uint32_t src_count, const uint32_t* src_gidx,
                         uint32_t* dst_dev, uint32_t dst_count, const uint32_t* dst_gidx, const int32_t* c_centered,
                         ck_stream stream);
/* ew_add / ew_sub / ew_mul over Q-prefix rows (poly.cpp:146-164) */
ck_status ck_ew_add(ck_context* ctx, const uint32_t* a, const uint32_t* b, uint32_t* out, uint32_t rows,
                    ck_stream stream);
ck_status ck_ew_sub(ck_context* ctx, const uint32_t* a, const uint32_t* b, uint32_t* out, uint32_t rows,
                    ck_stream stream);
ck_status ck_ew_mul(ck_context* ctx, const uint32_t* a, const uint32_t* b, uint32_t* out, uint32_t rows,
                    ck_stream stream);

/* ---- mechanisms (ckks.hpp:172-208) --------------------------------------- */
/* mod_up (ckks.cpp:680-731): d = level rows -> hoist D(level) x (level+alpha) rows.
 * Digit rows of each extension are the input rows (pass-through). */
ck_status ck_mod_up(ck_context* ctx, uint32_t level, const uint32_t* d, uint32_t* hoist, ck_stream stream);
/* key_mult (ckks.cpp:733-770): v = [v0; v1], each level+alpha rows. */
ck_status ck_key_mult(ck_context* ctx, uint32_t level, const uint32_t* hoist, const uint32_t* evk, uint32_t* v,
                      ck_stream stream);
/* mod_down (ckks.cpp:772-776): v (level+alpha rows) -> level rows. */
ck_status ck_mod_down(ck_context* ctx, uint32_t level, const uint32_t* v, uint32_t* out, ck_stream stream);
/* key_switch (ckks.cpp:778-787): d (level rows) -> [c0; c1] (2 x level rows). */
ck_status ck_key_switch(ck_context* ctx, uint32_t level, const uint32_t* d, const uint32_t* evk, uint32_t* out,
                        ck_stream stream);
/* rescale (ckks.cpp:789-802), batched: ct [B][2][level] -> out [B][2][level-2]. */
ck_status ck_rescale(ck_context* ctx, uint32_t level, uint32_t batch, const uint32_t* ct, uint32_t* out,
                     ck_stream stream);
/* hmult (ckks.cpp:804-865), batched over B ciphertext pairs sharing one relin key:
 * x, y [B][2][level] -> out [B][2][level-2] (merged) or [B][2][level] (lazy_rescale). */
ck_status ck_hmult(ck_context* ctx, uint32_t level, uint32_t batch, const uint32_t* x, const uint32_t* y,
                   const uint32_t* relin_evk, uint32_t* out, ck_stream stream);
/* hrot (ckks.cpp:890-897), batched over B ciphertexts sharing one rotation key. */
ck_status ck_hrot(ck_context* ctx, uint32_t level, uint32_t batch, const uint32_t* ct, int64_t r,
                  const uint32_t* rot_evk, uint32_t* out, ck_stream stream);
/* hadd / padd / pmult element-wise parts (ckks.cpp:557-600), batched:
 * ct [B][2][level]; pt [level] (shared by the batch). */
ck_status ck_hadd(ck_context* ctx, uint32_t level, uint32_t batch, const uint32_t* x, const uint32_t* y,
                  uint32_t* out, ck_stream stream);
ck_status ck_padd(ck_context* ctx, uint32_t level, uint32_t batch, const uint32_t* ct, const uint32_t* pt,
                  uint32_t* out, ck_stream stream);
ck_status ck_pmult(ck_context* ctx, uint32_t level, uint32_t batch, const uint32_t* ct, const uint32_t* pt,
                   uint32_t* out, ck_stream stream);
/* hoisted_rotations (ckks.cpp:899-925): one ModUp shared by `count` rotations;
 * out [count][2][level]; evks[i] ignored (identity) when rots[i] == 0. */
ck_status ck_hoisted_rotations(ck_context* ctx, uint32_t level, const uint32_t* ct, uint32_t count,
                               const int64_t* rots, const uint32_t* const* evks, uint32_t* out, ck_stream stream);
/* hoisted_rotate_accumulate (ckks.cpp:945-1012): sum_i pt_i * rot_{r_i}(ct) with
 * one ModUp and one ModDown; pts[i] are P-extended (level+alpha rows). */
ck_status ck_hoisted_rotate_accumulate(ck_context* ctx, uint32_t level, const uint32_t* ct, uint32_t count,
                                       const int64_t* rots, const uint32_t* const* pts,
                                       const uint32_t* const* evks, uint32_t* out, ck_stream stream);

/* encode (ckks.cpp:278-319): `count` <= n/2 complex slots (re, im doubles,
 * device memory) -> plaintext rows [level (+alpha if p_extend)][n] in the
 * evaluation domain, Montgomery form (canonical residues).  scale_log2 is
 * log2_rational(scale) (ckks.cpp:140-158); residues are bit-identical to the
 * reference at every scale (its powl / x87 long double rounding is replayed). */
ck_status ck_encode(ck_context* ctx, const double* slots_dev, uint32_t count, double scale_log2, uint32_t level,
                    int p_extend, uint32_t* out_dev, ck_stream stream);
/* decode (ckks.cpp:321-362): plaintext rows [level][n] (evaluation,
 * Montgomery) -> n/2 complex slots (re, im doubles, device memory).  The CRT
 * lift uses the minimal prime prefix covering scale_log2 + 40 bits (as the
 * reference), multi-precision, up to 16 primes.  Precision contract: the
 * reference rounds Rational(v) / scale to double once; here the centred lift
 * is rounded to double and multiplied by 2^-scale_log2: bit-identical to the
 * reference at power-of-two scales, within 2^-40 otherwise -- use
 * ck_decode_rational for bit-identical slots at every scale. */
ck_status ck_decode(ck_context* ctx, const uint32_t* pt_dev, uint32_t level, double scale_log2, double* slots_dev,
                    ck_stream stream);
/* decode with the scale as the exact rational num / den (32-bit limbs,
 * little endian, at most 8 words each, num > 0; scale_log2 as above selects
 * the prime prefix): every coefficient is the correctly rounded double of
 * Rational(v) / scale, as the reference computes it (ckks.cpp:353), so the
 * slots are bit-identical to the reference's decode at every scale
 * (tests/test_gpu_encode.py).  CK_ERR_ARG for more than 8 words or num = 0. */
ck_status ck_decode_rational(ck_context* ctx, const uint32_t* pt_dev, uint32_t level, double scale_log2,
                             const uint32_t* scale_num, uint32_t num_words, const uint32_t* scale_den,
                             uint32_t den_words, double* slots_dev, ck_stream stream);

/* Element-wise parts of decrypt / encrypt (ckks.cpp:497-553).  All operands
 * are evaluation-domain Montgomery rows (canonical); the randomness of
 * encrypt is supplied by the caller (the reference samples it on the host with
 * mt19937_64, ckks.cpp:390-430; ck_sample_* below replay that stream) and
 * turned into evaluation form with ck_coeffs_to_eval.
 *   decrypt     out [B][level]   = ct.b + ct.a * s        (ct [B][2][level], s [level])
 *   encrypt_sk  out [2][level]   = (m + e - a s, a)
 *   encrypt_pk  out [2][level]   = (v pk.b + e0 + m, v pk.a + e1)   (pk [2][level]) */
ck_status ck_decrypt(ck_context* ctx, uint32_t level, uint32_t batch, const uint32_t* ct, const uint32_t* s,
                     uint32_t* out, ck_stream stream);
ck_status ck_encrypt_sk(ck_context* ctx, uint32_t level, const uint32_t* pt, const uint32_t* a, const uint32_t* e,
                        const uint32_t* s, uint32_t* out, ck_stream stream);
ck_status ck_encrypt_pk(ck_context* ctx, uint32_t level, const uint32_t* pt, const uint32_t* v, const uint32_t* e0,
                        const uint32_t* e1, const uint32_t* pk, uint32_t* out, ck_stream stream);
/* One evaluation-key digit (evk_gen, ckks.cpp:459-474) over the full L+alpha
 * rows: out_b = e + s_src * g - a * s_dst (s_src squared first when
 * square_src: relinearisation).  g_mont: L+alpha host words, the digit's
 * gadget factor P * dhat * (dhat^-1 mod d_k) reduced mod every prime, in
 * Montgomery form; a, e and the secrets are evaluation-domain Montgomery rows. */
ck_status ck_evk_digit(ck_context* ctx, const uint32_t* s_src, const uint32_t* s_dst, const uint32_t* a,
                       const uint32_t* e, const uint32_t* g_mont, int square_src, uint32_t* out_b, ck_stream stream);
/* coeffs_to_eval (ckks.cpp:366-380): n signed int64 coefficients (device) ->
 * rows [level + p_rows][n], each reduced mod its prime then forward NTT. */
ck_status ck_coeffs_to_eval(ck_context* ctx, const int64_t* coeffs, uint32_t level, uint32_t p_rows, uint32_t* out,
                            ck_stream stream);

/* ---- wire formats, byte-compatible with the reference --
 * Blobs live in host memory; rows move directly between device memory and the
 * blob (device rows are canonical, exactly what the reference writes).
 * Writers: out == NULL only reports the length in *len; otherwise cap must
 * cover it.  Readers validate like the reference (magic, version, ring degree,
 * basis hash, truncation: CK_RUNTIME_ERROR for polynomial / basis blobs,
 * CK_INVALID_ARGUMENT for ciphertext / key headers) and additionally reject
 * residues >= q (the device only holds canonical values).  A ciphertext's
 * scale is its reduced Rational as two big-endian magnitudes (export_bits
 * order), numerator then denominator. */
/* serialize_basis / deserialize_basis (rns.cpp:188-216) */
ck_status ck_serialize_basis(const ck_context* ctx, uint8_t* out, size_t cap, size_t* len);
ck_status ck_deserialize_basis(const uint8_t* in, size_t len, ck_params* params, uint32_t* primes, uint32_t cap);
/* serialize_poly / deserialize_poly (poly.cpp:297-352); meta = {q_count, p_count, domain, mont} */
ck_status ck_serialize_poly(ck_context* ctx, const uint32_t* rows_dev, uint32_t q_count, uint32_t p_count, int domain,
                            int mont, uint8_t* out, size_t cap, size_t* len, ck_stream stream);
ck_status ck_deserialize_poly(ck_context* ctx, const uint8_t* in, size_t len, uint32_t* rows_dev, uint32_t cap_rows,
                              uint32_t meta[4], ck_stream stream);
/* serialize_ciphertext / deserialize_ciphertext (ckks.cpp:1092-1121): ct [2][level] */
ck_status ck_serialize_ciphertext(ck_context* ctx, const uint32_t* ct_dev, uint32_t level, int pending_rescale,
                                  const uint8_t* scale_num, size_t num_len, const uint8_t* scale_den, size_t den_len,
                                  uint8_t* out, size_t cap, size_t* len, ck_stream stream);
ck_status ck_deserialize_ciphertext(ck_context* ctx, const uint8_t* in, size_t len, uint32_t* ct_dev,
                                    uint32_t cap_level, uint32_t* level, int* pending_rescale, uint8_t* scale_num,
                                    size_t num_cap, size_t* num_len, uint8_t* scale_den, size_t den_cap,
                                    size_t* den_len, ck_stream stream);
/* serialize_evk / deserialize_evk (ckks.cpp:1123-1154): evk [D][2][L+alpha] */
ck_status ck_serialize_evk(ck_context* ctx, const uint32_t* evk_dev, uint32_t digits, int kind, int64_t rotation,
                           uint8_t* out, size_t cap, size_t* len, ck_stream stream);
ck_status ck_deserialize_evk(ck_context* ctx, const uint8_t* in, size_t len, uint32_t* evk_dev, uint32_t cap_digits,
                             int* kind, int64_t* rotation, uint32_t* digits, ck_stream stream);

/* Number of this library's kernel launches issued since context creation
 * (evidence for bench.py's gpu_launches). */
uint64_t ck_launch_count(const ck_context* ctx);

/* Per-kernel-class CUDA-event timing (no reference counterpart; the
 * reference times whole mechanisms with steady_clock, bench.cpp:105-110).
 * ck_profile(ctx, 1) clears and starts recording an event pair around every
 * launch group; ck_profile_read synchronises and returns one entry per class
 * (ntt_fwd, ntt_inv, bconv, key_mult, tensor, combine, hrot_tail) with the
 * summed device time and the algorithmic bytes of SURVEY.md §8(d). */
typedef struct {
  char name[16];
  uint64_t groups;   /* event-bracketed launch groups */
  uint64_t launches; /* kernel launches inside them */
  double ms;         /* summed event time */
  double bytes;      /* summed algorithmic bytes (read + write once) */
} ck_prof_stat;
ck_status ck_profile(ck_context* ctx, int enable);
ck_status ck_profile_read(ck_context* ctx, ck_prof_stat* out, uint32_t max_classes, uint32_t* count);

/* ---- limb-sharded key switching (BASELINE config 4) -------------------------
 * The reference runs one ciphertext on one host (key_switch, ckks.cpp:778-787;
 * mod_up ckks.cpp:680-731; drop_and_divide ckks.cpp:611-655); these entry
 * points split the same computation over `world` devices by RNS limb.  Rank s
 * owns Q primes [q_lo, q_hi) and P primes L + [p_lo, p_hi) (balanced blocks).
 * A shard-local polynomial at level l holds the owned Q rows below l (in
 * order), then — when it carries them — the owned P rows.  A shard-local key
 * is D x 2 x ((q_hi-q_lo) + (p_hi-p_lo)) rows: owned Q rows of every level,
 * then owned P rows.  Every *_begin leaves INTT'd source rows in `send`; the
 * host all-gathers the send buffers of all ranks (rank-major, equal sizes) and
 * passes the result as `recv` to the matching second phase:
 *   ModUp:   send [q_max][n]            recv [world][q_max][n]
 *   switch:  send [2][s_max][n]         recv [world][2][s_max][n]
 *            s_max = p_max (kind 0), 2 (kind 1), p_max + 2 (kind 2)
 * Outputs are bit-identical to the single-device mechanisms restricted to the
 * owned rows. */
typedef struct ck_shard ck_shard;
ck_status ck_shard_create(ck_context* ctx, uint32_t world, uint32_t rank, ck_shard** out);
ck_status ck_shard_destroy(ck_shard* sh);
/* out = {q_lo, q_hi, p_lo, p_hi, owned Q rows below level, q_max, p_max, world} */
ck_status ck_shard_layout(const ck_shard* sh, uint32_t level, uint32_t out[8]);
/* ModUp phase 1 (ckks.cpp:690-697): INTT + part 1 of the owned rows of d. */
ck_status ck_shard_modup_begin(ck_shard* sh, uint32_t level, const uint32_t* d, uint32_t* send, ck_stream stream);
/* ModUp phase 2 + KeyMult (ckks.cpp:698-770): BConv of every digit to the owned
 * rows, NTT, multiply-accumulate with the shard-local key; optional fold
 * v += P * (d0, d1) on the owned Q rows (fold = [2][owned Q rows], ckks.cpp:831-842).
 * v = [2][owned Q rows + owned P rows]. */
ck_status ck_shard_modup_keymult(ck_shard* sh, uint32_t level, const uint32_t* recv, const uint32_t* d,
                                 const uint32_t* evk, const uint32_t* fold, uint32_t* v, ck_stream stream);
/* drop_and_divide phase 1: INTT + part 1 of the owned source rows of v (two
 * polynomials).  kind 0 = mod_down (v carries P rows), 1 = rescale (v is a
 * shard-local ciphertext), 2 = merged ModDown + rescale (ckks.cpp:206-258). */
ck_status ck_shard_switch_begin(ck_shard* sh, int kind, uint32_t level, const uint32_t* v, uint32_t* send,
                                ck_stream stream);
/* drop_and_divide phase 2: BConv to the owned output rows, NTT, combine
 * (v - conv) * divisor^-1; then out_c += addend_c for bit c of add_mask (addend
 * [2][owned output rows]); then, if rotate, the automorphism of rotation r on
 * both polynomials (hrot tail, ckks.cpp:875-882). out = [2][owned output rows]. */
ck_status ck_shard_switch_end(ck_shard* sh, int kind, uint32_t level, const uint32_t* recv, const uint32_t* v,
                              const uint32_t* addend, uint32_t add_mask, int32_t rotate, int64_t r, uint32_t* out,
                              ck_stream stream);
/* The reference's randomness, host side as in the reference: a
 * std::mt19937_64(seed) consumed exactly as ckks.cpp does, so a seed
 * reproduces the reference's keys and ciphertexts bit for bit.
 *   ck_sample_gaussian   sample_gaussian x n   (ckks.cpp:33-47)
 *   ck_sample_ternary    ternary_coeffs        (ckks.cpp:51-60)
 *   ck_sample_uniform    uniform_eval residues (ckks.cpp:383-395), out [rows][n] host
 *   ck_rng_draws         raw 64-bit outputs (e.g. for std::uniform_real_distribution slots) */
typedef struct ck_rng ck_rng;
ck_status ck_rng_create(uint64_t seed, ck_rng** out);
ck_status ck_rng_destroy(ck_rng* rng);
ck_status ck_rng_draws(ck_rng* rng, uint64_t count, uint64_t* out);
ck_status ck_sample_gaussian(ck_rng* rng, uint32_t n, double sigma, int64_t* out);
ck_status ck_sample_ternary(ck_rng* rng, uint32_t n, uint32_t h, int64_t* out);
ck_status ck_sample_uniform(ck_rng* rng, const uint32_t* q, uint32_t rows, uint32_t n, uint32_t* out);

/* Peer exchange ("peer-mapped loads inside BConv"), replacing
 * the host all-gather: every rank allocates ONE exchange buffer, the ranks map
 * each other's buffers (CUDA IPC across processes: ck_ipc_*; plain pointers
 * for shards of one process) and pass all bases in rank order to
 * ck_shard_set_peers.  After that, send == NULL in *_begin and recv == NULL in
 * the second phases select the peer path: phase 1 INTTs into the rank's own
 * buffer and publishes an epoch flag to every peer (system-scope release);
 * phase 2 waits for all peers' flags (bounded: ck_shard_set_timeout, default
 * 10 s; a timeout sets the error word read by ck_shard_peer_error instead of
 * hanging) and its BConv loads the source rows straight from the peers'
 * buffers.  Every rank must issue every phase in the same order (as with a
 * collective) and on ONE stream per rank: the double-buffer reuse argument
 * (a buffer is rewritten only after all peers have finished reading it)
 * relies on each rank's phases being stream-ordered.  After a timeout the
 * phase-2 outputs are poisoned (0xFFFFFFFF, never a canonical residue) and
 * ck_shard_peer_error reports it; ck_shard_set_peers clears the flag and
 * error words (callers barrier after it).  The epochs and buffer parities
 * are kept in device memory, so a sequence of phases captured in a CUDA graph
 * on every rank replays correctly. */
ck_status ck_shard_exchange_buffer(ck_shard* sh, void** base, uint64_t* bytes);
ck_status ck_shard_set_peers(ck_shard* sh, const uint64_t* bases, uint32_t world);
ck_status ck_shard_set_timeout(ck_shard* sh, uint64_t timeout_ns);
ck_status ck_shard_peer_error(ck_shard* sh, uint32_t* err);
/* CUDA IPC of an exchange buffer (64-byte cudaIpcMemHandle_t) */
ck_status ck_ipc_get_handle(const void* base, unsigned char handle[64]);
ck_status ck_ipc_open_handle(const unsigned char handle[64], void** base);
ck_status ck_ipc_close(void* base);
/* hmult tensor (ckks.cpp:818-821) on the owned rows: d01 [2][lq], d2 [lq]. */
ck_status ck_shard_tensor(ck_shard* sh, uint32_t level, const uint32_t* x, const uint32_t* y, uint32_t* d01,
                          uint32_t* d2, ck_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* CK32_B200_H */
