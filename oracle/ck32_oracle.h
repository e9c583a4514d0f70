/* ORACLE TEST INFRASTRUCTURE ONLY — the CPU restatement used as the parity
 * checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.
 * Never linked into or called by the product path.
 *
 * Plain-C restatement of the reference's 32-bit RNS-CKKS hot path
 * (/root/reference/proj).  Every function cites the reference file:line it
 * follows.  Pinned against (1) the reference itself built from its own
 * sources (oracle/_ref/libckks32_ref*.so, oracle/Makefile) and (2) the golden
 * fixtures under tests/golden/ that the reference's serialisers wrote.
 *
 * Layout conventions (same as the reference's Polynomial, poly.hpp:74-119):
 * a polynomial is `rows x n` int32, row-major; rows [0, q_count) are the
 * Q-prefix, followed by P rows.  Evaluation keys are contiguous
 * [D][2 (b, a)][L + alpha][n] int32 over the full basis (ckks.hpp:79-84).
 */
#ifndef CK32_ORACLE_H
#define CK32_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cko_ctx cko_ctx;

/* mt19937_64 stream identical to std::mt19937_64 (random_poly, bench.cpp:121-129). */
typedef struct {
  uint64_t mt[312];
  int mti;
} cko_rng;
void cko_rng_seed(cko_rng* r, uint64_t seed);
uint64_t cko_rng_next(cko_rng* r);
/* rows x n residues rng() % q (row-major); gidx[i] = global prime index of row i. */
void cko_random_rows(const cko_ctx* c, cko_rng* r, uint32_t rows, const uint32_t* gidx, int32_t* out);

/* generate_basis (rns.cpp:63-117): writes l Q primes then alpha P primes. 0 on success. */
int cko_generate_basis(uint32_t n, uint32_t l, uint32_t alpha, uint32_t delta_bits, uint32_t* primes_out);
/* find_root_2n (modarith.cpp:30-40). */
uint32_t cko_find_root_2n(uint32_t q, uint32_t n);

cko_ctx* cko_create(uint32_t n, uint32_t l, uint32_t alpha, uint32_t delta_bits);
void cko_destroy(cko_ctx* c);
const uint32_t* cko_primes(const cko_ctx* c); /* l + alpha */
/* twiddles of prime gidx (ntt.cpp:100-135): fwd[n], inv[n], scalars {psi, fwd1_r2, exit_x, exit_y} */
void cko_twiddles(const cko_ctx* c, uint32_t gidx, uint32_t* fwd, uint32_t* inv, uint32_t* scalars);

/* Row transforms (forward_row_serial / inverse_row_serial, ntt.cpp:274-286). */
void cko_ntt_fwd_row(const cko_ctx* c, int32_t* row, uint32_t gidx);
void cko_intt_row(const cko_ctx* c, int32_t* row, uint32_t gidx, const uint32_t* epilogue_mont);

/* bconv_part2 (bconv.cpp:96-174) with make_bconv_table(src, dst) (bconv.cpp:13-46):
 * src is src_count x n canonical; dst rows written lazily in (-q, q). */
void cko_bconv(const cko_ctx* c, uint32_t src_count, const uint32_t* src_gidx, uint32_t dst_count,
               const uint32_t* dst_gidx, const int32_t* src, int32_t* dst);
/* part1 constants ((P/P_j)^-1 mod p_j, Montgomery), bconv.cpp:22-27 */
void cko_bconv_part1(const cko_ctx* c, uint32_t src_count, const uint32_t* src_gidx, uint32_t* part1_mont);

/* Mechanisms (ckks.cpp).  All inputs/outputs evaluation-domain Montgomery. */
/* mod_up (ckks.cpp:680-731): d is level x n; out is D(level) x (level+alpha) x n */
int cko_mod_up(const cko_ctx* c, uint32_t level, const int32_t* d, int32_t* out);
/* key_mult (ckks.cpp:733-770): hoist D x (level+alpha) x n; v0, v1 (level+alpha) x n */
int cko_key_mult(const cko_ctx* c, uint32_t level, const int32_t* hoist, const int32_t* evk, int32_t* v0,
                 int32_t* v1);
/* mod_down (ckks.cpp:772-776 via drop_and_divide :611-655): v (level+alpha) x n -> level x n */
int cko_mod_down(const cko_ctx* c, uint32_t level, const int32_t* v, int32_t* out);
int cko_key_switch(const cko_ctx* c, uint32_t level, const int32_t* d, const int32_t* evk, int32_t* c0,
                   int32_t* c1);
/* rescale (ckks.cpp:789-802): level -> level-2 */
int cko_rescale(const cko_ctx* c, uint32_t level, const int32_t* b, const int32_t* a, int32_t* ob, int32_t* oa);
/* hmult (ckks.cpp:804-865).  lazy=0: merged path, output level-2; lazy=1: output level. */
int cko_hmult(const cko_ctx* c, uint32_t level, const int32_t* xb, const int32_t* xa, const int32_t* yb,
              const int32_t* ya, const int32_t* evk, int lazy, int32_t* ob, int32_t* oa);
/* hrot (ckks.cpp:869-897) */
int cko_hrot(const cko_ctx* c, uint32_t level, const int32_t* b, const int32_t* a, int64_t r, const int32_t* evk,
             int32_t* ob, int32_t* oa);
/* rotation gather map src[] (automorphism.cpp:38-69) */
void cko_rotation_src_map(uint32_t n, int64_t r, uint32_t* src);
/* element-wise (poly.cpp:146-205, ckks.cpp:557-600) over `rows` Q-prefix rows */
void cko_ew_add(const cko_ctx* c, uint32_t rows, const int32_t* x, const int32_t* y, int32_t* o);
void cko_ew_mul(const cko_ctx* c, uint32_t rows, const int32_t* x, const int32_t* y, int32_t* o);
/* element-wise over rows at global primes gidx[]: op 0 add, 1 sub, 2 mul, 3 mul_const (consts[rows]) */
void cko_ew_rows(const cko_ctx* c, int op, uint32_t rows, const uint32_t* gidx, const int32_t* x, const int32_t* y,
                 const uint32_t* consts, int32_t* o);
/* apply_automorphism for Galois element g (inverse gi), evaluation or coefficient domain */
void cko_automorphism(const cko_ctx* c, uint32_t rows, uint64_t g, uint64_t gi, int coeff, const int32_t* in,
                      int32_t* o);
/* hoisted_rotate_accumulate (ckks.cpp:945-1012); pts are P-extended (level+alpha rows);
 * evks[i] ignored when rots[i]==0 */
int cko_hoisted_accumulate(const cko_ctx* c, uint32_t level, const int32_t* b, const int32_t* a, uint32_t count,
                           const int64_t* rots, const int32_t* const* pts, const int32_t* const* evks,
                           int32_t* ob, int32_t* oa);
/* canonical residues (correct, modarith.hpp:46-50) */
void cko_canonical(const cko_ctx* c, uint32_t rows, const uint32_t* gidx, const int32_t* in, uint32_t* out);

#ifdef __cplusplus
}
#endif
#endif
