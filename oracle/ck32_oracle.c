/* ORACLE TEST INFRASTRUCTURE ONLY — see ck32_oracle.h.  Plain-C restatement
 * of the reference hot path; each function cites the reference file:line it
 * follows (paths relative to /root/reference/proj). */
#include "ck32_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ rng -- */
#define MT_NN 312
#define MT_MM 156
void cko_rng_seed(cko_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_NN; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->mti = MT_NN;
}
uint64_t cko_rng_next(cko_rng* r) {
  static const uint64_t mag01[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (r->mti >= MT_NN) {
    int i;
    uint64_t x;
    for (i = 0; i < MT_NN - MT_MM; ++i) {
      x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + MT_MM] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    }
    for (; i < MT_NN - 1; ++i) {
      x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + (MT_MM - MT_NN)] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    }
    x = (r->mt[MT_NN - 1] & UM) | (r->mt[0] & LM);
    r->mt[MT_NN - 1] = r->mt[MT_MM - 1] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    r->mti = 0;
  }
  uint64_t x = r->mt[r->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* ------------------------------------------------------------- modarith -- */
typedef struct {
  uint32_t q;
  int32_t m;   /* q^-1 mod 2^32, signed (modarith.cpp:47-49) */
  uint32_t r2; /* 2^64 mod q (modarith.cpp:50) */
} ckp;

static uint64_t pow_mod(uint64_t b, uint64_t e, uint64_t m) { /* modarith.hpp:63-72 */
  unsigned __int128 acc = 1 % m;
  b %= m;
  while (e) {
    if (e & 1) acc = acc * b % m;
    b = (uint64_t)((unsigned __int128)b * b % m);
    e >>= 1;
  }
  return (uint64_t)acc;
}
static uint64_t inv_mod(uint64_t a, uint64_t p) { return pow_mod(a, p - 2, p); } /* modarith.hpp:74 */

static ckp make_prime(uint32_t q) { /* make_prime_context, modarith.cpp:42-54 */
  ckp c;
  uint32_t inv = q;
  for (int i = 0; i < 5; ++i) inv *= 2u - q * inv;
  c.q = q;
  c.m = (int32_t)inv;
  c.r2 = (uint32_t)((((unsigned __int128)1) << 64) % q);
  return c;
}

static inline int32_t mont_reduce(int64_t a, const ckp* c) { /* modarith.hpp:21-30 */
  int32_t a_hi = (int32_t)(a >> 32);
  uint32_t a_lo = (uint32_t)a;
  int32_t t = (int32_t)(a_lo * (uint32_t)c->m);
  int32_t u = (int32_t)(((int64_t)t * (int32_t)c->q) >> 32);
  return a_hi - u;
}
static inline int32_t mont_mul(int32_t a, int32_t b, const ckp* c) { /* modarith.hpp:34-36 */
  return mont_reduce((int64_t)a * b, c);
}
static inline uint32_t correct_lazy(int32_t a, uint32_t q) { /* modarith.hpp:39-43 */
  return a < 0 ? (uint32_t)(a + (int32_t)q) : (uint32_t)a;
}
static inline uint32_t correct64(int64_t a, uint32_t q) { /* modarith.hpp:46-50 */
  int64_t r = a % (int64_t)q;
  if (r < 0) r += q;
  return (uint32_t)r;
}
static inline uint32_t to_mont(uint32_t a, const ckp* c) { /* modarith.hpp:54-56 */
  return correct_lazy(mont_reduce((int64_t)a * c->r2, c), c->q);
}
/* narrow of poly.cpp:127-131 (one +-q step) */
static inline int32_t narrow1(int64_t v, int32_t q) {
  if (v >= q) v -= q;
  else if (v <= -q) v += q;
  return (int32_t)v;
}
/* narrow of ckks.cpp:25-32: (-4q, 4q) -> (-q, q) */
static inline int32_t narrow4(int32_t v, int32_t q) {
  const int32_t two_q = q << 1;
  if (v >= two_q) v -= two_q;
  if (v <= -two_q) v += two_q;
  if (v >= q) v -= q;
  if (v <= -q) v += q;
  return v;
}

static int is_prime_u64(uint64_t v) { /* modarith.cpp:7-28 */
  static const uint64_t bases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (v < 2) return 0;
  for (int i = 0; i < 12; ++i)
    if (v % bases[i] == 0) return v == bases[i];
  uint64_t d = v - 1;
  int s = 0;
  while ((d & 1) == 0) d >>= 1, ++s;
  for (int i = 0; i < 12; ++i) {
    uint64_t x = pow_mod(bases[i], d, v);
    if (x == 1 || x == v - 1) continue;
    int composite = 1;
    for (int k = 1; k < s; ++k) {
      x = (uint64_t)((unsigned __int128)x * x % v);
      if (x == v - 1) {
        composite = 0;
        break;
      }
    }
    if (composite) return 0;
  }
  return 1;
}

uint32_t cko_find_root_2n(uint32_t q, uint32_t n) { /* modarith.cpp:30-40 */
  const uint64_t order = 2ull * n;
  if ((q - 1) % order != 0) return 0;
  const uint64_t cof = (q - 1) / order;
  for (uint64_t g = 2; g < q; ++g) {
    uint64_t cand = pow_mod(g, cof, q);
    if (pow_mod(cand, n, q) == q - 1) return (uint32_t)cand;
  }
  return 0;
}

static uint32_t bit_reverse(uint32_t x, uint32_t bits) { /* ntt.hpp:24-28 */
  uint32_t r = 0;
  for (uint32_t i = 0; i < bits; ++i) r |= ((x >> i) & 1u) << (bits - 1 - i);
  return r;
}

/* ---------------------------------------------------------------- basis -- */
/* scan_down, rns.cpp:10-20 */
static size_t scan_down(uint64_t top, uint32_t two_n, size_t count, uint64_t stop_at, uint32_t* out, size_t cap) {
  size_t got = 0;
  uint64_t k = (top - 1) / two_n * two_n + 1;
  if (k >= top) k -= two_n;
  for (; k > two_n && k > stop_at && got < count; k -= two_n)
    if (is_prime_u64(k)) {
      if (got >= cap) return got;
      out[got++] = (uint32_t)k;
    }
  return got;
}

static int cmp_u32(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : x > y;
}

typedef struct {
  uint32_t a, b;
} dgroup;
static double dg_log2(const dgroup* g) { return log2((double)g->a) + log2((double)g->b); }

int cko_generate_basis(uint32_t n, uint32_t l, uint32_t alpha, uint32_t db, uint32_t* primes_out) {
  /* rns.cpp:63-117 */
  if (n == 0 || (n & (n - 1)) != 0) return -1;
  if (l == 0 || l % 2 != 0) return -1;
  const uint64_t two_n = 2ull * n;
  uint64_t cap = 1ull << 29;
  const uint64_t den = (alpha + 2 > 3) ? alpha + 2 : 3;
  if ((1ull << 32) / den < cap) cap = (1ull << 32) / den;
  const uint64_t slots = cap > two_n ? (cap - two_n) / two_n : 0;
  if (slots < l + alpha) return -2;
  uint32_t* p_list = (uint32_t*)malloc(sizeof(uint32_t) * (alpha + 1));
  size_t np = scan_down(cap, (uint32_t)two_n, alpha, 0, p_list, alpha + 1);
  if (np < alpha) {
    free(p_list);
    return -2;
  }
  const uint64_t p_min = alpha ? p_list[np - 1] : cap;
  uint64_t q_top = (uint64_t)sqrt(ldexp(1.0, (int)db + 1));
  if (cap < q_top) q_top = cap;
  if (p_min < q_top) q_top = p_min;
  size_t qcap = (size_t)(slots + l + 16);
  uint32_t* cands = (uint32_t*)malloc(sizeof(uint32_t) * qcap);
  size_t nc = scan_down(q_top, (uint32_t)two_n, l, 0, cands, qcap);
  if (nc < l) nc += scan_down(p_min, (uint32_t)two_n, (size_t)-1, q_top - 1, cands + nc, qcap - nc);
  qsort(cands, nc, sizeof(uint32_t), cmp_u32);
  size_t u = 0;
  for (size_t i = 0; i < nc; ++i)
    if (u == 0 || cands[i] != cands[u - 1]) cands[u++] = cands[i];
  nc = u;
  if (nc < l) {
    free(p_list);
    free(cands);
    return -2;
  }
  /* pair_delta_groups, rns.cpp:31-59 */
  const size_t need = l / 2;
  dgroup* groups = (dgroup*)malloc(sizeof(dgroup) * need);
  size_t ng = 0;
  double lo = ldexp(1.0, (int)db - 1), hi = ldexp(1.0, (int)db + 1);
  for (int widen = 0; ng < need && widen <= 12; ++widen) {
    size_t i = 0;
    while (i < nc && ng < need) {
      const double a = (double)cands[i];
      size_t j = nc - 1;
      while (j > i && a * (double)cands[j] >= hi) --j;
      if (j > i && a * (double)cands[j] >= lo) {
        uint32_t x = cands[i], y = cands[j];
        groups[ng].a = x > y ? x : y;
        groups[ng].b = x > y ? y : x;
        ++ng;
        memmove(cands + j, cands + j + 1, sizeof(uint32_t) * (nc - j - 1));
        --nc;
        memmove(cands + i, cands + i + 1, sizeof(uint32_t) * (nc - i - 1));
        --nc;
      } else {
        ++i;
      }
    }
    lo /= 2;
    hi *= 2;
  }
  if (ng < need) {
    free(p_list);
    free(cands);
    free(groups);
    return -2;
  }
  /* std::stable_sort by |log2(product) - db| descending (rns.cpp:100-104):
   * insertion sort is stable */
  for (size_t i = 1; i < ng; ++i) {
    dgroup g = groups[i];
    double kg = fabs(dg_log2(&g) - db);
    size_t j = i;
    while (j > 0 && fabs(dg_log2(&groups[j - 1]) - db) < kg) {
      groups[j] = groups[j - 1];
      --j;
    }
    groups[j] = g;
  }
  for (size_t i = 0; i < ng; ++i) {
    primes_out[2 * i] = groups[i].a;
    primes_out[2 * i + 1] = groups[i].b;
  }
  for (uint32_t i = 0; i < alpha; ++i) primes_out[l + i] = p_list[i];
  free(p_list);
  free(cands);
  free(groups);
  return 0;
}

/* -------------------------------------------------------------- context -- */
typedef struct {
  ckp ctx;
  uint32_t psi;
  uint32_t* fwd; /* psi^brev(i) * R */
  uint32_t* inv; /* psi^-brev(i) * R */
  uint32_t fwd1_r2, exit_x, exit_y;
} cko_table;

struct cko_ctx {
  uint32_t n, logn, l, alpha, db;
  uint32_t* primes; /* l + alpha */
  ckp* pc;
  cko_table* tw;
  uint32_t* p_mont; /* P mod q_i, Montgomery (ckks.cpp:171-175) */
};

static void build_table(cko_table* T, uint32_t q, uint32_t n, uint32_t logn) { /* ntt.cpp:100-135 */
  T->ctx = make_prime(q);
  T->psi = cko_find_root_2n(q, n);
  const uint64_t psi_inv = inv_mod(T->psi, q);
  uint32_t* pw = (uint32_t*)malloc(sizeof(uint32_t) * n);
  uint32_t* pwi = (uint32_t*)malloc(sizeof(uint32_t) * n);
  pw[0] = pwi[0] = 1;
  for (uint32_t k = 1; k < n; ++k) {
    pw[k] = (uint32_t)((uint64_t)pw[k - 1] * T->psi % q);
    pwi[k] = (uint32_t)((uint64_t)pwi[k - 1] * psi_inv % q);
  }
  T->fwd = (uint32_t*)calloc(n, sizeof(uint32_t));
  T->inv = (uint32_t*)calloc(n, sizeof(uint32_t));
  for (uint32_t i = 1; i < n; ++i) {
    const uint32_t e = bit_reverse(i, logn);
    T->fwd[i] = to_mont(pw[e], &T->ctx);
    T->inv[i] = to_mont(pwi[e], &T->ctx);
  }
  T->fwd1_r2 = to_mont(to_mont(pw[n / 2], &T->ctx), &T->ctx);
  const uint64_t n_inv = inv_mod(n % q, q);
  T->exit_x = (uint32_t)n_inv;
  T->exit_y = (uint32_t)(pwi[n / 2] * n_inv % q);
  free(pw);
  free(pwi);
}

cko_ctx* cko_create(uint32_t n, uint32_t l, uint32_t alpha, uint32_t db) {
  cko_ctx* c = (cko_ctx*)calloc(1, sizeof(cko_ctx));
  c->n = n;
  c->l = l;
  c->alpha = alpha;
  c->db = db;
  while ((1u << c->logn) < n) ++c->logn;
  c->primes = (uint32_t*)malloc(sizeof(uint32_t) * (l + alpha));
  if (cko_generate_basis(n, l, alpha, db, c->primes) != 0) {
    free(c->primes);
    free(c);
    return NULL;
  }
  c->pc = (ckp*)malloc(sizeof(ckp) * (l + alpha));
  c->tw = (cko_table*)calloc(l + alpha, sizeof(cko_table));
#pragma omp parallel for schedule(dynamic)
  for (int i = 0; i < (int)(l + alpha); ++i) build_table(&c->tw[i], c->primes[i], n, c->logn);
  for (uint32_t i = 0; i < l + alpha; ++i) c->pc[i] = c->tw[i].ctx;
  c->p_mont = (uint32_t*)malloc(sizeof(uint32_t) * l);
  for (uint32_t i = 0; i < l; ++i) {
    uint64_t pm = 1 % c->primes[i];
    for (uint32_t j = 0; j < alpha; ++j) pm = pm * (c->primes[l + j] % c->primes[i]) % c->primes[i];
    c->p_mont[i] = to_mont((uint32_t)pm, &c->pc[i]);
  }
  return c;
}

void cko_destroy(cko_ctx* c) {
  if (!c) return;
  for (uint32_t i = 0; i < c->l + c->alpha; ++i) {
    free(c->tw[i].fwd);
    free(c->tw[i].inv);
  }
  free(c->tw);
  free(c->pc);
  free(c->primes);
  free(c->p_mont);
  free(c);
}

const uint32_t* cko_primes(const cko_ctx* c) { return c->primes; }

void cko_twiddles(const cko_ctx* c, uint32_t g, uint32_t* fwd, uint32_t* inv, uint32_t* s) {
  memcpy(fwd, c->tw[g].fwd, sizeof(uint32_t) * c->n);
  memcpy(inv, c->tw[g].inv, sizeof(uint32_t) * c->n);
  s[0] = c->tw[g].psi;
  s[1] = c->tw[g].fwd1_r2;
  s[2] = c->tw[g].exit_x;
  s[3] = c->tw[g].exit_y;
}

void cko_random_rows(const cko_ctx* c, cko_rng* r, uint32_t rows, const uint32_t* gidx, int32_t* out) {
  for (uint32_t i = 0; i < rows; ++i) { /* bench.cpp:121-129 */
    const uint32_t q = c->primes[gidx[i]];
    for (uint32_t k = 0; k < c->n; ++k) out[(size_t)i * c->n + k] = (int32_t)(cko_rng_next(r) % q);
  }
}

void cko_canonical(const cko_ctx* c, uint32_t rows, const uint32_t* gidx, const int32_t* in, uint32_t* out) {
  for (uint32_t i = 0; i < rows; ++i)
    for (uint32_t k = 0; k < c->n; ++k)
      out[(size_t)i * c->n + k] = correct64(in[(size_t)i * c->n + k], c->primes[gidx[i]]);
}

/* ------------------------------------------------------------------ ntt -- */
/* fwd_stages (ntt.cpp:15-50) restricted to the serial single-segment path
 * forward_row_serial (ntt.cpp:274-279): one stage per call, entry merge at
 * stage 0, tighten at the last stage. */
void cko_ntt_fwd_row(const cko_ctx* c, int32_t* d, uint32_t gidx) {
  const cko_table* T = &c->tw[gidx];
  const ckp* pc = &T->ctx;
  const int32_t q = (int32_t)pc->q, q2 = 2 * q;
  const uint32_t n = c->n;
  for (uint32_t sl = 0; sl < c->logn; ++sl) {
    const size_t t = (size_t)n >> (sl + 1), m = (size_t)1 << sl;
    const int entry = sl == 0, tighten = sl == c->logn - 1;
    for (size_t g = 0; g < m; ++g) {
      const int32_t w = entry ? (int32_t)T->fwd1_r2 : (int32_t)T->fwd[m + g];
      int32_t* px = d + 2 * g * t;
      int32_t* py = px + t;
      for (size_t j = 0; j < t; ++j) {
        int32_t x = px[j];
        const int32_t y = mont_mul(py[j], w, pc);
        if (entry) x = mont_mul(x, (int32_t)pc->r2, pc);
        int64_t u = (int64_t)x + y, v = (int64_t)x - y;
        if (u >= q2) u -= q2; else if (u <= -q2) u += q2;
        if (v >= q2) v -= q2; else if (v <= -q2) v += q2;
        if (tighten) {
          if (u >= q) u -= q; else if (u <= -q) u += q;
          if (v >= q) v -= q; else if (v <= -q) v += q;
        }
        px[j] = (int32_t)u;
        py[j] = (int32_t)v;
      }
    }
  }
}

/* inv_stages (ntt.cpp:56-96) on the serial path inverse_row_serial
 * (ntt.cpp:281-286): exit constants at the m = 1 stage, optional fused
 * BConv part-1 epilogue with canonicalisation to [0, q). */
void cko_intt_row(const cko_ctx* c, int32_t* d, uint32_t gidx, const uint32_t* epilogue_mont) {
  const cko_table* T = &c->tw[gidx];
  const ckp* pc = &T->ctx;
  const int32_t q = (int32_t)pc->q, q2 = 2 * q;
  const uint32_t n = c->n;
  const uint32_t epi = epilogue_mont ? *epilogue_mont : 0;
  for (uint32_t v = 0; v < c->logn; ++v) {
    const size_t m = (size_t)n >> (1 + v), t = (size_t)1 << v;
    const int exit_stage = m == 1;
    for (size_t g = 0; g < m; ++g) {
      const int32_t w = exit_stage ? 0 : (int32_t)T->inv[m + g];
      int32_t* px = d + 2 * g * t;
      int32_t* py = px + t;
      for (size_t j = 0; j < t; ++j) {
        const int32_t x = px[j], y = py[j];
        int64_t u = (int64_t)x + y, v2 = (int64_t)x - y;
        if (exit_stage) {
          int32_t a0 = mont_reduce(u * (int32_t)T->exit_x, pc);
          int32_t a1 = mont_reduce(v2 * (int32_t)T->exit_y, pc);
          if (epi) {
            a0 = (int32_t)correct_lazy(mont_mul(a0, (int32_t)epi, pc), pc->q);
            a1 = (int32_t)correct_lazy(mont_mul(a1, (int32_t)epi, pc), pc->q);
          }
          px[j] = a0;
          py[j] = a1;
        } else {
          if (u >= q2) u -= q2; else if (u <= -q2) u += q2;
          px[j] = (int32_t)u;
          py[j] = mont_reduce(v2 * w, pc);
        }
      }
    }
  }
}

/* ---------------------------------------------------------------- bconv -- */
typedef struct {
  uint32_t sc, dc;
  const uint32_t* sg; /* global prime indices */
  const uint32_t* dg;
  int32_t* cm;        /* dc x sc centred Montgomery (P/P_j) mod q_i */
  uint32_t* part1;    /* sc */
  size_t interval;
} btable;

/* make_bconv_table, bconv.cpp:13-46 (the Boost big-int P/P_j is reduced
 * factor by factor mod each destination prime: same residue) */
static void make_btable(const cko_ctx* c, btable* t, uint32_t sc, const uint32_t* sg, uint32_t dc,
                        const uint32_t* dg) {
  t->sc = sc;
  t->dc = dc;
  t->sg = sg;
  t->dg = dg;
  t->cm = (int32_t*)malloc(sizeof(int32_t) * (size_t)sc * dc + 1);
  t->part1 = (uint32_t*)malloc(sizeof(uint32_t) * sc + 1);
  for (uint32_t j = 0; j < sc; ++j) {
    const uint32_t pj = c->primes[sg[j]];
    uint64_t ph = 1 % pj;
    for (uint32_t k = 0; k < sc; ++k)
      if (k != j) ph = ph * (c->primes[sg[k]] % pj) % pj;
    t->part1[j] = to_mont((uint32_t)inv_mod(ph, pj), &c->pc[sg[j]]);
  }
  for (uint32_t i = 0; i < dc; ++i) {
    const uint32_t q = c->primes[dg[i]];
    for (uint32_t j = 0; j < sc; ++j) {
      uint64_t ph = 1 % q;
      for (uint32_t k = 0; k < sc; ++k)
        if (k != j) ph = ph * (c->primes[sg[k]] % q) % q;
      const uint32_t m = to_mont((uint32_t)ph, &c->pc[dg[i]]);
      int64_t centred = m;
      if (centred > (int64_t)(q - 1) / 2) centred -= q;
      t->cm[(size_t)i * sc + j] = (int32_t)centred;
    }
  }
  uint32_t p_max = 0;
  for (uint32_t j = 0; j < sc; ++j)
    if (c->primes[sg[j]] > p_max) p_max = c->primes[sg[j]];
  const size_t k_max = (size_t)((1ull << 32) / p_max);
  t->interval = (size_t)-1;
  if (sc > k_max && k_max >= 1) t->interval = k_max - 1;
}
static void free_btable(btable* t) {
  free(t->cm);
  free(t->part1);
}

static inline int64_t centered_mod(int64_t v, uint32_t q) { /* bconv.cpp:86-92 */
  int64_t r = v % (int64_t)q;
  const int64_t half = ((int64_t)q - 1) / 2;
  if (r > half) r -= q;
  if (r < -half) r += q;
  return r;
}

/* bconv_part2, bconv.cpp:96-174 (untiled order of the same sums) */
static void bconv_part2(const cko_ctx* c, const btable* t, const int32_t* src, int32_t* const* dst) {
  const uint32_t n = c->n;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)t->dc; ++i) {
    const ckp* pc = &c->pc[t->dg[i]];
    for (uint32_t x = 0; x < n; ++x) {
      int64_t acc = 0;
      for (uint32_t k = 0; k < t->sc; ++k) {
        acc += (int64_t)t->cm[(size_t)i * t->sc + k] * src[(size_t)k * n + x];
        if ((size_t)(k + 1) % t->interval == 0 && k + 1 < t->sc) acc = centered_mod(acc, pc->q);
      }
      dst[i][x] = mont_reduce(acc, pc);
    }
  }
}

void cko_bconv_part1(const cko_ctx* c, uint32_t sc, const uint32_t* sg, uint32_t* part1_mont) {
  btable t;
  uint32_t dummy = 0;
  make_btable(c, &t, sc, sg, 0, &dummy);
  memcpy(part1_mont, t.part1, sizeof(uint32_t) * sc);
  free_btable(&t);
}

void cko_bconv(const cko_ctx* c, uint32_t sc, const uint32_t* sg, uint32_t dc, const uint32_t* dg, const int32_t* src,
               int32_t* dst) {
  btable t;
  make_btable(c, &t, sc, sg, dc, dg);
  int32_t** rows = (int32_t**)malloc(sizeof(int32_t*) * (dc + 1));
  for (uint32_t i = 0; i < dc; ++i) rows[i] = dst + (size_t)i * c->n;
  bconv_part2(c, &t, src, rows);
  free(rows);
  free_btable(&t);
}

/* ------------------------------------------------------------ mechanisms -- */
static uint32_t num_digits(const cko_ctx* c, uint32_t level) { return (level + c->alpha - 1) / c->alpha; }
/* global_prime_index, poly.hpp:103-106, for a (level Q + alpha P) polynomial */
static uint32_t gidx_of(const cko_ctx* c, uint32_t level, uint32_t row) {
  return row < level ? row : c->l + (row - level);
}

int cko_mod_up(const cko_ctx* c, uint32_t level, const int32_t* d, int32_t* out) { /* ckks.cpp:680-731 */
  const uint32_t n = c->n, alpha = c->alpha, D = num_digits(c, level), rows = level + alpha;
  uint32_t* sg = (uint32_t*)malloc(sizeof(uint32_t) * alpha);
  uint32_t* dg = (uint32_t*)malloc(sizeof(uint32_t) * rows);
  int32_t** dst = (int32_t**)malloc(sizeof(int32_t*) * rows);
  int32_t* scratch = (int32_t*)malloc(sizeof(int32_t) * (size_t)alpha * n);
  for (uint32_t k = 0; k < D; ++k) {
    const uint32_t b = k * alpha, e = (k + 1) * alpha < level ? (k + 1) * alpha : level, cnt = e - b;
    for (uint32_t j = 0; j < cnt; ++j) sg[j] = b + j;
    uint32_t nd = 0;
    for (uint32_t i = 0; i < level; ++i)
      if (i < b || i >= e) dg[nd++] = i;
    for (uint32_t j = 0; j < alpha; ++j) dg[nd++] = c->l + j;
    btable t; /* modup_table (ckks.cpp:188-202) */
    make_btable(c, &t, cnt, sg, nd, dg);
    for (uint32_t j = 0; j < cnt; ++j) {
      memcpy(scratch + (size_t)j * n, d + (size_t)(b + j) * n, sizeof(int32_t) * n);
      cko_intt_row(c, scratch + (size_t)j * n, b + j, &t.part1[j]);
    }
    int32_t* ext = out + (size_t)k * rows * n;
    memset(ext, 0, sizeof(int32_t) * (size_t)rows * n);
    for (uint32_t j = 0; j < cnt; ++j) memcpy(ext + (size_t)(b + j) * n, d + (size_t)(b + j) * n, sizeof(int32_t) * n);
    uint32_t di = 0;
    for (uint32_t i = 0; i < rows; ++i)
      if (i < b || i >= e) dst[di++] = ext + (size_t)i * n;
    bconv_part2(c, &t, scratch, dst);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)rows; ++i)
      if ((uint32_t)i < b || (uint32_t)i >= e) cko_ntt_fwd_row(c, ext + (size_t)i * n, gidx_of(c, level, (uint32_t)i));
    free_btable(&t);
  }
  free(sg);
  free(dg);
  free(dst);
  free(scratch);
  return 0;
}

int cko_key_mult(const cko_ctx* c, uint32_t level, const int32_t* hoist, const int32_t* evk, int32_t* v0,
                 int32_t* v1) { /* ckks.cpp:733-770 */
  const uint32_t n = c->n, rows = level + c->alpha, D = num_digits(c, level), L = c->l + c->alpha;
  memset(v0, 0, sizeof(int32_t) * (size_t)rows * n);
  memset(v1, 0, sizeof(int32_t) * (size_t)rows * n);
#pragma omp parallel for schedule(static)
  for (int64_t ii = 0; ii < (int64_t)rows; ++ii) {
    const uint32_t row = (uint32_t)ii, g = gidx_of(c, level, row);
    const ckp* pc = &c->pc[g];
    const int32_t q = (int32_t)pc->q;
    int32_t* o0 = v0 + (size_t)row * n;
    int32_t* o1 = v1 + (size_t)row * n;
    for (uint32_t k = 0; k < D; ++k) {
      const int32_t* dk = hoist + ((size_t)k * rows + row) * n;
      const int32_t* eb = evk + (((size_t)k * 2 + 0) * L + g) * n;
      const int32_t* ea = evk + (((size_t)k * 2 + 1) * L + g) * n;
      for (uint32_t x = 0; x < n; ++x) {
        o0[x] += mont_mul(dk[x], eb[x], pc);
        o1[x] += mont_mul(dk[x], ea[x], pc);
      }
      if (k % 3 == 2 || k + 1 == D)
        for (uint32_t x = 0; x < n; ++x) {
          o0[x] = narrow4(o0[x], q);
          o1[x] = narrow4(o1[x], q);
        }
    }
  }
  return 0;
}

/* drop_and_divide (ckks.cpp:611-655) with a switch table (ckks.cpp:206-220):
 * v has out_q + sc rows; tail source rows have global indices sg. */
static void drop_and_divide(const cko_ctx* c, const int32_t* v, uint32_t out_q, uint32_t sc, const uint32_t* sg,
                            int32_t* out) {
  const uint32_t n = c->n;
  uint32_t* dg = (uint32_t*)malloc(sizeof(uint32_t) * (out_q + 1));
  for (uint32_t i = 0; i < out_q; ++i) dg[i] = i;
  btable t;
  make_btable(c, &t, sc, sg, out_q, dg);
  /* divisor = product of the source primes; div_inv_mont per destination row */
  uint32_t* div_inv = (uint32_t*)malloc(sizeof(uint32_t) * (out_q + 1));
  for (uint32_t i = 0; i < out_q; ++i) {
    const uint32_t q = c->primes[i];
    uint64_t d = 1 % q;
    for (uint32_t j = 0; j < sc; ++j) d = d * (c->primes[sg[j]] % q) % q;
    div_inv[i] = to_mont((uint32_t)inv_mod(d, q), &c->pc[i]);
  }
  int32_t* scratch = (int32_t*)malloc(sizeof(int32_t) * (size_t)sc * n);
  for (uint32_t j = 0; j < sc; ++j) {
    memcpy(scratch + (size_t)j * n, v + (size_t)(out_q + j) * n, sizeof(int32_t) * n);
    cko_intt_row(c, scratch + (size_t)j * n, sg[j], &t.part1[j]);
  }
  int32_t** dst = (int32_t**)malloc(sizeof(int32_t*) * (out_q + 1));
  for (uint32_t i = 0; i < out_q; ++i) dst[i] = out + (size_t)i * n;
  bconv_part2(c, &t, scratch, dst);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)out_q; ++i) cko_ntt_fwd_row(c, out + (size_t)i * n, (uint32_t)i);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)out_q; ++i) {
    const ckp* pc = &c->pc[i];
    const int32_t inv = (int32_t)div_inv[i];
    const int32_t* vr = v + (size_t)i * n;
    int32_t* o = out + (size_t)i * n;
    for (uint32_t x = 0; x < n; ++x) o[x] = mont_mul(vr[x] - o[x], inv, pc);
  }
  free(scratch);
  free(dst);
  free(div_inv);
  free(dg);
  free_btable(&t);
}

int cko_mod_down(const cko_ctx* c, uint32_t level, const int32_t* v, int32_t* out) { /* ckks.cpp:224-232,657-661 */
  uint32_t* sg = (uint32_t*)malloc(sizeof(uint32_t) * c->alpha);
  for (uint32_t j = 0; j < c->alpha; ++j) sg[j] = c->l + j;
  drop_and_divide(c, v, level, c->alpha, sg, out);
  free(sg);
  return 0;
}

int cko_key_switch(const cko_ctx* c, uint32_t level, const int32_t* d, const int32_t* evk, int32_t* c0,
                   int32_t* c1) { /* ckks.cpp:778-787 */
  const size_t rows = level + c->alpha, n = c->n;
  int32_t* hoist = (int32_t*)malloc(sizeof(int32_t) * num_digits(c, level) * rows * n);
  int32_t* v0 = (int32_t*)malloc(sizeof(int32_t) * rows * n);
  int32_t* v1 = (int32_t*)malloc(sizeof(int32_t) * rows * n);
  cko_mod_up(c, level, d, hoist);
  cko_key_mult(c, level, hoist, evk, v0, v1);
  cko_mod_down(c, level, v0, c0);
  cko_mod_down(c, level, v1, c1);
  free(hoist);
  free(v0);
  free(v1);
  return 0;
}

int cko_rescale(const cko_ctx* c, uint32_t level, const int32_t* b, const int32_t* a, int32_t* ob, int32_t* oa) {
  /* ckks.cpp:234-244, 789-802 */
  if (level < 4) return -1;
  uint32_t sg[2] = {level - 2, level - 1};
  drop_and_divide(c, b, level - 2, 2, sg, ob);
  drop_and_divide(c, a, level - 2, 2, sg, oa);
  return 0;
}

void cko_ew_add(const cko_ctx* c, uint32_t rows, const int32_t* x, const int32_t* y, int32_t* o) {
  for (uint32_t i = 0; i < rows; ++i) /* ew_add, poly.cpp:146-150 */
    for (uint32_t k = 0; k < c->n; ++k) {
      const size_t e = (size_t)i * c->n + k;
      o[e] = narrow1((int64_t)x[e] + y[e], (int32_t)c->primes[i]);
    }
}

void cko_ew_mul(const cko_ctx* c, uint32_t rows, const int32_t* x, const int32_t* y, int32_t* o) {
  for (uint32_t i = 0; i < rows; ++i) /* ew_mul, poly.cpp:158-164 */
    for (uint32_t k = 0; k < c->n; ++k) {
      const size_t e = (size_t)i * c->n + k;
      o[e] = mont_mul(x[e], y[e], &c->pc[i]);
    }
}

int cko_hmult(const cko_ctx* c, uint32_t level, const int32_t* xb, const int32_t* xa, const int32_t* yb,
              const int32_t* ya, const int32_t* evk, int lazy, int32_t* ob, int32_t* oa) { /* ckks.cpp:804-865 */
  if (level < 4) return -1;
  const uint32_t n = c->n, rows = level + c->alpha;
  const size_t ln = (size_t)level * n;
  int32_t* d0 = (int32_t*)malloc(sizeof(int32_t) * ln);
  int32_t* d1 = (int32_t*)malloc(sizeof(int32_t) * ln);
  int32_t* d2 = (int32_t*)malloc(sizeof(int32_t) * ln);
  int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * ln);
  cko_ew_mul(c, level, xb, yb, d0);
  cko_ew_mul(c, level, xb, ya, d1);
  cko_ew_mul(c, level, xa, yb, tmp);
  for (uint32_t i = 0; i < level; ++i) /* ew_add_inplace, poly.cpp:183-193 */
    for (uint32_t k = 0; k < n; ++k) {
      const size_t e = (size_t)i * n + k;
      d1[e] = narrow1((int64_t)d1[e] + tmp[e], (int32_t)c->primes[i]);
    }
  cko_ew_mul(c, level, xa, ya, d2);
  int32_t* hoist = (int32_t*)malloc(sizeof(int32_t) * num_digits(c, level) * rows * (size_t)n);
  int32_t* v0 = (int32_t*)malloc(sizeof(int32_t) * rows * (size_t)n);
  int32_t* v1 = (int32_t*)malloc(sizeof(int32_t) * rows * (size_t)n);
  cko_mod_up(c, level, d2, hoist);
  cko_key_mult(c, level, hoist, evk, v0, v1);
  if (!lazy) {
    for (uint32_t i = 0; i < level; ++i) { /* fold P*d, ckks.cpp:831-842 */
      const int32_t pm = (int32_t)c->p_mont[i];
      for (uint32_t k = 0; k < n; ++k) {
        const size_t e = (size_t)i * n + k;
        v0[e] += mont_mul(d0[e], pm, &c->pc[i]);
        v1[e] += mont_mul(d1[e], pm, &c->pc[i]);
      }
    }
    uint32_t* sg = (uint32_t*)malloc(sizeof(uint32_t) * (2 + c->alpha)); /* merged_table, ckks.cpp:246-258 */
    sg[0] = level - 2;
    sg[1] = level - 1;
    for (uint32_t j = 0; j < c->alpha; ++j) sg[2 + j] = c->l + j;
    drop_and_divide(c, v0, level - 2, 2 + c->alpha, sg, ob);
    drop_and_divide(c, v1, level - 2, 2 + c->alpha, sg, oa);
    free(sg);
  } else { /* ckks.cpp:853-863 */
    cko_mod_down(c, level, v0, tmp);
    cko_ew_add(c, level, d0, tmp, ob);
    cko_mod_down(c, level, v1, tmp);
    cko_ew_add(c, level, d1, tmp, oa);
  }
  free(d0);
  free(d1);
  free(d2);
  free(tmp);
  free(hoist);
  free(v0);
  free(v1);
  return 0;
}

/* element-wise over a polynomial whose row i lives at global prime gidx[i]
 * (Q-prefix then P rows, poly.hpp:103-106): op 0 ew_add, 1 ew_sub (narrow to
 * (-q, q), poly.cpp:121-156), 2 ew_mul (Montgomery, poly.cpp:158-164),
 * 3 ew_mul_const with one Montgomery constant per row (poly.cpp:166-180). */
void cko_ew_rows(const cko_ctx* c, int op, uint32_t rows, const uint32_t* gidx, const int32_t* x, const int32_t* y,
                 const uint32_t* consts, int32_t* o) {
  for (uint32_t i = 0; i < rows; ++i) {
    const ckp* P = &c->pc[gidx[i]];
    for (uint32_t k = 0; k < c->n; ++k) {
      const size_t e = (size_t)i * c->n + k;
      if (op == 0) o[e] = narrow1((int64_t)x[e] + y[e], (int32_t)P->q);
      else if (op == 1) o[e] = narrow1((int64_t)x[e] - y[e], (int32_t)P->q);
      else if (op == 2) o[e] = mont_mul(x[e], y[e], P);
      else o[e] = mont_mul(x[e], (int32_t)consts[i], P);
    }
  }
}

/* apply_automorphism for Galois element g with inverse gi (automorphism.cpp:
 * 38-61, 76-100): evaluation domain o[j] = in[src(j)], src the inverse of
 * dest(i) = brev(phi_g(brev(i))); coefficient domain: coefficient k goes to
 * k gi mod 2n, negated past n. */
void cko_automorphism(const cko_ctx* c, uint32_t rows, uint64_t g, uint64_t gi, int coeff, const int32_t* in,
                      int32_t* o) {
  const uint32_t n = c->n;
  uint32_t bits = 0;
  while ((1u << bits) < n) ++bits;
  uint32_t* src = (uint32_t*)malloc(sizeof(uint32_t) * n);
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t ph = (uint32_t)((((2ull * bit_reverse(i, bits) + 1) * g) % (2ull * n) - 1) / 2);
    src[bit_reverse(ph, bits)] = i;
  }
  for (uint32_t r = 0; r < rows; ++r) {
    const int32_t* a = in + (size_t)r * n;
    int32_t* b = o + (size_t)r * n;
    if (!coeff) {
      for (uint32_t j = 0; j < n; ++j) b[j] = a[src[j]];
    } else {
      for (uint32_t k = 0; k < n; ++k) {
        const uint64_t e = (uint64_t)k * gi % (2ull * n);
        if (e < n) b[e] = a[k];
        else b[e - n] = -a[k];
      }
    }
  }
  free(src);
}

/* -------------------------------------------------------- automorphism -- */
void cko_rotation_src_map(uint32_t n, int64_t r, uint32_t* src) { /* automorphism.cpp:11-69 */
  uint32_t bits = 0;
  while ((1u << bits) < n) ++bits;
  const int64_t half = (int64_t)n / 2;
  int64_t e = (-r) % half;
  if (e < 0) e += half;
  uint64_t g = 1;
  const uint64_t mod = 2ull * n;
  for (int64_t i = 0; i < e; ++i) g = g * 5 % mod;
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t bi = bit_reverse(i, bits);
    const uint32_t phi = (uint32_t)((((2ull * bi + 1) * g) % mod - 1) / 2);
    src[bit_reverse(phi, bits)] = i;
  }
}

static void automorph(uint32_t n, uint32_t rows, const uint32_t* src, const int32_t* in, int32_t* out) {
  for (uint32_t i = 0; i < rows; ++i) /* apply_automorphism gather, automorphism.cpp:82-87 */
    for (uint32_t j = 0; j < n; ++j) out[(size_t)i * n + j] = in[(size_t)i * n + src[j]];
}

int cko_hrot(const cko_ctx* c, uint32_t level, const int32_t* b, const int32_t* a, int64_t r, const int32_t* evk,
             int32_t* ob, int32_t* oa) { /* ckks.cpp:869-897 */
  const uint32_t n = c->n, rows = level + c->alpha;
  const size_t ln = (size_t)level * n;
  int32_t* hoist = (int32_t*)malloc(sizeof(int32_t) * num_digits(c, level) * rows * (size_t)n);
  int32_t* v0 = (int32_t*)malloc(sizeof(int32_t) * rows * (size_t)n);
  int32_t* v1 = (int32_t*)malloc(sizeof(int32_t) * rows * (size_t)n);
  int32_t* c0 = (int32_t*)malloc(sizeof(int32_t) * ln);
  int32_t* c1 = (int32_t*)malloc(sizeof(int32_t) * ln);
  uint32_t* src = (uint32_t*)malloc(sizeof(uint32_t) * n);
  cko_mod_up(c, level, a, hoist);
  cko_key_mult(c, level, hoist, evk, v0, v1);
  cko_mod_down(c, level, v0, c0);
  cko_mod_down(c, level, v1, c1);
  for (uint32_t i = 0; i < level; ++i) /* ew_add_inplace(c0, ct.b), ckks.cpp:880 */
    for (uint32_t k = 0; k < n; ++k) {
      const size_t e = (size_t)i * n + k;
      c0[e] = narrow1((int64_t)c0[e] + b[e], (int32_t)c->primes[i]);
    }
  cko_rotation_src_map(n, r, src);
  automorph(n, level, src, c0, ob);
  automorph(n, level, src, c1, oa);
  free(hoist);
  free(v0);
  free(v1);
  free(c0);
  free(c1);
  free(src);
  return 0;
}

/* addmul_rows, ckks.cpp:930-941 */
static void addmul_rows(const cko_ctx* c, uint32_t level, uint32_t rows, int32_t* acc, const int32_t* x,
                        const int32_t* y) {
  for (uint32_t i = 0; i < rows; ++i) {
    const ckp* pc = &c->pc[gidx_of(c, level, i)];
    const int32_t q = (int32_t)pc->q;
    for (uint32_t k = 0; k < c->n; ++k) {
      const size_t e = (size_t)i * c->n + k;
      acc[e] = narrow4(acc[e] + mont_mul(x[e], y[e], pc), q);
    }
  }
}

int cko_hoisted_accumulate(const cko_ctx* c, uint32_t level, const int32_t* b, const int32_t* a, uint32_t count,
                           const int64_t* rots, const int32_t* const* pts, const int32_t* const* evks, int32_t* ob,
                           int32_t* oa) { /* ckks.cpp:945-1012 */
  const uint32_t n = c->n, rows = level + c->alpha;
  const size_t rn = (size_t)rows * n, ln = (size_t)level * n;
  int32_t* hoist = (int32_t*)malloc(sizeof(int32_t) * num_digits(c, level) * rn);
  int32_t* acc0 = (int32_t*)calloc(rn, sizeof(int32_t));
  int32_t* acc1 = (int32_t*)calloc(rn, sizeof(int32_t));
  int32_t* v0 = (int32_t*)malloc(sizeof(int32_t) * rn);
  int32_t* v1 = (int32_t*)malloc(sizeof(int32_t) * rn);
  int32_t* w = (int32_t*)malloc(sizeof(int32_t) * rn);
  uint32_t* src = (uint32_t*)malloc(sizeof(uint32_t) * n);
  int used_pq = 0;
  memset(ob, 0, sizeof(int32_t) * ln);
  memset(oa, 0, sizeof(int32_t) * ln);
  cko_mod_up(c, level, a, hoist);
  for (uint32_t i = 0; i < count; ++i) {
    if (rots[i] == 0) {
      addmul_rows(c, level, level, ob, b, pts[i]);
      addmul_rows(c, level, level, oa, a, pts[i]);
      continue;
    }
    cko_key_mult(c, level, hoist, evks[i], v0, v1);
    cko_rotation_src_map(n, rots[i], src);
    automorph(n, rows, src, v0, w);
    addmul_rows(c, level, rows, acc0, w, pts[i]);
    automorph(n, rows, src, v1, w);
    addmul_rows(c, level, rows, acc1, w, pts[i]);
    automorph(n, level, src, b, w);
    addmul_rows(c, level, level, ob, w, pts[i]);
    used_pq = 1;
  }
  if (used_pq) {
    cko_mod_down(c, level, acc0, v0);
    cko_mod_down(c, level, acc1, v1);
    for (uint32_t i = 0; i < level; ++i)
      for (uint32_t k = 0; k < n; ++k) {
        const size_t e = (size_t)i * n + k;
        ob[e] = narrow1((int64_t)ob[e] + v0[e], (int32_t)c->primes[i]);
        oa[e] = narrow1((int64_t)oa[e] + v1[e], (int32_t)c->primes[i]);
      }
  }
  free(hoist);
  free(acc0);
  free(acc1);
  free(v0);
  free(v1);
  free(w);
  free(src);
  return 0;
}
