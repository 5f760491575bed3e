/* oracle.c — CPU reference for arXiv 1310.3809's hot path.  TEST INFRASTRUCTURE ONLY:
 * see oracle.h for who may call this and for the conventions.  Nothing here is tuned; every
 * routine is the plain definition or the paper's algorithm, step by step, cited by
 * PAPER.md line.  No code is shared with paper_1310_3809_b200/csrc.
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu") check every function below against Python
 * arbitrary-precision integers, closed forms, brute force on tiny moduli, curve group
 * orders counted by brute force, and the paper's printed values — see DESIGN.md §4.
 */
#include "oracle.h"
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------ */
/* plain multiprecision helpers (little-endian 32-bit words)                            */
/* ------------------------------------------------------------------------------------ */
static void zero(uint32_t *a, int w) { memset(a, 0, sizeof(uint32_t) * (size_t)w); }
static void copy(uint32_t *d, const uint32_t *s, int w) { memcpy(d, s, sizeof(uint32_t) * (size_t)w); }

static int is_zero(const uint32_t *a, int w) {
  for (int i = 0; i < w; ++i)
    if (a[i]) return 0;
  return 1;
}
static int is_one(const uint32_t *a, int w) {
  if (a[0] != 1) return 0;
  for (int i = 1; i < w; ++i)
    if (a[i]) return 0;
  return 1;
}
/* -1, 0, +1 */
static int cmp(const uint32_t *a, const uint32_t *b, int w) {
  for (int i = w - 1; i >= 0; --i) {
    if (a[i] < b[i]) return -1;
    if (a[i] > b[i]) return 1;
  }
  return 0;
}
/* d = a + b, returns carry out */
static uint32_t add(uint32_t *d, const uint32_t *a, const uint32_t *b, int w) {
  uint64_t c = 0;
  for (int i = 0; i < w; ++i) {
    c += (uint64_t)a[i] + b[i];
    d[i] = (uint32_t)c;
    c >>= 32;
  }
  return (uint32_t)c;
}
/* d = a - b, returns borrow out (1 if a < b) */
static uint32_t sub(uint32_t *d, const uint32_t *a, const uint32_t *b, int w) {
  int64_t br = 0;
  for (int i = 0; i < w; ++i) {
    int64_t t = (int64_t)a[i] - b[i] - br;
    br = t < 0;
    d[i] = (uint32_t)t;
  }
  return (uint32_t)br;
}
static int bit(const uint32_t *a, uint32_t i) { return (a[i >> 5] >> (i & 31)) & 1; }
static void shr1(uint32_t *a, int w, uint32_t topbit) {
  for (int i = 0; i < w; ++i) {
    uint32_t hi = (i + 1 < w) ? a[i + 1] : topbit;
    a[i] = (a[i] >> 1) | (hi << 31);
  }
}

/* ------------------------------------------------------------------------------------ */
/* schoolbook product                                                 */
/* ------------------------------------------------------------------------------------ */
void orc_mul(const uint32_t *a, const uint32_t *b, uint32_t *t, int L) {
  zero(t, 2 * L);
  for (int i = 0; i < L; ++i) {
    uint64_t c = 0;
    for (int j = 0; j < L; ++j) {
      c += (uint64_t)a[i] * b[j] + t[i + j];
      t[i + j] = (uint32_t)c;
      c >>= 32;
    }
    t[i + L] = (uint32_t)c;
  }
}

/* low half of a product: d = a*b mod R (R = 2^(32L)) */
static void mul_low(const uint32_t *a, const uint32_t *b, uint32_t *d, int L) {
  uint32_t t[2 * ORC_MAXL];
  orc_mul(a, b, t, L);
  copy(d, t, L);
}

/* m' with m*m' = -1 mod R.  Hensel/Newton lifting x <- x(2 - n x) of n^{-1},
 * starting from x = n (n*n = 1 mod 8 for odd n), doubling the correct bits per step. */
void orc_nprime(const uint32_t *n, uint32_t *np, int L) {
  uint32_t x[ORC_MAXL], t[ORC_MAXL], two[ORC_MAXL], u[ORC_MAXL];
  copy(x, n, L);
  zero(two, L);
  two[0] = 2;
  for (int correct = 3; correct < 32 * L; correct *= 2) {
    mul_low(n, x, t, L);      /* t = n x           */
    sub(u, two, t, L);        /* u = 2 - n x mod R */
    mul_low(x, u, t, L);      /* x = x (2 - n x)   */
    copy(x, t, L);
  }
  /* np = -x mod R */
  uint32_t z[ORC_MAXL];
  zero(z, L);
  sub(np, z, x, L);
}

/* REDC steps 1-2: b = a m' mod R; r = (a + b m)/R over the integers.
 * r is returned in L+1 words (r < 2R always when a < R m). */
static void redc_steps12(const uint32_t *T, const uint32_t *n, const uint32_t *np, uint32_t *r, int L) {
  uint32_t q[ORC_MAXL], qn[2 * ORC_MAXL], s[2 * ORC_MAXL + 1];
  mul_low(T, np, q, L);                 /* step 1: q = (T mod R) m' mod R            */
  orc_mul(q, n, qn, L);                 /* q*m, 2L words                              */
  s[2 * L] = add(s, T, qn, 2 * L);      /* T + q m, exact (2L+1 words)                */
  /* low L words of s are zero by construction; r = s / R */
  copy(r, s + L, L + 1);
}

void orc_redc_raw(const uint32_t *T, const uint32_t *n, const uint32_t *np, uint32_t *out, int L) {
  uint32_t r[ORC_MAXL + 1];
  redc_steps12(T, n, np, r, L);
  copy(out, r, L); /* caller guarantees r < R (lazy precondition, reading G3) */
}

void orc_redc(const uint32_t *T, const uint32_t *n, const uint32_t *np, uint32_t *out, int L) {
  uint32_t r[ORC_MAXL + 1], n1[ORC_MAXL + 1], d[ORC_MAXL + 1];
  redc_steps12(T, n, np, r, L);
  copy(n1, n, L);
  n1[L] = 0;
  /* step 3: if r >= m return r - m else r */
  if (cmp(r, n1, L + 1) >= 0) {
    sub(d, r, n1, L + 1);
    copy(out, d, L);
  } else {
    copy(out, r, L);
  }
}

void orc_mulmod_chain(const uint32_t *a, const uint32_t *b, const uint32_t *n, uint32_t *out,
                      size_t count, int L, uint32_t iters, int square, int canonical) {
  for (size_t i = 0; i < count; ++i) {
    const uint32_t *ai = a + i * (size_t)L, *bi = b + i * (size_t)L, *ni = n + i * (size_t)L;
    uint32_t np[ORC_MAXL], x[ORC_MAXL], T[2 * ORC_MAXL];
    orc_nprime(ni, np, L);
    copy(x, ai, L);
    for (uint32_t t = 0; t < iters; ++t) {
      orc_mul(x, square ? x : bi, T, L);
      orc_redc_raw(T, ni, np, x, L); /* lazy chain, no intermediate reduction */
    }
    if (canonical && cmp(x, ni, L) >= 0) sub(x, x, ni, L);
    copy(out + i * (size_t)L, x, L);
  }
}

/* Reduction after Addition with 2m: domain [0, 2n). */
void orc_add_lazy(const uint32_t *x, const uint32_t *y, const uint32_t *n, uint32_t *out, int L) {
  uint32_t s[ORC_MAXL + 1], n2[ORC_MAXL + 1], x1[ORC_MAXL + 1], y1[ORC_MAXL + 1];
  copy(x1, x, L); x1[L] = 0;
  copy(y1, y, L); y1[L] = 0;
  copy(n2, n, L); n2[L] = 0;
  add(n2, n2, n2, L + 1);
  add(s, x1, y1, L + 1);
  if (cmp(s, n2, L + 1) >= 0) sub(s, s, n2, L + 1);
  copy(out, s, L);
}
/* Reduction after Subtraction (condition as read in G4) with 2m. */
void orc_sub_lazy(const uint32_t *x, const uint32_t *y, const uint32_t *n, uint32_t *out, int L) {
  uint32_t d[ORC_MAXL], n2[ORC_MAXL];
  add(n2, n, n, L);
  if (sub(d, x, y, L)) add(d, d, n2, L); /* a < 0: return a + 2m */
  copy(out, d, L);
}

/* ------------------------------------------------------------------------------------ */
/* residue system of PAPER.md:104 over one modulus, canonical representatives            */
/* ------------------------------------------------------------------------------------ */
typedef struct {
  int L;
  uint32_t n[ORC_MAXL], np[ORC_MAXL], r2[ORC_MAXL];
} ctx_t;

/* r = x mod n for an arbitrary-width x, by shift-and-subtract (binary long division). */
static void mod_n(const uint32_t *x, int xw, const uint32_t *n, uint32_t *r, int L) {
  uint32_t acc[ORC_MAXL + 1], n1[ORC_MAXL + 1];
  zero(acc, L + 1);
  copy(n1, n, L);
  n1[L] = 0;
  for (int i = 32 * xw - 1; i >= 0; --i) {
    add(acc, acc, acc, L + 1);
    acc[0] |= (uint32_t)bit(x, (uint32_t)i);
    if (cmp(acc, n1, L + 1) >= 0) sub(acc, acc, n1, L + 1);
  }
  copy(r, acc, L);
}

static void ctx_init(ctx_t *c, const uint32_t *n, int L) {
  uint32_t R2[2 * ORC_MAXL + 1];
  c->L = L;
  copy(c->n, n, L);
  orc_nprime(n, c->np, L);
  zero(R2, 2 * L + 1);
  R2[2 * L] = 1; /* 2^(64L) = R^2 */
  mod_n(R2, 2 * L + 1, n, c->r2, L);
}
static void mmul(const ctx_t *c, const uint32_t *x, const uint32_t *y, uint32_t *out) {
  uint32_t T[2 * ORC_MAXL];
  orc_mul(x, y, T, c->L);
  orc_redc(T, c->n, c->np, out, c->L);
}
static void to_mont(const ctx_t *c, const uint32_t *x, uint32_t *out) { mmul(c, x, c->r2, out); }
static void from_mont(const ctx_t *c, const uint32_t *x, uint32_t *out) {
  uint32_t T[2 * ORC_MAXL];
  zero(T, 2 * c->L);
  copy(T, x, c->L);
  orc_redc(T, c->n, c->np, out, c->L);
}
/* canonical add / sub mod n (PAPER.md:156-168 with m) */
static void madd(const ctx_t *c, const uint32_t *x, const uint32_t *y, uint32_t *out) {
  int L = c->L;
  uint32_t s[ORC_MAXL + 1], x1[ORC_MAXL + 1], y1[ORC_MAXL + 1], n1[ORC_MAXL + 1];
  copy(x1, x, L); x1[L] = 0;
  copy(y1, y, L); y1[L] = 0;
  copy(n1, c->n, L); n1[L] = 0;
  add(s, x1, y1, L + 1);
  if (cmp(s, n1, L + 1) >= 0) sub(s, s, n1, L + 1);
  copy(out, s, L);
}
static void msub(const ctx_t *c, const uint32_t *x, const uint32_t *y, uint32_t *out) {
  uint32_t d[ORC_MAXL];
  if (sub(d, x, y, c->L)) add(d, d, c->n, c->L);
  copy(out, d, c->L);
}
static void small_mont(const ctx_t *c, uint64_t v, uint32_t *out) {
  uint32_t w[2] = {(uint32_t)v, (uint32_t)(v >> 32)}, r[ORC_MAXL];
  mod_n(w, 2, c->n, r, c->L);
  to_mont(c, r, out);
}

/* g = gcd(a, n) and, when g == 1, inv = a^{-1} mod n.  Binary extended Euclid for odd n with
 * the invariants x1*a = u, x2*a = v (mod n); halving mod n is (x + n)/2 for odd x.
 * a and n canonical (a < n), n odd.  Returns 1 iff invertible. */
static int inv_gcd(const uint32_t *a, const uint32_t *n, int L, uint32_t *g, uint32_t *inv) {
  uint32_t u[ORC_MAXL], v[ORC_MAXL], x1[ORC_MAXL], x2[ORC_MAXL];
  copy(u, a, L);
  copy(v, n, L);
  zero(x1, L); x1[0] = 1;
  zero(x2, L);
  if (is_zero(u, L)) { /* gcd(0, n) = n */
    copy(g, n, L);
    if (inv) zero(inv, L);
    return 0;
  }
  while (!is_zero(u, L) && !is_zero(v, L)) {
    while (!(u[0] & 1)) {
      shr1(u, L, 0);
      uint32_t c = 0;
      if (x1[0] & 1) c = add(x1, x1, n, L);
      shr1(x1, L, c);
    }
    while (!(v[0] & 1)) {
      shr1(v, L, 0);
      uint32_t c = 0;
      if (x2[0] & 1) c = add(x2, x2, n, L);
      shr1(x2, L, c);
    }
    if (cmp(u, v, L) >= 0) {
      sub(u, u, v, L);
      if (sub(x1, x1, x2, L)) add(x1, x1, n, L);
    } else {
      sub(v, v, u, L);
      if (sub(x2, x2, x1, L)) add(x2, x2, n, L);
    }
  }
  /* one of u, v is zero; the other is the gcd, and its x is the Bezout coefficient */
  if (is_zero(u, L)) {
    copy(g, v, L);
    if (inv) copy(inv, x2, L);
  } else {
    copy(g, u, L);
    if (inv) copy(inv, x1, L);
  }
  return is_one(g, L);
}

/* status of a gcd g of N (§8(b)) */
static int classify(const uint32_t *g, const uint32_t *N, int L) {
  if (is_one(g, L)) return 0;
  if (cmp(g, N, L) == 0) return 2;
  return 1;
}

/* ------------------------------------------------------------------------------------ */
/* ECM stage 1                                                        */
/* ------------------------------------------------------------------------------------ */
uint32_t orc_stage1_k(uint64_t B1, uint32_t *k_words, size_t cap) {
  if (B1 < 2 || B1 > 0xffffffffull || cap == 0) return 0;
  char *comp = (char *)calloc((size_t)B1 + 1, 1);
  if (!comp) return 0;
  memset(k_words, 0, cap * sizeof(uint32_t));
  k_words[0] = 1;
  size_t used = 1;
  for (uint64_t p = 2; p <= B1; ++p) {
    if (comp[p]) continue;
    for (uint64_t m = p * p; m <= B1; m += p) comp[m] = 1;
    uint64_t q = p;                 /* step 1: p^e <= B1 < p^(e+1) (reading G8) */
    while (q * p <= B1) q *= p;
    uint64_t c = 0;                 /* k *= q (q < 2^32) */
    for (size_t i = 0; i < used; ++i) {
      c += (uint64_t)k_words[i] * q;
      k_words[i] = (uint32_t)c;
      c >>= 32;
    }
    if (c) {
      if (used == cap) { free(comp); return 0; }
      k_words[used++] = (uint32_t)c;
    }
  }
  free(comp);
  uint32_t top = k_words[used - 1], b = 0;
  while (top) { ++b; top >>= 1; }
  return (uint32_t)(32 * (used - 1) + b);
}

typedef struct { uint32_t X[ORC_MAXL], Z[ORC_MAXL]; } pt_t;

/* xDBL (reading G9 / SURVEY §8(c) c6): s=(X+Z)^2, d=(X-Z)^2, t=s-d, X'=s d, Z'=t (d + a24 t) */
static void xdbl(const ctx_t *c, const pt_t *P, const uint32_t *a24, pt_t *out) {
  uint32_t s[ORC_MAXL], d[ORC_MAXL], t[ORC_MAXL], w[ORC_MAXL];
  madd(c, P->X, P->Z, w); mmul(c, w, w, s);
  msub(c, P->X, P->Z, w); mmul(c, w, w, d);
  msub(c, s, d, t);
  mmul(c, s, d, out->X);
  mmul(c, a24, t, w);
  madd(c, d, w, w);
  mmul(c, t, w, out->Z);
}
/* xADD with difference (x0:1): U=(X0-Z0)(X1+Z1), V=(X0+Z0)(X1-Z1), X'=(U+V)^2, Z'=x0 (U-V)^2 */
static void xadd(const ctx_t *c, const pt_t *P0, const pt_t *P1, const uint32_t *x0, pt_t *out) {
  uint32_t U[ORC_MAXL], V[ORC_MAXL], w1[ORC_MAXL], w2[ORC_MAXL];
  msub(c, P0->X, P0->Z, w1); madd(c, P1->X, P1->Z, w2); mmul(c, w1, w2, U);
  madd(c, P0->X, P0->Z, w1); msub(c, P1->X, P1->Z, w2); mmul(c, w1, w2, V);
  madd(c, U, V, w1); mmul(c, w1, w1, out->X);
  msub(c, U, V, w1); mmul(c, w1, w1, w2); mmul(c, x0, w2, out->Z);
}

/* Brent-Suyama (formulas: reading G10): u = s^2-5, v = 4s,
 * x0 = u^3/v^3, a24 = (v-u)^3 (3u+v)/(16 u^3 v), through one inverse of D = 16 u^3 v^4.
 * Montgomery-form outputs x0m, a24m; returns status 0, 3 (gcd(D,N)=N) or 4. */
static int suyama_mont(const ctx_t *c, uint64_t sigma, uint32_t *x0m, uint32_t *a24m, uint32_t *g) {
  int L = c->L;
  uint32_t s[ORC_MAXL], u[ORC_MAXL], v[ORC_MAXL], k5[ORC_MAXL], k3[ORC_MAXL], k16[ORC_MAXL];
  uint32_t u2[ORC_MAXL], u3[ORC_MAXL], v2[ORC_MAXL], v3[ORC_MAXL], v4[ORC_MAXL], D[ORC_MAXL];
  uint32_t Dn[ORC_MAXL], wn[ORC_MAXL], w[ORC_MAXL], t1[ORC_MAXL], t2[ORC_MAXL], t3[ORC_MAXL];
  small_mont(c, sigma, s);
  small_mont(c, 5, k5);
  small_mont(c, 3, k3);
  small_mont(c, 16, k16);
  mmul(c, s, s, u);
  msub(c, u, k5, u);                              /* u = s^2 - 5 */
  madd(c, s, s, v); madd(c, v, v, v);             /* v = 4 s     */
  mmul(c, u, u, u2); mmul(c, u2, u, u3);
  mmul(c, v, v, v2); mmul(c, v2, v, v3); mmul(c, v3, v, v4);
  mmul(c, k16, u3, t1); mmul(c, t1, v4, D);      /* D = 16 u^3 v^4 */
  from_mont(c, D, Dn);
  if (!inv_gcd(Dn, c->n, L, g, wn)) return is_zero(Dn, L) || cmp(g, c->n, L) == 0 ? 3 : 4;
  to_mont(c, wn, w);
  /* x0 = 16 u^6 v w */
  mmul(c, t1, u3, t2); mmul(c, t2, v, t3); mmul(c, t3, w, x0m);
  /* a24 = (v-u)^3 (3u+v) v^3 w */
  msub(c, v, u, t1); mmul(c, t1, t1, t2); mmul(c, t2, t1, t3);    /* (v-u)^3 */
  mmul(c, k3, u, t1); madd(c, t1, v, t1);                         /* 3u + v  */
  mmul(c, t3, t1, t2); mmul(c, t2, v3, t3); mmul(c, t3, w, a24m);
  return 0;
}

int orc_suyama(const uint32_t *N, int L, uint64_t sigma, uint32_t *x0, uint32_t *a24, uint32_t *g) {
  if (L < 1 || L > ORC_MAXL || !(N[0] & 1)) return -1;
  ctx_t c;
  ctx_init(&c, N, L);
  uint32_t x0m[ORC_MAXL], a24m[ORC_MAXL], gg[ORC_MAXL];
  zero(gg, L); gg[0] = 1;
  int st = suyama_mont(&c, sigma, x0m, a24m, gg);
  if (g) copy(g, gg, L);
  if (st == 0) {
    if (x0) from_mont(&c, x0m, x0);
    if (a24) from_mont(&c, a24m, a24);
  }
  return st;
}

/* Montgomery ladder over k (reading G9): R0 = P = (x0:1), R1 = xDBL(P); then for bits
 * k_{l-2}..k_0: bit 1: (R0,R1) <- (xADD(R0,R1), xDBL(R1)); bit 0: (xDBL(R0), xADD(R0,R1)).
 * If trace != NULL, the canonical normal-domain state after every step is appended. */
static void ladder(const ctx_t *c, const uint32_t *x0m, const uint32_t *a24m, const uint32_t *k,
                   uint32_t k_bits, pt_t *R0out, uint32_t *trace) {
  int L = c->L;
  pt_t R0, R1, T0, T1;
  uint32_t one[ORC_MAXL];
  small_mont(c, 1, one);
  copy(R0.X, x0m, L);
  copy(R0.Z, one, L);
  xdbl(c, &R0, a24m, &R1);
  uint32_t rec = 0;
#define TRACE_STATE()                                                                 \
  if (trace) {                                                                        \
    from_mont(c, R0.X, trace + (size_t)rec * 4 * L);                                 \
    from_mont(c, R0.Z, trace + (size_t)rec * 4 * L + L);                             \
    from_mont(c, R1.X, trace + (size_t)rec * 4 * L + 2 * L);                         \
    from_mont(c, R1.Z, trace + (size_t)rec * 4 * L + 3 * L);                         \
    ++rec;                                                                            \
  }
  if (k_bits == 1) { /* k = 1: R0 = P */
    TRACE_STATE();
    *R0out = R0;
    return;
  }
  TRACE_STATE();
  for (int i = (int)k_bits - 2; i >= 0; --i) {
    if (bit(k, (uint32_t)i)) {
      xadd(c, &R0, &R1, x0m, &T0);
      xdbl(c, &R1, a24m, &T1);
    } else {
      xdbl(c, &R0, a24m, &T0);
      xadd(c, &R0, &R1, x0m, &T1);
    }
    R0 = T0;
    R1 = T1;
    TRACE_STATE();
  }
#undef TRACE_STATE
  *R0out = R0;
}

/* xADD with a projective difference D = (Xd:Zd) (reading G9b):
 * U=(X0-Z0)(X1+Z1), V=(X0+Z0)(X1-Z1), X'=Zd (U+V)^2, Z'=Xd (U-V)^2 */
static void xadd_d(const ctx_t *c, const pt_t *P0, const pt_t *P1, const pt_t *D, pt_t *out) {
  uint32_t U[ORC_MAXL], V[ORC_MAXL], w1[ORC_MAXL], w2[ORC_MAXL];
  msub(c, P0->X, P0->Z, w1); madd(c, P1->X, P1->Z, w2); mmul(c, w1, w2, U);
  madd(c, P0->X, P0->Z, w1); msub(c, P1->X, P1->Z, w2); mmul(c, w1, w2, V);
  madd(c, U, V, w1); mmul(c, w1, w1, w2); mmul(c, D->Z, w2, out->X);
  msub(c, U, V, w1); mmul(c, w1, w1, w2); mmul(c, D->X, w2, out->Z);
}

/* Q <- [p]Q by a Montgomery ladder with difference Q: R0 = Q, R1 = xDBL(Q), then the bits of p
 * below the top one, MSB first, as in ladder() (reading G9b). */
static void ladder_prime(const ctx_t *c, pt_t *Q, const uint32_t *a24m, uint32_t p) {
  pt_t D = *Q, R0 = *Q, R1, T0, T1;
  xdbl(c, &R0, a24m, &R1);
  int top = 31;
  while (!((p >> top) & 1)) --top;
  for (int i = top - 1; i >= 0; --i) {
    if ((p >> i) & 1) {
      xadd_d(c, &R0, &R1, &D, &T0);
      xdbl(c, &R1, a24m, &T1);
    } else {
      xdbl(c, &R0, a24m, &T0);
      xadd_d(c, &R0, &R1, &D, &T1);
    }
    R0 = T0;
    R1 = T1;
  }
  *Q = R0;
}

int orc_ecm_stage1_primes(const uint32_t *N, int L, uint64_t B1, const uint64_t *sigmas, size_t count,
                          uint32_t *X, uint32_t *Z, uint32_t *g, uint8_t *status, uint32_t *xaff) {
  if (!N || L < 1 || L > ORC_MAXL || !(N[0] & 1) || B1 < 2 || B1 > 0xffffffffull) return -1;
  /* the prime schedule: p ascending, each repeated e times with p^e <= B1 < p^(e+1) */
  char *comp = (char *)calloc((size_t)B1 + 1, 1);
  uint32_t *plist = (uint32_t *)malloc(sizeof(uint32_t) * ((size_t)B1 + 1));
  if (!comp || !plist) { free(comp); free(plist); return -1; }
  size_t np = 0;
  for (uint64_t p = 2; p <= B1; ++p) {
    if (comp[p]) continue;
    for (uint64_t m = p * p; m <= B1; m += p) comp[m] = 1;
    for (uint64_t q = p; q <= B1; q *= p) plist[np++] = (uint32_t)p;
  }
  free(comp);
  ctx_t c;
  ctx_init(&c, N, L);
  for (size_t i = 0; i < count; ++i) {
    uint32_t x0m[ORC_MAXL], a24m[ORC_MAXL], gg[ORC_MAXL], Xn[ORC_MAXL], Zn[ORC_MAXL], xa[ORC_MAXL];
    zero(gg, L); gg[0] = 1;
    zero(Xn, L); zero(Zn, L); zero(xa, L);
    int st = suyama_mont(&c, sigmas[i], x0m, a24m, gg);
    if (st == 0) {
      pt_t Q;
      copy(Q.X, x0m, L);
      small_mont(&c, 1, Q.Z);
      for (size_t j = 0; j < np; ++j) ladder_prime(&c, &Q, a24m, plist[j]);
      from_mont(&c, Q.X, Xn);
      from_mont(&c, Q.Z, Zn);
      uint32_t zi[ORC_MAXL];
      if (inv_gcd(Zn, c.n, L, gg, zi)) {
        uint32_t xm[ORC_MAXL], zim[ORC_MAXL], pm[ORC_MAXL];
        to_mont(&c, Xn, xm);
        to_mont(&c, zi, zim);
        mmul(&c, xm, zim, pm);
        from_mont(&c, pm, xa);
      }
      st = classify(gg, N, L);
    }
    if (X) copy(X + i * (size_t)L, Xn, L);
    if (Z) copy(Z + i * (size_t)L, Zn, L);
    if (g) copy(g + i * (size_t)L, gg, L);
    if (status) status[i] = (uint8_t)st;
    if (xaff) copy(xaff + i * (size_t)L, xa, L);
  }
  free(plist);
  return 0;
}

static int check_args(const uint32_t *N, int L, const uint32_t *k_words, uint32_t k_bits) {
  if (!N || L < 1 || L > ORC_MAXL || !(N[0] & 1) || !k_words || k_bits == 0) return -1;
  if (!bit(k_words, k_bits - 1)) return -1; /* k_bits must be exact */
  return 0;
}

/* One curve after its setup: ladder over k, tail, outputs written at index i. */
static void stage1_curve(const ctx_t *c, const uint32_t *N, const uint32_t *k_words, uint32_t k_bits, int st,
                         const uint32_t *x0m, const uint32_t *a24m, uint32_t *gg, size_t i, uint32_t *X,
                         uint32_t *Z, uint32_t *g, uint8_t *status, uint32_t *xaff) {
  int L = c->L;
  uint32_t Xn[ORC_MAXL], Zn[ORC_MAXL], xa[ORC_MAXL];
  zero(Xn, L); zero(Zn, L); zero(xa, L);
  if (st == 0) {
    pt_t R0;
    ladder(c, x0m, a24m, k_words, k_bits, &R0, NULL);
    from_mont(c, R0.X, Xn);
    from_mont(c, R0.Z, Zn);
    /* tail: the gcd of the final denominator gives the factor */
    uint32_t zi[ORC_MAXL];
    if (inv_gcd(Zn, c->n, L, gg, zi)) {
      uint32_t xm[ORC_MAXL], zim[ORC_MAXL], pm[ORC_MAXL];
      to_mont(c, Xn, xm);
      to_mont(c, zi, zim);
      mmul(c, xm, zim, pm);
      from_mont(c, pm, xa);
    }
    st = classify(gg, N, L);
  }
  if (X) copy(X + i * (size_t)L, Xn, L);
  if (Z) copy(Z + i * (size_t)L, Zn, L);
  if (g) copy(g + i * (size_t)L, gg, L);
  if (status) status[i] = (uint8_t)st;
  if (xaff) copy(xaff + i * (size_t)L, xa, L);
}

int orc_ecm_stage1(const uint32_t *N, int L, const uint32_t *k_words, uint32_t k_bits,
                   const uint64_t *sigmas, size_t count, uint32_t *X, uint32_t *Z, uint32_t *g,
                   uint8_t *status, uint32_t *xaff) {
  if (check_args(N, L, k_words, k_bits)) return -1;
  ctx_t c;
  ctx_init(&c, N, L);
  for (size_t i = 0; i < count; ++i) {
    uint32_t x0m[ORC_MAXL], a24m[ORC_MAXL], gg[ORC_MAXL];
    zero(gg, L); gg[0] = 1;
    int st = suyama_mont(&c, sigmas[i], x0m, a24m, gg);
    stage1_curve(&c, N, k_words, k_bits, st, x0m, a24m, gg, i, X, Z, g, status, xaff);
  }
  return 0;
}

/* Small-parameter family (reading G16 — not the paper's curves): for a seed
 * s in [1, 2^30), the curve B y^2 = x^3 + A x^2 + x with a24 = (A+2)/4 = s / 2^32 mod N and the
 * base point x0 = 2.  Out-of-range seeds get status 3 (no curve). */
static int small_mont_setup(const ctx_t *c, uint64_t s, uint32_t *x0m, uint32_t *a24m) {
  int L = c->L;
  if (s < 1 || s >= ((uint64_t)1 << 30)) return 3;
  uint32_t w[2] = {0u, 1u}, t[ORC_MAXL], inv[ORC_MAXL], g[ORC_MAXL], sm[ORC_MAXL], im[ORC_MAXL];
  mod_n(w, 2, c->n, t, L);                     /* 2^32 mod N */
  if (!inv_gcd(t, c->n, L, g, inv)) return 3;  /* N odd: never */
  small_mont(c, s, sm);                        /* s R        */
  to_mont(c, inv, im);                         /* 2^-32 R    */
  mmul(c, sm, im, a24m);                       /* a24 R = s 2^-32 R */
  small_mont(c, 2, x0m);                       /* x0 = 2     */
  return 0;
}

int orc_ecm_stage1_small(const uint32_t *N, int L, const uint32_t *k_words, uint32_t k_bits,
                         const uint64_t *seeds, size_t count, uint32_t *X, uint32_t *Z, uint32_t *g,
                         uint8_t *status, uint32_t *xaff) {
  if (check_args(N, L, k_words, k_bits)) return -1;
  ctx_t c;
  ctx_init(&c, N, L);
  for (size_t i = 0; i < count; ++i) {
    uint32_t x0m[ORC_MAXL], a24m[ORC_MAXL], gg[ORC_MAXL];
    zero(gg, L); gg[0] = 1;
    int st = small_mont_setup(&c, seeds[i], x0m, a24m);
    if (st) copy(gg, N, L); /* no curve: g = N */
    stage1_curve(&c, N, k_words, k_bits, st, x0m, a24m, gg, i, X, Z, g, status, xaff);
  }
  return 0;
}

int orc_ladder_trace(const uint32_t *N, int L, const uint32_t *k_words, uint32_t k_bits,
                     uint64_t sigma, uint32_t *trace) {
  if (check_args(N, L, k_words, k_bits) || !trace) return -1;
  ctx_t c;
  ctx_init(&c, N, L);
  uint32_t x0m[ORC_MAXL], a24m[ORC_MAXL], gg[ORC_MAXL];
  int st = suyama_mont(&c, sigma, x0m, a24m, gg);
  if (st) return st;
  pt_t R0;
  ladder(&c, x0m, a24m, k_words, k_bits, &R0, trace);
  return 0;
}
