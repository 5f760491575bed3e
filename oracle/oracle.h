/* oracle.h — CPU reference ("oracle") for the hot path of W. Trei, "Efficient Modular
 * Arithmetic for SIMD Devices" (arXiv 1310.3809).
 *
 * THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load or call it.  It shares no code,
 * headers, tables or constants with the CUDA path (paper_1310_3809_b200/csrc); the only
 * thing both sides consume is the seeded input generator in workload/.
 *
 * Plain, slow, obviously correct: schoolbook 32-bit-limb integers, REDC exactly as the
 * paper's Algorithm "Montgomery Reduction", ECM stage 1 exactly as the
 * paper's Algorithm on Montgomery-form curves with the Brent-Suyama
 * parametrisation.  Readings of the paper where it is silent or garbled
 * are listed in DESIGN.md §3 (G1..G15) and cited at each function.
 *
 * Conventions: integers are little-endian arrays of uint32 limbs, L limbs (L <= ORC_MAXL),
 * R = 2^(32L) (reading G2), bitlen(N) <= 32L-2 for the lazy routines (reading G3).
 * Arrays of many integers are "AoS": element i occupies words [i*L, i*L+L).
 */
#ifndef ECM_ORACLE_H
#define ECM_ORACLE_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAXL 16

/* ---- multiprecision primitives (PAPER.md:112-116 schoolbook) ---- */
/* t[0..2L) = a*b, schoolbook over 32-bit words. */
void orc_mul(const uint32_t *a, const uint32_t *b, uint32_t *t, int L);
/* np = -n^{-1} mod R (the paper's m').  n must be odd. */
void orc_nprime(const uint32_t *n, uint32_t *np, int L);
/* out = (T + q*n)/R with q = (T mod R)*np mod R: steps 1-2 of PAPER.md:97-98, WITHOUT the
 * final subtraction of step 3 (lazy).  T has 2L words, out has L words; the
 * result must fit L words (true when T < R*n, e.g. T = x*y with x, y < 2n and R >= 4n). */
void orc_redc_raw(const uint32_t *T, const uint32_t *n, const uint32_t *np, uint32_t *out, int L);
/* full algorithm incl. step 3: out in [0, n). Requires T < R*n. */
void orc_redc(const uint32_t *T, const uint32_t *n, const uint32_t *np, uint32_t *out, int L);

/* ---- batched mulmod chain (SURVEY §8(b) ecm_mulmod_batch semantics) ----
 * For each i: x_0 = a_i, x_{t+1} = redc_raw(x_t * b_i) (or redc_raw(x_t^2) if square),
 * out_i = x_iters; canonical != 0 subtracts n_i once if out_i >= n_i. */
void orc_mulmod_chain(const uint32_t *a, const uint32_t *b, const uint32_t *n, uint32_t *out,
                      size_t count, int L, uint32_t iters, int square, int canonical);

/* ---- lazy add / sub in [0, 2n) (reading G4) ---- */
void orc_add_lazy(const uint32_t *x, const uint32_t *y, const uint32_t *n, uint32_t *out, int L);
void orc_sub_lazy(const uint32_t *x, const uint32_t *y, const uint32_t *n, uint32_t *out, int L);

/* ---- ECM stage 1 ---- */
/* k = prod_{p prime <= B1} p^e, p^e <= B1 < p^(e+1) (reading G8).
 * Writes k little-endian into k_words (capacity cap words); returns bit length of k, or 0 if
 * the capacity is too small or B1 < 2. */
uint32_t orc_stage1_k(uint64_t B1, uint32_t *k_words, size_t cap);

/* Stage 1 on one shared odd N (L limbs) for count curves with Suyama seeds sigmas[i].
 * Scalar k given as little-endian words with k_bits significant bits (k >= 1).
 * Per curve outputs (any output pointer may be NULL):
 *   X, Z   : R0 of the ladder, canonical in [0, N), normal (non-Montgomery) domain
 *   g      : gcd(Z, N) (g = N when Z == 0); for status 3/4 the setup gcd
 *   status : 0 no factor, 1 factor (1<g<N), 2 g == N, 3 setup gcd == N, 4 setup factor
 *   xaff   : X/Z mod N when status == 0, else 0
 * For status 3/4, X = Z = xaff = 0.  Returns 0, or -1 on bad arguments. */
int orc_ecm_stage1(const uint32_t *N, int L, const uint32_t *k_words, uint32_t k_bits,
                   const uint64_t *sigmas, size_t count, uint32_t *X, uint32_t *Z, uint32_t *g,
                   uint8_t *status, uint32_t *xaff);

/* Stage 1 with the paper-comparable schedule (reading G9b): instead of one
 * ladder over k, Q <- [p]Q for every prime p <= B1 in ascending order, each repeated e_p times
 * (p^e_p <= B1), each by a Montgomery ladder whose differential addition uses the projective
 * difference Q (11 products per step).  Same outputs/conventions as orc_ecm_stage1; [k]P and so
 * xaff and status equal orc_ecm_stage1's, X and Z differ by a projective factor. */
int orc_ecm_stage1_primes(const uint32_t *N, int L, uint64_t B1, const uint64_t *sigmas, size_t count,
                          uint32_t *X, uint32_t *Z, uint32_t *g, uint8_t *status, uint32_t *xaff);

/* Stage 1 on the small-parameter family (reading G16 — not the paper's curve
 * model): seed s in [1, 2^30) gives a24 = s / 2^32 mod N and x0 = 2; same ladder, tail and
 * outputs as orc_ecm_stage1.  A seed outside [1, 2^30) gives status 3 with g = N. */
int orc_ecm_stage1_small(const uint32_t *N, int L, const uint32_t *k_words, uint32_t k_bits,
                         const uint64_t *seeds, size_t count, uint32_t *X, uint32_t *Z, uint32_t *g,
                         uint8_t *status, uint32_t *xaff);

/* Suyama setup only (reading G10): returns status 0/3/4; on 0 writes the
 * canonical normal-domain x0 = u^3/v^3 and a24 = (v-u)^3(3u+v)/(16u^3 v). */
int orc_suyama(const uint32_t *N, int L, uint64_t sigma, uint32_t *x0, uint32_t *a24, uint32_t *g);

/* Ladder with a trace: like orc_ecm_stage1 for one curve, but also writes the canonical
 * normal-domain ladder state (X0,Z0,X1,Z1) after the initial doubling and after every step
 * into trace (4*L words per state, k_bits states).  Used by the per-step invariant test
 * (SURVEY §8(c) c6(i)).  Returns the setup status. */
int orc_ladder_trace(const uint32_t *N, int L, const uint32_t *k_words, uint32_t k_bits,
                     uint64_t sigma, uint32_t *trace);

#ifdef __cplusplus
}
#endif
#endif
