/* ecmgpu.h — C ABI of libecmgpu: the data-parallel hot path of W. Trei, "Efficient Modular
 * Arithmetic for SIMD Devices" (arXiv 1310.3809), built for NVIDIA B200 (sm_100a).
 *
 * Two operations, following the paper's statement of the problem:
 *   ecm_mulmod_batch  — batched lazy Montgomery multiplication, one independent modulus and
 *                       operand set per lane (PAPER.md:93-104 REDC and residue system;
 *                       PAPER.md:174-189 Lemma / lazy reduction; PAPER.md:239-258 Theorem).
 *   ecm_stage1_batch  — ECM stage 1, one curve per thread on a shared N: "Calculate the
 *                       constant k ... Pick a random elliptic curve ... Calculate kP ... its gcd
 *                       gives a factor of n", Montgomery-form curves with the
 *                       Brent-Suyama parametrisation, one work item per curve
 *                       (PAPER.md:310-312).
 *
 * Conventions (all entry points)
 *   - Integers are little-endian arrays of uint32 limbs; L limbs per integer: L in {4,6,8,12,16}
 *     for every entry point ("b-bit" = 32L bits of storage, moduli of at most 32L-2 bits:
 *     PAPER.md:189; 510-bit moduli at L = 16, "510 bit arithmetic should work").
 *     R = 2^(32L).
 *   - Arrays of `count` integers are AoS by default: element i occupies words [i*L, i*L+L).
 *     With ECM_LAYOUT_SLICED (mulmod only) limb j of element i is at word [j*count + i].
 *   - Memory: the caller owns every buffer.  Array arguments are DEVICE pointers on the current
 *     device (16-byte aligned) unless ECM_HOST_BUFFERS is set, in which case they are host
 *     pointers (pinned memory recommended) and the library stages them through device scratch
 *     with copies on `stream` and synchronises the stream before returning.  `N_host` and
 *     `k_words` are always host pointers.
 *   - Execution: calls enqueue work on `stream` (a cudaStream_t; NULL = legacy default stream)
 *     and return without waiting, except with ECM_HOST_BUFFERS or ECM_CHECK.
 *   - Errors: no C++ exception crosses the ABI.  Argument errors return before anything is
 *     enqueued.  Outputs are unspecified when the return value is not ECM_OK.
 *   - Thread safety: calls may be made concurrently from several host threads; the only
 *     library state is a mutex-guarded cache of per-device scratch and scalar plans.
 */
#ifndef ECMGPU_H
#define ECMGPU_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ECM_OK = 0,
  ECM_E_ARG = 1,     /* null pointer, count == 0 or > 2^40, unsupported L, misaligned pointer, bad flags */
  ECM_E_MODULUS = 2, /* N even or N < 3 (ECM_CHECK for mulmod; always for stage 1) */
  ECM_E_WIDTH = 3,   /* bitlen(N) > 32L-2: no two spare bits */
  ECM_E_B1 = 4,      /* B1 < 2 or B1 >= 2^32, or k_bits == 0 */
  ECM_E_RANGE = 5,   /* an operand >= 2N (only detected with ECM_CHECK) */
  ECM_E_CUDA = 6,    /* a CUDA runtime error (launch failure, no device) */
  ECM_E_NOMEM = 7    /* device or host allocation failed */
} ecm_status;

/* flags */
#define ECM_CANONICAL 0x1u      /* mulmod: outputs reduced to [0, n_i) instead of lazy [0, 2n_i) */
#define ECM_SQUARE 0x2u         /* mulmod: x_{t+1} = REDC(x_t^2); b is ignored (may be NULL) */
#define ECM_LAYOUT_SLICED 0x4u  /* mulmod: limb-sliced layout [j*count + i] for a, b, n, out */
#define ECM_CHECK 0x8u          /* validate per-element preconditions on the device first */
#define ECM_HOST_BUFFERS 0x10u  /* array arguments are host pointers (see conventions) */
#define ECM_NO_XAFF 0x20u       /* stage 1: skip the affine x (xaff may then be NULL) */
#define ECM_EAGER 0x40u         /* stage 1, ablation (L = 6, 8): canonicalise after every product and
                                   reduce add/sub mod N — the paper's baseline without the lazy
                                   reduction of PAPER.md:172-191.  Outputs are identical. */
#define ECM_PRIME_LADDERS 0x80u /* stage 1 (L = 6, 8): the paper-comparable schedule (G9b) —
                                   Q <- [p]Q for every prime p <= B1 ascending, each e_p times, by
                                   ladders with a projective difference (11 products per step)
                                   instead of one ladder over k.  Same [k]P, status and affine x;
                                   X and Z differ by a projective factor. */
/* REDC variant (bits 8..10): all give the SAME raw lazy value, which is a function of (T, N, R).
   ecm_mulmod_batch accepts all five; ecm_stage1/ladder_batch accept WORD for every L and
   KNOWNLOW / BLOCKTHM / CLASSIC for L = 6 and 8 (ECM_E_ARG otherwise). */
#define ECM_REDC_WORD (0u << 8)     /* default: word-serial CIOS, fused IMAD.WIDE carry chains */
#define ECM_REDC_KNOWNLOW (1u << 8) /* the paper's Theorem per word: lo(m_i N_0) = -t_0 not multiplied */
#define ECM_REDC_BLOCKTHM (2u << 8) /* block SOS with the Theorem: 3 of 4 quadrant products of q*N */
#define ECM_REDC_CLASSIC (3u << 8)  /* block SOS, q*N as a full product (PAPER.md:93-99 as written) */
#define ECM_REDC_KARATSUBA (4u << 8) /* Karatsuba products; q*N with 2 instead of 3 half-size products by
                                        the paper's second Theorem — mulmod only */
#define ECM_REDC_MASK (7u << 8)
/* mulmod kernel choice (diagnostic; the default picks by `iters`): the CTA-tile
   streaming kernel (bulk-copy ring, the memory-bound regime, default for iters <= 4) or the
   warp-tile kernel (default for longer chains).  Outputs are identical.  Sliced layouts fall
   back to the warp-tile kernel unless count % 4 == 0 and every array is 16-byte aligned. */
#define ECM_KERNEL_STREAM 0x800u
#define ECM_KERNEL_WARP 0x1000u
/* stage 1 kernel choice (diagnostic; the default picks by batch size): one curve
   per thread (throughput kernel) or four lanes per curve (latency kernel: the ladder step's 10
   products as three rounds of independent products spread over the lanes of a 4-lane group,
   default for count <= 64 x SMs).  Outputs are identical.  LANES4 needs the default REDC_WORD
   lazy full-k ladder (ECM_E_ARG with ECM_EAGER, ECM_PRIME_LADDERS or another REDC variant). */
#define ECM_KERNEL_LANES4 0x2000u
#define ECM_KERNEL_LANES1 0x4000u
/* stage 1 curve family (NOT the paper's curves, reading G16): seed s_i
   in [1, 2^30) (passed in `sigmas`) selects B y^2 = x^3 + A x^2 + x with a24 = (A+2)/4 = s_i / 2^32
   mod N and base point x0 = 2, so a24*t is one word-level REDC and x0*t an addition (8 instead of
   10 full products per ladder step).  No setup inversion; a seed outside [1, 2^30) gives status
   ECM_CURVE_BAD_SIGMA with g = N.  Default lazy full-k ladder only (ECM_E_ARG with ECM_EAGER,
   ECM_PRIME_LADDERS or another REDC variant). */
#define ECM_CURVE_SMALL 0x8000u

/* Status values written per curve by ecm_stage1_batch / ecm_ladder_batch. */
#define ECM_CURVE_NO_FACTOR 0    /* g == 1 */
#define ECM_CURVE_FACTOR 1       /* 1 < g < N: g is a proper factor */
#define ECM_CURVE_ALL 2          /* g == N (Z == 0 mod every prime factor) */
#define ECM_CURVE_BAD_SIGMA 3    /* setup: gcd(16 u^3 v^4, N) == N */
#define ECM_CURVE_SETUP_FACTOR 4 /* setup: 1 < gcd(16 u^3 v^4, N) < N, g = that gcd */

/* ecm_mulmod_batch — batched lazy Montgomery multiplication chains.
 *   For each i < count, modulo n_i:  x_0 = a_i;  x_{t+1} = REDC(x_t * b_i)  (or REDC(x_t^2) with
 *   ECM_SQUARE);  out_i = x_iters.  REDC(T) = (T + q n_i)/R with q = T (-n_i^{-1}) mod R, the
 *   paper's Algorithm WITHOUT the final subtraction (lazy), so
 *   out_i is the unique raw value in [0, 2 n_i); with ECM_CANONICAL it is reduced to [0, n_i).
 *   iters >= 1 (iters = 1: one batched Montgomery product a_i b_i R^{-1}).
 *   Preconditions per element: n_i odd, bitlen(n_i) <= 32L-2, a_i < 2n_i, b_i < 2n_i.  They are
 *   validated only with ECM_CHECK (then ECM_E_MODULUS / ECM_E_WIDTH / ECM_E_RANGE are returned
 *   after a stream synchronisation and nothing else is launched).
 *   a, b, n, out: `count` integers each (b unused with ECM_SQUARE); out may alias a. */
ecm_status ecm_mulmod_batch(const uint32_t *a, const uint32_t *b, const uint32_t *n, uint32_t *out,
                            size_t count, int L, uint32_t iters, uint32_t flags, void *stream);

/* ecm_stage1_batch — ECM stage 1 on one shared N for `count` curves.
 *   N_host: host pointer to N (L limbs); N odd, N >= 3 (ECM_E_MODULUS), bitlen(N) <= 32L-2
 *   (ECM_E_WIDTH).  B1 in [2, 2^32) (ECM_E_B1); k = prod_{p<=B1} p^e, p^e <= B1 < p^(e+1).
 *   sigmas: `count` Suyama seeds (uint64, >= 6 recommended); curve i uses u = s^2-5, v = 4s,
 *   s = sigma_i mod N, x0 = u^3/v^3, a24 = (v-u)^3(3u+v)/(16u^3 v), P = (x0 : 1).
 *   The scalar multiple (X:Z) = [k]P is the R0 of the Montgomery ladder with the pinned
 *   schedule of DESIGN.md §3 (G9).  Outputs per curve (device arrays unless ECM_HOST_BUFFERS):
 *     X, Z   : L words each, canonical in [0, N), normal (non-Montgomery) domain
 *     g      : L words, gcd(Z, N) (N when Z == 0); for status 3/4 the setup gcd
 *     status : 1 byte, ECM_CURVE_*
 *     xaff   : L words, X/Z mod N when status == 0, else 0 (may be NULL with ECM_NO_XAFF)
 *   For status 3/4, X = Z = xaff = 0.  X, Z, g may be NULL when not wanted; status may not. */
ecm_status ecm_stage1_batch(const uint32_t *N_host, int L, uint64_t B1, const uint64_t *sigmas,
                            size_t count, uint32_t *X, uint32_t *Z, uint32_t *g, uint8_t *status,
                            uint32_t *xaff, uint32_t flags, void *stream);

/* ecm_ladder_batch — as ecm_stage1_batch with an explicit scalar k instead of B1:
 *   k_words: host pointer, little-endian words of k; k_bits = bitlen(k) >= 1 exactly
 *   (ECM_E_B1 otherwise).  Used to check [#E(F_p)]P = O on small p and prefix states. */
ecm_status ecm_ladder_batch(const uint32_t *N_host, int L, const uint32_t *k_words, uint32_t k_bits,
                            const uint64_t *sigmas, size_t count, uint32_t *X, uint32_t *Z,
                            uint32_t *g, uint8_t *status, uint32_t *xaff, uint32_t flags,
                            void *stream);

/* bit length of k(B1) (0 on bad B1); the plan the library uses, for callers that size work. */
uint32_t ecm_stage1_kbits(uint64_t B1);

/* Static description of an ecm_status. */
const char *ecm_strerror(ecm_status s);

/* Library build identity, e.g. "libecmgpu sm_100a <git-describe>". */
const char *ecm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ECMGPU_H */
