#pragma once
// ecm_kernels.cuh — ECM stage 1, one curve per thread, sm_100a.
//
// Per thread (one curve, no inter-thread synchronisation: PAPER.md:312):
//   setup  : Brent-Suyama curve from sigma (formulas: DESIGN.md reading G10)
//            u = s^2-5, v = 4s, D = 16u^3v^4, one inversion w = D^{-1} (per-thread binary
//            extended gcd), x0 = 16u^6 v w, a24 = (v-u)^3(3u+v) v^3 w.  gcd(D, N) != 1 ->
//            status 3 / 4 (the setup denominator "is not invertible").
//   ladder : R0 = (x0:1), R1 = xDBL(R0); for each further bit of k (MSB first) one combined
//            xADD + xDBL step, 6M + 4S + 8 lazy add/sub.  k is shared by every
//            curve, so the bit is warp-uniform: the conditional swap is a uniform select and
//            the k words are broadcast across the warp with __shfl_sync.
//   tail   : X, Z out of Montgomery form, canonical; g = gcd(Z, N) by the same binary extended
//            gcd, which also yields Z^{-1} for the affine x = X/Z ("its gcd gives a factor of n",
//            PAPER.md:302).
// N, 2N, R^2 mod N, R mod N and -N^{-1} mod 2^32 are shared by all curves and live in the kernel
// parameter (constant) bank, so the hot loop reads N directly as IMAD constant operands.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"
#include "mont.cuh"

namespace ecm {

constexpr int kEcmTPB = 128;
// Build-time experiment knobs (tools/ecm_ab.py builds variant libraries; defaults = the product):
//   ECM_MIN_BLOCKS  : __launch_bounds__ min CTAs/SM for the ladder kernel (0 = unconstrained)
//   ECM_SWAP_BRANCH : 1 = no conditional swap; a warp-uniform branch picks which slot is doubled
#ifndef ECM_MIN_BLOCKS
#define ECM_MIN_BLOCKS -1  // -1: ecm_min_blocks' per-instantiation default
#endif
#ifndef ECM_SWAP_BRANCH
#define ECM_SWAP_BRANCH 0
#endif
//   ECM_SWAP_SEL    : 1 = no state swap; the doubling's input sums are selected (ladder_step_sel,
//                     2L instead of 4L selects per step); 0 = conditional swap; -1 = per-width default
#ifndef ECM_SWAP_SEL
#define ECM_SWAP_SEL -1
#endif
//   ECM_LADDER_SQR  : square form in the ladder (mont_sqr FORM; -1 = per-width default below)
#ifndef ECM_LADDER_SQR
#define ECM_LADDER_SQR -1
#endif
// Per-width ladder forms, each the measured best (tools/ecm_ab.py, profiles/r02b/e/f/i_ab*.jsonl): the
// swap-free step at L <= 8 (L = 12 and 16 keep the conditional swap: their 168 / 254-register ladders
// schedule worse with the extra live sums, -11 % / -5 %); the square on offset chains (mont.cuh FORMs
// 2..5) instead of rows: FORM 4 at L = 4 and 8, FORM 3 at L = 6 and 16, FORM 5 at L = 12 — against the
// round-1 row forms about +3.6 / +0.9 / +2.6 / +3.4 / +1.7 % curves/s at L = 4 / 6 / 8 / 12 / 16 (across
// boxes, +-1 %).
__host__ __device__ constexpr bool ladder_swap_sel(int L) { return ECM_SWAP_SEL >= 0 ? ECM_SWAP_SEL != 0 : L <= 8; }
__host__ __device__ constexpr int ladder_sqr_form(int L) {
  return ECM_LADDER_SQR >= 0 ? ECM_LADDER_SQR : (L == 4 || L == 8) ? 4 : L == 12 ? 5 : 3;
}
//   ECM_MULADD      : 1 = d + a24 t as one REDC frame with d injected (Field::mul_add)
#ifndef ECM_MULADD
#define ECM_MULADD 0
#endif
//   ECM_CONST_SMEM  : 1 = x0 and a24 live in shared memory during the ladder (loaded per use)
#ifndef ECM_CONST_SMEM
#define ECM_CONST_SMEM 0
#endif
//   ECM_LADDER_UNROLL : unroll factor of the one-lane ladder loop
//   ECM_SQR_CANON   : 1 = the ladder squares canonicalise their input and use the CIOS square
#ifndef ECM_SQR_CANON
#define ECM_SQR_CANON 0
#endif
#ifndef ECM_LADDER_UNROLL
#define ECM_LADDER_UNROLL 1
#endif
constexpr int kLadderUnroll = ECM_LADDER_UNROLL;
// Occupancy of the default ladder (tools/ecm_ab.py, profiles/r01_ecm_ab.jsonl): L <= 6 is held to
// 80 registers = 6 CTAs x 4 warps per SM (at 81..88 the 256-register warp allocation granule leaves
// 5; the cap costs one spill load per step); L = 12 to 168 = 3 CTAs (+6 % over 182 registers and 2
// CTAs, no spills).  L = 8 (138 registers, 3 CTAs) measured the same at 4 CTAs; L = 4 and 16 are
// left to ptxas.
__host__ __device__ constexpr int ecm_min_blocks(int L, int V, bool eager, bool primes) {
  return ECM_MIN_BLOCKS >= 0 ? ECM_MIN_BLOCKS
         : (V != 0 || eager || primes) ? 0
         : L <= 6 ? 6 : L == 12 ? 3 : 0;
}

template <int L>
__device__ __forceinline__ const uint32_t (&cref(const uint32_t* p))[L] {
  return *reinterpret_cast<const uint32_t(*)[L]>(p);
}

template <int L>
__device__ __forceinline__ void copy(uint32_t (&d)[L], const uint32_t (&s)[L]) {
#pragma unroll
  for (int k = 0; k < L; ++k) d[k] = s[k];
}

template <int L>
__device__ __forceinline__ bool is_zero(const uint32_t (&a)[L]) {
  uint32_t o = 0;
#pragma unroll
  for (int k = 0; k < L; ++k) o |= a[k];
  return o == 0;
}

template <int L>
__device__ __forceinline__ bool is_one(const uint32_t (&a)[L]) {
  uint32_t o = a[0] ^ 1u;
#pragma unroll
  for (int k = 1; k < L; ++k) o |= a[k];
  return o == 0;
}

template <int L>
__device__ __forceinline__ bool equal(const uint32_t (&a)[L], const uint32_t (&b)[L]) {
  uint32_t o = 0;
#pragma unroll
  for (int k = 0; k < L; ++k) o |= a[k] ^ b[k];
  return o == 0;
}

// a >= b ?
template <int L>
__device__ __forceinline__ bool geq(const uint32_t (&a)[L], const uint32_t (&b)[L]) {
  (void)ptx::sub_cc(a[0], b[0]);
#pragma unroll
  for (int k = 1; k < L; ++k) (void)ptx::subc_cc(a[k], b[k]);
  return ptx::subc(0u, 0u) == 0u;
}

template <int L>
__device__ __forceinline__ void sub_plain(uint32_t (&d)[L], const uint32_t (&a)[L], const uint32_t (&b)[L]) {
  d[0] = ptx::sub_cc(a[0], b[0]);
#pragma unroll
  for (int k = 1; k < L - 1; ++k) d[k] = ptx::subc_cc(a[k], b[k]);
  d[L - 1] = ptx::subc(a[L - 1], b[L - 1]);
}

// x = x/2 mod N for x < N (N odd): add N when x is odd, then shift the (L*32+1)-bit sum.
template <int L>
__device__ __forceinline__ void half_mod(uint32_t (&x)[L], const uint32_t (&N)[L]) {
  const uint32_t mask = 0u - (x[0] & 1u);
  uint32_t s[L];
  s[0] = ptx::add_cc(x[0], N[0] & mask);
#pragma unroll
  for (int k = 1; k < L; ++k) s[k] = ptx::addc_cc(x[k], N[k] & mask);
  const uint32_t top = ptx::addc(0u, 0u);
#pragma unroll
  for (int k = 0; k < L - 1; ++k) x[k] = __funnelshift_r(s[k], s[k + 1], 1);
  x[L - 1] = __funnelshift_r(s[L - 1], top, 1);
}

template <int L>
__device__ __forceinline__ void shr1(uint32_t (&x)[L]) {
#pragma unroll
  for (int k = 0; k < L - 1; ++k) x[k] = __funnelshift_r(x[k], x[k + 1], 1);
  x[L - 1] >>= 1;
}

// d = a - b mod N for a, b < N
template <int L>
__device__ __forceinline__ void sub_modN(uint32_t (&d)[L], const uint32_t (&a)[L], const uint32_t (&b)[L],
                                         const uint32_t (&N)[L]) {
  uint32_t t[L];
  t[0] = ptx::sub_cc(a[0], b[0]);
#pragma unroll
  for (int k = 1; k < L; ++k) t[k] = ptx::subc_cc(a[k], b[k]);
  const uint32_t mask = ptx::subc(0u, 0u);
  d[0] = ptx::add_cc(t[0], N[0] & mask);
#pragma unroll
  for (int k = 1; k < L - 1; ++k) d[k] = ptx::addc_cc(t[k], N[k] & mask);
  d[L - 1] = ptx::addc(t[L - 1], N[L - 1] & mask);
}

// Constant-iteration binary extended gcd, no data-dependent branch (PAPER.md:152-154 asks SIMD
// code to avoid them; the lanes of a warp hold different curves):
//   u = a, v = N (odd), A = 1, C = 0 with A a = u, C a = v (mod N).  Each iteration
//     if u odd:  if u < v: (u, A) <-> (v, C);  u -= v;  A -= C (mod N)       [masks and selects]
//     u /= 2;  A /= 2 (mod N)
//   keeps v odd.  While u != 0 every iteration lowers bitlen(u) + bitlen(v) (<= 2 bitlen(N)
//   initially, >= 2 while u != 0) by at least one, so after 64L - 4 >= 2(32L - 2) iterations
//   u = 0; from then on v and C no longer change: v = gcd(a, N) and, if v = 1, C = a^{-1} mod N.
// a < N canonical (a = 0 gives g = N).  Returns true iff invertible.  The trip count is the same
// for every lane (setup and tail only).
template <int L>
__device__ bool xgcd(const uint32_t (&a)[L], const uint32_t (&N)[L], uint32_t (&g)[L], uint32_t (&inv)[L]) {
  uint32_t u[L], v[L], A[L], C[L];
  copy(u, a);
  copy(v, N);
#pragma unroll
  for (int k = 0; k < L; ++k) { A[k] = 0; C[k] = 0; }
  A[0] = 1;
#pragma unroll 1
  for (int it = 0; it < 64 * L - 4; ++it) {
    const uint32_t odd = 0u - (u[0] & 1u);
    (void)ptx::sub_cc(u[0], v[0]);
#pragma unroll
    for (int k = 1; k < L; ++k) (void)ptx::subc_cc(u[k], v[k]);
    const uint32_t sw = odd & ptx::subc(0u, 0u);  // u odd and u < v
#pragma unroll
    for (int k = 0; k < L; ++k) {
      const uint32_t du = (u[k] ^ v[k]) & sw, dA = (A[k] ^ C[k]) & sw;
      u[k] ^= du;
      v[k] ^= du;
      A[k] ^= dA;
      C[k] ^= dA;
    }
    // u -= v (u >= v now), A -= C (mod N): both only when u was odd
    u[0] = ptx::sub_cc(u[0], v[0] & odd);
#pragma unroll
    for (int k = 1; k < L - 1; ++k) u[k] = ptx::subc_cc(u[k], v[k] & odd);
    u[L - 1] = ptx::subc(u[L - 1], v[L - 1] & odd);
    uint32_t t[L];
    t[0] = ptx::sub_cc(A[0], C[0] & odd);
#pragma unroll
    for (int k = 1; k < L; ++k) t[k] = ptx::subc_cc(A[k], C[k] & odd);
    const uint32_t br = ptx::subc(0u, 0u);
    A[0] = ptx::add_cc(t[0], N[0] & br);
#pragma unroll
    for (int k = 1; k < L - 1; ++k) A[k] = ptx::addc_cc(t[k], N[k] & br);
    A[L - 1] = ptx::addc(t[L - 1], N[L - 1] & br);
    shr1(u);
    half_mod(A, N);
  }
  copy(g, v);
  copy(inv, C);
  return is_one(v);
}

// d = m ? a : b for an all-ones / zero mask m
template <int L>
__device__ __forceinline__ void select(uint32_t (&d)[L], uint32_t m, const uint32_t (&a)[L], const uint32_t (&b)[L]) {
#pragma unroll
  for (int k = 0; k < L; ++k) d[k] = (a[k] & m) | (b[k] & ~m);
}

// ---------------------------------------------------------------------------------------
// Field products of the ladder, templated for the paper's ablation (Table 5 analogue, §8(f) N1):
//   V     : REDC variant (mont.cuh); all give the same raw value.
//   EAGER : canonicalise after every product and reduce add/sub modulo N (the "without
//           Section 2.2" baseline: 18 conditional reductions per step instead of 8).
// ---------------------------------------------------------------------------------------
template <int L, int V, bool EAGER>
struct Field {
  const uint32_t (&N)[L];
  const uint32_t (&M)[L];   // add/sub modulus: 2N (lazy) or N (eager)
  const uint32_t (&NP)[L];  // -N^{-1} mod R (block variants)
  uint32_t n0inv;
  __device__ __forceinline__ void mul(uint32_t (&r)[L], const uint32_t (&x)[L], const uint32_t (&y)[L]) const {
    if (V == REDC_WORD || V == REDC_KNOWNLOW) mont_mul_cios<L, V>(r, x, y, N, n0inv);
    else mont_mul_block<L, V>(r, x, y, N, NP);
    debug_lazy_bound<L>(r, N);
    if (EAGER) canonicalize<L>(r, r, N);
  }
  __device__ __forceinline__ void sqr(uint32_t (&r)[L], const uint32_t (&x)[L]) const {
    if (V == REDC_WORD && ECM_SQR_CANON) {
      uint32_t xc[L];
      canonicalize<L>(xc, x, N);  // x < N: the CIOS square's bound holds
      mont_sqr_cios<L>(r, xc, N, n0inv);
    } else if (V == REDC_WORD) mont_sqr<L, ladder_sqr_form(L)>(r, x, N, n0inv);
    else if (V == REDC_KNOWNLOW) mont_mul_cios<L, V>(r, x, x, N, n0inv);
    else mont_mul_block<L, V>(r, x, x, N, NP);
    debug_lazy_bound<L>(r, N);
    if (EAGER) canonicalize<L>(r, r, N);
  }
  __device__ __forceinline__ void add(uint32_t (&r)[L], const uint32_t (&x)[L], const uint32_t (&y)[L]) const {
    add_lazy<L>(r, x, y, M);
  }
  // r = d + x y: with ECM_MULADD the addend enters the product's REDC frame (mont_mul_add, no add
  // instructions) and only the conditional subtraction of 2N remains
  __device__ __forceinline__ void mul_add(uint32_t (&r)[L], const uint32_t (&x)[L], const uint32_t (&y)[L],
                                          const uint32_t (&d)[L]) const {
    if constexpr (V == REDC_WORD && !EAGER && ECM_MULADD != 0) {
      mont_mul_add<L>(r, x, y, d, N, n0inv);
      reduce_2n<L>(r, M);
      debug_lazy_bound<L>(r, N);
    } else {
      uint32_t t[L];
      mul(t, x, y);
      add(r, d, t);
    }
  }
  __device__ __forceinline__ void sub(uint32_t (&r)[L], const uint32_t (&x)[L], const uint32_t (&y)[L]) const {
    sub_lazy<L>(r, x, y, M);
  }
};

// ---------------------------------------------------------------------------------------
// One combined ladder step on (X0:Z0) [doubled] and (X1:Z1) [added], difference (x0:1):
//   t1 = X0+Z0, t2 = X0-Z0, t3 = X1+Z1, t4 = X1-Z1
//   U = t2 t3, V = t1 t4, s = t1^2, d = t2^2
//   X0' = s d,  t = s - d,  Z0' = t (d + a24 t)
//   X1' = (U+V)^2,  Z1' = x0 (U-V)^2
// ---------------------------------------------------------------------------------------
template <int L, class F>
__device__ __forceinline__ void ladder_step(uint32_t (&X0)[L], uint32_t (&Z0)[L], uint32_t (&X1)[L],
                                            uint32_t (&Z1)[L], const uint32_t (&x0)[L], const uint32_t (&a24)[L],
                                            const F& f) {
  uint32_t t1[L], t2[L], t3[L], t4[L], U[L], V[L], s[L], d[L];
  f.add(t1, X0, Z0);
  f.sub(t2, X0, Z0);
  f.add(t3, X1, Z1);
  f.sub(t4, X1, Z1);
  f.mul(U, t2, t3);
  f.mul(V, t1, t4);
  f.sqr(s, t1);
  f.sqr(d, t2);
  f.mul(X0, s, d);
  f.sub(t1, s, d);   // t
  f.mul_add(t2, a24, t1, d);  // d + a24 t
  f.mul(Z0, t1, t2);
  f.add(t3, U, V);
  f.sub(t4, U, V);
  f.sqr(X1, t3);
  f.sqr(t4, t4);
  f.mul(Z1, x0, t4);
}

// The same step without a state swap: the slots are not exchanged; `c` picks which slot's sums
// (t1, t2) or (t3, t4) feed the doubling.  The addition is symmetric in its two inputs — swapping
// the slots exchanges U and V, leaves U + V and flips the sign of U - V, which is squared — so the
// doubled point always lands in slot 0 and the sum in slot 1: 2L selects per step instead of the
// 4L of a conditional swap of (X0:Z0) and (X1:Z1).  Every product is congruent mod N to the one
// ladder_step computes, so the canonical outputs are identical.
template <int L, class F>
__device__ __forceinline__ void ladder_step_sel(uint32_t (&X0)[L], uint32_t (&Z0)[L], uint32_t (&X1)[L],
                                                uint32_t (&Z1)[L], const uint32_t (&x0)[L], const uint32_t (&a24)[L],
                                                const F& f, bool c) {
  uint32_t t1[L], t2[L], t3[L], t4[L], U[L], V[L], s[L], d[L];
  f.add(t1, X0, Z0);
  f.sub(t2, X0, Z0);
  f.add(t3, X1, Z1);
  f.sub(t4, X1, Z1);
  f.mul(U, t2, t3);
  f.mul(V, t1, t4);
#pragma unroll
  for (int k = 0; k < L; ++k) {
    t1[k] = c ? t3[k] : t1[k];
    t2[k] = c ? t4[k] : t2[k];
  }
  f.sqr(s, t1);
  f.sqr(d, t2);
  f.mul(X0, s, d);
  f.sub(t1, s, d);   // t
  f.mul_add(t2, a24, t1, d);  // d + a24 t
  f.mul(Z0, t1, t2);
  f.add(t3, U, V);
  f.sub(t4, U, V);
  f.sqr(X1, t3);
  f.sqr(t4, t4);
  f.mul(Z1, x0, t4);
}

// ECM_CONST_SMEM: the step with x0 and a24 read from shared memory ([word][thread], conflict-free)
// right before their products, so they are not live in registers across the step.
__device__ __forceinline__ uint32_t lds_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)));
  return v;
}
template <int L, int TPB>
__device__ __forceinline__ void lds_res(uint32_t (&d)[L], const uint32_t* base) {
#pragma unroll
  for (int k = 0; k < L; ++k) d[k] = lds_u32(base + k * TPB);
}
// SEL: the swap-free form of ladder_step_sel (`csel` picks the doubling's input sums).
template <int L, int TPB, bool SEL = false, class F>
__device__ __forceinline__ void ladder_step_sm(uint32_t (&X0)[L], uint32_t (&Z0)[L], uint32_t (&X1)[L],
                                               uint32_t (&Z1)[L], const uint32_t* sx0, const uint32_t* sa24,
                                               const F& f, bool csel = false) {
  uint32_t t1[L], t2[L], t3[L], t4[L], U[L], V[L], s[L], d[L], c[L];
  f.add(t1, X0, Z0);
  f.sub(t2, X0, Z0);
  f.add(t3, X1, Z1);
  f.sub(t4, X1, Z1);
  f.mul(U, t2, t3);
  f.mul(V, t1, t4);
  if constexpr (SEL) {
#pragma unroll
    for (int k = 0; k < L; ++k) {
      t1[k] = csel ? t3[k] : t1[k];
      t2[k] = csel ? t4[k] : t2[k];
    }
  }
  f.sqr(s, t1);
  f.sqr(d, t2);
  f.mul(X0, s, d);
  f.sub(t1, s, d);
  lds_res<L, TPB>(c, sa24);
  f.mul(t2, c, t1);
  f.add(t2, d, t2);
  f.mul(Z0, t1, t2);
  f.add(t3, U, V);
  f.sub(t4, U, V);
  f.sqr(X1, t3);
  f.sqr(t4, t4);
  lds_res<L, TPB>(c, sx0);
  f.mul(Z1, c, t4);
}

// The step on the small-parameter family (FAM 1): a24 t = c t / 2^32 by one word-level REDC
// (mont_smul, 2L products) and x0 (U-V)^2 = 2 (U-V)^2 by a lazy addition — 8 full products per step.
template <int L, class F>
__device__ __forceinline__ void ladder_step_small(uint32_t (&X0)[L], uint32_t (&Z0)[L], uint32_t (&X1)[L],
                                                  uint32_t (&Z1)[L], uint32_t c, const uint32_t (&N)[L],
                                                  uint32_t n0inv, const F& f) {
  uint32_t t1[L], t2[L], t3[L], t4[L], U[L], V[L], s[L], d[L];
  f.add(t1, X0, Z0);
  f.sub(t2, X0, Z0);
  f.add(t3, X1, Z1);
  f.sub(t4, X1, Z1);
  f.mul(U, t2, t3);
  f.mul(V, t1, t4);
  f.sqr(s, t1);
  f.sqr(d, t2);
  f.mul(X0, s, d);
  f.sub(t1, s, d);                  // t
  mont_smul<L>(t2, c, t1, N, n0inv);  // a24 t
  f.add(t2, d, t2);                 // d + a24 t
  f.mul(Z0, t1, t2);
  f.add(t3, U, V);
  f.sub(t4, U, V);
  f.sqr(X1, t3);
  f.sqr(t4, t4);
  f.add(Z1, t4, t4);                // x0 (U-V)^2 with x0 = 2
}

// The same step with a projective difference D = (Xd:Zd) (the paper-comparable prime-by-prime
// schedule, reading G9b): X1' = Zd (U+V)^2, Z1' = Xd (U-V)^2 — 7M + 4S.
template <int L, class F>
__device__ __forceinline__ void ladder_step_d(uint32_t (&X0)[L], uint32_t (&Z0)[L], uint32_t (&X1)[L],
                                              uint32_t (&Z1)[L], const uint32_t (&Xd)[L], const uint32_t (&Zd)[L],
                                              const uint32_t (&a24)[L], const F& f) {
  uint32_t t1[L], t2[L], t3[L], t4[L], U[L], V[L], s[L], d[L];
  f.add(t1, X0, Z0);
  f.sub(t2, X0, Z0);
  f.add(t3, X1, Z1);
  f.sub(t4, X1, Z1);
  f.mul(U, t2, t3);
  f.mul(V, t1, t4);
  f.sqr(s, t1);
  f.sqr(d, t2);
  f.mul(X0, s, d);
  f.sub(t1, s, d);
  f.mul(t2, a24, t1);
  f.add(t2, d, t2);
  f.mul(Z0, t1, t2);
  f.add(t3, U, V);
  f.sub(t4, U, V);
  f.sqr(t3, t3);
  f.sqr(t4, t4);
  f.mul(X1, Zd, t3);
  f.mul(Z1, Xd, t4);
}

template <int L, class F>
__device__ __forceinline__ void xdbl(uint32_t (&Xo)[L], uint32_t (&Zo)[L], const uint32_t (&X)[L], const uint32_t (&Z)[L],
                                     const uint32_t (&a24)[L], const F& f) {
  uint32_t t1[L], t2[L], sd[L], dd[L], tt[L];
  f.add(t1, X, Z);
  f.sub(t2, X, Z);
  f.sqr(sd, t1);
  f.sqr(dd, t2);
  f.mul(Xo, sd, dd);
  f.sub(tt, sd, dd);
  f.mul(t1, a24, tt);
  f.add(t1, dd, t1);
  f.mul(Zo, tt, t1);
}

template <int L>
__device__ __forceinline__ void cswap(uint32_t (&a)[L], uint32_t (&b)[L], bool c) {
#pragma unroll
  for (int k = 0; k < L; ++k) {
    const uint32_t ta = c ? b[k] : a[k];
    const uint32_t tb = c ? a[k] : b[k];
    a[k] = ta;
    b[k] = tb;
  }
}

// curve i's L words when `on` (a predicated store; dst == nullptr: not wanted, kernel-uniform)
template <int L>
__device__ __forceinline__ void store_if(uint32_t* dst, size_t i, const uint32_t (&v)[L], bool on) {
  if (!dst) return;
  uint2* d2 = reinterpret_cast<uint2*>(dst + i * L);
#pragma unroll
  for (int k = 0; k < L / 2; ++k)
    if (on) d2[k] = make_uint2(v[2 * k], v[2 * k + 1]);
}

// ---------------------------------------------------------------------------------------
// Setup (Brent-Suyama, reading G10): sigma -> (x0, a24) in Montgomery form; gg = gcd(D, N) when
// the setup denominator D = 16 u^3 v^4 is not invertible (status 3 / 4).
// ---------------------------------------------------------------------------------------
template <int L>
__device__ __forceinline__ uint8_t ecm_setup(const EcmParams& p, uint64_t sigma, uint32_t (&x0)[L], uint32_t (&a24)[L],
                                             uint32_t (&gg)[L]) {
  const uint32_t(&N)[L] = cref<L>(p.N);
  const uint32_t(&N2)[L] = cref<L>(p.N2);
  const uint32_t(&R2)[L] = cref<L>(p.R2);
  const uint32_t(&ONE)[L] = cref<L>(p.ONE);
  const uint32_t n0inv = p.n0inv;
  uint32_t s[L], u[L], v[L], t[L], w[L], c[L];
#pragma unroll
  for (int k = 0; k < L; ++k) t[k] = 0;
  t[0] = (uint32_t)sigma;
  t[1] = (uint32_t)(sigma >> 32);
  mont_mul<L>(s, t, R2, N, n0inv);                 // s = sigma R mod N (any sigma < 2^64)
  // small Montgomery constants from ONE by lazy additions: 2, 4, 5, 3, 16
  uint32_t two[L], four[L], five[L], three[L], sixteen[L];
  add_lazy<L>(two, ONE, ONE, N2);
  add_lazy<L>(four, two, two, N2);
  add_lazy<L>(five, four, ONE, N2);
  add_lazy<L>(three, two, ONE, N2);
  add_lazy<L>(t, four, four, N2);
  add_lazy<L>(sixteen, t, t, N2);
  mont_mul<L>(t, s, s, N, n0inv);
  sub_lazy<L>(u, t, five, N2);                     // u = s^2 - 5
  add_lazy<L>(t, s, s, N2);
  add_lazy<L>(v, t, t, N2);                        // v = 4 s
  uint32_t u3[L], v3[L], D[L];
  mont_mul<L>(t, u, u, N, n0inv);
  mont_mul<L>(u3, t, u, N, n0inv);                 // u^3
  mont_mul<L>(t, v, v, N, n0inv);
  mont_mul<L>(v3, t, v, N, n0inv);                 // v^3
  mont_mul<L>(t, sixteen, u3, N, n0inv);           // 16 u^3
  mont_mul<L>(w, t, v3, N, n0inv);
  mont_mul<L>(D, w, v, N, n0inv);                  // D = 16 u^3 v^4
  // D out of Montgomery form, canonical, then invert
  uint32_t Dn[L], Di[L];
#pragma unroll
  for (int k = 0; k < L; ++k) c[k] = 0;
  c[0] = 1;
  mont_mul<L>(Dn, D, c, N, n0inv);
  canonicalize<L>(Dn, Dn, N);
  const bool ok = xgcd<L>(Dn, N, gg, Di);
  // both outcomes are computed and selected (no divergent branch): with D not invertible the
  // curve's (x0, a24) = (1, 0) keep the discarded ladder arithmetic well-defined
  mont_mul<L>(w, Di, R2, N, n0inv);                // w = D^{-1} (Montgomery form)
  // x0 = 16 u^3 * u^3 * v * w
  mont_mul<L>(c, t, u3, N, n0inv);
  mont_mul<L>(c, c, v, N, n0inv);
  mont_mul<L>(x0, c, w, N, n0inv);
  // a24 = (v-u)^3 (3u+v) v^3 w
  sub_lazy<L>(t, v, u, N2);
  mont_mul<L>(c, t, t, N, n0inv);
  mont_mul<L>(c, c, t, N, n0inv);
  mont_mul<L>(t, three, u, N, n0inv);
  add_lazy<L>(t, t, v, N2);
  mont_mul<L>(c, c, t, N, n0inv);
  mont_mul<L>(c, c, v3, N, n0inv);
  mont_mul<L>(a24, c, w, N, n0inv);
  const uint32_t okm = 0u - (uint32_t)ok;
  select<L>(x0, okm, x0, ONE);
#pragma unroll
  for (int k = 0; k < L; ++k) a24[k] &= okm;
  // gcd(D, N) == N (D == 0 mod N) -> 3; proper factor -> 4 (both tests evaluated: no branch)
  const uint32_t eqN = equal(gg, N), okv = ok;
  return (uint8_t)((1u - okv) * (4u - eqN));
}

// Small-parameter family (reading G16 — not the paper's curves): a
// seed s in [1, 2^30) gives a24 = s / 2^32 mod N and x0 = 2, both in Montgomery form; no
// inversion.  Seeds outside the range get status 3 (g = N).
template <int L>
__device__ __forceinline__ uint8_t ecm_setup_small(const EcmParams& p, uint64_t seed, uint32_t (&x0)[L],
                                                   uint32_t (&a24)[L]) {
  const uint32_t(&N)[L] = cref<L>(p.N);
  const uint32_t(&N2)[L] = cref<L>(p.N2);
  const uint32_t(&ONE)[L] = cref<L>(p.ONE);
  const bool ok = seed >= 1 && seed < (1ull << 30);
  add_lazy<L>(x0, ONE, ONE, N2);                                 // 2 R mod N
  mont_smul<L>(a24, ok ? (uint32_t)seed : 1u, ONE, N, p.n0inv);  // (s / 2^32) R mod N
  return ok ? 0 : 3;
}

// setup, and g = gcd(D, N) of a curve whose setup failed written at once (ecm_tail skips it);
// FAM 0: Brent-Suyama (the paper's), FAM 1: the small-parameter family
template <int L, int FAM = 0>
__device__ __forceinline__ uint8_t ecm_setup_store(const EcmParams& p, uint64_t sigma, uint32_t (&x0)[L],
                                                   uint32_t (&a24)[L], bool live, size_t i, uint32_t* g) {
  uint32_t gg[L];
  uint8_t st;
  if (FAM == 1) {
    st = ecm_setup_small<L>(p, sigma, x0, a24);
    copy(gg, cref<L>(p.N));
  } else {
    st = ecm_setup<L>(p, sigma, x0, a24, gg);
  }
  store_if<L>(g, i, gg, live && st != 0);
  return st;
}

// ---------------------------------------------------------------------------------------
// Tail: X, Z out of Montgomery form and canonical; g = gcd(Z, N) and Z^{-1} by one binary xgcd;
// status; affine x = X Z^{-1}.  Writes curve i's outputs (dead lanes compute and
// store nothing).  Branch-free: the gcd and the affine x are computed for every curve and the
// outputs selected by status.
// ---------------------------------------------------------------------------------------
// A curve whose setup failed (st = 3 / 4) had its g written by ecm_setup_store already, so the
// setup gcd is not live across the ladder.
template <int L>
__device__ __forceinline__ void ecm_tail(const EcmParams& p, const uint32_t (&X0)[L], const uint32_t (&Z0)[L], uint8_t st,
                                         bool live, size_t i, uint32_t* X, uint32_t* Z, uint32_t* g,
                                         uint8_t* status, uint32_t* xaff, uint32_t flags) {
  uint32_t gg[L], Zi[L];
  const uint32_t(&N)[L] = cref<L>(p.N);
  const uint32_t(&R2)[L] = cref<L>(p.R2);
  const uint32_t n0inv = p.n0inv;
  uint32_t c[L], t[L];
  uint32_t Xn[L], Zn[L], xa[L];
#pragma unroll
  for (int k = 0; k < L; ++k) c[k] = 0;
  c[0] = 1;
  mont_mul<L>(Xn, X0, c, N, n0inv);
  canonicalize<L>(Xn, Xn, N);
  mont_mul<L>(Zn, Z0, c, N, n0inv);
  canonicalize<L>(Zn, Zn, N);
  const bool inv = xgcd<L>(Zn, N, gg, Zi);
  const bool want_x = xaff && !(flags & 0x20u);  // kernel-uniform
  if (want_x) {
    mont_mul<L>(t, Xn, R2, N, n0inv);  // X R
    mont_mul<L>(xa, t, Zi, N, n0inv);  // X Z^{-1}
    canonicalize<L>(xa, xa, N);
  }
  // status: the setup's (3 / 4) if it failed, else 0 (Z invertible), 2 (g = N) or 1 (proper factor)
  const uint32_t eqN = equal(gg, N), invv = inv, stv = st;
  const uint8_t so = (uint8_t)(stv + (stv == 0u) * (1u - invv) * (1u + eqN));
  const uint32_t keep = 0u - (uint32_t)(st == 0), xkeep = 0u - (uint32_t)(so == 0);
#pragma unroll
  for (int k = 0; k < L; ++k) {
    Xn[k] &= keep;
    Zn[k] &= keep;
    xa[k] &= xkeep;
  }
  store_if<L>(X, i, Xn, live);
  store_if<L>(Z, i, Zn, live);
  store_if<L>(g, i, gg, live && so <= 2);
  if (want_x) store_if<L>(xaff, i, xa, live);
  if (live) status[i] = so;
}

template <int L, int VAR, bool EAGER, bool PRIMES, int FAM>
__global__ void __launch_bounds__(kEcmTPB, ecm_min_blocks(L, VAR, EAGER, PRIMES)) ecm_stage1_kernel(const __grid_constant__ EcmParams p,
                                                             const uint32_t* __restrict__ kwords, uint32_t k_bits,
                                                             const uint64_t* __restrict__ sigmas, size_t count,
                                                             uint32_t* X, uint32_t* Z, uint32_t* g, uint8_t* status,
                                                             uint32_t* xaff, uint32_t flags) {
  const uint32_t(&N)[L] = cref<L>(p.N);
  const uint32_t(&N2)[L] = cref<L>(p.N2);
  const uint32_t(&ONE)[L] = cref<L>(p.ONE);
  const uint32_t(&NP)[L] = cref<L>(p.NP);
  const uint32_t n0inv = p.n0inv;
  const Field<L, VAR, EAGER> fld{N, EAGER ? N : N2, NP, n0inv};
  const int lane = threadIdx.x & 31;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = i < count;
  const uint64_t sigma = live ? sigmas[i] : 6ull;

  uint32_t X0[L], Z0[L], X1[L], Z1[L], x0[L], a24[L];
  const uint8_t st = ecm_setup_store<L, FAM>(p, sigma, x0, a24, live, i, g);
  const uint32_t cs = st == 0 ? (uint32_t)sigma : 1u;  // FAM 1: a24 = cs / 2^32

  // ---------------- ladder over k (warp-uniform bits) ----------------
  if (EAGER) {
    canonicalize<L>(x0, x0, N);
    canonicalize<L>(a24, a24, N);
  }
  copy(X0, x0);
  copy(Z0, ONE);
  if (!PRIMES) xdbl<L>(X1, Z1, X0, Z0, a24, fld);  // R1 = xDBL(P)
#if ECM_CONST_SMEM
  __shared__ uint32_t sm_c[2][L][kEcmTPB];
#pragma unroll
  for (int k = 0; k < L; ++k) { sm_c[0][k][threadIdx.x] = x0[k]; sm_c[1][k][threadIdx.x] = a24[k]; }
#endif
  if (!PRIMES) {
    bool swapped = false;
    if (k_bits >= 2) {
      int idx = (int)k_bits - 2;
      int chunk = idx >> 10;  // 32 words = 1024 bits per warp-wide load
      uint32_t kreg = kwords[(chunk << 5) + lane];
#pragma unroll kLadderUnroll
      for (; idx >= 0; --idx) {
        if ((idx >> 10) != chunk) {
          chunk = idx >> 10;
          kreg = kwords[(chunk << 5) + lane];
        }
        const uint32_t word = __shfl_sync(0xffffffffu, kreg, (idx >> 5) & 31);
        const bool bit = (word >> (idx & 31)) & 1u;
#if ECM_SWAP_BRANCH
        // bit 1: R1 <- xDBL(R1), R0 <- xADD(R0, R1); bit 0: R0 <- xDBL(R0), R1 <- xADD.  The
        // bit is warp-uniform, so this is a uniform branch between two copies of the step.
        if (bit) ladder_step<L>(X1, Z1, X0, Z0, x0, a24, fld);
        else ladder_step<L>(X0, Z0, X1, Z1, x0, a24, fld);
#else
        if constexpr (ladder_swap_sel(L) && FAM == 0) {
          // slot 0 holds R_swapped: double slot (bit != swapped), write the double to slot 0
#if ECM_CONST_SMEM
          ladder_step_sm<L, kEcmTPB, true>(X0, Z0, X1, Z1, &sm_c[0][0][threadIdx.x], &sm_c[1][0][threadIdx.x], fld,
                                           bit != swapped);
#else
          ladder_step_sel<L>(X0, Z0, X1, Z1, x0, a24, fld, bit != swapped);
#endif
          swapped = bit;
          continue;
        }
        // bit 1: (R0, R1) <- (xADD, xDBL(R1)); bit 0: (xDBL(R0), xADD).  Double the point in the
        // (X0,Z0) slot: swap so that slot holds R_bit, swap back lazily on the next change.
        cswap<L>(X0, X1, bit != swapped);
        cswap<L>(Z0, Z1, bit != swapped);
        swapped = bit;
#if ECM_CONST_SMEM
        ladder_step_sm<L, kEcmTPB>(X0, Z0, X1, Z1, &sm_c[0][0][threadIdx.x], &sm_c[1][0][threadIdx.x], fld);
#else
        if (FAM == 1) ladder_step_small<L>(X0, Z0, X1, Z1, cs, N, n0inv, fld);
        else ladder_step<L>(X0, Z0, X1, Z1, x0, a24, fld);
#endif
#endif
      }
    }
    cswap<L>(X0, X1, swapped);
    cswap<L>(Z0, Z1, swapped);
  } else {
    // prime-by-prime: kwords holds the list of primes p <= B1 (each repeated e_p times),
    // k_bits its length; Q <- [p]Q by a ladder with difference Q for every entry.
    uint32_t QX[L], QZ[L];
    copy(QX, x0);
    copy(QZ, ONE);
    for (int c0 = 0; c0 < (int)k_bits; c0 += 32) {
      const uint32_t preg = kwords[c0 + lane];
      const int nt = ((int)k_bits - c0) < 32 ? ((int)k_bits - c0) : 32;
      for (int t = 0; t < nt; ++t) {
        const uint32_t pr = __shfl_sync(0xffffffffu, preg, t);
        copy(X0, QX);
        copy(Z0, QZ);
        xdbl<L>(X1, Z1, QX, QZ, a24, fld);
        bool swapped = false;
        for (int i = 30 - __clz(pr); i >= 0; --i) {
          const bool bit = (pr >> i) & 1u;
          cswap<L>(X0, X1, bit != swapped);
          cswap<L>(Z0, Z1, bit != swapped);
          swapped = bit;
          ladder_step_d<L>(X0, Z0, X1, Z1, QX, QZ, a24, fld);
        }
        cswap<L>(X0, X1, swapped);
        cswap<L>(Z0, Z1, swapped);
        copy(QX, X0);
        copy(QZ, Z0);
      }
    }
  }

  ecm_tail<L>(p, X0, Z0, st, live, i, X, Z, g, status, xaff, flags);
}

// ---------------------------------------------------------------------------------------
// Latency kernel: four lanes per curve (small batches, e.g. C1's 256 curves, where one warp per
// SM sub-partition leaves the one-curve-per-thread ladder bound by dependency latency).  The 10
// products of a ladder step form three rounds of independent products (4, 4, 2); lane q of the
// curve's 4-lane group computes product q of each round and the group exchanges the results
// with __shfl_sync (width 4).  The additions, the swap and the scalar bits are replicated in all
// four lanes, so every lane holds the whole state and every instruction stays warp-uniform.
// Squares go through the multiply (mont_mul(x, x) == mont_sqr(x), the unique raw REDC value), so
// the outputs are bit-identical to ecm_stage1_kernel's.
// ---------------------------------------------------------------------------------------
constexpr int kCoopLanes = 4;
constexpr int kCoopTPB = 128;

// d = a_q, branch-free (lanes of a warp hold different q): bit masks of q, 3 LOP3 per word
template <int L>
__device__ __forceinline__ void pick4(uint32_t (&d)[L], int q, const uint32_t (&a0)[L], const uint32_t (&a1)[L],
                                      const uint32_t (&a2)[L], const uint32_t (&a3)[L]) {
  const uint32_t m1 = 0u - (uint32_t)(q & 1), m2 = 0u - (uint32_t)((q >> 1) & 1);
#pragma unroll
  for (int k = 0; k < L; ++k) {
    const uint32_t lo = (a0[k] & ~m1) | (a1[k] & m1);
    const uint32_t hi = (a2[k] & ~m1) | (a3[k] & m1);
    d[k] = (lo & ~m2) | (hi & m2);
  }
}

// d = c ? a1 : a0 with an all-ones/zero mask c, 1 LOP3 per word
template <int L>
__device__ __forceinline__ void pick2(uint32_t (&d)[L], uint32_t c, const uint32_t (&a0)[L], const uint32_t (&a1)[L]) {
#pragma unroll
  for (int k = 0; k < L; ++k) d[k] = (a0[k] & ~c) | (a1[k] & c);
}

template <int L>
__device__ __forceinline__ void from_lane(uint32_t (&d)[L], const uint32_t (&r)[L], int q) {
#pragma unroll
  for (int k = 0; k < L; ++k) d[k] = __shfl_sync(0xffffffffu, r[k], q, kCoopLanes);
}

template <int L>
__device__ __forceinline__ void ladder_step_coop(uint32_t (&X0)[L], uint32_t (&Z0)[L], uint32_t (&X1)[L],
                                                 uint32_t (&Z1)[L], const uint32_t (&x0)[L], const uint32_t (&a24)[L],
                                                 const uint32_t (&N)[L], const uint32_t (&N2)[L], uint32_t n0inv,
                                                 int q) {
  uint32_t t1[L], t2[L], t3[L], t4[L], a[L], b[L], r[L];
  add_lazy<L>(t1, X0, Z0, N2);
  sub_lazy<L>(t2, X0, Z0, N2);
  add_lazy<L>(t3, X1, Z1, N2);
  sub_lazy<L>(t4, X1, Z1, N2);
  // round A: U = t2 t3, V = t1 t4, s = t1^2, d = t2^2
  pick2<L>(a, 0u - (uint32_t)((q ^ (q >> 1)) & 1), t2, t1);  // t1 for q = 1, 2
  pick4<L>(b, q, t3, t4, t1, t2);
  mont_mul<L>(r, a, b, N, n0inv);
  uint32_t U[L], V[L], sd[L], dd[L];
  from_lane<L>(U, r, 0);
  from_lane<L>(V, r, 1);
  from_lane<L>(sd, r, 2);
  from_lane<L>(dd, r, 3);
  uint32_t tt[L], w1[L], w2[L];
  sub_lazy<L>(tt, sd, dd, N2);  // t = s - d
  add_lazy<L>(w1, U, V, N2);
  sub_lazy<L>(w2, U, V, N2);
  // round B: X0' = s d, a24 t, X1' = (U+V)^2, (U-V)^2
  pick4<L>(a, q, sd, a24, w1, w2);
  pick4<L>(b, q, dd, tt, w1, w2);
  mont_mul<L>(r, a, b, N, n0inv);
  uint32_t at[L], sq[L];
  from_lane<L>(X0, r, 0);
  from_lane<L>(at, r, 1);
  from_lane<L>(X1, r, 2);
  from_lane<L>(sq, r, 3);
  add_lazy<L>(w1, dd, at, N2);  // d + a24 t
  // round C: Z0' = t (d + a24 t), Z1' = x0 (U-V)^2 (lanes 2, 3 repeat lanes 0, 1)
  const uint32_t odd = 0u - (uint32_t)(q & 1);
  pick2<L>(a, odd, tt, x0);
  pick2<L>(b, odd, w1, sq);
  mont_mul<L>(r, a, b, N, n0inv);
  from_lane<L>(Z0, r, 0);
  from_lane<L>(Z1, r, 1);
}

template <int L, int FAM>
__global__ void __launch_bounds__(kCoopTPB) ecm_stage1_coop_kernel(const __grid_constant__ EcmParams p,
                                                                   const uint32_t* __restrict__ kwords, uint32_t k_bits,
                                                                   const uint64_t* __restrict__ sigmas, size_t count,
                                                                   uint32_t* X, uint32_t* Z, uint32_t* g,
                                                                   uint8_t* status, uint32_t* xaff, uint32_t flags) {
  const uint32_t(&N)[L] = cref<L>(p.N);
  const uint32_t(&N2)[L] = cref<L>(p.N2);
  const uint32_t(&ONE)[L] = cref<L>(p.ONE);
  const uint32_t(&NP)[L] = cref<L>(p.NP);
  const uint32_t n0inv = p.n0inv;
  const Field<L, REDC_WORD, false> fld{N, N2, NP, n0inv};
  const int lane = threadIdx.x & 31;
  const int q = lane & (kCoopLanes - 1);
  const size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) / kCoopLanes;
  const bool live = i < count;
  const uint64_t sigma = live ? sigmas[i] : 6ull;

  uint32_t X0[L], Z0[L], X1[L], Z1[L], x0[L], a24[L];
  const uint8_t st = ecm_setup_store<L, FAM>(p, sigma, x0, a24, live, i, g);
  copy(X0, x0);
  copy(Z0, ONE);
  xdbl<L>(X1, Z1, X0, Z0, a24, fld);  // R1 = xDBL(P), replicated
  bool swapped = false;
  if (k_bits >= 2) {
    int idx = (int)k_bits - 2;
    int chunk = idx >> 10;
    uint32_t kreg = kwords[(chunk << 5) + lane];
    for (; idx >= 0; --idx) {
      if ((idx >> 10) != chunk) {
        chunk = idx >> 10;
        kreg = kwords[(chunk << 5) + lane];
      }
      const uint32_t word = __shfl_sync(0xffffffffu, kreg, (idx >> 5) & 31);
      const bool bit = (word >> (idx & 31)) & 1u;
      cswap<L>(X0, X1, bit != swapped);
      cswap<L>(Z0, Z1, bit != swapped);
      swapped = bit;
      ladder_step_coop<L>(X0, Z0, X1, Z1, x0, a24, N, N2, n0inv, q);
    }
  }
  cswap<L>(X0, X1, swapped);
  cswap<L>(Z0, Z1, swapped);
  ecm_tail<L>(p, X0, Z0, st, live && q == 0, i, X, Z, g, status, xaff, flags);
}

// Batches up to this many curves per SM take the 4-lane kernel by default: below ~80 curves/SM
// (≈2.6 four-lane warps per SM sub-partition) it beats the one-lane kernel, which stays
// latency-bound up to one warp per sub-partition (profiles/r01_ecm_lat.jsonl).
constexpr size_t kCoopMaxCurvesPerSM = 64;

template <int L, int VAR, bool EAGER, bool PRIMES = false, int FAM = 0>
static cudaError_t launch_ecm_LV(const EcmParams& p, const uint32_t* kw, uint32_t k_bits, const uint64_t* sigmas,
                                 size_t count, uint32_t* X, uint32_t* Z, uint32_t* g, uint8_t* status, uint32_t* xaff,
                                 uint32_t flags, cudaStream_t s) {
  if (VAR == REDC_WORD && !EAGER && !PRIMES && !(flags & 0x4000u)) {
    bool coop = (flags & 0x2000u) != 0;  // ECM_KERNEL_LANES4 forces it, ECM_KERNEL_LANES1 forbids it
    if (!coop) {
      int dev = 0, sms = 0;
      cudaError_t e = cudaGetDevice(&dev);
      if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (e != cudaSuccess) return e;
      coop = count <= (size_t)sms * kCoopMaxCurvesPerSM;
    }
    if (coop) {
      const size_t threads = count * kCoopLanes;
      const size_t blocks = (threads + kCoopTPB - 1) / kCoopTPB;
      ecm_stage1_coop_kernel<L, FAM><<<(unsigned)blocks, kCoopTPB, 0, s>>>(p, kw, k_bits, sigmas, count, X, Z, g,
                                                                           status, xaff, flags);
      return cudaGetLastError();
    }
  }
  const size_t blocks = (count + kEcmTPB - 1) / kEcmTPB;
  ecm_stage1_kernel<L, VAR, EAGER, PRIMES, FAM><<<(unsigned)blocks, kEcmTPB, 0, s>>>(p, kw, k_bits, sigmas, count, X,
                                                                             Z, g, status, xaff, flags);
  return cudaGetLastError();
}

// Ablation variants (REDC form x eager/lazy) are instantiated for L = 6 and 8 (192/256-bit,
// the paper's 254-bit setting); every width gets the default lazy word-serial kernel.
template <int L>
cudaError_t launch_ecm_L(const EcmParams& p, const uint32_t* kw, uint32_t k_bits, const uint64_t* sigmas,
                                size_t count, uint32_t* X, uint32_t* Z, uint32_t* g, uint8_t* status, uint32_t* xaff,
                                uint32_t flags, cudaStream_t s) {
  const uint32_t var = (flags >> 8) & 7u;
  const bool eager = flags & 0x40u;
  if (flags & 0x8000u) {  // small-parameter family: default lazy full-k ladder only
    if (var == REDC_WORD && !eager && !(flags & 0x80u))
      return launch_ecm_LV<L, REDC_WORD, false, false, 1>(p, kw, k_bits, sigmas, count, X, Z, g, status, xaff, flags, s);
    return cudaErrorInvalidValue;
  }
  if (flags & 0x80u) {  // prime-by-prime schedule (paper-comparable)
    if constexpr (L == 8) {
#define ECM_PCASE(V, E) \
      if (var == V && eager == E) return launch_ecm_LV<L, V, E, true>(p, kw, k_bits, sigmas, count, X, Z, g, status, xaff, flags, s);
      ECM_PCASE(REDC_WORD, false)
      ECM_PCASE(REDC_WORD, true)
      ECM_PCASE(REDC_BLOCKTHM, false)
      ECM_PCASE(REDC_BLOCKTHM, true)
      ECM_PCASE(REDC_CLASSIC, false)
      ECM_PCASE(REDC_CLASSIC, true)
#undef ECM_PCASE
    }
    if constexpr (L == 6) {
      if (var == REDC_WORD && !eager) return launch_ecm_LV<L, REDC_WORD, false, true>(p, kw, k_bits, sigmas, count, X, Z, g, status, xaff, flags, s);
    }
    return cudaErrorInvalidValue;
  }
  if (var == REDC_WORD && !eager) return launch_ecm_LV<L, REDC_WORD, false>(p, kw, k_bits, sigmas, count, X, Z, g, status, xaff, flags, s);
  if constexpr (L == 6 || L == 8) {
#define ECM_CASE(V, E) \
    if (var == V && eager == E) return launch_ecm_LV<L, V, E>(p, kw, k_bits, sigmas, count, X, Z, g, status, xaff, flags, s);
    ECM_CASE(REDC_WORD, true)
    ECM_CASE(REDC_KNOWNLOW, false)
    ECM_CASE(REDC_KNOWNLOW, true)
    ECM_CASE(REDC_BLOCKTHM, false)
    ECM_CASE(REDC_BLOCKTHM, true)
    ECM_CASE(REDC_CLASSIC, false)
    ECM_CASE(REDC_CLASSIC, true)
#undef ECM_CASE
  }
  return cudaErrorInvalidValue;
}

}  // namespace ecm
