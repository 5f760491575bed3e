// mont.cuh — sm_100a multi-precision Montgomery arithmetic (device side of libecmgpu).
//
// Implements, per lane, the paper's modular arithmetic (arXiv 1310.3809 §2):
//   * REDC in word-serial CIOS form, LAZY: no final subtraction, values stay
//     in [0, 2N) by the Lemma because R = 2^(32L) >= 4N (reading G2/G3).
//   * the paper's Theorem applied per word (REDC_KNOWNLOW): the low word of
//     m_i*N_0 is known to be -t_0 (mod 2^32), so it is not multiplied; carry = (t_0 != 0).
//     And block forms (REDC_CLASSIC: q = T*N' mod R, T + q*N with 4 quadrant products;
//     REDC_BLOCKTHM: the Theorem literally, m0*b0 recovered from the congruence, 3 quadrants).
//   * branch-free Reduction after Addition / Subtraction with 2N.
//
// Hardware mapping (measured, profiles/r01_imad_rates.jsonl): on sm_100a a PTX pair
//   mad.lo.cc  d0, a, b, c0;  madc.hi.cc d1, a, b, c1;
// is fused by ptxas into ONE `IMAD.WIDE.U32 {d1,d0}, P, a, b, {c1,c0}` with carry-in/out
// predicates; it issues at 32 lanes/clk/SM (same pipe time as IMAD.HI, twice IMAD.LO).
// One IMAD.WIDE = one 32x32->64 partial product ("FPE").  The schedule below therefore keeps
// every product as an adjacent lo/hi pair into an even-aligned 64-bit accumulator:
//   even products a_i*b_j (j even) land on word pairs (j, j+1)      -> accumulator E[0..L)
//   odd  products a_i*b_j (j odd)  land on word pairs (j, j+1)      -> accumulator O[0..L)
// (O[k] has weight 2^(32(k+1))).  Within a row no two pairs overlap, so each accumulator is
// ONE carry chain of L/2 IMAD.WIDE.  The division by 2^32 at the end of a CIOS row is pure
// register renaming: the next row's odd chain reads E[2..L) as its addends (the "shift").
// L must be even (L in {4, 6, 8, 12, 16}).
#pragma once
#include <cstdint>

namespace ecm {

enum RedcVariant : int { REDC_WORD = 0, REDC_KNOWNLOW = 1, REDC_BLOCKTHM = 2, REDC_CLASSIC = 3, REDC_KARATSUBA = 4 };

// ------------------------------------------------------------------------------------------
// PTX carry-chain primitives.  The carry flag (CC.CF) is implicit state that links
// consecutive statements; every wrapper is `asm volatile` so the compiler keeps their order.
// ------------------------------------------------------------------------------------------
namespace ptx {
__device__ __forceinline__ uint32_t mul_lo(uint32_t a, uint32_t b) { uint32_t d; asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d; }
__device__ __forceinline__ uint32_t mul_hi(uint32_t a, uint32_t b) { uint32_t d; asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d; }
__device__ __forceinline__ uint32_t mad_lo_cc(uint32_t a, uint32_t b, uint32_t c) { uint32_t d; asm volatile("mad.lo.cc.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
__device__ __forceinline__ uint32_t madc_lo_cc(uint32_t a, uint32_t b, uint32_t c) { uint32_t d; asm volatile("madc.lo.cc.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
__device__ __forceinline__ uint32_t mad_hi_cc(uint32_t a, uint32_t b, uint32_t c) { uint32_t d; asm volatile("mad.hi.cc.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
__device__ __forceinline__ uint32_t madc_hi_cc(uint32_t a, uint32_t b, uint32_t c) { uint32_t d; asm volatile("madc.hi.cc.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
__device__ __forceinline__ uint32_t madc_hi(uint32_t a, uint32_t b, uint32_t c) { uint32_t d; asm volatile("madc.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
__device__ __forceinline__ uint32_t madc_lo(uint32_t a, uint32_t b, uint32_t c) { uint32_t d; asm volatile("madc.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
__device__ __forceinline__ uint32_t add_cc(uint32_t a, uint32_t b) { uint32_t d; asm volatile("add.cc.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d; }
__device__ __forceinline__ uint32_t addc_cc(uint32_t a, uint32_t b) { uint32_t d; asm volatile("addc.cc.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d; }
__device__ __forceinline__ uint32_t addc(uint32_t a, uint32_t b) { uint32_t d; asm volatile("addc.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d; }
__device__ __forceinline__ uint32_t sub_cc(uint32_t a, uint32_t b) { uint32_t d; asm volatile("sub.cc.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d; }
__device__ __forceinline__ uint32_t subc_cc(uint32_t a, uint32_t b) { uint32_t d; asm volatile("subc.cc.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d; }
__device__ __forceinline__ uint32_t subc(uint32_t a, uint32_t b) { uint32_t d; asm volatile("subc.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d; }
}  // namespace ptx

// n0inv = -N0^{-1} mod 2^32 (the word-level m' of PAPER.md:94): Newton/Hensel lifting,
// x <- x(2 - N0 x) doubles the correct low bits; x0 = (3 N0) ^ 2 is correct to 5 bits.
__device__ __forceinline__ uint32_t neg_inv32(uint32_t n0) {
  uint32_t x = (3u * n0) ^ 2u;
  x *= 2u - n0 * x;
  x *= 2u - n0 * x;
  x *= 2u - n0 * x;
  return 0u - x;
}

// ------------------------------------------------------------------------------------------
// Chains.  acc += a * v[par], par = 0 (even j) or 1 (odd j), as L/2 fused IMAD.WIDE.U32.
// `cin` selects madc (consume a pending carry) vs mad for the first pair; `cout_free`
// promises the chain cannot carry out (so the last op does not write CC).
// ------------------------------------------------------------------------------------------
template <int L, int PAR, bool CIN, bool COUT>
__device__ __forceinline__ void chain(uint32_t (&d)[L], const uint32_t (&c)[L], uint32_t a, const uint32_t (&v)[L]) {
#pragma unroll
  for (int j = 0; j < L; j += 2) {
    const uint32_t b = v[j + PAR];
    if (j == 0 && !CIN) d[j] = ptx::mad_lo_cc(a, b, c[j]);
    else d[j] = ptx::madc_lo_cc(a, b, c[j]);
    if (j + 2 == L && !COUT) d[j + 1] = ptx::madc_hi(a, b, c[j + 1]);
    else d[j + 1] = ptx::madc_hi_cc(a, b, c[j + 1]);
  }
}

// Known-low even reduction chain: E += m*N_even where the low word of m*N_0 is the known
// value -E_0 (b*m = -a mod R).  E_0 + lo(m N_0) = 0 (mod 2^32) carries iff
// E_0 != 0, produced here by E_0 + 0xffffffff.  IMAD.HI replaces the first IMAD.WIDE.
template <int L>
__device__ __forceinline__ void chain_even_knownlow(uint32_t (&E)[L], uint32_t m, const uint32_t (&n)[L]) {
  (void)ptx::add_cc(E[0], 0xffffffffu);
  E[1] = ptx::madc_hi_cc(m, n[0], E[1]);
#pragma unroll
  for (int j = 2; j < L; j += 2) {
    E[j] = ptx::madc_lo_cc(m, n[j], E[j]);
    E[j + 1] = ptx::madc_hi_cc(m, n[j], E[j + 1]);
  }
  E[0] = 0;
}

// ------------------------------------------------------------------------------------------
// Lazy Montgomery multiplication, word-serial (CIOS) with even/odd accumulators.
// r = (x*y + q*N)/R, q = x*y*(-N^{-1}) mod R — the unique raw REDC value (no final
// subtraction).  Preconditions: N odd, N < R/4, x, y < 2N  =>  r < 2N (Lemma, reading G3).
// Invariant (start of row i): running value t = E + O*2^32 + cc*2^32 with t < y + N, so
// every partial sum is < (3/4) 2^(32(L+1)): the odd chain never carries out and the even
// chain's carry fits in O[L-1].
// ------------------------------------------------------------------------------------------
template <int L, int V>
__device__ __forceinline__ void mont_mul_cios(uint32_t (&r)[L], const uint32_t (&x)[L], const uint32_t (&y)[L],
                                              const uint32_t (&n)[L], uint32_t n0inv) {
  static_assert(L % 2 == 0 && L >= 2, "L must be even");
  uint32_t E[L], O[L], Z[L];
#pragma unroll
  for (int j = 0; j < L; ++j) Z[j] = 0;
  // row 0: products only (pairs are disjoint: no carries)
  chain<L, 1, false, false>(O, Z, x[0], y);
  chain<L, 0, false, false>(E, Z, x[0], y);
#pragma unroll
  for (int i = 0; i < L; ++i) {
    if (i > 0) {
      // t += x_i * y.  O holds the shifted even accumulator; the pending carry of the
      // shift add (weight 2^32) enters the odd chain's first pair.
      chain<L, 1, true, false>(O, O, x[i], y);
      chain<L, 0, false, true>(E, E, x[i], y);
      O[L - 1] = ptx::addc(O[L - 1], 0);
    }
    // m_i = t_0 * (-N^{-1}) mod 2^32;  t += m_i * N
    const uint32_t m = E[0] * n0inv;
    chain<L, 1, false, false>(O, O, m, n);
    if (V == REDC_KNOWNLOW) chain_even_knownlow<L>(E, m, n);
    else chain<L, 0, false, true>(E, E, m, n);
    O[L - 1] = ptx::addc(O[L - 1], 0);
    // t /= 2^32: E[0] == 0.  New even accumulator = O (+ E[1] at weight 1, carry pending);
    // new odd accumulator = E[2..L) (weights 2^32..), top two words zero.
    uint32_t nE[L], nO[L];
#pragma unroll
    for (int k = 0; k < L; ++k) nE[k] = O[k];
    nE[0] = ptx::add_cc(nE[0], E[1]);
#pragma unroll
    for (int k = 0; k < L; ++k) nO[k] = (k + 2 < L) ? E[k + 2] : 0u;
    if (i + 1 < L) {
#pragma unroll
      for (int k = 0; k < L; ++k) { E[k] = nE[k]; O[k] = nO[k]; }
    } else {
      // merge: r = nE + nO*2^32 + carry
      r[0] = nE[0];
#pragma unroll
      for (int k = 1; k < L - 1; ++k) r[k] = ptx::addc_cc(nE[k], nO[k - 1]);
      r[L - 1] = ptx::addc(nE[L - 1], nO[L - 2]);
    }
  }
}

// r = REDC(x*y) + d (< 4N for d < 2N) with no addition instructions: REDC(x y + d R) = REDC(x y) + d
// because q depends only on x y mod R, and word d_i (original weight R 2^(32i)) is placed into the
// slot that is zero after row i's shift (O[L-2], weight L-1), as in mont_sqr_inj.  Frame bound: the
// running value stays < y + N + R, and a row adds < 2^32 (y + N): < (3/4) 2^(32(L+1)) for y < 2N.
template <int L>
__device__ __forceinline__ void mont_mul_add(uint32_t (&r)[L], const uint32_t (&x)[L], const uint32_t (&y)[L],
                                             const uint32_t (&d)[L], const uint32_t (&n)[L], uint32_t n0inv) {
  uint32_t E[L], O[L], Z[L];
#pragma unroll
  for (int j = 0; j < L; ++j) Z[j] = 0;
  chain<L, 1, false, false>(O, Z, x[0], y);
  chain<L, 0, false, false>(E, Z, x[0], y);
#pragma unroll
  for (int i = 0; i < L; ++i) {
    if (i > 0) {
      chain<L, 1, true, false>(O, O, x[i], y);
      chain<L, 0, false, true>(E, E, x[i], y);
      O[L - 1] = ptx::addc(O[L - 1], 0);
    }
    const uint32_t m = E[0] * n0inv;
    chain<L, 1, false, false>(O, O, m, n);
    chain<L, 0, false, true>(E, E, m, n);
    O[L - 1] = ptx::addc(O[L - 1], 0);
    uint32_t nE[L], nO[L];
#pragma unroll
    for (int k = 0; k < L; ++k) nE[k] = O[k];
    nE[0] = ptx::add_cc(nE[0], E[1]);
#pragma unroll
    for (int k = 0; k < L; ++k) nO[k] = (k + 2 < L) ? E[k + 2] : (k == L - 2) ? d[i] : 0u;
    if (i + 1 < L) {
#pragma unroll
      for (int k = 0; k < L; ++k) { E[k] = nE[k]; O[k] = nO[k]; }
    } else {
      r[0] = nE[0];
#pragma unroll
      for (int k = 1; k < L - 1; ++k) r[k] = ptx::addc_cc(nE[k], nO[k - 1]);
      r[L - 1] = ptx::addc(nE[L - 1], nO[L - 2]);
    }
  }
}

// ------------------------------------------------------------------------------------------
// Block (SOS) forms of REDC, for the paper's ablation (Table 5).
// T = x*y (2L words); q = (T mod R) * N' mod R; r = (T + q*N)/R.
//   CLASSIC : q*N as a full product (4 half-size quadrants).
//   BLOCKTHM: the Theorem: with q = q1 h + q0, N = N1 h + N0, h = 2^(32 L/2), only
//             q1 N1, q1 N0, q0 N1 are multiplied; q0 N0 = -(T + (q1 N0 + q0 N1) h) mod R.
// Both return the same unique raw value as mont_mul_cios.
// ------------------------------------------------------------------------------------------
// Schoolbook product built from the same fused IMAD.WIDE chains as the word-serial kernel:
// each row a_i * b is split by the parity of the product offset i+j into an even-offset chain
// (accumulator EV) and an odd-offset chain (OD); the pairs of one chain are disjoint, and with
// rows in increasing i each chain's carry-out lands in a word that so far holds only earlier
// carries, absorbed by one add.  t = EV + OD at the end.
template <int A, int B>
__device__ __forceinline__ void mul_full(uint32_t (&t)[A + B], const uint32_t* a, const uint32_t* b) {
  uint32_t EV[A + B + 1], OD[A + B + 1];
#pragma unroll
  for (int k = 0; k <= A + B; ++k) { EV[k] = 0; OD[k] = 0; }
#pragma unroll
  for (int i = 0; i < A; ++i) {
#pragma unroll
    for (int par = 0; par < 2; ++par) {
      uint32_t* acc = par ? OD : EV;
      const int j0 = ((i & 1) == par) ? 0 : 1;
      int last = -1;
#pragma unroll
      for (int j = j0; j < B; j += 2) {
        const int o = i + j;
        if (last < 0) acc[o] = ptx::mad_lo_cc(a[i], b[j], acc[o]);
        else acc[o] = ptx::madc_lo_cc(a[i], b[j], acc[o]);
        acc[o + 1] = ptx::madc_hi_cc(a[i], b[j], acc[o + 1]);
        last = o;
      }
      if (last >= 0) acc[last + 2] = ptx::addc(acc[last + 2], 0u);
    }
  }
  t[0] = EV[0];
  t[1] = ptx::add_cc(EV[1], OD[1]);
#pragma unroll
  for (int k = 2; k < A + B - 1; ++k) t[k] = ptx::addc_cc(EV[k], OD[k]);
  t[A + B - 1] = ptx::addc(EV[A + B - 1], OD[A + B - 1]);
}

// q = a*b mod 2^(32L): the same chains, truncated — a product at offset L-1 contributes only
// its low word (IMAD, no high half), pairs above are not formed.
template <int L>
__device__ __forceinline__ void mul_low_half(uint32_t (&q)[L], const uint32_t* a, const uint32_t* b) {
  uint32_t EV[L + 1], OD[L + 1];
#pragma unroll
  for (int k = 0; k <= L; ++k) { EV[k] = 0; OD[k] = 0; }
#pragma unroll
  for (int i = 0; i < L; ++i) {
#pragma unroll
    for (int par = 0; par < 2; ++par) {
      uint32_t* acc = par ? OD : EV;
      const int j0 = ((i & 1) == par) ? 0 : 1;
      int last = -1;
      bool closed = false;
#pragma unroll
      for (int j = j0; i + j < L; j += 2) {
        const int o = i + j;
        if (o == L - 1) {
          acc[o] = (last < 0) ? acc[o] + a[i] * b[j] : ptx::madc_lo(a[i], b[j], acc[o]);
          closed = true;
        } else {
          if (last < 0) acc[o] = ptx::mad_lo_cc(a[i], b[j], acc[o]);
          else acc[o] = ptx::madc_lo_cc(a[i], b[j], acc[o]);
          acc[o + 1] = ptx::madc_hi_cc(a[i], b[j], acc[o + 1]);
        }
        last = o;
      }
      if (last >= 0 && !closed && last + 2 < L) acc[last + 2] = ptx::addc(acc[last + 2], 0u);
    }
  }
  q[0] = EV[0];
  q[1] = ptx::add_cc(EV[1], OD[1]);
#pragma unroll
  for (int k = 2; k < L - 1; ++k) q[k] = ptx::addc_cc(EV[k], OD[k]);
  q[L - 1] = ptx::addc(EV[L - 1], OD[L - 1]);
}

template <int L, int V>
__device__ __forceinline__ void mont_mul_block(uint32_t (&r)[L], const uint32_t (&x)[L], const uint32_t (&y)[L],
                                               const uint32_t (&n)[L], const uint32_t (&nprime)[L]) {
  constexpr int H = L / 2;
  uint32_t T[2 * L], q[L];
  mul_full<L, L>(T, x, y);
  mul_low_half<L>(q, T, nprime);  // step 1
  uint32_t QN[2 * L];
  if (V == REDC_CLASSIC) {
    mul_full<L, L>(QN, q, n);
  } else {
    // q N = q1 N1 h^2 + (q1 N0 + q0 N1) h + q0 N0,  h = 2^(32H)
    uint32_t hh[2 * H], m10[2 * H], m01[2 * H];
    mul_full<H, H>(hh, q + H, n + H);
    mul_full<H, H>(m10, q + H, n);
    mul_full<H, H>(m01, q, n + H);
    // mid = q1 N0 + q0 N1  (2H words + carry)
    uint32_t mid[2 * H + 1];
    mid[0] = ptx::add_cc(m10[0], m01[0]);
#pragma unroll
    for (int k = 1; k < 2 * H; ++k) mid[k] = ptx::addc_cc(m10[k], m01[k]);
    mid[2 * H] = ptx::addc(0u, 0u);
    // q0 N0 = -(T + mid h) mod R  (the congruence of the Theorem)
    uint32_t s[L], q0n0[L];
    s[0] = T[0];
#pragma unroll
    for (int k = 1; k < H; ++k) s[k] = T[k];
    s[H] = ptx::add_cc(T[H], mid[0]);
#pragma unroll
    for (int k = H + 1; k < L; ++k) s[k] = ptx::addc_cc(T[k], mid[k - H]);
    q0n0[0] = ptx::sub_cc(0u, s[0]);
#pragma unroll
    for (int k = 1; k < L; ++k) q0n0[k] = ptx::subc_cc(0u, s[k]);
    // QN = q0n0 + mid h + hh h^2
#pragma unroll
    for (int k = 0; k < 2 * L; ++k) QN[k] = (k < L) ? q0n0[k] : 0u;
    QN[H] = ptx::add_cc(QN[H], mid[0]);
#pragma unroll
    for (int k = H + 1; k < 2 * L; ++k) QN[k] = ptx::addc_cc(QN[k], (k - H <= 2 * H) ? mid[k - H] : 0u);
    QN[L] = ptx::add_cc(QN[L], hh[0]);
#pragma unroll
    for (int k = L + 1; k < 2 * L; ++k) QN[k] = ptx::addc_cc(QN[k], hh[k - L]);
  }
  // r = (T + QN) / R  (low half is zero by construction; only its carry matters)
  uint32_t lo = ptx::add_cc(T[0], QN[0]);
#pragma unroll
  for (int k = 1; k < L; ++k) lo = ptx::addc_cc(T[k], QN[k]);
  (void)lo;
#pragma unroll
  for (int k = 0; k < L - 1; ++k) r[k] = ptx::addc_cc(T[L + k], QN[L + k]);
  r[L - 1] = ptx::addc(T[2 * L - 1], QN[2 * L - 1]);
}

// ------------------------------------------------------------------------------------------
// Karatsuba-level REDC with the paper's second Theorem (Table 3: 2k-2 instead
// of 2k-1 sub-products for k = 2).  L = 2H words, B = 2^(32H), R = B^2.
//   T = x*y by subtractive Karatsuba: z0 = x0 y0, z2 = x1 y1, D = (x0-x1)(y1-y0) = |.||.|(+-),
//       x0 y1 + x1 y0 = z0 + z2 + D                                   (3 H x H products)
//   q = (T mod R) N' mod R                                           (low half)
//   q N = w_inf B^2 + M B + w0 with w_inf = q1 N1, D2 = (q0-q1)(N1-N0), M = D2 + w0 + w_inf;
//       w0 = q0 N0 is NOT multiplied: q N = -T (mod R) gives
//         w0L = -T0L mod B,  w0H = ((-(T0 + w0L))/B - D2 - w0L - w_inf) mod B   (2 products)
//   r = (T + q N)/R = T1 + w_inf + (T0 + w0 + M B)/B^2                 (exact)
// |N1 - N0| and its sign are per-modulus constants (dN, sn), computed once per element.
// ------------------------------------------------------------------------------------------
// d = |a - b| over W words; returns 1 if a < b
template <int W>
__device__ __forceinline__ uint32_t absdiff(uint32_t (&d)[W], const uint32_t* a, const uint32_t* b) {
  d[0] = ptx::sub_cc(a[0], b[0]);
#pragma unroll
  for (int k = 1; k < W; ++k) d[k] = ptx::subc_cc(a[k], b[k]);
  const uint32_t m = ptx::subc(0u, 0u);  // all ones iff a < b
  // conditional two's complement negate: (d ^ m) + (m & 1)
  d[0] = ptx::add_cc(d[0] ^ m, m & 1u);
#pragma unroll
  for (int k = 1; k < W - 1; ++k) d[k] = ptx::addc_cc(d[k] ^ m, 0u);
  if (W > 1) d[W - 1] = ptx::addc(d[W - 1] ^ m, 0u);
  return m & 1u;
}

template <int L>
__device__ __forceinline__ void kara_consts(uint32_t (&dN)[L / 2], uint32_t& sn, const uint32_t (&n)[L]) {
  sn = absdiff<L / 2>(dN, n + L / 2, n);  // |N1 - N0|, sn = (N1 < N0)
}

template <int L>
__device__ __forceinline__ void mont_mul_kara(uint32_t (&r)[L], const uint32_t (&x)[L], const uint32_t (&y)[L],
                                              const uint32_t (&n)[L], const uint32_t (&np)[L],
                                              const uint32_t (&dN)[L / 2], uint32_t sn) {
  constexpr int H = L / 2;
  // ---- T = x*y ----
  uint32_t T[2 * L];
  {
    uint32_t z0[2 * H], z2[2 * H], dx[H], dy[H], Dm[2 * H];
    mul_full<H, H>(z0, x, y);
    mul_full<H, H>(z2, x + H, y + H);
    const uint32_t sx = absdiff<H>(dx, x, x + H);   // |x0 - x1|
    const uint32_t sy = absdiff<H>(dy, y + H, y);   // |y1 - y0|
    mul_full<H, H>(Dm, dx, dy);
    const uint32_t m = 0u - (sx ^ sy);              // D = -Dm when the signs differ
    // mid = z0 + z2 + D  (2H+1 words, >= 0)
    uint32_t mid[2 * H + 1];
    mid[0] = ptx::add_cc(z0[0], z2[0]);
#pragma unroll
    for (int k = 1; k < 2 * H; ++k) mid[k] = ptx::addc_cc(z0[k], z2[k]);
    mid[2 * H] = ptx::addc(0u, 0u);
    mid[0] = ptx::add_cc(mid[0], Dm[0] ^ m);
#pragma unroll
    for (int k = 1; k < 2 * H; ++k) mid[k] = ptx::addc_cc(mid[k], Dm[k] ^ m);
    mid[2 * H] = ptx::addc(mid[2 * H], m);
    mid[0] = ptx::add_cc(mid[0], m & 1u);
#pragma unroll
    for (int k = 1; k < 2 * H; ++k) mid[k] = ptx::addc_cc(mid[k], 0u);
    mid[2 * H] = ptx::addc(mid[2 * H], 0u);
    // T = z0 + z2 B^2 + mid B
#pragma unroll
    for (int k = 0; k < 2 * H; ++k) { T[k] = z0[k]; T[2 * H + k] = z2[k]; }
    T[H] = ptx::add_cc(T[H], mid[0]);
#pragma unroll
    for (int k = 1; k <= 2 * H; ++k) T[H + k] = ptx::addc_cc(T[H + k], mid[k]);
#pragma unroll
    for (int k = 3 * H + 1; k < 4 * H - 1; ++k) T[k] = ptx::addc_cc(T[k], 0u);
    if (3 * H + 1 <= 4 * H - 1) T[4 * H - 1] = ptx::addc(T[4 * H - 1], 0u);
  }
  // ---- q = T0 N' mod R ----
  uint32_t q[L];
  mul_low_half<L>(q, T, np);
  // ---- q N with two products ----
  uint32_t dq[H], Dm2[2 * H], winf[2 * H];
  const uint32_t sq = absdiff<H>(dq, q, q + H);  // |q0 - q1|
  mul_full<H, H>(Dm2, dq, dN);
  mul_full<H, H>(winf, q + H, n + H);
  const uint32_t m2 = 0u - (sq ^ sn);            // D2 = -Dm2 when the signs differ
  // w0L = -T0L mod B; the low half of T0 + w0L is 0 and carries c = (T0L != 0) into word H
  uint32_t w0[2 * H];
  w0[0] = ptx::sub_cc(0u, T[0]);
#pragma unroll
  for (int k = 1; k < H; ++k) w0[k] = ptx::subc_cc(0u, T[k]);
  const uint32_t c = ptx::subc(0u, 0u) & 1u;    // borrow iff T0L != 0
  // U_H = -(T[H..2H) + c) mod B;  w0H = U_H - D2 - w0L - w_inf (mod B)
  {
    uint32_t u[H];
    u[0] = ptx::add_cc(T[H], c);
#pragma unroll
    for (int k = 1; k < H; ++k) u[k] = ptx::addc_cc(T[H + k], 0u);
    // u <- -u - w0L - winf_low  (mod B)
    uint32_t s[H];
    s[0] = ptx::add_cc(u[0], w0[0]);
#pragma unroll
    for (int k = 1; k < H; ++k) s[k] = ptx::addc_cc(u[k], w0[k]);
    s[0] = ptx::add_cc(s[0], winf[0]);
#pragma unroll
    for (int k = 1; k < H; ++k) s[k] = ptx::addc_cc(s[k], winf[k]);
    // + D2_low = +-(Dm2 low) : add (Dm2 ^ m2) + (m2 & 1)
    s[0] = ptx::add_cc(s[0], Dm2[0] ^ m2);
#pragma unroll
    for (int k = 1; k < H; ++k) s[k] = ptx::addc_cc(s[k], Dm2[k] ^ m2);
    s[0] = ptx::add_cc(s[0], m2 & 1u);
#pragma unroll
    for (int k = 1; k < H; ++k) s[k] = ptx::addc_cc(s[k], 0u);
    // w0H = -s mod B
    w0[H] = ptx::sub_cc(0u, s[0]);
#pragma unroll
    for (int k = 1; k < H; ++k) w0[H + k] = ptx::subc_cc(0u, s[k]);
  }
  // ---- M = D2 + w0 + w_inf  (2H+1 words, >= 0) ----
  uint32_t M[2 * H + 1];
  M[0] = ptx::add_cc(w0[0], winf[0]);
#pragma unroll
  for (int k = 1; k < 2 * H; ++k) M[k] = ptx::addc_cc(w0[k], winf[k]);
  M[2 * H] = ptx::addc(0u, 0u);
  M[0] = ptx::add_cc(M[0], Dm2[0] ^ m2);
#pragma unroll
  for (int k = 1; k < 2 * H; ++k) M[k] = ptx::addc_cc(M[k], Dm2[k] ^ m2);
  M[2 * H] = ptx::addc(M[2 * H], m2);
  M[0] = ptx::add_cc(M[0], m2 & 1u);
#pragma unroll
  for (int k = 1; k < 2 * H; ++k) M[k] = ptx::addc_cc(M[k], 0u);
  M[2 * H] = ptx::addc(M[2 * H], 0u);
  // ---- V = T0 + w0 + M B  (words 0..3H+1); only words >= 2H are needed ----
  uint32_t V[3 * H + 2];
  V[0] = ptx::add_cc(T[0], w0[0]);
#pragma unroll
  for (int k = 1; k < 2 * H; ++k) V[k] = ptx::addc_cc(T[k], w0[k]);
  V[2 * H] = ptx::addc(0u, 0u);
#pragma unroll
  for (int k = 2 * H + 1; k < 3 * H + 2; ++k) V[k] = 0u;
  V[H] = ptx::add_cc(V[H], M[0]);
#pragma unroll
  for (int k = 1; k <= 2 * H; ++k) V[H + k] = ptx::addc_cc(V[H + k], M[k]);
  V[3 * H + 1] = ptx::addc(0u, 0u);
  // ---- r = T1 + w_inf + V[2H ..] ----
  r[0] = ptx::add_cc(T[2 * H], winf[0]);
#pragma unroll
  for (int k = 1; k < 2 * H; ++k) r[k] = ptx::addc_cc(T[2 * H + k], winf[k]);
  r[0] = ptx::add_cc(r[0], V[2 * H]);
#pragma unroll
  for (int k = 1; k < 2 * H; ++k) r[k] = ptx::addc_cc(r[k], (k <= H + 1) ? V[2 * H + k] : 0u);
}

// ------------------------------------------------------------------------------------------
// Lazy Montgomery squaring: the same unique raw value as mont_mul_cios(x, x), with
// (3L^2 + L)/2 partial products instead of 2L^2.
//   T = x^2 = sum_r x_r * V_r * 2^(64r),  V_r = [x_r, 2x_{r+1}, 2x_{r+2}, ...] taken from
//   Y = 2x (fits L words because x < 2N < 2^(32L-1)); word r+1 of Y carries bit 31 of x_r,
//   which does not belong to row r and is masked off.  Row r = L-r products at offset 2r.
//   Even/odd product offsets go to accumulators EV/OD (disjoint pairs -> one carry chain
//   each); rows run in increasing r, so each chain's carry lands in a word that so far holds
//   only earlier carries and is absorbed by one add, never rippled.
//   Reduction: the even/odd CIOS frame of mont_mul_cios on T mod R, plus T's high half.
// ------------------------------------------------------------------------------------------
//   FORM 1 (default): the triangle's even/odd accumulators are not merged — their low halves enter
//   the reduction frame directly and their high halves are added at the end (5 fewer additions at
//   L = 6; measured +2.3 % in square mode at L = 4 and 6, profiles/r02a_ab*.jsonl).  FORM 0: T is
//   merged first.  Both give the same raw value.
//   FORM 2: the same products regrouped into offset chains (sqr_triangle) and T's high half fed into
//   the reduction frame's free top slot one word per row (see mont_sqr_inj).
template <int L, bool INJ = true, int ORD = 0>
__device__ __forceinline__ void mont_sqr_inj(uint32_t (&r)[L], const uint32_t (&x)[L], const uint32_t (&n)[L],
                                             uint32_t n0inv);

template <int L, int FORM = 1>
__device__ __forceinline__ void mont_sqr(uint32_t (&r)[L], const uint32_t (&x)[L], const uint32_t (&n)[L], uint32_t n0inv) {
  static_assert(L % 2 == 0 && L >= 2, "L must be even");
  if constexpr (FORM >= 2 && FORM <= 5) {
    // 2 / 3: chain order 0, high half injected / added at the end; 4 / 5: chain order 1, added / injected
    mont_sqr_inj<L, FORM == 2 || FORM == 5, (FORM >= 4) ? 1 : 0>(r, x, n, n0inv);
    return;
  }
  uint32_t Y[L];
  Y[0] = x[0] << 1;
#pragma unroll
  for (int k = 1; k < L; ++k) Y[k] = __funnelshift_l(x[k - 1], x[k], 1);
  uint32_t EV[2 * L + 1], OD[2 * L + 1];
#pragma unroll
  for (int k = 0; k <= 2 * L; ++k) { EV[k] = 0; OD[k] = 0; }
#pragma unroll
  for (int row = 0; row < L; ++row) {
    const uint32_t xr = x[row];
    // even k -> EV pairs (2row+k, 2row+k+1)
#pragma unroll
    for (int k = 0; k < L - row; k += 2) {
      const uint32_t v = (k == 0) ? xr : Y[row + k];
      const int w = 2 * row + k;
      if (k == 0) EV[w] = ptx::mad_lo_cc(xr, v, EV[w]);
      else EV[w] = ptx::madc_lo_cc(xr, v, EV[w]);
      EV[w + 1] = ptx::madc_hi_cc(xr, v, EV[w + 1]);
    }
    {
      const int klast = ((L - row - 1) / 2) * 2;
      const int w = 2 * row + klast + 2;
      EV[w] = ptx::addc(EV[w], 0u);
    }
    // odd k -> OD pairs
    if (L - row > 1) {
#pragma unroll
      for (int k = 1; k < L - row; k += 2) {
        const uint32_t v = (k == 1) ? (Y[row + 1] & 0xfffffffeu) : Y[row + k];
        const int w = 2 * row + k;
        if (k == 1) OD[w] = ptx::mad_lo_cc(xr, v, OD[w]);
        else OD[w] = ptx::madc_lo_cc(xr, v, OD[w]);
        OD[w + 1] = ptx::madc_hi_cc(xr, v, OD[w + 1]);
      }
      const int klast = ((L - row - 2) / 2) * 2 + 1;
      const int w = 2 * row + klast + 2;
      OD[w] = ptx::addc(OD[w], 0u);
    }
  }
  if constexpr (FORM == 1) {
  // T = A + B R with A = EV mod R + OD mod R (< 2R, not merged) and B = EV div R + OD div R.
  // q depends only on A mod R = T mod R, so REDC(T) = (A + qN)/R + B.  The frame starts from
  // E = EV[0..L), O = OD[1..L) (O[k] has weight k+1; OD[0] = 0), O[L-1] = 0: its running value
  // stays < 2R + 2^32 N < (3/4) 2^(32(L+1)), so the chains' carry bounds of mont_mul_cios hold.
  {
    uint32_t E[L], O[L];
#pragma unroll
    for (int k = 0; k < L; ++k) { E[k] = EV[k]; O[k] = (k + 1 < L) ? OD[k + 1] : 0u; }
#pragma unroll
    for (int i = 0; i < L; ++i) {
      const uint32_t m = E[0] * n0inv;
      if (i == 0) chain<L, 1, false, false>(O, O, m, n);
      else chain<L, 1, true, false>(O, O, m, n);
      chain<L, 0, false, true>(E, E, m, n);
      O[L - 1] = ptx::addc(O[L - 1], 0u);
      uint32_t nE[L], nO[L];
#pragma unroll
      for (int k = 0; k < L; ++k) nE[k] = O[k];
      nE[0] = ptx::add_cc(nE[0], E[1]);
#pragma unroll
      for (int k = 0; k < L; ++k) nO[k] = (k + 2 < L) ? E[k + 2] : 0u;
#pragma unroll
      for (int k = 0; k < L; ++k) { E[k] = nE[k]; O[k] = nO[k]; }
    }
    uint32_t q[L];
    q[0] = E[0];
#pragma unroll
    for (int k = 1; k < L - 1; ++k) q[k] = ptx::addc_cc(E[k], O[k - 1]);
    q[L - 1] = ptx::addc(E[L - 1], O[L - 2]);
    q[0] = ptx::add_cc(q[0], EV[L]);
#pragma unroll
    for (int k = 1; k < L - 1; ++k) q[k] = ptx::addc_cc(q[k], EV[L + k]);
    q[L - 1] = ptx::addc(q[L - 1], EV[2 * L - 1]);
    r[0] = ptx::add_cc(q[0], OD[L]);
#pragma unroll
    for (int k = 1; k < L - 1; ++k) r[k] = ptx::addc_cc(q[k], OD[L + k]);
    r[L - 1] = ptx::addc(q[L - 1], OD[2 * L - 1]);
    return;
  }
  }
  // T = EV + OD (< 2^(64L): the top carry and EV/OD[2L] are zero)
  uint32_t T[2 * L];
  T[0] = EV[0];
  T[1] = ptx::add_cc(EV[1], OD[1]);
#pragma unroll
  for (int k = 2; k < 2 * L - 1; ++k) T[k] = ptx::addc_cc(EV[k], OD[k]);
  T[2 * L - 1] = ptx::addc(EV[2 * L - 1], OD[2 * L - 1]);
  // Word-serial reduction of T_low = T mod R in the even/odd frame of mont_mul_cios (E =
  // T_low, O = 0, no product rows), then r = (T_low + q N)/R + T_high: q depends only on
  // T mod R, so this is exactly (T + q N)/R.  (T_low + qN)/R < N + 1, so the window bounds
  // of mont_mul_cios hold and the final sum is the unique raw value < 2N.
  uint32_t E[L], O[L];
#pragma unroll
  for (int k = 0; k < L; ++k) { E[k] = T[k]; O[k] = 0; }
#pragma unroll
  for (int i = 0; i < L; ++i) {
    const uint32_t m = E[0] * n0inv;
    if (i == 0) chain<L, 1, false, false>(O, O, m, n);
    else chain<L, 1, true, false>(O, O, m, n);
    chain<L, 0, false, true>(E, E, m, n);
    O[L - 1] = ptx::addc(O[L - 1], 0u);
    uint32_t nE[L], nO[L];
#pragma unroll
    for (int k = 0; k < L; ++k) nE[k] = O[k];
    nE[0] = ptx::add_cc(nE[0], E[1]);
#pragma unroll
    for (int k = 0; k < L; ++k) nO[k] = (k + 2 < L) ? E[k + 2] : 0u;
#pragma unroll
    for (int k = 0; k < L; ++k) { E[k] = nE[k]; O[k] = nO[k]; }
  }
  uint32_t q[L];
  q[0] = E[0];
#pragma unroll
  for (int k = 1; k < L - 1; ++k) q[k] = ptx::addc_cc(E[k], O[k - 1]);
  q[L - 1] = ptx::addc(E[L - 1], O[L - 2]);
  r[0] = ptx::add_cc(q[0], T[L]);
#pragma unroll
  for (int k = 1; k < L - 1; ++k) r[k] = ptx::addc_cc(q[k], T[L + k]);
  r[L - 1] = ptx::addc(q[L - 1], T[2 * L - 1]);
}

// ------------------------------------------------------------------------------------------
// FORM 2 of the lazy square (same unique raw value, same (3L^2+L)/2 partial products).
//   Triangle by offset chains: the products P(i,j) = x_i b_ij (i <= j; b_ii = x_i, b_i,i+1 =
//   Y_{i+1} & ~1, b_ij = Y_j beyond) sit at word offset o = i + j.  An IMAD.WIDE carry chain may
//   change both factors at every link, so chain c of parity p takes, at every offset o = p, p+2, ...
//   that still has more than c products, the product with i = floor(o/2) - c: consecutive links
//   are disjoint pairs (o, o+1), (o+2, o+3), and every chain runs over a contiguous range of
//   offsets (the count per offset is unimodal).  A carry absorb is needed only where a chain
//   stops below the top — ceil(L/2) - 1 + L/2 absorbs instead of the rows' 2L - 1 (L = 6: 5 vs 11).
//   Each accumulator's partial sums stay <= its final value <= x^2 < 2^(64L), so the even
//   accumulator's top link never carries out.
//   Reduction with the high half injected: T = A + B R with A = EV mod R + OD mod R and
//   B = EV div R + OD div R (< N, since T < 4N^2 <= R N).  q depends only on A mod R, and
//   (A + qN)/R + B is computed in the CIOS frame of mont_mul_cios by placing word B_i into the
//   slot that is zero after row i's shift (O[L-2], weight L-1 = original weight R 2^(32i)): no
//   addition at all.  Frame bound: before row i+1 the frame holds at most
//   (A + q_{<=i} N)/2^(32(i+1)) + (B mod 2^(32(i+1))) 2^(32(L-i-1)) < 2R/2^32 + N + R, and the row
//   adds m N < 2^32 N: < (3/4) 2^(32(L+1)), so the chains' carry bounds of mont_mul_cios hold.
//   Against FORM 1 this saves the triangle's surplus absorbs and the final B + A merge (L adds
//   remain, for B = EV_high + OD_high).
// ------------------------------------------------------------------------------------------
//   Chain order ORD 0: shortest chains first — when chain c stops at offset e, word e + 2 has so far
//   received only the carries of the (shorter) chains already run, so a one-word absorb cannot
//   overflow; but that word and its pair partner are then fresh registers, and the longer chain that
//   later passes over the pair needs an explicit zero for the partner (ptxas emits HFMA2 / IMAD.MOV
//   zeros on the fma pipe — the square's bottleneck).
//   ORD 1: chain 0 (the diagonal, the longest) first, then the others shortest to longest.  Chain 0
//   writes every pair fresh (RZ addends, no zero registers), and when a later chain c stops at e, the
//   pair (e+2, e+3) holds chain 0's one product plus at most a carry-in and the +1s of the shorter
//   chains' absorbs (chains 1..c-1 run after c): <= 2^64 - 2^33 + 2 + L, so the carry is absorbed as
//   a 64-bit add into the pair (two ALU instructions) and can never carry out of it.
template <int L, int PAR, int ORD = 0>
__device__ __forceinline__ void sqr_triangle(uint32_t (&acc)[2 * L], const uint32_t (&x)[L], const uint32_t (&Y)[L],
                                             const uint32_t (&Ym)[L]) {
#pragma unroll
  for (int k = 0; k < L; ++k) {
    const int c = (ORD == 0) ? L - 1 - k : (k == 0) ? 0 : L - k;
    int last = -1;
#pragma unroll
    for (int o = PAR; o <= 2 * L - 2; o += 2) {
      const int i = o / 2 - c, j = o - i;
      if (i < 0 || j > L - 1) continue;  // offset o has at most c products
      const uint32_t a = x[i];
      const uint32_t b = (i == j) ? x[i] : (j == i + 1) ? Ym[j] : Y[j];
      if (last < 0) acc[o] = ptx::mad_lo_cc(a, b, acc[o]);
      else acc[o] = ptx::madc_lo_cc(a, b, acc[o]);
      if (o + 1 == 2 * L - 1) acc[o + 1] = ptx::madc_hi(a, b, acc[o + 1]);
      else acc[o + 1] = ptx::madc_hi_cc(a, b, acc[o + 1]);
      last = o;
    }
    if (last < 0 || last + 2 > 2 * L - 1) continue;
    if (ORD == 1 && c > 0 && last + 3 <= 2 * L - 1) {
      acc[last + 2] = ptx::addc_cc(acc[last + 2], 0u);
      acc[last + 3] = ptx::addc(acc[last + 3], 0u);
    } else {
      acc[last + 2] = ptx::addc(acc[last + 2], 0u);
    }
  }
}

template <int L, bool INJ, int ORD>
__device__ __forceinline__ void mont_sqr_inj(uint32_t (&r)[L], const uint32_t (&x)[L], const uint32_t (&n)[L],
                                             uint32_t n0inv) {
  uint32_t Y[L], Ym[L];
  Y[0] = x[0] << 1;
#pragma unroll
  for (int k = 1; k < L; ++k) {
    Y[k] = __funnelshift_l(x[k - 1], x[k], 1);
    Ym[k] = Y[k] & 0xfffffffeu;
  }
  Ym[0] = Y[0];
  uint32_t EV[2 * L], OD[2 * L];
#pragma unroll
  for (int k = 0; k < 2 * L; ++k) { EV[k] = 0; OD[k] = 0; }
  sqr_triangle<L, 0, ORD>(EV, x, Y, Ym);
  sqr_triangle<L, 1, ORD>(OD, x, Y, Ym);
  uint32_t B[L];
  B[0] = ptx::add_cc(EV[L], OD[L]);
#pragma unroll
  for (int k = 1; k < L - 1; ++k) B[k] = ptx::addc_cc(EV[L + k], OD[L + k]);
  B[L - 1] = ptx::addc(EV[2 * L - 1], OD[2 * L - 1]);
  uint32_t E[L], O[L];
#pragma unroll
  for (int k = 0; k < L; ++k) { E[k] = EV[k]; O[k] = (k + 1 < L) ? OD[k + 1] : 0u; }
#pragma unroll
  for (int i = 0; i < L; ++i) {
    const uint32_t m = E[0] * n0inv;
    if (i == 0) chain<L, 1, false, false>(O, O, m, n);
    else chain<L, 1, true, false>(O, O, m, n);
    chain<L, 0, false, true>(E, E, m, n);
    O[L - 1] = ptx::addc(O[L - 1], 0u);
    uint32_t nE[L], nO[L];
#pragma unroll
    for (int k = 0; k < L; ++k) nE[k] = O[k];
    nE[0] = ptx::add_cc(nE[0], E[1]);
#pragma unroll
    for (int k = 0; k < L; ++k) nO[k] = (k + 2 < L) ? E[k + 2] : (INJ && k == L - 2) ? B[i] : 0u;
#pragma unroll
    for (int k = 0; k < L; ++k) { E[k] = nE[k]; O[k] = nO[k]; }
  }
  r[0] = E[0];  // + O 2^32 + the last shift's pending carry (at word 1)
#pragma unroll
  for (int k = 1; k < L - 1; ++k) r[k] = ptx::addc_cc(E[k], O[k - 1]);
  r[L - 1] = ptx::addc(E[L - 1], O[L - 2]);
  if constexpr (!INJ) {  // FORM 3: B added at the end (no injected words: the frame's top pairs stay zero)
    r[0] = ptx::add_cc(r[0], B[0]);
#pragma unroll
    for (int k = 1; k < L - 1; ++k) r[k] = ptx::addc_cc(r[k], B[k]);
    r[L - 1] = ptx::addc(r[L - 1], B[L - 1]);
  }
}

// ------------------------------------------------------------------------------------------
// Row-interleaved (CIOS) Montgomery squaring for a CANONICAL input x < N (ECM ladder only; the
// mulmod API squares lazy inputs with mont_sqr).  Same unique raw value REDC(x^2) < 2N with
// (3L^2 + L)/2 partial products and the multiply's per-row carry handling:
//   x^2 = sum_i x_i V_i 2^(32 i), V_i = x_i + 2 sum_{j>i} x_j 2^(32(j-i)) (words of Y = 2x, bit 0
//   of Y_{i+1} masked): row i is a CIOS row of x_i times V_i, whose pairs start at word i; rows
//   i >= 1 leave word 0 alone, so m_i = E_0 n0' is known first and the reduction chain (which
//   consumes the shift's pending carry) runs before the row's short product chains.
// Bound: every row adds at most 2^32 (2x + N) before its shift, and with x < N that is
// < 2^32 3N < (3/4) 2^(32(L+1)) (N < R/4): the odd chains cannot carry out and the even chains'
// carries fit in O[L-1], as in mont_mul_cios.  (With a lazy x < 2N the sum can reach 2^32 5N,
// beyond R 2^32 when N is near R/4 — why the lazy square keeps the split form.)
// ------------------------------------------------------------------------------------------
template <int L, int PAR, int S, bool COUT>
__device__ __forceinline__ void chain_from(uint32_t (&d)[L], uint32_t a, const uint32_t (&v)[L]) {
  constexpr int j0 = (S % 2 == PAR) ? S : S + 1;
#pragma unroll
  for (int j = j0; j < L; j += 2) {
    if (j == j0) d[j - PAR] = ptx::mad_lo_cc(a, v[j], d[j - PAR]);
    else d[j - PAR] = ptx::madc_lo_cc(a, v[j], d[j - PAR]);
    if (j + 2 >= L && !COUT) d[j - PAR + 1] = ptx::madc_hi(a, v[j], d[j - PAR + 1]);
    else d[j - PAR + 1] = ptx::madc_hi_cc(a, v[j], d[j - PAR + 1]);
  }
}

template <int L, int I>
__device__ __forceinline__ void sqr_row_products(uint32_t (&E)[L], uint32_t (&O)[L], const uint32_t (&x)[L],
                                                 const uint32_t (&Y)[L]) {
  uint32_t v[L];
#pragma unroll
  for (int j = 0; j < L; ++j) v[j] = (j < I) ? 0u : (j == I) ? x[I] : (j == I + 1) ? (Y[j] & 0xfffffffeu) : Y[j];
  constexpr int je = (I % 2 == 0) ? I : I + 1;  // first even pair
  constexpr int jo = (I % 2 == 1) ? I : I + 1;  // first odd pair
  if (jo < L) chain_from<L, 1, jo, false>(O, x[I], v);
  if (je < L) {
    chain_from<L, 0, je, true>(E, x[I], v);
    O[L - 1] = ptx::addc(O[L - 1], 0u);
  }
}

template <int L, int I>
__device__ __forceinline__ void sqr_rows(uint32_t (&E)[L], uint32_t (&O)[L], const uint32_t (&x)[L],
                                         const uint32_t (&Y)[L], const uint32_t (&n)[L], uint32_t n0inv) {
  if constexpr (I < L) {
    if (I == 0) sqr_row_products<L, 0>(E, O, x, Y);
    const uint32_t m = E[0] * n0inv;
    chain<L, 1, (I > 0), false>(O, O, m, n);  // rows >= 1: consumes the pending shift carry
    chain<L, 0, false, true>(E, E, m, n);
    O[L - 1] = ptx::addc(O[L - 1], 0u);
    if (I > 0) sqr_row_products<L, I>(E, O, x, Y);
    uint32_t nE[L], nO[L];
#pragma unroll
    for (int k = 0; k < L; ++k) nE[k] = O[k];
    nE[0] = ptx::add_cc(nE[0], E[1]);
#pragma unroll
    for (int k = 0; k < L; ++k) nO[k] = (k + 2 < L) ? E[k + 2] : 0u;
#pragma unroll
    for (int k = 0; k < L; ++k) { E[k] = nE[k]; O[k] = nO[k]; }
    sqr_rows<L, I + 1>(E, O, x, Y, n, n0inv);
  }
}

template <int L>
__device__ __forceinline__ void mont_sqr_cios(uint32_t (&r)[L], const uint32_t (&x)[L], const uint32_t (&n)[L],
                                              uint32_t n0inv) {
  static_assert(L % 2 == 0 && L >= 2, "L must be even");
  uint32_t Y[L];
  Y[0] = x[0] << 1;
#pragma unroll
  for (int k = 1; k < L; ++k) Y[k] = __funnelshift_l(x[k - 1], x[k], 1);
  uint32_t E[L], O[L];
#pragma unroll
  for (int k = 0; k < L; ++k) { E[k] = 0; O[k] = 0; }
  sqr_rows<L, 0>(E, O, x, Y, n, n0inv);
  r[0] = E[0];  // + O 2^32 + the last shift's pending carry (at word 1)
#pragma unroll
  for (int k = 1; k < L - 1; ++k) r[k] = ptx::addc_cc(E[k], O[k - 1]);
  r[L - 1] = ptx::addc(E[L - 1], O[L - 2]);
}

// -N^{-1} mod R over the full width, for the block (SOS) REDC variants: Newton lifting
// x <- x (2 - N x) of N^{-1} from the 32-bit inverse, doubling the correct words.
template <int L>
__device__ __forceinline__ void nprime_full(uint32_t (&np)[L], const uint32_t (&n)[L]) {
  uint32_t x[L];
#pragma unroll
  for (int k = 0; k < L; ++k) x[k] = 0;
  x[0] = 0u - neg_inv32(n[0]);  // N^{-1} mod 2^32
#pragma unroll
  for (int correct = 1; correct < L; correct *= 2) {
    uint32_t t[L], u[L];
    mul_low_half<L>(t, n, x);  // t = N x
    // u = 2 - t  (mod R)
    u[0] = ptx::sub_cc(2u, t[0]);
#pragma unroll
    for (int k = 1; k < L; ++k) u[k] = ptx::subc_cc(0u, t[k]);
    mul_low_half<L>(t, x, u);
#pragma unroll
    for (int k = 0; k < L; ++k) x[k] = t[k];
  }
  np[0] = ptx::sub_cc(0u, x[0]);
#pragma unroll
  for (int k = 1; k < L; ++k) np[k] = ptx::subc_cc(0u, x[k]);
}

// ------------------------------------------------------------------------------------------
// Lazy add / sub in [0, 2N) with a precomputed 2N: both candidates
// are formed and the carry/borrow bit selects — no data-dependent branch.
// ------------------------------------------------------------------------------------------
template <int L>
__device__ __forceinline__ void add_lazy(uint32_t (&r)[L], const uint32_t (&x)[L], const uint32_t (&y)[L], const uint32_t (&n2)[L]) {
  uint32_t s[L], d[L];
  s[0] = ptx::add_cc(x[0], y[0]);
#pragma unroll
  for (int k = 1; k < L; ++k) s[k] = ptx::addc_cc(x[k], y[k]);
  // x + y < 4N < R: no carry out of s.  d = s - 2N; keep s if it borrowed.
  d[0] = ptx::sub_cc(s[0], n2[0]);
#pragma unroll
  for (int k = 1; k < L; ++k) d[k] = ptx::subc_cc(s[k], n2[k]);
  const uint32_t borrow = ptx::subc(0u, 0u);  // 0 or 0xffffffff
#pragma unroll
  for (int k = 0; k < L; ++k) r[k] = borrow ? s[k] : d[k];
}

template <int L>
__device__ __forceinline__ void sub_lazy(uint32_t (&r)[L], const uint32_t (&x)[L], const uint32_t (&y)[L], const uint32_t (&n2)[L]) {
  uint32_t d[L];
  d[0] = ptx::sub_cc(x[0], y[0]);
#pragma unroll
  for (int k = 1; k < L; ++k) d[k] = ptx::subc_cc(x[k], y[k]);
  const uint32_t mask = ptx::subc(0u, 0u);  // all ones iff x < y (reading G4: add 2N then)
  r[0] = ptx::add_cc(d[0], n2[0] & mask);
#pragma unroll
  for (int k = 1; k < L - 1; ++k) r[k] = ptx::addc_cc(d[k], n2[k] & mask);
  r[L - 1] = ptx::addc(d[L - 1], n2[L - 1] & mask);
}

// x in [0, 4N) -> [0, 2N): subtract 2N when x >= 2N (the reduction half of add_lazy)
template <int L>
__device__ __forceinline__ void reduce_2n(uint32_t (&x)[L], const uint32_t (&n2)[L]) {
  uint32_t d[L];
  d[0] = ptx::sub_cc(x[0], n2[0]);
#pragma unroll
  for (int k = 1; k < L; ++k) d[k] = ptx::subc_cc(x[k], n2[k]);
  const uint32_t borrow = ptx::subc(0u, 0u);
#pragma unroll
  for (int k = 0; k < L; ++k) x[k] = borrow ? x[k] : d[k];
}

// r = x - N if x >= N else x  (canonical representative of a lazy value in [0, 2N))
template <int L>
__device__ __forceinline__ void canonicalize(uint32_t (&r)[L], const uint32_t (&x)[L], const uint32_t (&n)[L]) {
  uint32_t d[L];
  d[0] = ptx::sub_cc(x[0], n[0]);
#pragma unroll
  for (int k = 1; k < L; ++k) d[k] = ptx::subc_cc(x[k], n[k]);
  const uint32_t borrow = ptx::subc(0u, 0u);
#pragma unroll
  for (int k = 0; k < L; ++k) r[k] = borrow ? x[k] : d[k];
}

// Debug builds (-DECM_DEBUG_BOUNDS=1, tools/debug_bounds.py) check the Lemma's lazy bound r < 2N
// (reading G3) after every Montgomery product and trap if it fails.
#ifndef ECM_DEBUG_BOUNDS
#define ECM_DEBUG_BOUNDS 0
#endif
template <int L>
__device__ __forceinline__ void debug_lazy_bound(const uint32_t (&r)[L], const uint32_t (&n)[L]) {
#if ECM_DEBUG_BOUNDS
  uint32_t n2[L], c = 0;
#pragma unroll
  for (int k = 0; k < L; ++k) {
    n2[k] = (n[k] << 1) | c;
    c = n[k] >> 31;
  }
  int cmp = 0;  // sign of r - 2N, decided from the top word down
#pragma unroll
  for (int k = L - 1; k >= 0; --k)
    if (cmp == 0 && r[k] != n2[k]) cmp = r[k] < n2[k] ? -1 : 1;
  if (cmp >= 0) __trap();
#else
  (void)r;
  (void)n;
#endif
}

template <int L>
__device__ __forceinline__ void mont_mul(uint32_t (&r)[L], const uint32_t (&x)[L], const uint32_t (&y)[L],
                                         const uint32_t (&n)[L], uint32_t n0inv) {
  mont_mul_cios<L, REDC_WORD>(r, x, y, n, n0inv);
  debug_lazy_bound<L>(r, n);
}

// r = c t / 2^32 mod N by one word-level REDC step, c < 2^30 a plain word, t < 2N: the product
// of t (Montgomery form) with the field element c / 2^32 (the small-parameter family's a24,
// SURVEY §8(f) N4) — 2L partial products instead of 2L^2.  c t + m N < 2^32 (1.5 N) < 2^32 R,
// so the odd chains cannot carry out, and r < 1.5 N < 2N (lazy domain).
template <int L>
__device__ __forceinline__ void mont_smul(uint32_t (&r)[L], uint32_t c, const uint32_t (&t)[L],
                                          const uint32_t (&n)[L], uint32_t n0inv) {
  uint32_t E[L], O[L], Z[L];
#pragma unroll
  for (int k = 0; k < L; ++k) Z[k] = 0;
  chain<L, 1, false, false>(O, Z, c, t);  // disjoint pairs on zero: no carries
  chain<L, 0, false, false>(E, Z, c, t);
  const uint32_t m = E[0] * n0inv;
  chain<L, 1, false, false>(O, O, m, n);
  chain<L, 0, false, true>(E, E, m, n);
  O[L - 1] = ptx::addc(O[L - 1], 0u);
  // (E + O 2^32) / 2^32 with E[0] == 0
  r[0] = ptx::add_cc(O[0], E[1]);
#pragma unroll
  for (int k = 1; k < L - 1; ++k) r[k] = ptx::addc_cc(O[k], E[k + 1]);
  r[L - 1] = ptx::addc(O[L - 1], 0u);
  debug_lazy_bound<L>(r, n);
}

}  // namespace ecm
