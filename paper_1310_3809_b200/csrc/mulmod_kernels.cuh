#pragma once
// mulmod_kernels.cuh — batched lazy Montgomery multiplication chains (ecm_mulmod_batch), sm_100a.
//
// One lane = one independent (a_i, b_i, n_i) triple (north_star: "one independent modulus and
// operand set per lane").  Stage-in (AoS): for a full 32-element tile one lane issues bulk
// asynchronous copies (cp.async.bulk, the TMA engine) of the a, b and n tiles — 32*L contiguous
// words each — into warp-private shared memory, completing on a per-warp mbarrier; each lane then
// reads its own L words.  Hot loop:
// `iters` dependent Montgomery products entirely in registers (mont.cuh).  Stage-out: lanes write
// their words back into the tile and one lane issues a bulk store.  Limb-sliced tiles move with
// 128-bit loads through the tile (load_sliced); ragged tiles and unaligned sliced rows take a
// 32-bit load path.
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <utility>

#include "kernels.h"
#include "mont.cuh"

namespace ecm {

constexpr int kMulmodTPB = 256;
// Internal flag (never accepted from callers: abi.cu rejects unknown bits before it is set): every
// limb-sliced row is 16-byte aligned — count % 4 == 0 and a, b, n, out 16-byte aligned — so the
// warp-tile kernel may move sliced tiles with 128-bit accesses.
constexpr uint32_t kVec16 = 1u << 30;
// Occupancy floor for the headline kernels (AoS, word-serial REDC, L <= 6): 6 CTAs x 8 warps per
// SM needs <= 40 registers, which the hot loop fits; other instantiations are left unconstrained.
// Chain-loop unroll and the limb-sliced L <= 6 kernels' occupancy (tools/ecm_ab.py variants,
// DESIGN.md §6.2): unrolled by 8 and held to 64 registers (4 CTAs x 8 warps per SM), the L = 6
// sliced chains measured +0.6 % (multiply) and +3.5 % (square) over unroll 4 / 76 registers.
// Per width (multiply / square, word REDC): L = 4: 8 / 16, L = 6: 8 / 16, L = 8: 2 / 8,
// L = 12, 16: 2 / 2 — each the best of {2, 4, 8, 16} measured; other REDC variants keep 4.  (L = 6 square:
// 8 until the n0' slot; with it, 16 measured 0.862 -> 0.869 — 8 HFMA2 zeros per 8 squares left on the fma
// pipe instead of 12 IMAD.X + 4 IMAD.MOV + 6 HFMA2; profiles/r02s_ab.jsonl.)
// MULMOD_UNROLL / MULMOD_SLICED_MINB override them for experiments.
#ifndef MULMOD_UNROLL
#define MULMOD_UNROLL 0  // 0: per-width default below
#endif
// Square form of the chains (mont.cuh mont_sqr: 1 = split rows; 2..5 = offset-chain triangle with chain
// order 0 (2, 3) or 1 (4, 5), the high half injected into the reduction frame (2, 5) or added at the end
// (3, 4)), per width the measured best (tools/ecm_ab.py; profiles/r02e/f/i_ab*.jsonl): FORM 4 at L <= 8
// (square mode L = 4 / 6: 0.746 / 0.824 with FORM 1 -> 0.796 / 0.857), FORM 1 at L = 12, FORM 2 at L = 16.
#ifndef MULMOD_SQR_FORM
#define MULMOD_SQR_FORM -1
#endif
__host__ __device__ constexpr int mulmod_sqr_form(int L) {
  return MULMOD_SQR_FORM >= 0 ? MULMOD_SQR_FORM : L <= 8 ? 4 : L == 12 ? 1 : 2;
}
#ifndef MULMOD_SLICED_MINB
#define MULMOD_SLICED_MINB 4
#endif
__host__ __device__ constexpr int mulmod_unroll(int L, int V, bool square) {
  return MULMOD_UNROLL > 0 ? MULMOD_UNROLL
         : V != 0        ? 4
         : L <= 6        ? (square ? 16 : 8)
         : L <= 8        ? (square ? 8 : 2)
                         : 2;
}
__host__ __device__ constexpr int mulmod_min_blocks(int L, int V, bool sliced) {
  return (!sliced && V == 0 && L <= 6) ? 6 : (sliced && V == 0 && L <= 6) ? MULMOD_SLICED_MINB : 1;
}


// ---- bulk asynchronous copies (the TMA engine: cp.async.bulk -> SASS UBLKCP) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  } while (!done);
}
// global -> shared, completes on the mbarrier (size and addresses multiples of 16 bytes)
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// shared -> global, tracked by bulk groups
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Warp-cooperative AoS tile load: words [e0*L, e0*L + nvalid*L) -> smem tile, then lane's L words.
template <int L>
__device__ __forceinline__ void load_aos(uint32_t (&v)[L], const uint32_t* __restrict__ g, uint32_t* tile,
                                         size_t e0, int nvalid, int lane) {
  const uint32_t* src = g + e0 * L;
  if (nvalid == 32) {
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* t4 = reinterpret_cast<uint4*>(tile);
#pragma unroll
    for (int k = lane; k < 8 * L; k += 32) t4[k] = __ldcs(s4 + k);
  } else {
    for (int k = lane; k < nvalid * L; k += 32) tile[k] = __ldcs(src + k);
  }
  __syncwarp();
  const uint2* t2 = reinterpret_cast<const uint2*>(tile) + lane * (L / 2);
  const bool valid = lane < nvalid;  // dead lanes of a ragged tile do not read unwritten words
#pragma unroll
  for (int k = 0; k < L / 2; ++k) {
    const uint2 w = valid ? t2[k] : make_uint2(0u, 0u);
    v[2 * k] = w.x;
    v[2 * k + 1] = w.y;
  }
  __syncwarp();
}

// Limb-sliced tile (ECM_LAYOUT_SLICED): limb j of the warp's 32 elements is the 128-byte row
// g[j*count + e0 .. +32).  With 16-byte-aligned rows (`vec`: count % 4 == 0 and every array
// 16-byte aligned, decided on the host: kVec16) the warp moves the L rows with 128-bit loads, 8
// lanes per row, into smem tile[j*32 + lane]; each lane then reads its limb j at tile[j*32 + lane]
// (consecutive lanes, consecutive banks: conflict-free).  Otherwise 32-bit loads.
template <int L>
__device__ __forceinline__ void load_sliced(uint32_t (&v)[L], const uint32_t* __restrict__ g, uint32_t* tile,
                                            size_t count, size_t e0, int nvalid, int lane, bool vec) {
  if (nvalid == 32 && vec) {
    uint4* t4 = reinterpret_cast<uint4*>(tile);
#pragma unroll
    for (int k = lane; k < 8 * L; k += 32) {
      const int row = k >> 3, col = k & 7;
      t4[k] = __ldcs(reinterpret_cast<const uint4*>(g + (size_t)row * count + e0) + col);
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < L; ++j) v[j] = tile[j * 32 + lane];
    __syncwarp();
  } else {
#pragma unroll
    for (int j = 0; j < L; ++j) v[j] = lane < nvalid ? __ldcs(g + (size_t)j * count + e0 + lane) : 0u;
  }
}

template <int L>
__device__ __forceinline__ void store_sliced(uint32_t* __restrict__ g, const uint32_t (&v)[L], uint32_t* tile,
                                             size_t count, size_t e0, int nvalid, int lane, bool vec) {
  if (nvalid == 32 && vec) {
#pragma unroll
    for (int j = 0; j < L; ++j) tile[j * 32 + lane] = v[j];
    __syncwarp();
    const uint4* t4 = reinterpret_cast<const uint4*>(tile);
#pragma unroll
    for (int k = lane; k < 8 * L; k += 32) {
      const int row = k >> 3, col = k & 7;
      __stcs(reinterpret_cast<uint4*>(g + (size_t)row * count + e0) + col, t4[k]);
    }
    __syncwarp();
  } else if (lane < nvalid) {
#pragma unroll
    for (int j = 0; j < L; ++j) __stcs(g + (size_t)j * count + e0 + lane, v[j]);
  }
}

template <int L>
__device__ __forceinline__ void store_aos(uint32_t* __restrict__ g, const uint32_t (&v)[L], uint32_t* tile,
                                          size_t e0, int nvalid, int lane) {
  uint2* t2 = reinterpret_cast<uint2*>(tile) + lane * (L / 2);
#pragma unroll
  for (int k = 0; k < L / 2; ++k) t2[k] = make_uint2(v[2 * k], v[2 * k + 1]);
  __syncwarp();
  uint32_t* dst = g + e0 * L;
  if (nvalid == 32) {
    const uint4* t4 = reinterpret_cast<const uint4*>(tile);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int k = lane; k < 8 * L; k += 32) __stcs(d4 + k, t4[k]);
  } else {
    for (int k = lane; k < nvalid * L; k += 32) dst[k] = tile[k];
  }
  __syncwarp();
}

// The hot loop of one lane: x <- REDC(x*y) (or REDC(x^2)) `iters` times, all in registers,
// then the optional canonicalisation.  Unrolled per width (mulmod_unroll): ptxas then keeps the carry
// absorbs on the ALU pipe and renames instead of copying (SASS: at most 2 IMAD.X per 4 products instead
// of 5-7 per product; tools/loopcount.py, tests/test_sass.py).
// n0' = -N^{-1} mod 2^32 parked in a per-thread shared-memory slot and re-read once per product (an
// LDS on the MIO pipe): under the register cap ptxas otherwise rematerialises the Newton iteration
// (5 IMAD on the fma pipe, the chains' bottleneck) at the top of every unrolled block.  Limb-sliced
// warp-tile kernels only, per width the measured best (profiles/r02o_ab.jsonl, r02p_ab.jsonl: same
// process and box, alternating rounds, fractions of the IMAD.WIDE peak): L = 6 multiply 0.907 -> 0.911,
// square 0.856 -> 0.861; L = 4 square 0.795 -> 0.797; L = 12 square 0.898 -> 0.900; L = 16 multiply
// 0.932 -> 0.934, square 0.874 -> 0.879.  Kept in a register: L = 4 multiply (-0.5 %), L = 8 square
// (-0.7 %), L = 8 / 12 multiply (no change) and the AoS kernels (L = 6: -0.2 % / -1 %).
// MULMOD_N0_SMEM=0/1 forces it.
#ifndef MULMOD_N0_SMEM
#define MULMOD_N0_SMEM -1
#endif
__host__ __device__ constexpr bool mulmod_n0_smem(int L, int V, bool square) {
  return MULMOD_N0_SMEM >= 0 ? MULMOD_N0_SMEM != 0
                             : V == REDC_WORD && (L == 6 || L == 16 || (square && (L == 4 || L == 12)));
}
__device__ __forceinline__ uint32_t ld_volatile_shared(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)));
  return v;
}
// N0SLOT: the caller is the limb-sliced warp-tile kernel (the streaming kernel, K <= 4, keeps n0' in a
// register and its shared memory for the copy ring).
template <int L, int V, bool SQUARE, bool N0SLOT = false>
__device__ __forceinline__ void mulmod_chain(uint32_t (&x)[L], const uint32_t (&y)[L], const uint32_t (&nn)[L],
                                             uint32_t iters, bool canon) {
  constexpr bool kN0Smem = N0SLOT && mulmod_n0_smem(L, V, SQUARE);
  __shared__ uint32_t s_n0inv[kN0Smem ? kMulmodTPB : 1];
  const uint32_t n0reg = neg_inv32(nn[0]);
  if (kN0Smem) s_n0inv[threadIdx.x] = n0reg;
  uint32_t np[L], dN[L / 2], sn = 0;
  if (V == REDC_BLOCKTHM || V == REDC_CLASSIC || V == REDC_KARATSUBA) nprime_full<L>(np, nn);
  if (V == REDC_KARATSUBA) kara_consts<L>(dN, sn, nn);
  constexpr int kUnroll = mulmod_unroll(L, V, SQUARE);
#pragma unroll kUnroll
  for (uint32_t t = iters; t != 0; --t) {
    const uint32_t n0inv = kN0Smem ? ld_volatile_shared(&s_n0inv[threadIdx.x]) : n0reg;
    uint32_t r[L];
    if (V == REDC_WORD || V == REDC_KNOWNLOW) {
      if (SQUARE && V == REDC_WORD) mont_sqr<L, mulmod_sqr_form(L)>(r, x, nn, n0inv);
      else if (SQUARE) mont_mul_cios<L, V>(r, x, x, nn, n0inv);
      else mont_mul_cios<L, V>(r, x, y, nn, n0inv);
    } else if (V == REDC_KARATSUBA) {
      if (SQUARE) mont_mul_kara<L>(r, x, x, nn, np, dN, sn);
      else mont_mul_kara<L>(r, x, y, nn, np, dN, sn);
    } else {
      if (SQUARE) mont_mul_block<L, V>(r, x, x, nn, np);
      else mont_mul_block<L, V>(r, x, y, nn, np);
    }
    debug_lazy_bound<L>(r, nn);
#pragma unroll
    for (int k = 0; k < L; ++k) x[k] = r[k];
  }
  if (canon) {
    uint32_t r[L];
    canonicalize<L>(r, x, nn);
#pragma unroll
    for (int k = 0; k < L; ++k) x[k] = r[k];
  }
}

// One thread = one element; the layout (AoS or limb-sliced) is a template parameter so that
// each kernel carries only its own staging code (register allocation is per kernel: sharing one
// kernel raised the AoS kernel from 40 to 56 registers and cost 3 % at C2).  Two independent
// chains per thread were measured at +0.5 % only: the kernel is bound by the IMAD.WIDE pipe,
// not by dependency latency.
template <int L, int V, bool SQUARE, bool SLICED>
__global__ void __launch_bounds__(kMulmodTPB, mulmod_min_blocks(L, V, SLICED)) mulmod_batch_kernel(const uint32_t* __restrict__ a,
                                                                  const uint32_t* __restrict__ b,
                                                                  const uint32_t* __restrict__ n,
                                                                  uint32_t* out, size_t count, uint32_t iters,
                                                                  uint32_t flags) {
  // per warp: tiles A, B, N (32*L words each; A is reused for the output) + one mbarrier
  extern __shared__ __align__(128) uint32_t smem[];
  constexpr int TW = 32 * L;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  uint32_t* tA = smem + warp * 3 * TW;
  uint32_t* tB = tA + TW;
  uint32_t* tN = tB + TW;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (kMulmodTPB / 32) * 3 * TW) + warp;
  const bool canon = flags & 0x1u;
  const bool vec = flags & kVec16;
  // bulk-copy path: AoS full tiles (one 32*L-word copy per array).  Limb-sliced tiles would need
  // L 128-byte copies per array: measured slower than 128-bit loads (48.7 % vs 55.8 % of HBM at
  // K = 1), and so was issuing all three arrays' 128-bit loads before one sync (51 %, 94
  // registers), so sliced tiles use load_sliced (per array, 128-bit loads through the tile).
  const bool bulk_ok = !SLICED;
  if (lane == 0) mbar_init(bar);
  __syncwarp();
  uint32_t phase = 0;
  const size_t ntiles = (count + 31) / 32;
  const size_t warps_total = (size_t)gridDim.x * (kMulmodTPB / 32);
  for (size_t wt = (size_t)blockIdx.x * (kMulmodTPB / 32) + warp; wt < ntiles; wt += warps_total) {
    const size_t e0 = wt * 32;
    const int nvalid = (int)((count - e0) < 32 ? (count - e0) : 32);
    uint32_t x[L], y[L], nn[L];
    const bool bulk = bulk_ok && nvalid == 32;
    if (bulk) {
      // stage-in: one lane issues the bulk copies of all three tiles at once (TMA engine)
      if (lane == 0) {
        bulk_wait_read();  // the previous tile's output store has finished reading tile A
        constexpr uint32_t bytes = 4u * TW;
        mbar_expect_tx(bar, (SQUARE ? 2u : 3u) * bytes);
        bulk_load(tA, a + e0 * L, bytes, bar);
        if (!SQUARE) bulk_load(tB, b + e0 * L, bytes, bar);
        bulk_load(tN, n + e0 * L, bytes, bar);
      }
      mbar_wait(bar, phase);
      phase ^= 1u;
#pragma unroll
      for (int k = 0; k < L; ++k) {
        const int idx = lane * L + k;
        x[k] = tA[idx];
        y[k] = SQUARE ? 0u : tB[idx];
        nn[k] = tN[idx];
      }
    } else if (SLICED) {
      load_sliced<L>(x, a, tA, count, e0, nvalid, lane, vec);
      if (!SQUARE) load_sliced<L>(y, b, tA, count, e0, nvalid, lane, vec);
      load_sliced<L>(nn, n, tA, count, e0, nvalid, lane, vec);
    } else {
      load_aos<L>(x, a, tA, e0, nvalid, lane);
      if (!SQUARE) load_aos<L>(y, b, tA, e0, nvalid, lane);
      load_aos<L>(nn, n, tA, e0, nvalid, lane);
    }
    if (lane >= nvalid) nn[0] |= 1u;  // keep dead lanes' arithmetic well-defined
    mulmod_chain<L, V, SQUARE, SLICED>(x, y, nn, iters, canon);
    if (bulk) {
      // stage-out: each lane writes its own words of tile A (the ones it read), then one lane
      // issues the bulk store; generic-proxy writes are fenced for the async proxy first.
#pragma unroll
      for (int k = 0; k < L; ++k) tA[lane * L + k] = x[k];
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        bulk_store(out + e0 * L, tA, 4u * TW);
        bulk_commit();
      }
    } else if (SLICED) {
      store_sliced<L>(out, x, tA, count, e0, nvalid, lane, vec);
    } else {
      store_aos<L>(out, x, tA, e0, nvalid, lane);
    }
    // every lane's reads of tiles B and N precede the next bulk writes into them
    fence_async_smem();
    __syncwarp();
  }
  if (lane == 0) bulk_wait_all();
}


// ---- CTA-tile streaming kernel: the memory-bound regime (short chains, K = 1 in C2) ----
// A persistent CTA of 256 threads walks the tiles blockIdx.x, blockIdx.x + gridDim.x, ... of
// 256 elements each through an S-stage ring of shared-memory buffers: thread 0 keeps S tiles'
// bulk copies (cp.async.bulk, the TMA engine) in flight, so the HBM reads of tile i+S overlap
// the products of tile i; outputs leave through two shared tiles by bulk stores.  AoS tiles
// are one contiguous 256*L-word copy per array; limb-sliced tiles are L copies of 1 KiB rows
// per array (row j = words [j*count + e0, +256)), so both layouts move in >= 1 KiB transfers
// and each thread then reads its words from shared memory (sliced: conflict-free).
constexpr int kStreamTPB = 256;
template <int L>
__host__ __device__ constexpr int stream_stages() { return L <= 6 ? 3 : 2; }
template <int L>
__host__ __device__ constexpr size_t stream_smem() {
  return (size_t)(3 * stream_stages<L>() + 2) * kStreamTPB * L * sizeof(uint32_t) + 8 * stream_stages<L>();
}

template <int L, bool SQUARE, bool SLICED>
__device__ __forceinline__ void stream_issue(uint32_t* st, uint64_t* bar, const uint32_t* __restrict__ a,
                                             const uint32_t* __restrict__ b, const uint32_t* __restrict__ n,
                                             size_t count, size_t e0) {
  constexpr int TW = kStreamTPB * L;
  constexpr uint32_t bytes = 4u * TW;
  mbar_expect_tx(bar, (SQUARE ? 2u : 3u) * bytes);
  if (!SLICED) {
    bulk_load(st, a + e0 * L, bytes, bar);
    if (!SQUARE) bulk_load(st + TW, b + e0 * L, bytes, bar);
    bulk_load(st + 2 * TW, n + e0 * L, bytes, bar);
  } else {
    constexpr uint32_t row = 4u * kStreamTPB;
#pragma unroll
    for (int j = 0; j < L; ++j) {
      const size_t off = (size_t)j * count + e0;
      bulk_load(st + j * kStreamTPB, a + off, row, bar);
      if (!SQUARE) bulk_load(st + TW + j * kStreamTPB, b + off, row, bar);
      bulk_load(st + 2 * TW + j * kStreamTPB, n + off, row, bar);
    }
  }
}

template <int L, int V, bool SQUARE, bool SLICED>
__global__ void __launch_bounds__(kStreamTPB) mulmod_stream_kernel(const uint32_t* __restrict__ a,
                                                                   const uint32_t* __restrict__ b,
                                                                   const uint32_t* __restrict__ n, uint32_t* out,
                                                                   size_t count, uint32_t iters, uint32_t flags) {
  extern __shared__ __align__(128) uint32_t smem[];
  constexpr int S = stream_stages<L>();
  constexpr int T = kStreamTPB, TW = T * L;
  uint32_t* obuf = smem + S * 3 * TW;  // two output tiles
  uint64_t* bars = reinterpret_cast<uint64_t*>(obuf + 2 * TW);
  const int tid = threadIdx.x;
  const bool canon = flags & 0x1u;
  const size_t nfull = count / T;
  const size_t my_n = nfull > blockIdx.x ? (nfull - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) mbar_init(&bars[s]);
    for (int s = 0; s < S && (size_t)s < my_n; ++s)
      stream_issue<L, SQUARE, SLICED>(smem + s * 3 * TW, &bars[s], a, b, n, count,
                                      ((size_t)blockIdx.x + (size_t)s * gridDim.x) * T);
  }
  __syncthreads();
  for (size_t i = 0; i < my_n; ++i) {
    const int s = (int)(i % S);
    uint32_t* st = smem + s * 3 * TW;
    mbar_wait(&bars[s], (uint32_t)((i / S) & 1u));
    uint32_t x[L], y[L], nn[L];
#pragma unroll
    for (int k = 0; k < L; ++k) {
      const int idx = SLICED ? k * T + tid : tid * L + k;
      x[k] = st[idx];
      y[k] = SQUARE ? 0u : st[TW + idx];
      nn[k] = st[2 * TW + idx];
    }
    fence_async_smem();
    if (tid == 0) bulk_wait_read1();  // output tile (i & 1) is free: the store of tile i-2 has read it
    __syncthreads();                  // every thread has read stage s
    if (tid == 0 && i + S < my_n)
      stream_issue<L, SQUARE, SLICED>(st, &bars[s], a, b, n, count, ((size_t)blockIdx.x + (i + S) * gridDim.x) * T);
    mulmod_chain<L, V, SQUARE>(x, y, nn, iters, canon);
    uint32_t* ob = obuf + (i & 1) * TW;
#pragma unroll
    for (int k = 0; k < L; ++k) ob[SLICED ? k * T + tid : tid * L + k] = x[k];
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      const size_t e0 = ((size_t)blockIdx.x + i * gridDim.x) * T;
      if (!SLICED) {
        bulk_store(out + e0 * L, ob, 4u * TW);
      } else {
#pragma unroll
        for (int j = 0; j < L; ++j) bulk_store(out + (size_t)j * count + e0, ob + j * T, 4u * T);
      }
      bulk_commit();
    }
  }
  // ragged tail (count % 256 elements): one CTA, direct loads
  if (nfull * T < count && blockIdx.x == nfull % gridDim.x) {
    const size_t e = nfull * T + tid;
    if (e < count) {
      uint32_t x[L], y[L], nn[L];
#pragma unroll
      for (int k = 0; k < L; ++k) {
        const size_t off = SLICED ? (size_t)k * count + e : e * L + k;
        x[k] = a[off];
        y[k] = SQUARE ? 0u : b[off];
        nn[k] = n[off];
      }
      mulmod_chain<L, V, SQUARE>(x, y, nn, iters, canon);
#pragma unroll
      for (int k = 0; k < L; ++k) out[SLICED ? (size_t)k * count + e : e * L + k] = x[k];
    }
  }
  if (tid == 0) bulk_wait_all();
}

// Which kernel runs a chain: the CTA-tile streaming kernel for short (memory-bound) chains,
// the warp-tile kernel for long (IMAD-bound) ones.  Sliced streaming needs
// 16-byte-aligned rows.  ECM_KERNEL_STREAM / ECM_KERNEL_WARP force one (diagnostic flags).
constexpr uint32_t kStreamMaxIters = 4;
static inline bool use_stream_kernel(const uint32_t* a, const uint32_t* b, const uint32_t* n, const uint32_t* out,
                              size_t count, uint32_t iters, uint32_t flags) {
  if (flags & 0x4u) {
    const auto al = [](const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
    if ((count & 3u) || !al(a) || !al(b) || !al(n) || !al(out)) return false;
  }
  if (flags & 0x800u) return true;    // ECM_KERNEL_STREAM
  if (flags & 0x1000u) return false;  // ECM_KERNEL_WARP
  return iters <= kStreamMaxIters;
}

// Resident CTAs per SM of a streaming kernel, cached per (device, kernel); also raises the
// kernel's dynamic shared memory limit (once per device and kernel).
static inline cudaError_t stream_occupancy(const void* kern, size_t smem, int* occ) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> cache;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_pair(dev, kern);
  const auto it = cache.find(key);
  if (it != cache.end()) {
    *occ = it->second;
    return cudaSuccess;
  }
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, kern, kStreamTPB, smem);
  if (e != cudaSuccess) return e;
  cache[key] = *occ;
  return cudaSuccess;
}

// wave != nullptr: launch nothing, return in *wave the elements one full wave of the kernel this
// call would run processes (SMs x resident CTAs x elements per CTA), for wave-multiple chunking.
template <int L, int V>
static cudaError_t launch_mulmod_LV(const uint32_t* a, const uint32_t* b, const uint32_t* n, uint32_t* out,
                                    size_t count, uint32_t iters, uint32_t flags, cudaStream_t s, size_t* wave) {
  const size_t ntiles = (count + 31) / 32;
  size_t blocks = (ntiles + (kMulmodTPB / 32) - 1) / (kMulmodTPB / 32);
  if (blocks > 0x7fffffffull) blocks = 0x7fffffffull;
  const unsigned g = (unsigned)blocks;
  const bool sq = flags & 0x2u, sl = flags & 0x4u;
  {
    const auto al = [](const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
    flags &= ~kVec16;
    if (sl && (count & 3u) == 0 && al(a) && al(b) && al(n) && al(out)) flags |= kVec16;
  }
  constexpr size_t smem = (size_t)(kMulmodTPB / 32) * (3 * 32 * L * sizeof(uint32_t) + sizeof(uint64_t));
  static_assert(smem <= 200 * 1024, "tile staging does not fit shared memory");
  auto sm_count = [](int* sms) -> cudaError_t {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, dev);
    return e;
  };
  auto go = [&](auto kern) -> cudaError_t {
    if (smem > 48 * 1024) {
      const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    if (wave) {
      int occ = 0, sms = 0;
      cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kMulmodTPB, smem);
      if (e == cudaSuccess) e = sm_count(&sms);
      *wave = (size_t)sms * (size_t)(occ > 0 ? occ : 1) * kMulmodTPB;
      return e;
    }
    kern<<<g, kMulmodTPB, smem, s>>>(a, b, n, out, count, iters, flags);
    return cudaGetLastError();
  };
  if (V == REDC_WORD && use_stream_kernel(a, b, n, out, count, iters, flags)) {
    constexpr size_t ssm = stream_smem<L>();
    auto gs = [&](auto kern) -> cudaError_t {
      int occ = 0;
      cudaError_t e = stream_occupancy(reinterpret_cast<const void*>(kern), ssm, &occ);
      if (e != cudaSuccess) return e;
      int sms = 0;
      e = sm_count(&sms);
      if (e != cudaSuccess) return e;
      const size_t nfull = count / kStreamTPB;
      size_t grid = (size_t)sms * (size_t)(occ > 0 ? occ : 1);
      if (wave) {
        *wave = grid * kStreamTPB;
        return cudaSuccess;
      }
      if (grid > nfull) grid = nfull > 0 ? nfull : 1;
      kern<<<(unsigned)grid, kStreamTPB, ssm, s>>>(a, b, n, out, count, iters, flags);
      return cudaGetLastError();
    };
    if (sq && sl) return gs(mulmod_stream_kernel<L, V, true, true>);
    if (sq) return gs(mulmod_stream_kernel<L, V, true, false>);
    if (sl) return gs(mulmod_stream_kernel<L, V, false, true>);
    return gs(mulmod_stream_kernel<L, V, false, false>);
  }
  if (sq && sl) return go(mulmod_batch_kernel<L, V, true, true>);
  if (sq) return go(mulmod_batch_kernel<L, V, true, false>);
  if (sl) return go(mulmod_batch_kernel<L, V, false, true>);
  return go(mulmod_batch_kernel<L, V, false, false>);
}

template <int L>
cudaError_t launch_mulmod_L(const uint32_t* a, const uint32_t* b, const uint32_t* n, uint32_t* out,
                                   size_t count, uint32_t iters, uint32_t flags, cudaStream_t s, size_t* wave) {
  switch ((flags >> 8) & 7u) {
    case REDC_WORD: return launch_mulmod_LV<L, REDC_WORD>(a, b, n, out, count, iters, flags, s, wave);
    case REDC_KNOWNLOW: return launch_mulmod_LV<L, REDC_KNOWNLOW>(a, b, n, out, count, iters, flags, s, wave);
    case REDC_BLOCKTHM: return launch_mulmod_LV<L, REDC_BLOCKTHM>(a, b, n, out, count, iters, flags, s, wave);
    case REDC_CLASSIC: return launch_mulmod_LV<L, REDC_CLASSIC>(a, b, n, out, count, iters, flags, s, wave);
    case REDC_KARATSUBA: return launch_mulmod_LV<L, REDC_KARATSUBA>(a, b, n, out, count, iters, flags, s, wave);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ecm
