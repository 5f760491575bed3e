// abi.cu — extern "C" entry points of libecmgpu (declared and documented in include/ecmgpu.h).
//
// Host responsibilities: argument validation (before anything is enqueued), the per-modulus
// constants shared by all curves (R mod N, R^2 mod N, 2N, -N^{-1} mod 2^32), the stage-1
// scalar k = prod p^e (reading G8) as little-endian words cached per (device, B1),
// optional host<->device staging (ECM_HOST_BUFFERS) and optional device-side precondition
// checks (ECM_CHECK).  All device work is stream ordered on the caller's stream.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "../../include/ecmgpu.h"
#include "kernels.h"

#ifndef ECMGPU_VERSION
#define ECMGPU_VERSION "dev"
#endif

namespace {

using ecm::EcmParams;

constexpr uint32_t kKnownFlags = ECM_CANONICAL | ECM_SQUARE | ECM_LAYOUT_SLICED | ECM_CHECK | ECM_HOST_BUFFERS |
                                 ECM_NO_XAFF | ECM_EAGER | ECM_PRIME_LADDERS | ECM_REDC_MASK |
                                 ECM_KERNEL_STREAM | ECM_KERNEL_WARP | ECM_KERNEL_LANES4 | ECM_KERNEL_LANES1 |
                                 ECM_CURVE_SMALL;

// widths: L in {4, 6, 8, 12, 16} for mulmod and ECM (510-bit moduli at L = 16; the
// L = 16 ladder kernel holds its six-residue state in 254 registers without spilling)
bool valid_L(int L) { return L == 4 || L == 6 || L == 8 || L == 12 || L == 16; }
bool valid_L_mulmod(int L) { return valid_L(L); }
// count small enough that every byte size the calls form (4 arrays x count x L words, and the
// kernels' element indices) fits size_t with room: 2^40 elements (far beyond device memory)
bool valid_count(size_t count) { return count != 0 && count <= ((size_t)1 << 40); }

// ---- host multiprecision helpers (little-endian 32-bit words, fixed width W) ----
int bitlen(const uint32_t* a, int W) {
  for (int k = W - 1; k >= 0; --k)
    if (a[k]) return 32 * k + (32 - __builtin_clz(a[k]));
  return 0;
}

// 2^e mod N by repeated doubling with a conditional subtraction (N odd, N >= 3).
void pow2_mod(uint32_t* out, int e, const uint32_t* N, int L) {
  std::vector<uint64_t> x(L + 1, 0), n(L + 1, 0);
  for (int k = 0; k < L; ++k) n[k] = N[k];
  x[0] = 1;
  for (int step = 0; step < e; ++step) {
    uint64_t c = 0;
    for (int k = 0; k <= L; ++k) {
      const uint64_t t = (x[k] << 1) | c;
      c = x[k] >> 31;
      x[k] = t & 0xffffffffull;
    }
    // if x >= N: x -= N
    int cmp = 0;
    for (int k = L; k >= 0 && !cmp; --k) cmp = (x[k] > n[k]) - (x[k] < n[k]);
    if (cmp >= 0) {
      int64_t br = 0;
      for (int k = 0; k <= L; ++k) {
        const int64_t t = (int64_t)x[k] - (int64_t)n[k] - br;
        br = t < 0;
        x[k] = (uint64_t)(t + (br ? (int64_t)1 << 32 : 0));
      }
    }
  }
  for (int k = 0; k < L; ++k) out[k] = (uint32_t)x[k];
}

ecm_status make_params(EcmParams& p, const uint32_t* N, int L) {
  std::memset(&p, 0, sizeof(p));
  if (!(N[0] & 1u)) return ECM_E_MODULUS;
  const int bl = bitlen(N, L);
  if (bl < 2 || (bl == 2 && N[0] < 3)) return ECM_E_MODULUS;
  if (bl > 32 * L - 2) return ECM_E_WIDTH;
  p.L = L;
  std::memcpy(p.N, N, sizeof(uint32_t) * L);
  uint32_t c = 0;
  for (int k = 0; k < L; ++k) {
    p.N2[k] = (N[k] << 1) | c;
    c = N[k] >> 31;
  }
  pow2_mod(p.ONE, 32 * L, N, L);
  pow2_mod(p.R2, 64 * L, N, L);
  // -N0^{-1} mod 2^32 by Newton iteration
  uint32_t x = N[0];  // correct to 3 bits
  for (int i = 0; i < 5; ++i) x *= 2u - N[0] * x;
  p.n0inv = 0u - x;
  // -N^{-1} mod R word by word: choose word i of X so that word i of N*X is 0xffffffff
  std::vector<uint64_t> S(L + 1, 0);
  for (int i = 0; i < L; ++i) {
    const uint32_t xi = (uint32_t)((0xffffffffull - S[i]) & 0xffffffffull) * p.n0inv * 0xffffffffu;  // * N0^{-1}
    p.NP[i] = xi;
    uint64_t c = 0;
    for (int j = 0; i + j < L; ++j) {
      const uint64_t t = S[i + j] + (uint64_t)xi * N[j] + c;
      S[i + j] = t & 0xffffffffull;
      c = t >> 32;
    }
  }
  return ECM_OK;
}

// ---- stage-1 scalar k(B1), little-endian words, padded to a multiple of 32 words ----
std::vector<uint32_t> stage1_scalar(uint64_t B1, uint32_t* bits_out) {
  std::vector<uint8_t> sieve(B1 + 1, 1);
  std::vector<uint32_t> k{1};
  for (uint64_t p = 2; p <= B1; ++p) {
    if (!sieve[p]) continue;
    for (uint64_t q = p * p; q <= B1; q += p) sieve[q] = 0;
    uint64_t pe = p;
    while (pe <= B1 / p) pe *= p;  // largest p^e <= B1
    uint64_t carry = 0;
    for (auto& w : k) {
      const uint64_t t = (uint64_t)w * pe + carry;
      w = (uint32_t)t;
      carry = t >> 32;
    }
    while (carry) {
      k.push_back((uint32_t)carry);
      carry >>= 32;
    }
  }
  *bits_out = (uint32_t)bitlen(k.data(), (int)k.size());
  k.resize(((k.size() + 31) / 32) * 32, 0u);
  return k;
}

struct PlanCache {
  std::mutex mu;
  std::map<std::pair<int, uint64_t>, std::pair<uint32_t*, uint32_t>> plans;  // (device, B1) -> (words, bits)
};
PlanCache& cache() {
  static PlanCache* c = new PlanCache();  // intentionally leaked: device memory lives for the process
  return *c;
}

ecm_status cuda_err(cudaError_t e) {
  if (e == cudaSuccess) return ECM_OK;
  if (e == cudaErrorMemoryAllocation) return ECM_E_NOMEM;
  return ECM_E_CUDA;
}

// ablation variants of the ECM kernel exist for L = 6 and 8 only (csrc/ecm.cu)
bool ecm_variant_ok(int L, uint32_t flags) {
  if ((flags & ECM_REDC_MASK) > ECM_REDC_CLASSIC) return false;  // Karatsuba REDC: mulmod only
  const bool ablation = (flags & ECM_REDC_MASK) || (flags & ECM_EAGER);
  if ((flags & ECM_KERNEL_LANES4) && (flags & ECM_KERNEL_LANES1)) return false;
  if ((flags & ECM_KERNEL_LANES4) && (ablation || (flags & ECM_PRIME_LADDERS))) return false;
  if ((flags & ECM_CURVE_SMALL) && (ablation || (flags & ECM_PRIME_LADDERS))) return false;
  if (flags & ECM_PRIME_LADDERS) {
    if (L == 8) return (flags & ECM_REDC_MASK) != ECM_REDC_KNOWNLOW;
    return L == 6 && !ablation;
  }
  return !ablation || L == 6 || L == 8;
}

// prime schedule: p <= B1 ascending, each repeated e_p times (p^e_p <= B1), padded to 32 words
std::vector<uint32_t> stage1_primes(uint64_t B1, uint32_t* n_out) {
  std::vector<uint8_t> sieve(B1 + 1, 1);
  std::vector<uint32_t> list;
  for (uint64_t p = 2; p <= B1; ++p) {
    if (!sieve[p]) continue;
    for (uint64_t q = p * p; q <= B1; q += p) sieve[q] = 0;
    for (uint64_t q = p; q <= B1; q *= p) list.push_back((uint32_t)p);
  }
  *n_out = (uint32_t)list.size();
  list.resize(((list.size() + 31) / 32) * 32, 0u);
  return list;
}

bool aligned(const void* p, size_t a) { return ((uintptr_t)p % a) == 0; }

// Stream-ordered scratch from the device's default memory pool.  The pool keeps freed memory
// (release threshold = max) so repeated ECM_HOST_BUFFERS calls do not re-map pages each time.
template <class T>
cudaError_t dev_alloc(T** p, size_t bytes, cudaStream_t s) {
  static std::once_flag once[64];
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess && dev >= 0 && dev < 64) {
    std::call_once(once[dev], [dev] {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
    });
  }
  return cudaMallocAsync(reinterpret_cast<void**>(p), bytes, s);
}

ecm_status run_ecm(const uint32_t* N_host, int L, const uint32_t* kw_dev, uint32_t k_bits, const uint64_t* sigmas,
                   size_t count, uint32_t* X, uint32_t* Z, uint32_t* g, uint8_t* status, uint32_t* xaff,
                   uint32_t flags, cudaStream_t s) {
  EcmParams p;
  ecm_status st = make_params(p, N_host, L);
  if (st != ECM_OK) return st;
  const bool host = flags & ECM_HOST_BUFFERS;
  if (!host) {
    if (!aligned(sigmas, 8) || (X && !aligned(X, 8)) || (Z && !aligned(Z, 8)) || (g && !aligned(g, 8)) ||
        (xaff && !aligned(xaff, 8)))
      return ECM_E_ARG;
    return cuda_err(ecm::launch_ecm(p, kw_dev, k_bits, sigmas, count, X, Z, g, status, xaff, flags, s));
  }
  // host staging: one device block for sigmas and all outputs
  const size_t res = count * L * sizeof(uint32_t);
  const size_t bytes = count * 8 + 4 * res + count;
  uint8_t* d = nullptr;
  cudaError_t e = dev_alloc(&d, bytes, s);
  if (e != cudaSuccess) return cuda_err(e);
  uint64_t* dsig = reinterpret_cast<uint64_t*>(d);
  uint32_t* dX = reinterpret_cast<uint32_t*>(d + count * 8);
  uint32_t* dZ = reinterpret_cast<uint32_t*>(d + count * 8 + res);
  uint32_t* dg = reinterpret_cast<uint32_t*>(d + count * 8 + 2 * res);
  uint32_t* dx = reinterpret_cast<uint32_t*>(d + count * 8 + 3 * res);
  uint8_t* dst = d + count * 8 + 4 * res;
  e = cudaMemcpyAsync(dsig, sigmas, count * 8, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess)
    e = ecm::launch_ecm(p, kw_dev, k_bits, dsig, count, X ? dX : nullptr, Z ? dZ : nullptr, g ? dg : nullptr, dst,
                        xaff ? dx : nullptr, flags, s);
  if (e == cudaSuccess && X) e = cudaMemcpyAsync(X, dX, res, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && Z) e = cudaMemcpyAsync(Z, dZ, res, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && g) e = cudaMemcpyAsync(g, dg, res, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && xaff) e = cudaMemcpyAsync(xaff, dx, res, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(status, dst, count, cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(d, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  return cuda_err(e);
}

// ECM_HOST_BUFFERS without ECM_CHECK (AoS or limb-sliced): the batch is cut into chunks that cycle
// through three internal streams, so the host->device copy of chunk c+1, the kernel of chunk c and
// the device->host copy of chunk c-1 overlap (copy engines and SMs run concurrently).  Chunks are
// whole waves of the kernel that runs them (SMs x resident CTAs x elements per CTA), so no chunk
// ends in a partly filled wave.  Chunk sizes ramp up from one wave by about 1.5x per chunk to the
// cap (about count/32): a chunk's host->device copy must fit in the previous chunk's kernel time, or
// the SMs idle (at L = 6, K = 256 a wave copies in ~0.2 ms and computes in ~0.33 ms); the last chunks
// are one wave and the ragged rest, so the final device->host copy is short.
std::vector<size_t> pipeline_chunks(size_t count, size_t wave) {
  const size_t nw = count / wave, ragged = count % wave;
  size_t capw = (count / 32 + wave - 1) / wave;  // cap in waves
  if (capw < 1) capw = 1;
  std::vector<size_t> sizes;
  size_t rem = nw, gw = 1;  // waves per chunk: 1, 1, 2, 3, 4, 6, 9, ... up to the cap; the last one is 1
  while (rem > 1) {
    size_t t = gw < capw ? gw : capw;
    if (t > rem - 1) t = rem - 1;
    sizes.push_back(t * wave);
    rem -= t;
    if (sizes.size() >= 2) gw = (gw * 3 / 2 > gw + 1) ? gw * 3 / 2 : gw + 1;
  }
  if (rem) sizes.push_back(rem * wave);  // the last whole wave
  if (ragged) sizes.push_back(ragged);   // the ragged rest on its own: a limb-sliced chunk whose count is
                                         // not a multiple of 4 takes the slower unaligned path
  return sizes;
}
constexpr int kPipeStreams = 3;
cudaError_t mulmod_host_pipelined(const uint32_t* a, const uint32_t* b, const uint32_t* n, uint32_t* out,
                                  size_t count, int L, uint32_t iters, uint32_t flags, cudaStream_t s) {
  const bool square = flags & ECM_SQUARE;
  const bool sliced = flags & ECM_LAYOUT_SLICED;
  size_t wave = 0;
  cudaError_t e = ecm::launch_mulmod(nullptr, nullptr, nullptr, nullptr, (size_t)1 << 24, L, iters, flags, s, &wave);
  if (e != cudaSuccess) return e;
  if (wave == 0) wave = 1u << 16;
  const std::vector<size_t> plan = pipeline_chunks(count, wave);
  size_t chunk = 0;
  for (size_t m : plan) chunk = m > chunk ? m : chunk;
  // words per array per slot, rounded up to 128 bytes: the last chunk carries the ragged rest (any
  // count), and every sub-array must stay 16-byte aligned for the bulk copies and 128-bit accesses
  const size_t cw = (chunk * (size_t)L + 31) & ~(size_t)31;
  uint32_t* scratch = nullptr;
  e = dev_alloc(&scratch, kPipeStreams * 4 * cw * sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  cudaStream_t st[kPipeStreams] = {};
  cudaEvent_t start = nullptr, done[kPipeStreams] = {};
  for (int i = 0; i < kPipeStreams && e == cudaSuccess; ++i) e = cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
  for (int i = 0; i < kPipeStreams && e == cudaSuccess; ++i) e = cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(start, s);
  for (int i = 0; i < kPipeStreams && e == cudaSuccess; ++i) e = cudaStreamWaitEvent(st[i], start, 0);
  for (size_t c0 = 0, c = 0; c < plan.size() && e == cudaSuccess; ++c) {
    const size_t m = plan[c];
    const size_t by = m * (size_t)L * sizeof(uint32_t);
    cudaStream_t q = st[c % kPipeStreams];
    uint32_t* base = scratch + (c % kPipeStreams) * 4 * cw;
    uint32_t *ta = base, *tb = base + cw, *tn = base + 2 * cw, *to = base + 3 * cw;
    if (!sliced) {
      e = cudaMemcpyAsync(ta, a + c0 * L, by, cudaMemcpyHostToDevice, q);
      if (e == cudaSuccess && !square) e = cudaMemcpyAsync(tb, b + c0 * L, by, cudaMemcpyHostToDevice, q);
      if (e == cudaSuccess) e = cudaMemcpyAsync(tn, n + c0 * L, by, cudaMemcpyHostToDevice, q);
    } else {
      // limb j of the chunk is the row [j*count + c0, +m) of the host array: one 2-D copy of L
      // rows per array into a chunk-local sliced tile [j*m + i]
      const size_t hp = count * sizeof(uint32_t), dp = m * sizeof(uint32_t);
      e = cudaMemcpy2DAsync(ta, dp, a + c0, hp, dp, L, cudaMemcpyHostToDevice, q);
      if (e == cudaSuccess && !square) e = cudaMemcpy2DAsync(tb, dp, b + c0, hp, dp, L, cudaMemcpyHostToDevice, q);
      if (e == cudaSuccess) e = cudaMemcpy2DAsync(tn, dp, n + c0, hp, dp, L, cudaMemcpyHostToDevice, q);
    }
    if (e == cudaSuccess) e = ecm::launch_mulmod(ta, square ? nullptr : tb, tn, to, m, L, iters, flags, q);
    if (e == cudaSuccess) {
      if (!sliced)
        e = cudaMemcpyAsync(out + c0 * L, to, by, cudaMemcpyDeviceToHost, q);
      else
        e = cudaMemcpy2DAsync(out + c0, count * sizeof(uint32_t), to, m * sizeof(uint32_t), m * sizeof(uint32_t), L,
                              cudaMemcpyDeviceToHost, q);
    }
    c0 += m;
  }
  for (int i = 0; i < kPipeStreams; ++i) {
    if (done[i] && st[i]) {
      cudaEventRecord(done[i], st[i]);
      cudaStreamWaitEvent(s, done[i], 0);
    }
  }
  cudaFreeAsync(scratch, s);
  const cudaError_t e2 = cudaStreamSynchronize(s);
  for (int i = 0; i < kPipeStreams; ++i) {
    if (st[i]) cudaStreamDestroy(st[i]);
    if (done[i]) cudaEventDestroy(done[i]);
  }
  if (start) cudaEventDestroy(start);
  return e != cudaSuccess ? e : e2;
}

}  // namespace

extern "C" {

const char* ecm_strerror(ecm_status s) {
  switch (s) {
    case ECM_OK: return "ok";
    case ECM_E_ARG: return "invalid argument (null pointer, count 0, unsupported L, misalignment or flags)";
    case ECM_E_MODULUS: return "modulus must be odd and >= 3";
    case ECM_E_WIDTH: return "modulus wider than 32L-2 bits (two spare bits required)";
    case ECM_E_B1: return "B1 must be in [2, 2^32) / scalar must be >= 1";
    case ECM_E_RANGE: return "operand >= 2N";
    case ECM_E_CUDA: return "CUDA runtime error";
    case ECM_E_NOMEM: return "out of memory";
  }
  return "unknown status";
}

const char* ecm_version(void) { return "libecmgpu sm_100a " ECMGPU_VERSION; }

uint32_t ecm_stage1_kbits(uint64_t B1) {
  if (B1 < 2 || B1 >= (1ull << 32)) return 0;
  uint32_t bits = 0;
  (void)stage1_scalar(B1, &bits);
  return bits;
}

ecm_status ecm_mulmod_batch(const uint32_t* a, const uint32_t* b, const uint32_t* n, uint32_t* out, size_t count,
                            int L, uint32_t iters, uint32_t flags, void* stream) {
  const bool square = flags & ECM_SQUARE;
  if (!a || !n || !out || (!b && !square) || !valid_count(count) || !valid_L_mulmod(L) || iters == 0 ||
      (flags & ~kKnownFlags))
    return ECM_E_ARG;
  if (flags & (ECM_NO_XAFF | ECM_EAGER | ECM_PRIME_LADDERS | ECM_KERNEL_LANES4 | ECM_KERNEL_LANES1 | ECM_CURVE_SMALL))
    return ECM_E_ARG;
  if ((flags & ECM_REDC_MASK) > ECM_REDC_KARATSUBA) return ECM_E_ARG;
  if ((flags & ECM_KERNEL_STREAM) && (flags & ECM_KERNEL_WARP)) return ECM_E_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool host = flags & ECM_HOST_BUFFERS;
  const size_t bytes = count * (size_t)L * sizeof(uint32_t);
  const uint32_t* da = a;
  const uint32_t* db = b;
  const uint32_t* dn = n;
  uint32_t* dout = out;
  uint8_t* scratch = nullptr;
  cudaError_t e = cudaSuccess;
  if (host && !(flags & ECM_CHECK))
    return cuda_err(mulmod_host_pipelined(a, b, n, out, count, L, iters, flags, s));
  if (host) {
    // four sub-buffers, each starting on a 16-byte boundary (the AoS kernels move tiles with bulk
    // copies and 128-bit accesses, which need it): stride rounded up to a multiple of 4 words
    const size_t stride = (count * (size_t)L + 3) & ~(size_t)3;
    e = dev_alloc(&scratch, 4 * stride * sizeof(uint32_t), s);
    if (e != cudaSuccess) return cuda_err(e);
    uint32_t* base = reinterpret_cast<uint32_t*>(scratch);
    uint32_t* ta = base;
    uint32_t* tb = base + stride;
    uint32_t* tn = base + 2 * stride;
    dout = base + 3 * stride;
    e = cudaMemcpyAsync(ta, a, bytes, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && !square) e = cudaMemcpyAsync(tb, b, bytes, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(tn, n, bytes, cudaMemcpyHostToDevice, s);
    da = ta;
    db = square ? nullptr : tb;
    dn = tn;
  } else {
    const size_t al = (flags & ECM_LAYOUT_SLICED) ? 4 : 16;
    if (!aligned(a, al) || !aligned(n, al) || !aligned(out, al) || (b && !square && !aligned(b, al))) return ECM_E_ARG;
  }
  ecm_status result = ECM_OK;
  if (e == cudaSuccess && (flags & ECM_CHECK)) {
    uint32_t* derr = nullptr;
    e = dev_alloc(&derr, sizeof(uint32_t), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(derr, 0, sizeof(uint32_t), s);
    if (e == cudaSuccess) e = ecm::launch_mulmod_check(da, db, dn, count, L, flags, derr, s);
    uint32_t herr = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&herr, derr, sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (derr) cudaFreeAsync(derr, s);
    if (e == cudaSuccess && herr) result = (ecm_status)herr;
  }
  if (e == cudaSuccess && result == ECM_OK) e = ecm::launch_mulmod(da, db, dn, dout, count, L, iters, flags, s);
  if (host) {
    if (e == cudaSuccess && result == ECM_OK) e = cudaMemcpyAsync(out, dout, bytes, cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(scratch, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  }
  if (e != cudaSuccess) return cuda_err(e);
  return result;
}

ecm_status ecm_stage1_batch(const uint32_t* N_host, int L, uint64_t B1, const uint64_t* sigmas, size_t count,
                            uint32_t* X, uint32_t* Z, uint32_t* g, uint8_t* status, uint32_t* xaff, uint32_t flags,
                            void* stream) {
  if (!N_host || !sigmas || !status || !valid_count(count) || !valid_L(L) || (flags & ~kKnownFlags)) return ECM_E_ARG;
  if (flags & (ECM_SQUARE | ECM_LAYOUT_SLICED | ECM_CANONICAL | ECM_KERNEL_STREAM | ECM_KERNEL_WARP)) return ECM_E_ARG;
  if (!ecm_variant_ok(L, flags)) return ECM_E_ARG;
  if (!xaff && !(flags & ECM_NO_XAFF)) flags |= ECM_NO_XAFF;
  if (B1 < 2 || B1 >= (1ull << 32)) return ECM_E_B1;
  EcmParams probe;
  ecm_status st = make_params(probe, N_host, L);
  if (st != ECM_OK) return st;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_err(e);
  uint32_t* kw = nullptr;
  uint32_t kb = 0;
  {
    PlanCache& c = cache();
    std::lock_guard<std::mutex> lock(c.mu);
    const uint64_t key = B1 | ((flags & ECM_PRIME_LADDERS) ? (1ull << 40) : 0ull);
    auto it = c.plans.find({dev, key});
    if (it == c.plans.end()) {
      std::vector<uint32_t> words = (flags & ECM_PRIME_LADDERS) ? stage1_primes(B1, &kb) : stage1_scalar(B1, &kb);
      e = cudaMalloc(&kw, words.size() * sizeof(uint32_t));
      if (e == cudaSuccess) e = cudaMemcpy(kw, words.data(), words.size() * sizeof(uint32_t), cudaMemcpyHostToDevice);
      if (e != cudaSuccess) return cuda_err(e);
      c.plans[{dev, key}] = {kw, kb};
    } else {
      kw = it->second.first;
      kb = it->second.second;
    }
  }
  return run_ecm(N_host, L, kw, kb, sigmas, count, X, Z, g, status, xaff, flags, static_cast<cudaStream_t>(stream));
}

ecm_status ecm_ladder_batch(const uint32_t* N_host, int L, const uint32_t* k_words, uint32_t k_bits,
                            const uint64_t* sigmas, size_t count, uint32_t* X, uint32_t* Z, uint32_t* g,
                            uint8_t* status, uint32_t* xaff, uint32_t flags, void* stream) {
  if (!N_host || !k_words || !sigmas || !status || !valid_count(count) || !valid_L(L) || (flags & ~kKnownFlags))
    return ECM_E_ARG;
  if (flags & (ECM_SQUARE | ECM_LAYOUT_SLICED | ECM_CANONICAL | ECM_KERNEL_STREAM | ECM_KERNEL_WARP)) return ECM_E_ARG;
  if (!ecm_variant_ok(L, flags)) return ECM_E_ARG;
  if (!xaff && !(flags & ECM_NO_XAFF)) flags |= ECM_NO_XAFF;
  if (flags & ECM_PRIME_LADDERS) return ECM_E_ARG;
  if (k_bits == 0) return ECM_E_B1;
  const size_t nw = (k_bits + 31) / 32;
  if (bitlen(k_words, (int)nw) != (int)k_bits) return ECM_E_B1;
  EcmParams probe;
  ecm_status st = make_params(probe, N_host, L);
  if (st != ECM_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t padded = ((nw + 31) / 32) * 32;
  std::vector<uint32_t> words(padded, 0u);
  std::memcpy(words.data(), k_words, nw * sizeof(uint32_t));
  uint32_t* kw = nullptr;
  cudaError_t e = dev_alloc(&kw, padded * sizeof(uint32_t), s);
  if (e != cudaSuccess) return cuda_err(e);
  e = cudaMemcpyAsync(kw, words.data(), padded * sizeof(uint32_t), cudaMemcpyHostToDevice, s);
  // pageable source: the copy is complete when cudaMemcpyAsync returns, `words` may die after
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    cudaFreeAsync(kw, s);
    return cuda_err(e);
  }
  st = run_ecm(N_host, L, kw, k_bits, sigmas, count, X, Z, g, status, xaff, flags, s);
  cudaFreeAsync(kw, s);
  return st;
}

}  // extern "C"
