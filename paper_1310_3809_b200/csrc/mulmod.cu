// mulmod.cu — dispatch of ecm_mulmod_batch by width, and the ECM_CHECK precondition kernel.
// The chain kernels are in mulmod_kernels.cuh, instantiated per width in mulmod_l<L>.cu.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace ecm {

template <int L>
cudaError_t launch_mulmod_L(const uint32_t* a, const uint32_t* b, const uint32_t* n, uint32_t* out, size_t count,
                            uint32_t iters, uint32_t flags, cudaStream_t s, size_t* wave);

// ---- precondition check (ECM_CHECK): n odd, bitlen(n) <= 32L-2, a, b < 2n ----
template <int L>
__global__ void mulmod_check_kernel(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                                    const uint32_t* __restrict__ n, size_t count, uint32_t flags,
                                    uint32_t* err) {
  const bool sliced = flags & 0x4u, square = flags & 0x2u;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t x[L], y[L], nn[L], n2[L + 1];
#pragma unroll
    for (int k = 0; k < L; ++k) {
      const size_t off = sliced ? (size_t)k * count + i : i * L + k;
      x[k] = a[off];
      y[k] = square ? 0u : b[off];
      nn[k] = n[off];
    }
    uint32_t code = 0;
    uint32_t upper = 0;
#pragma unroll
    for (int k = 1; k < L; ++k) upper |= nn[k];
    if (!(nn[0] & 1u) || (upper == 0 && nn[0] < 3)) code = 2;  // ECM_E_MODULUS: even, or N = 1
    else if (nn[L - 1] >> 30) code = 3;                    // ECM_E_WIDTH
    else {
      // 2n (fits L words since n < 2^(32L-2))
      uint32_t c = 0;
#pragma unroll
      for (int k = 0; k < L; ++k) {
        n2[k] = (nn[k] << 1) | c;
        c = nn[k] >> 31;
      }
      // x < 2n and y < 2n ?
      bool xlt = false, ylt = false, xd = false, yd = false;
#pragma unroll
      for (int k = L - 1; k >= 0; --k) {
        if (!xd && x[k] != n2[k]) { xlt = x[k] < n2[k]; xd = true; }
        if (!yd && y[k] != n2[k]) { ylt = y[k] < n2[k]; yd = true; }
      }
      if (!xlt || !ylt) code = 5;  // ECM_E_RANGE
    }
    if (code) atomicMax(err, code);
  }
}

cudaError_t launch_mulmod(const uint32_t* a, const uint32_t* b, const uint32_t* n, uint32_t* out, size_t count,
                          int L, uint32_t iters, uint32_t flags, cudaStream_t s, size_t* wave) {
#ifdef ECM_ONLY_L  // single-width build (tools/ecm_ab.py variant libraries)
  if (L == ECM_ONLY_L) return launch_mulmod_L<ECM_ONLY_L>(a, b, n, out, count, iters, flags, s, wave);
  return cudaErrorInvalidValue;
#endif
  switch (L) {
    case 6: return launch_mulmod_L<6>(a, b, n, out, count, iters, flags, s, wave);
    case 4: return launch_mulmod_L<4>(a, b, n, out, count, iters, flags, s, wave);
    case 8: return launch_mulmod_L<8>(a, b, n, out, count, iters, flags, s, wave);
    case 12: return launch_mulmod_L<12>(a, b, n, out, count, iters, flags, s, wave);
    case 16: return launch_mulmod_L<16>(a, b, n, out, count, iters, flags, s, wave);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_mulmod_check(const uint32_t* a, const uint32_t* b, const uint32_t* n, size_t count, int L,
                                uint32_t flags, uint32_t* err, cudaStream_t s) {
  const unsigned blocks = (unsigned)((count + 255) / 256 < 4096 ? (count + 255) / 256 : 4096);
  switch (L) {
    case 4: mulmod_check_kernel<4><<<blocks, 256, 0, s>>>(a, b, n, count, flags, err); break;
    case 6: mulmod_check_kernel<6><<<blocks, 256, 0, s>>>(a, b, n, count, flags, err); break;
    case 8: mulmod_check_kernel<8><<<blocks, 256, 0, s>>>(a, b, n, count, flags, err); break;
    case 12: mulmod_check_kernel<12><<<blocks, 256, 0, s>>>(a, b, n, count, flags, err); break;
    case 16: mulmod_check_kernel<16><<<blocks, 256, 0, s>>>(a, b, n, count, flags, err); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace ecm
