// kernels.h — host-side launchers of the sm_100a kernels (internal to libecmgpu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace ecm {

cudaError_t launch_mulmod(const uint32_t* a, const uint32_t* b, const uint32_t* n, uint32_t* out, size_t count,
                          int L, uint32_t iters, uint32_t flags, cudaStream_t s);
cudaError_t launch_mulmod_check(const uint32_t* a, const uint32_t* b, const uint32_t* n, size_t count, int L,
                                uint32_t flags, uint32_t* err, cudaStream_t s);

// ECM stage 1: N, 2N, n0inv, R^2 mod N and the scalar bits (MSB first) are uploaded by the
// host into a per-call parameter block (struct below), then three kernels run:
//   setup (Suyama + inverse), ladder (hot loop), tail (gcd, affine x, canonical X, Z).
struct EcmParams {
  int L;
  uint32_t n0inv;
  uint32_t N[16], N2[16], R2[16], ONE[16], NP[16];  // N, 2N, R^2 mod N, R mod N (Montgomery 1), -N^{-1} mod R
};

cudaError_t launch_ecm(const EcmParams& p, const uint32_t* kbits_dev, uint32_t k_bits, const uint64_t* sigmas,
                       size_t count, uint32_t* X, uint32_t* Z, uint32_t* g, uint8_t* status, uint32_t* xaff,
                       uint32_t flags, cudaStream_t s);

}  // namespace ecm
