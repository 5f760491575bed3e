// kernels.h — host-side launchers of the sm_100a kernels (internal to libecmgpu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace ecm {

// wave != nullptr: launch nothing; *wave = elements per full wave of the kernel the call would run
cudaError_t launch_mulmod(const uint32_t* a, const uint32_t* b, const uint32_t* n, uint32_t* out, size_t count,
                          int L, uint32_t iters, uint32_t flags, cudaStream_t s, size_t* wave = nullptr);
cudaError_t launch_mulmod_check(const uint32_t* a, const uint32_t* b, const uint32_t* n, size_t count, int L,
                                uint32_t flags, uint32_t* err, cudaStream_t s);

// ECM stage 1: N, 2N, n0inv, R^2 mod N, R mod N and -N^{-1} mod R go to the kernel as a parameter
// block (struct below, constant bank); the scalar plan (bits of k, or the prime list) is a device
// buffer.  One kernel per call runs setup, ladder and tail (ecm_kernels.cuh).
struct EcmParams {
  int L;
  uint32_t n0inv;
  uint32_t N[16], N2[16], R2[16], ONE[16], NP[16];  // N, 2N, R^2 mod N, R mod N (Montgomery 1), -N^{-1} mod R
};

cudaError_t launch_ecm(const EcmParams& p, const uint32_t* kbits_dev, uint32_t k_bits, const uint64_t* sigmas,
                       size_t count, uint32_t* X, uint32_t* Z, uint32_t* g, uint8_t* status, uint32_t* xaff,
                       uint32_t flags, cudaStream_t s);

}  // namespace ecm
