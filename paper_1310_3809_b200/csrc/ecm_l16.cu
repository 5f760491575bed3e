// ecm_l16.cu — ECM stage-1 kernels for L = 16 (one translation unit per width so the build
// compiles the widths in parallel; the kernels are in ecm_kernels.cuh).
#include "ecm_kernels.cuh"

namespace ecm {
template cudaError_t launch_ecm_L<16>(const EcmParams& p, const uint32_t* kw, uint32_t k_bits, const uint64_t* sigmas,
                                       size_t count, uint32_t* X, uint32_t* Z, uint32_t* g, uint8_t* status,
                                       uint32_t* xaff, uint32_t flags, cudaStream_t s);
}  // namespace ecm
