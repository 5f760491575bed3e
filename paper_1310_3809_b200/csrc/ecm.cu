// ecm.cu — dispatch of the ECM stage-1 kernels by width.  The kernels are in ecm_kernels.cuh,
// instantiated per width in ecm_l<L>.cu.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace ecm {

template <int L>
cudaError_t launch_ecm_L(const EcmParams& p, const uint32_t* kw, uint32_t k_bits, const uint64_t* sigmas, size_t count,
                         uint32_t* X, uint32_t* Z, uint32_t* g, uint8_t* status, uint32_t* xaff, uint32_t flags,
                         cudaStream_t s);

cudaError_t launch_ecm(const EcmParams& p, const uint32_t* kw, uint32_t k_bits, const uint64_t* sigmas, size_t count,
                       uint32_t* X, uint32_t* Z, uint32_t* g, uint8_t* status, uint32_t* xaff, uint32_t flags,
                       cudaStream_t s) {
#ifdef ECM_ONLY_L  // single-width build (tools/ecm_ab.py variant libraries)
  if (p.L == ECM_ONLY_L) return launch_ecm_L<ECM_ONLY_L>(p, kw, k_bits, sigmas, count, X, Z, g, status, xaff, flags, s);
  return cudaErrorInvalidValue;
#endif
  switch (p.L) {
    case 4: return launch_ecm_L<4>(p, kw, k_bits, sigmas, count, X, Z, g, status, xaff, flags, s);
    case 6: return launch_ecm_L<6>(p, kw, k_bits, sigmas, count, X, Z, g, status, xaff, flags, s);
    case 8: return launch_ecm_L<8>(p, kw, k_bits, sigmas, count, X, Z, g, status, xaff, flags, s);
    case 12: return launch_ecm_L<12>(p, kw, k_bits, sigmas, count, X, Z, g, status, xaff, flags, s);
    case 16: return launch_ecm_L<16>(p, kw, k_bits, sigmas, count, X, Z, g, status, xaff, flags, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ecm
